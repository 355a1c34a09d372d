"""The device log (paper_2302_05176_b200/csrc/gm_glibc_log.cuh) is a
restatement of the host C library's log (what CPython's math.log -- the
reference's log, randgen.py:186 -- calls).  CPU check: the same source
compiled for the host, every operation explicit, against libm's log on
keyed uniforms, the near-1 interval and arbitrary positive doubles.  (The
device build is checked against glibc in tests/test_gpu_parity.py.)"""

import os
import subprocess

import pytest

SRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native", "glibc_log_check.cc")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("glog") / "glibc_log_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-o", exe, SRC, "-lm"], check=True)
    return exe


def test_clone_equals_libm_log(checker):
    res = subprocess.run([checker, "3000000", "7"], capture_output=True, text=True)
    bad = [int(x) for x in res.stdout.split()]
    assert res.returncode == 0 and bad[:4] == [0, 0, 0, 0], res.stdout + res.stderr
    assert bad[5] > 0  # the near-1 branch was exercised


def test_table_matches_this_libm():
    """gm_glibc_logtab.h was generated from this image's libm (the GPU box
    runs the same image): regenerate in memory and compare."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "gen_glibc_log", os.path.join(os.path.dirname(os.path.dirname(SRC)), "..", "tools", "gen_glibc_log.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    _, poly, poly1, tab = mod.extract(mod.find_libm())
    text = open(mod.OUT).read()
    for c, lc in tab:
        assert f"{{{c.hex()}, {lc.hex()}}}" in text
    for i, a in enumerate(poly):
        assert f"GM_GLOG_A{i} {a.hex()}" in text
