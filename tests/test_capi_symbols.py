"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/*.h declares (no compute calls: there is no GPU here)."""

import ctypes
import glob
import os
import re

from paper_2302_05176_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(gm_[a-z0-9_]+)\s*\(", text))
    return names


def test_header_declares_the_engine():
    names = declared_symbols()
    assert {"gm_sketch_csr", "gm_sketch_elements", "gm_merge", "gm_match_count", "gm_last_error"} <= names


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(declared_symbols()) if not hasattr(L, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert declared_symbols() == set(_lib.SIGNATURES)


def test_version_and_error_string_without_gpu():
    L = _lib.load()
    assert L.gm_version() >= 100
    assert isinstance(_lib.last_error(), str)


def test_bad_parameters_rejected_before_touching_the_device():
    L = _lib.load()
    # k out of range and bad bit widths fail argument checks (no CUDA call)
    assert L.gm_sketch_csr(None, 32, None, 32, None, 1, 0, 1, 2, 0, None, None, None, None) == _lib.GM_ERR_INVALID_PARAMETER
    assert "k must be >= 1" in _lib.last_error()
    assert L.gm_sketch_csr(None, 16, None, 32, None, 1, 8, 1, 2, 0, None, None, None, None) == _lib.GM_ERR_INVALID_PARAMETER
    assert L.gm_sketch_elements(None, 32, None, 8, 1, 8, 1, 2, 0, None, None, None, None) == _lib.GM_ERR_INVALID_PARAMETER
    assert L.gm_merge(None, None, 0, 8, None, None, None) == _lib.GM_ERR_MISMATCHED


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        return  # cuobjdump unavailable
    assert "sm_100a" in out.stdout
