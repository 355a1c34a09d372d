"""Pins the CPU oracle (oracle/gm_oracle.c) to the reference's own outputs.

The fixtures were produced by importing the reference package in the
build container (tests/golden/make_golden.py); every comparison here is
bit-exact (y via float.hex, s, emitted counts), so the oracle can stand in
for the reference on the GPU box and at sizes Python cannot reach.
"""

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_io import hexs, load_json, load_npz, sketch_arrays, vector_case


@pytest.fixture(scope="module")
def kats():
    return load_json("rng_kats.json")


@pytest.fixture(scope="module")
def cases():
    return load_json("sketch_cases.json")


def test_uniform_open_kats(kats):
    for seed, e, z, want in kats["uniform_open"]:
        assert O.uniform_open(seed, e, z) == float.fromhex(want)


def test_survey_appendix_b_kats():
    # SURVEY Appendix B, uniform_open(SeedScheme(1), 1, z)
    assert O.uniform_open(1, 1, 1).hex() == "0x1.67113a4f020dap-1"
    assert O.uniform_open(1, 1, 2).hex() == "0x1.94bdfaaa3e252p-1"
    assert O.uniform_open(1, 1, 3).hex() == "0x1.f06f2ca7cacaep-1"
    assert O.fingerprint(1) == 0xD10756E2BF1ACDBA


def test_rand_int_between_kats(kats):
    for pseed, e, z, lo, hi, want in kats["rand_int_between"]:
        assert O.rand_int_between(pseed, e, z, lo, hi) == want


def test_fingerprint_and_derive(kats):
    for seed, salt, fp, perm in kats["fingerprint"]:
        assert O.fingerprint(seed, salt) == fp
        assert (seed ^ salt) & ((1 << 64) - 1) == perm
    lib = O.lib()
    for m, t, want in kats["derive_seed"]:
        assert lib.gmo_derive_seed(m, t) == want


def test_full_queues(kats):
    for q in kats["queues"]:
        seed = q["seed"]
        t, s = O.run_queue_full(seed, O.DEFAULT_STREAM_SALT, q["element"], float.fromhex(q["weight"]), q["k"])
        assert t.tolist() == hexs(q["times"]).tolist()
        assert s.tolist() == q["servers"]


def test_sketch_fast_and_naive(cases):
    for case in cases["vectors"]:
        ids, w = vector_case(case)
        rc, y, s, em = O.sketch_fast(ids, w, case["k"], case["seed"])
        wy, ws = sketch_arrays(case["fast"])
        assert rc == 0
        assert y.tolist() == wy.tolist() and np.array_equal(s, ws)
        assert em == case["fast"]["emitted"]  # same FastSearch schedule as the reference
        if "naive_emitted" in case:
            rc, y2, s2, em2 = O.sketch_naive(ids, w, case["k"], case["seed"])
            assert y2.tolist() == wy.tolist() and np.array_equal(s2, ws)
            assert em2 == case["naive_emitted"]


def test_sketch_stream(cases):
    for case in cases["streams"]:
        ids = np.array([int(e) & 0xFFFFFFFFFFFFFFFF for e in case["ids"]], dtype=np.uint64)
        w = hexs(case["w"])
        rc, y, s, em, _ = O.sketch_stream(ids, w, case["k"], case["seed"])
        wy, ws = sketch_arrays(case["sketch"])
        assert rc == 0
        assert y.tolist() == wy.tolist() and np.array_equal(s, ws)
        assert em == case["sketch"]["emitted"]


def test_merge_partition_law(cases):
    for case in cases["merges"]:
        ys = np.array([sketch_arrays(p)[0] for p in case["parts"]])
        ss = np.array([sketch_arrays(p)[1] for p in case["parts"]])
        y, s = O.merge(ys, ss)
        wy, ws = sketch_arrays(case["merged"])
        assert y.tolist() == wy.tolist() and np.array_equal(s, ws)


def test_bench_golden():
    """test_bench.py:67-82 golden through the oracle: 9 matches, c = 1.76291929033662."""
    g = load_json("bench_golden.json")
    sks = []
    for vec in g["vectors"]:
        ids = np.array([e for e, _ in vec], dtype=np.uint64)
        w = np.array([x for _, x in vec], dtype=np.float64)
        rc, y, s, _ = O.sketch_fast(ids, w, g["k"], g["seed"])
        sks.append((y, s))
    assert int(np.sum(sks[0][1] == sks[1][1])) == g["matches"] == 9
    card = (g["k"] - 1) / O.fsum(sks[2][0])
    assert card == float.fromhex(g["cardinality"])
    assert card == pytest.approx(1.76291929033662, rel=1e-12)


def test_config1_golden():
    g = load_npz("config1.npz")
    rc, y, s, _, _ = O.sketch_stream(g["ids"].astype(np.uint64), g["w"], int(g["k"]), int(g["seed"]))
    assert rc == 0
    assert y.tolist() == g["y"].tolist() and np.array_equal(s, g["s"])


def test_config2_sample_golden():
    g = load_npz("config2_sample.npz")
    rc, y, s, em = O.sketch_csr(g["ids"].astype(np.uint64), g["w"].astype(np.float64), g["offsets"],
                                int(g["k"]), int(g["seed"]), mode=0, threads=2)
    assert rc == 0
    assert y.tolist() == g["y"].tolist() and np.array_equal(s, g["s"])
    assert em.tolist() == g["emitted"].tolist()


def test_oracle_errors():
    rc, *_ = O.sketch_fast(np.array([], np.uint64), np.array([], np.float64), 4, 1)
    assert rc == O.EMPTY_VECTOR
    rc, *_ = O.sketch_fast(np.array([1], np.uint64), np.array([0.0]), 4, 1)
    assert rc == O.INVALID_WEIGHT
    rc, y, s, em, ei = O.sketch_stream(np.array([1, 1], np.uint64), np.array([0.5, 0.75]), 4, 1)
    assert rc == O.INCONSISTENT_WEIGHT and ei == 1
    rc, *_ = O.sketch_stream(np.array([], np.uint64), np.array([], np.float64), 3, 1)
    assert rc == O.INCOMPLETE
