"""Host-side logic of the drop-in package, mirroring the reference's own
unit tests for the types (test_sketch.py:49-109, test_randgen.py:153-177,
test_estimate.py host algebra).  No GPU: sketch calls must fail loudly."""

import math

import numpy as np
import pytest
import torch

import paper_2302_05176_b200 as gm
from paper_2302_05176_b200 import shard
from paper_2302_05176_b200.errors import raise_for
from tests.golden_io import load_json

SCHEME = gm.SeedScheme(20240601)
EXAMPLE_WEIGHTS = (0.3, 0.1, 0.05, 0.05, 0.2, 0.07, 0.1, 0.03)
EXAMPLE_VECTOR = gm.WeightedVector({i + 1: w for i, w in enumerate(EXAMPLE_WEIGHTS)})


class TestWeightedVector:
    def test_rejects_bad_weights(self):
        for bad in (0.0, -1.0, float("nan"), float("inf"), 1e-310):
            with pytest.raises(gm.InvalidWeightError):
                gm.WeightedVector({1: bad})

    def test_rejects_bad_indices(self):
        with pytest.raises(gm.InvalidWeightError):
            gm.WeightedVector({0: 1.0})

    def test_sums_and_counts(self):
        v = gm.WeightedVector({3: 0.5, 1: 0.25, 7: 0.25})
        assert v.n_plus == 3
        assert v.weight_sum == pytest.approx(1.0, rel=1e-12)
        assert v.items() == ((1, 0.25), (3, 0.5), (7, 0.25))
        assert v[3] == 0.5 and v.get(99) == 0.0
        with pytest.raises(gm.MissingElementError):
            v[99]
        ids, w = v.arrays()
        assert ids.tolist() == [1, 3, 7] and w.tolist() == [0.25, 0.5, 0.25]

    def test_equality_and_scaled(self):
        assert gm.WeightedVector({1: 0.5, 2: 1.5}) == gm.WeightedVector({2: 1.5, 1: 0.5})
        v = gm.WeightedVector({1: 0.5, 2: 1.5}).scaled(2.0)
        assert v[1] == 1.0 and v[2] == 3.0
        with pytest.raises(gm.InvalidWeightError):
            v.scaled(0.0)


def test_compute_ri_worked_example():
    """sketch.py:160-169 sizing KAT (test_sketch.py:82-86)."""
    assert [gm.compute_ri(17, EXAMPLE_VECTOR, e) for e in range(1, 9)] == [6, 2, 1, 1, 4, 2, 2, 1]
    with pytest.raises(gm.InvalidParameterError):
        gm.compute_ri(-1, EXAMPLE_VECTOR, 1)


def test_generation_params():
    assert gm.GenerationParams(k=32, scheme=SCHEME).delta == 32
    with pytest.raises(gm.InvalidParameterError):
        gm.GenerationParams(k=0, scheme=SCHEME)
    with pytest.raises(gm.InvalidParameterError):
        gm.GenerationParams(k=4, scheme=SCHEME, delta=0)


def test_seed_scheme_matches_reference_kats():
    kats = load_json("rng_kats.json")
    for seed, salt, fp, perm in kats["fingerprint"]:
        sc = gm.SeedScheme(seed, salt)
        assert sc.fingerprint == fp and sc.perm_seed == perm
    for m, t, want in kats["derive_seed"]:
        assert gm.derive_seed(m, t) == want
    assert gm.SeedScheme(1).fingerprint == 0xD10756E2BF1ACDBA
    assert 0 <= gm.SeedScheme(-1).global_seed < 1 << 64


def test_lazy_permutation():
    perm = gm.LazyPermutation()
    assert perm[0] == 1 and perm[10] == 11
    perm[0], perm[10] = perm[10], perm[0]
    assert perm[0] == 11 and perm[10] == 1 and perm[5] == 6


def test_json_round_trip_bit_exact():
    sk = gm.GumbelMaxSketch(3, (5, 9, 5), (0.1, 1 / 3, 2.0 ** -1070), gm.SeedScheme(1).fingerprint)
    again = gm.sketch_from_json(gm.sketch_to_json(sk))
    assert again == sk
    with pytest.raises(gm.MismatchedSketchError):
        gm.sketch_from_json("not json")
    with pytest.raises(gm.MismatchedSketchError):
        gm.sketch_from_json('{"format": "something/9", "k": 1}')
    with pytest.raises(gm.InvalidParameterError):
        gm.GumbelMaxSketch(k=3, s=(1, 2), y=(0.1, 0.2), fingerprint=0)


def test_estimators_host_arithmetic():
    g = load_json("bench_golden.json")
    sks = [gm.GumbelMaxSketch(16, tuple(d["s"]), tuple(float.fromhex(v) for v in d["y"]), d["fingerprint"])
           for d in g["sketches"]]
    sim = gm.estimate_jaccard_p(sks[0], sks[1])
    assert sim.matches == 9 and sim.value == 0.5625 and sim.k == 16
    assert gm.estimate_cardinality(sks[2]).value == float.fromhex(g["cardinality"])
    with pytest.raises(gm.InvalidParameterError):
        gm.estimate_cardinality(gm.GumbelMaxSketch(1, (1,), (0.5,), 0))
    with pytest.raises(gm.MismatchedSketchError):
        gm.estimate_jaccard_p(sks[0], gm.GumbelMaxSketch(16, sks[1].s, sks[1].y, 0))


def test_exact_similarities():
    u = gm.WeightedVector({1: 0.5, 2: 0.5})
    assert gm.exact_jaccard_p(u, u) == pytest.approx(1.0)
    assert gm.exact_jaccard_w(u, gm.WeightedVector({3: 1.0})) == 0.0
    assert gm.exact_jaccard_w(u, gm.WeightedVector({1: 0.5, 2: 1.0})) == pytest.approx(1.0 / 1.5)


def test_error_code_mapping():
    for rc, cls in [(1, gm.EmptyVectorError), (2, gm.InvalidWeightError), (3, gm.InvalidParameterError),
                    (4, gm.InconsistentWeightError), (5, gm.IncompleteSketchError),
                    (6, gm.MismatchedSketchError), (100, gm.DeviceError), (101, gm.DeviceError)]:
        with pytest.raises(cls):
            raise_for(rc, "x")
    raise_for(0, "")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Without a GPU the product path raises; it never computes on the CPU."""
    with pytest.raises(gm.DeviceError):
        gm.sketch_fast(EXAMPLE_VECTOR, gm.GenerationParams(k=8, scheme=SCHEME))
    with pytest.raises(gm.DeviceError):
        gm.sketch_csr(np.array([1], np.uint32), np.array([1.0]), np.array([0, 1]), 8, SCHEME)
    with pytest.raises(gm.DeviceError):
        gm.uniform_open(SCHEME, 1, 1)
    with pytest.raises(gm.DeviceError):
        gm.merge([gm.GumbelMaxSketch(1, (1,), (0.5,), 0)])


def test_shard_element_ranges_cover():
    for n, world in [(10, 3), (10**9, 8), (5, 8), (0, 2)]:
        rs = [shard.element_range(n, world, r) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
        sizes = [b - a for a, b in rs]
        assert max(sizes) - min(sizes) <= 1


def test_shard_vector_ranges_balance_elements():
    rng = np.random.default_rng(3)
    sizes = np.clip(np.rint(rng.lognormal(6, 1, 10000)), 1, 50000).astype(np.int64)
    off = np.zeros(sizes.size + 1, np.int64)
    off[1:] = np.cumsum(sizes)
    for world in (1, 2, 4, 8):
        rs = shard.vector_ranges(off, world)
        assert rs[0][0] == 0 and rs[-1][1] == sizes.size
        loads = [int(off[b] - off[a]) for a, b in rs]
        assert max(loads) <= off[-1] / world + sizes.max()


def test_wire_records_match_reference_bytes():
    """sketch_to_json / sketch_from_json (sketch.py:325-357) against records
    the reference itself wrote (tests/golden/wire_records.json): the sketches
    of the golden sketch_cases (sketch_fast) and a merge, rebuilt from the
    fixture values, serialise to the same bytes and parse back equal."""
    cases = load_json("sketch_cases.json")["vectors"]
    for rec in load_json("wire_records.json"):
        if "case" in rec:
            c = cases[rec["case"]]["fast"]
            k = cases[rec["case"]]["k"]
            sk = gm.GumbelMaxSketch(k, tuple(int(x) for x in c["s"]), tuple(float.fromhex(v) for v in c["y"]),
                                    int(c["fingerprint"]))
            assert gm.sketch_to_json(sk) == rec["record"]
        back = gm.sketch_from_json(rec["record"])
        assert gm.sketch_to_json(back) == rec["record"]
