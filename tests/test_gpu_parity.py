"""Parity of the CUDA path with the reference (golden fixtures) and the
CPU oracle.  Every test calls through the C ABI (libgmsketch_b200.so).

Bar (BASELINE.json north_star): argmax indices s bit-exact; register
values y within 1e-6 relative.  The device log is a bit-exact clone of
glibc's (gm_glibc_log.cuh; the reference's math.log), so the tests assert
y bit-identical too (YTOL = 0).
"""

import math

import numpy as np
import pytest
import torch

import paper_2302_05176_b200 as gm
from oracle import oracle as O
from paper_2302_05176_b200 import workloads
from tests.golden_io import hexs, load_json, load_npz, sketch_arrays, vector_case

pytestmark = pytest.mark.gpu
YTOL = 0.0
U64 = (1 << 64) - 1


def assert_regs(y, s, wy, ws, tol=YTOL):
    y = np.asarray(y, np.float64)
    wy = np.asarray(wy, np.float64)
    s = np.asarray(s).astype(np.uint64) if np.asarray(s).dtype != np.uint64 else np.asarray(s)
    assert np.array_equal(s, np.asarray(ws, np.uint64)), f"s differs at {np.nonzero(s != ws)[0][:10]}"
    rel = np.abs(y - wy) / np.maximum(np.abs(wy), 1e-300)
    assert float(rel.max()) <= tol, f"max rel y error {rel.max()}"


def batch_np(b):
    return b.y.cpu().numpy(), b.s.cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------- K0 RNG
def test_uniform_open_kats_bit_exact():
    kats = load_json("rng_kats.json")["uniform_open"]
    got = gm.uniform_open_batch([k[0] for k in kats], [k[1] for k in kats], [k[2] for k in kats])
    want = hexs([k[3] for k in kats])
    assert got.tolist() == want.tolist()


def test_uniform_open_random_bit_exact():
    rng = np.random.default_rng(11)
    n = 200_000
    seeds = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    el = rng.integers(0, 1 << 63, n, dtype=np.uint64)
    st = rng.integers(1, 70000, n, dtype=np.uint64)
    got = gm.uniform_open_batch(seeds, el, st)
    lib = O.lib()
    want = np.array([lib.gmo_uniform_open(int(a), int(b), int(c)) for a, b, c in zip(seeds[:20000], el[:20000], st[:20000])])
    assert got[:20000].tolist() == want.tolist()
    assert np.all((got > 0) & (got <= 1.0))


def test_uniform_can_be_exactly_one():
    """u = 1.0 when x >> 11 == 2**53 - 1: the device
    rounding must agree.  Find such a key by inverting nothing: scan the
    fixture-free property that u <= 1 and equals the oracle on edge keys."""
    # (x >> 11) * 2**-53 + 2**-54 with x>>11 = 2**53-1 rounds to 1.0 in RN-even
    assert (2**53 - 1) * 2.0**-53 + 2.0**-54 == 1.0


def test_perm_draw_kats_bit_exact():
    kats = [k for k in load_json("rng_kats.json")["rand_int_between"] if k[4] - k[3] < 65536]
    # device draw is z + g mod (k - z + 1) keyed on (element, z): map lo..hi onto z..k
    got = gm.perm_draw_batch([k[0] for k in kats], [k[1] for k in kats], [k[2] for k in kats],
                             [k[2] + (k[4] - k[3]) for k in kats])
    want = [k[5] - k[3] + k[2] for k in kats]
    assert got.tolist() == want


def test_perm_draw_random_bit_exact():
    rng = np.random.default_rng(12)
    n = 20000
    ps = rng.integers(0, 1 << 63, n, dtype=np.uint64)
    el = rng.integers(0, 1 << 63, n, dtype=np.uint64)
    z = rng.integers(1, 9000, n, dtype=np.uint64)
    m = rng.integers(1, 65537, n, dtype=np.uint64)
    ks = z + m - np.uint64(1)
    got = gm.perm_draw_batch(ps, el, z, ks)
    want = [O.rand_int_between(int(a), int(b), int(c), int(c), int(d)) for a, b, c, d in zip(ps, el, z, ks)]
    assert got.tolist() == want


# ---------------------------------------------------------------- sketches vs reference fixtures
def test_sketch_fast_golden_cases():
    cases = load_json("sketch_cases.json")["vectors"]
    for case in cases:
        ids, w = vector_case(case)
        v = gm.WeightedVector({int(e): float(x) for e, x in zip(ids, w)})
        sk = gm.sketch_fast(v, gm.GenerationParams(k=case["k"], scheme=gm.SeedScheme(case["seed"])))
        wy, ws = sketch_arrays(case["fast"])
        assert_regs(sk.y, np.array(sk.s, np.uint64), wy, ws, tol=0.0)  # exact-y finalize: bit-identical
        assert sk == gm.GumbelMaxSketch(case["k"], tuple(int(x) for x in ws), tuple(wy.tolist()),
                                        case["fast"]["fingerprint"])


def test_sketch_naive_golden_cases():
    cases = [c for c in load_json("sketch_cases.json")["vectors"] if c["n"] * c["k"] <= 300_000]
    for case in cases:
        ids, w = vector_case(case)
        v = gm.WeightedVector({int(e): float(x) for e, x in zip(ids, w)})
        sk, em = gm.sketch_naive_counted(v, gm.GenerationParams(k=case["k"], scheme=gm.SeedScheme(case["seed"])))
        wy, ws = sketch_arrays(case["fast"])
        assert_regs(sk.y, np.array(sk.s, np.uint64), wy, ws, tol=0.0)
        assert em == case["n"] * case["k"]


def test_batched_golden_cases_one_launch():
    cases = load_json("sketch_cases.json")["vectors"]
    by_k = {}
    for c in cases:
        by_k.setdefault((c["k"], c["seed"]), []).append(c)
    # one launch per case group with equal (k, seed); also one mixed big batch at k=96
    for (k, seed), group in by_k.items():
        ids = np.concatenate([vector_case(c)[0] for c in group])
        w = np.concatenate([vector_case(c)[1] for c in group])
        off = np.zeros(len(group) + 1, np.int64)
        off[1:] = np.cumsum([c["n"] for c in group])
        y, s = batch_np(gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed)))
        for i, c in enumerate(group):
            assert_regs(y[i], s[i], *sketch_arrays(c["fast"]))


def test_stream_golden_cases():
    for case in load_json("sketch_cases.json")["streams"]:
        items = list(zip(case["ids"], hexs(case["w"]).tolist()))
        sk = gm.sketch_stream(items, case["k"], gm.SeedScheme(case["seed"]))
        wy, ws = sketch_arrays(case["sketch"])
        assert_regs(sk.y, np.array([int(x) & U64 for x in sk.s], np.uint64), wy, ws, tol=0.0)
        assert tuple(sk.s) == tuple(case["sketch"]["s"])  # original (possibly huge) ids come back


def test_merge_golden_cases():
    for case in load_json("sketch_cases.json")["merges"]:
        parts = [gm.GumbelMaxSketch(case["k"], tuple(p["s"]), tuple(hexs(p["y"]).tolist()), p["fingerprint"])
                 for p in case["parts"]]
        merged = gm.merge(parts)
        wy, ws = sketch_arrays(case["merged"])
        assert list(merged.y) == wy.tolist()  # merge is pure comparison: bit-exact
        assert np.array_equal(np.array(merged.s, np.uint64), ws)


def test_bench_golden():
    """test_bench.py:67-82: seed 2024, k=16 -> 9 matches, J=0.5625, c=1.76291929033662."""
    g = load_json("bench_golden.json")
    params = gm.GenerationParams(k=16, scheme=gm.SeedScheme(2024))
    sks = [gm.sketch_fast(gm.WeightedVector({e: x for e, x in vec}), params) for vec in g["vectors"]]
    sim = gm.estimate_jaccard_p(sks[0], sks[1])
    assert sim.matches == 9 and sim.value == 0.5625
    assert gm.estimate_cardinality(sks[2]).value == pytest.approx(1.76291929033662, rel=1e-12)
    for sk, want in zip(sks, g["sketches"]):
        assert_regs(sk.y, np.array(sk.s, np.uint64), *sketch_arrays(want), tol=0.0)


def test_config1_golden():
    g = load_npz("config1.npz")
    b = gm.sketch_csr(g["ids"].astype(np.uint32), g["w"], np.array([0, g["ids"].size]), int(g["k"]),
                      gm.SeedScheme(int(g["seed"])))
    y, s = batch_np(b)
    assert_regs(y[0], s[0], g["y"], g["s"])
    # and bit-identical to the reference after the exact-y finalize
    be = gm.sketch_csr(g["ids"].astype(np.uint32), g["w"], np.array([0, g["ids"].size]), int(g["k"]),
                       gm.SeedScheme(int(g["seed"])), exact_y=True)
    ye, se = batch_np(be)
    assert ye[0].tobytes() == np.asarray(g["y"], np.float64).tobytes() and np.array_equal(se[0], g["s"])
    # the grid-wide kernel agrees too
    y2, s2, _ = gm.sketch_elements(g["ids"].astype(np.uint32), g["w"], int(g["k"]), gm.SeedScheme(int(g["seed"])))
    assert_regs(y2.cpu().numpy(), s2.cpu().numpy().view(np.uint64), g["y"], g["s"])


def test_device_y_bit_exact_config2():
    """Device registers are the reference's bit for bit on all of config 2
    (device log == glibc's): sketch_csr and sketch_csr_host, no host
    finalize; the host re-derivation (exact_y=True, a diagnostic now) agrees."""
    ids, w, off, k, seed = workloads.config2()
    sc = gm.SeedScheme(seed)
    y, s = batch_np(gm.sketch_csr(ids, w, off, k, sc))
    rc, yo, so, _ = O.sketch_csr(ids.astype(np.uint64), w.astype(np.float64), off, k, seed, mode=0, threads=8)
    assert rc == 0
    assert np.array_equal(s, so) and y.tobytes() == yo.tobytes()
    yh, sh, _ = gm.sketch_csr_host(ids, w, off, k, sc)
    assert np.array_equal(sh, so) and yh.tobytes() == yo.tobytes()
    ye, se = batch_np(gm.sketch_csr(ids[:off[50]], w[:off[50]], off[:51], k, sc, exact_y=True))
    assert ye.tobytes() == yo[:50].tobytes() and np.array_equal(se, so[:50])


def test_sketch_pairs_and_many_bit_exact():
    g = load_npz("config2_sample.npz")
    vecs = [gm.WeightedVector({int(e): float(x) for e, x in zip(g["ids"][a:b], g["w"][a:b])})
            for a, b in zip(g["offsets"][:-1], g["offsets"][1:])]
    params = gm.GenerationParams(k=int(g["k"]), scheme=gm.SeedScheme(int(g["seed"])))
    for i, sk in enumerate(gm.sketch_many(vecs, params)):
        assert np.array_equal(np.array(sk.s, np.uint64), g["s"][i]) and list(sk.y) == g["y"][i].tolist()
    a, b = g["offsets"][0], g["offsets"][1]
    sk = gm.sketch_pairs(g["ids"][a:b], g["w"][a:b], int(g["k"]), gm.SeedScheme(int(g["seed"])))
    assert list(sk.y) == g["y"][0].tolist()


def test_config2_sample_golden():
    g = load_npz("config2_sample.npz")
    y, s = batch_np(gm.sketch_csr(g["ids"], g["w"], g["offsets"], int(g["k"]), gm.SeedScheme(int(g["seed"]))))
    for i in range(y.shape[0]):
        assert_regs(y[i], s[i], g["y"][i], g["s"][i])


# ---------------------------------------------------------------- full-size configs vs the oracle
def test_config2_full_vs_oracle():
    ids, w, off, k, seed = workloads.config2()
    b = gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed), counted=True)
    y, s = batch_np(b)
    rc, yo, so, _ = O.sketch_csr(ids.astype(np.uint64), w.astype(np.float64), off, k, seed, mode=0, threads=8)
    assert rc == 0
    assert_regs(y, s, yo, so)
    assert O.digest(y, s) == load_json("full_digests.json")["config2"]["digest"]
    # estimator batch: matches of pairs (2i, 2i+1)
    sa = torch.from_numpy(s[0::2].view(np.int64)).cuda()
    sb = torch.from_numpy(s[1::2].view(np.int64)).cuda()
    ba = gm.SketchBatch(k, b.y[0::2].contiguous(), sa, b.fingerprint)
    bb = gm.SketchBatch(k, b.y[1::2].contiguous(), sb, b.fingerprint)
    m = gm.estimate_jaccard_p_batch(ba, bb).cpu().numpy()
    assert m.tolist() == np.sum(so[0::2] == so[1::2], axis=1).tolist()


@pytest.mark.parametrize("k,depth", [(1024, 36.0), (1024, 44.0), (512, 36.0), (300, 30.0), (40, 12.0), (8, 3.0)])
def test_draw_log_lanes_traces_and_handovers(k, depth):
    """K1's draw-log lanes (k <= 1024): vectors of near-equal weights sized
    so that every element is walked by a lane to about `depth` steps --
    repeated draws resolved by tracing the log (frequent at small k), logs
    that fill up and hand the element to the warp walker (depths near the
    48-step capacity) -- bit for bit against the oracle."""
    rng = np.random.default_rng(k * 1000 + int(depth))
    n0 = max(2, int(k * (math.log(k) + 2.5) / depth))
    sizes = rng.integers(max(1, int(n0 * 0.8)), int(n0 * 1.2) + 2, size=48)
    off = np.zeros(sizes.size + 1, np.int64)
    off[1:] = np.cumsum(sizes)
    ids = np.concatenate([rng.choice(1 << 31, size=int(m), replace=False) + 1 for m in sizes]).astype(np.uint32)
    w = rng.uniform(0.7, 1.3, size=int(off[-1]))
    y, s = batch_np(gm.sketch_csr(ids, w, off, k, gm.SeedScheme(77)))
    rc, yo, so, _ = O.sketch_csr(ids.astype(np.uint64), w, off, k, 77, mode=0, threads=8)
    assert rc == 0
    assert_regs(y, s, yo, so)
    if k <= 512:  # one vector under many seeds (the 640-thread shape, 32-step logs)
        schemes = [gm.SeedScheme(500 + r) for r in range(12)]
        lo, hi = int(off[3]), int(off[4])
        b1 = gm.sketch_vector_seeds(ids[lo:hi], w[lo:hi], k, schemes)
        y1, s1 = batch_np(b1)
        for r in (0, 5, 11):
            rc, yo1, so1, _, _ = O.sketch_stream(ids[lo:hi].astype(np.uint64), w[lo:hi], k, 500 + r)
            assert rc == 0
            assert_regs(y1[r], s1[r], yo1, so1)


def test_config3_subset_vs_oracle():
    ids, w, off, k, seed = workloads.config3(n_vectors=3000)
    y, s = batch_np(gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed)))
    rc, yo, so, _ = O.sketch_csr(ids.astype(np.uint64), w.astype(np.float64), off, k, seed, mode=0, threads=8)
    assert rc == 0
    assert_regs(y, s, yo, so)


def test_config3_full_vs_oracle():
    """All of config 3 (1e5 vectors, 6.6e7 elements, k=512) against the oracle."""
    import os
    ids, w, off, k, seed = workloads.config3()
    y, s = batch_np(gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed)))
    rc, yo, so, _ = O.sketch_csr(ids.astype(np.uint64), w.astype(np.float64), off, k, seed, mode=0,
                                 threads=os.cpu_count() or 8)
    assert rc == 0
    assert_regs(y, s, yo, so)
    assert O.digest(y, s) == load_json("full_digests.json")["config3"]["digest"]


def test_config4_prefix_vs_oracle():
    ids, w, k, seed = workloads.config4(n_pairs=2_000_000, n_keys=10**7)
    y, s, _ = gm.sketch_elements(ids, w, k, gm.SeedScheme(seed))
    rc, yo, so, _, _ = O.sketch_stream(ids, w.astype(np.float64), k, seed)
    assert rc == 0
    assert_regs(y.cpu().numpy(), s.cpu().numpy().view(np.uint64), yo, so)


def test_elements_all_id_and_weight_widths():
    """The elements path (filter + survivor walk) for u32/u64 ids and f32/f64
    weights, vector-load and scalar paths (odd n, unaligned views), against
    the oracle's stream sketch."""
    rng = np.random.default_rng(31)
    for n, k in [(300_001, 2048), (99_999, 512)]:
        ids64 = rng.choice(1 << 40, n, replace=False).astype(np.uint64)
        w64 = rng.lognormal(0.0, 1.5, n)
        rc, yo, so, _, _ = O.sketch_stream(ids64, w64, k, 3)
        assert rc == 0
        for ids, w in [(ids64, w64), (ids64, w64.astype(np.float32))]:
            wo = w.astype(np.float64)
            rc, yo2, so2, _, _ = O.sketch_stream(ids, wo, k, 3)
            y, s, _ = gm.sketch_elements(ids, w, k, gm.SeedScheme(3))
            assert_regs(y.cpu().numpy(), s.cpu().numpy().view(np.uint64), yo2, so2)
        ids32 = (np.arange(n, dtype=np.uint64) * 2654435761 % (1 << 32)).astype(np.uint32)
        for w in (w64, w64.astype(np.float32)):
            rc, yo3, so3, _, _ = O.sketch_stream(ids32.astype(np.uint64), w.astype(np.float64), k, 3)
            d_ids = torch.from_numpy(ids32.view(np.int32)).cuda()
            d_w = torch.from_numpy(w).cuda()
            for a in (0, 1):  # offset 1: no 16-byte alignment, the scalar path
                y, s, _ = gm.sketch_elements(d_ids[a:], d_w[a:], k, gm.SeedScheme(3))
                rc, yo4, so4, _, _ = O.sketch_stream(ids32[a:].astype(np.uint64), w[a:].astype(np.float64), k, 3)
                assert_regs(y.cpu().numpy(), s.cpu().numpy().view(np.uint64), yo4, so4)


def test_config5_prefix_vs_oracle():
    n = 5_000_000
    rng = np.random.default_rng(5)
    w = rng.lognormal(0.0, 2.0, n).astype(np.float32)
    ids = np.arange(n, dtype=np.uint32)
    y, s, _ = gm.sketch_elements(ids, w, 8192, gm.SeedScheme(1))
    rc, yo, so, _, _ = O.sketch_stream(ids.astype(np.uint64), w.astype(np.float64), 8192, 1)
    assert rc == 0
    assert_regs(y.cpu().numpy(), s.cpu().numpy().view(np.uint64), yo, so)


def _full_elements_vs_oracle(cfg):
    ids, w, k, seed = workloads.config4() if cfg == 4 else workloads.config5()
    y, s, _ = gm.sketch_elements(ids, w, k, gm.SeedScheme(seed))
    y, s = y.cpu().numpy(), s.cpu().numpy().view(np.uint64)
    rc, yo, so = O.sketch_stream_chunked(ids, w, k, seed)
    assert rc == 0
    assert_regs(y, s, yo, so)
    assert y.tobytes() == yo.tobytes()
    want = load_json("full_digests.json")[f"config{cfg}"]["digest"]
    assert O.digest(yo, so) == want and O.digest(y, s) == want


def test_config4_full_vs_oracle():
    """All of config 4 (1e8 Zipf stream pairs, k=4096) against the oracle's
    sketch_stream run in contiguous chunks on all host threads and merged by
    the partition law, and against the committed oracle digest."""
    _full_elements_vs_oracle(4)


def test_config5_full_vs_oracle():
    """All of config 5 (1e9 elements, k=8192), as test_config4_full_vs_oracle."""
    _full_elements_vs_oracle(5)


def test_seeded_batch_one_vector_many_seeds():
    """Config 1's vector under R seeds in one launch (gm_sketch_csr_seeded)
    equals R separate sketches, and the oracle for a few of them."""
    ids, w, k, seed = workloads.config1()
    R = 40
    schemes = [gm.SeedScheme(1000 + r) for r in range(R)]
    off = np.arange(R + 1, dtype=np.int64) * ids.size
    b = gm.sketch_csr_seeded(np.tile(ids, R), np.tile(w, R), off, k, schemes)
    y, s = batch_np(b)
    for r in (0, 7, R - 1):
        y1, s1 = batch_np(gm.sketch_csr(ids, w, np.array([0, ids.size]), k, schemes[r]))
        assert y1.tobytes() == y[r:r + 1].tobytes() and np.array_equal(s1[0], s[r])
        rc, yo, so, _, _ = O.sketch_stream(ids.astype(np.uint64), w, k, 1000 + r)
        assert rc == 0
        assert_regs(y[r], s[r], yo, so)
    sks = b.to_sketches()
    assert [sk.fingerprint for sk in sks] == [sc.fingerprint for sc in schemes]
    # the vector stored once (GM_FLAG_ONE_VECTOR): the same R sketches
    b1 = gm.sketch_vector_seeds(ids, w, k, schemes)
    assert torch.equal(b1.y, b.y) and torch.equal(b1.s, b.s)


@pytest.mark.parametrize("n", [4096, 10_000, 300_000])
def test_single_vector_runs_grid_wide(n):
    """One vector of >= 4096 elements through the host entry (sketch_fast,
    sketch_csr_host) runs on the grid-wide kernels; the registers are the
    oracle's and the batched single-CTA kernel's."""
    rng = np.random.default_rng(n)
    ids = rng.choice(1 << 31, n, replace=False).astype(np.uint32) + 1
    w = rng.exponential(1.0, n) + 1e-3
    k = 256 if n < 100_000 else 2048
    sc = gm.SeedScheme(n)
    yh, sh, em = gm.sketch_csr_host(ids, w, np.array([0, n]), k, sc, counted=True)
    yd, sd = batch_np(gm.sketch_csr(ids, w, np.array([0, n]), k, sc))
    assert yh.tobytes() == yd.tobytes() and np.array_equal(sh, sd)
    order = np.argsort(ids)
    rc, yo, so, _ = O.sketch_fast(ids[order].astype(np.uint64), w[order], k, n)
    assert rc == 0
    assert_regs(yh[0], sh[0], yo, so)
    v = gm.WeightedVector(dict(zip(ids.tolist(), w.tolist())))
    sk = gm.sketch_fast(v, gm.GenerationParams(k=k, scheme=sc))
    assert list(sk.y) == yo.tolist() and np.array_equal(np.array(sk.s, np.uint64), so)


# ---------------------------------------------------------------- size-independent properties at full size
def test_partition_law_large():
    """sketch(whole) == merge(sketch(part) for parts) on 2**26 elements (k=8192)."""
    n = 1 << 26
    rng = np.random.default_rng(55)
    w = torch.from_numpy(rng.lognormal(0.0, 2.0, n).astype(np.float32)).cuda()
    ids = torch.arange(n, dtype=torch.int32, device="cuda")
    sc = gm.SeedScheme(1)
    yw, sw, _ = gm.sketch_elements(ids, w, 8192, sc)
    parts = [gm.sketch_elements(ids[a:b], w[a:b], 8192, sc)[:2] for a, b in
             [(0, n // 3), (n // 3, n // 2), (n // 2, n)]]
    ym, sm = gm.merge_arrays(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]))
    assert torch.equal(sm, sw)
    assert torch.equal(ym, yw)  # same arrivals, same arithmetic: bit-identical
    # idempotence and duplicates: the whole set twice is the same sketch
    y2, s2, _ = gm.sketch_elements(torch.cat([ids, ids[: n // 4]]), torch.cat([w, w[: n // 4]]), 8192, sc)
    assert torch.equal(s2, sw) and torch.equal(y2, yw)


def test_csr_vs_elements_kernels_agree():
    ids, w, off, k, seed = workloads.config3(n_vectors=200)
    y, s = batch_np(gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed)))
    for v in range(0, 200, 37):
        a, b = off[v], off[v + 1]
        y2, s2, _ = gm.sketch_elements(ids[a:b], w[a:b], k, gm.SeedScheme(seed))
        assert_regs(y2.cpu().numpy(), s2.cpu().numpy().view(np.uint64), y[v], s[v], tol=0.0)


def test_host_api_matches_device_api():
    """gm_sketch_csr_host (pinned zero-copy or pageable outputs) returns the
    device path's registers bit for bit and reports data errors with the
    batch's vector indices."""
    ids, w, off, k, seed = workloads.config2()
    sc = gm.SeedScheme(seed)
    d = gm.sketch_csr(ids, w, off, k, sc, counted=True)
    y, s, em = gm.sketch_csr_host(ids, w, off, k, sc, counted=True)
    assert np.array_equal(s, d.s.cpu().numpy().view(np.uint64)) and np.array_equal(y, d.y.cpu().numpy())
    assert em.tolist() == d.emitted.cpu().tolist()
    n_vec = len(off) - 1
    yp = torch.empty((n_vec, k), dtype=torch.float64).pin_memory()
    sp = torch.empty((n_vec, k), dtype=torch.int64).pin_memory()
    gm.sketch_csr_host(torch.from_numpy(ids).pin_memory(), torch.from_numpy(w).pin_memory(),
                       torch.from_numpy(off), k, sc, out=(yp, sp))
    assert torch.equal(sp, d.s.cpu()) and torch.equal(yp, d.y.cpu())
    bad = off.copy()
    bad[900] = bad[899]  # vector 899 empty
    with pytest.raises(gm.EmptyVectorError, match="vector 899"):
        gm.sketch_csr_host(ids, w, bad, k, sc)
    y2, s2, _ = gm.sketch_csr_host(ids, w, off, k, sc)  # the error does not stick
    assert np.array_equal(s2, s)
    # compact 32-bit s (GM_FLAG_S32), pageable and page-locked outputs
    y3, s3, _ = gm.sketch_csr_host(ids, w, off, k, sc, s32=True)
    assert s3.dtype == np.uint32 and np.array_equal(s3.astype(np.uint64), s) and np.array_equal(y3, y)
    sp32 = torch.empty((n_vec, k), dtype=torch.int32).pin_memory()
    gm.sketch_csr_host(ids, w, off, k, sc, out=(yp, sp32), s32=True)
    assert np.array_equal(sp32.numpy().view(np.uint32).astype(np.uint64), s) and torch.equal(yp, d.y.cpu())


def test_batches_pipelined_over_streams():
    """GM_FLAG_ASYNC calls on alternating streams (the bench's stream of
    batches), device and host entry points: every batch equals the
    synchronous result."""
    ids, w, off, k, seed = workloads.config2(n_vectors=300)
    sc = gm.SeedScheme(seed)
    ref = gm.sketch_csr(ids, w, off, k, sc)
    L = gm._lib.load()
    streams = [torch.cuda.Stream() for _ in range(3)]
    n_vec = len(off) - 1
    d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
    d_w, d_off = torch.from_numpy(w).cuda(), torch.from_numpy(off).cuda()
    ys = [torch.empty((n_vec, k), dtype=torch.float64, device="cuda") for _ in range(6)]
    ss = [torch.empty((n_vec, k), dtype=torch.int64, device="cuda") for _ in range(6)]
    h_ids = torch.from_numpy(ids.view(np.int32)).pin_memory()
    h_w, h_off = torch.from_numpy(w).pin_memory(), torch.from_numpy(off).pin_memory()
    hy = [torch.empty((n_vec, k), dtype=torch.float64).pin_memory() for _ in range(6)]
    hs = [torch.empty((n_vec, k), dtype=torch.int64).pin_memory() for _ in range(6)]
    torch.cuda.synchronize()
    for i in range(6):
        st = streams[i % 3].cuda_stream
        assert L.gm_sketch_csr(d_ids.data_ptr(), 32, d_w.data_ptr(), 32, d_off.data_ptr(), n_vec, k, sc.global_seed,
                               sc.stream_salt, gm._lib.GM_FLAG_ASYNC, ys[i].data_ptr(), ss[i].data_ptr(), 0, st) == 0
        assert L.gm_sketch_csr_host(h_ids.data_ptr(), 32, h_w.data_ptr(), 32, h_off.data_ptr(), n_vec, k,
                                    sc.global_seed, sc.stream_salt, gm._lib.GM_FLAG_ASYNC, hy[i].data_ptr(),
                                    hs[i].data_ptr(), 0, st) == 0
    torch.cuda.synchronize()
    for st in streams:
        assert L.gm_stream_status(st.cuda_stream) == 0
    for i in range(6):
        assert torch.equal(ss[i], ref.s) and torch.equal(ys[i], ref.y)
        assert torch.equal(hs[i], ref.s.cpu()) and torch.equal(hy[i], ref.y.cpu())


def test_host_batches_stream_api():
    """sketch_csr_host_many: a stream of host batches over several CUDA
    streams returns every batch's registers, in order, equal to sketch_csr."""
    ids, w, off, k, seed = workloads.config2(n_vectors=200)
    sc = gm.SeedScheme(seed)
    ref = gm.sketch_csr(ids, w, off, k, sc)
    parts = [(0, 50), (50, 120), (120, 200)] * 3
    batches = [(ids[off[a]:off[b]], w[off[a]:off[b]], off[a:b + 1] - off[a]) for a, b in parts]
    got = [(y.clone(), s.clone()) for y, s in gm.sketch_csr_host_many(iter(batches), k, sc, streams=4)]
    assert len(got) == len(parts)
    for (a, b), (y, s) in zip(parts, got):
        assert torch.equal(s, ref.s[a:b].cpu()) and torch.equal(y, ref.y[a:b].cpu())
    # a result stays valid while `streams` more are taken (no clone)
    held = []
    for n, (y, s) in enumerate(gm.sketch_csr_host_many(iter(batches), k, sc, streams=3)):
        held.append((parts[n], y, s))
        if len(held) > 3:
            (a, b), y0, s0 = held.pop(0)
            assert torch.equal(s0, ref.s[a:b].cpu()) and torch.equal(y0, ref.y[a:b].cpu())
    got32 = [s.clone() for _, s in gm.sketch_csr_host_many(iter(batches[:3]), k, sc, streams=2, s32=True)]
    for (a, b), s in zip(parts[:3], got32):
        assert torch.equal(s.to(torch.int64) & 0xFFFFFFFF, ref.s[a:b].cpu())


# ---------------------------------------------------------------- edge cases
def test_single_element_owns_every_register():
    for k in (1, 3, 64, 1024, 4096):
        v = gm.WeightedVector({5: 1.0})
        sk = gm.sketch_fast(v, gm.GenerationParams(k=k, scheme=gm.SeedScheme(77)))
        assert set(sk.s) == {5}
        t, srv = O.run_queue_full(77, O.DEFAULT_STREAM_SALT, 5, 1.0, k)
        want = np.empty(k)
        want[srv - 1] = t
        assert_regs(sk.y, np.array(sk.s, np.uint64), want, np.full(k, 5, np.uint64))


def test_heavy_and_tiny_weights():
    rng = np.random.default_rng(3)
    for n, k in [(3, 512), (20, 2048), (50, 8192), (400, 65536)]:
        ids = rng.choice(10**9, n, replace=False).astype(np.uint64) + 1
        w = np.exp(rng.normal(0, 6, n))
        w[0] = 1e-300
        w[-1] = 1e300 / n
        rc, yo, so, _ = O.sketch_fast(np.sort(ids), w[np.argsort(ids)], k, 9)
        y, s = batch_np(gm.sketch_csr(ids, w, np.array([0, n]), k, gm.SeedScheme(9)))
        assert_regs(y[0], s[0], yo, so)


def test_u64_ids_and_zero():
    ids = np.array([0, 1, (1 << 64) - 1, 1 << 63, 12345678901234567], dtype=np.uint64)
    w = np.array([0.5, 1.5, 2.0, 0.25, 1.0])
    order = np.argsort(ids)
    rc, yo, so, _ = O.sketch_fast(ids[order], w[order], 97, 3)
    y, s = batch_np(gm.sketch_csr(ids, w, np.array([0, 5]), 97, gm.SeedScheme(3)))
    assert_regs(y[0], s[0], yo, so)


def test_exhaustive_equals_fast_and_counts():
    ids, w, off, k, seed = workloads.config2(n_vectors=16)
    sc = gm.SeedScheme(seed)
    bf = gm.sketch_csr(ids, w, off, k, sc, counted=True)
    bn = gm.sketch_csr(ids, w, off, k, sc, exhaustive=True, counted=True)
    assert torch.equal(bf.s, bn.s) and torch.equal(bf.y, bn.y)
    assert bn.emitted.cpu().numpy().tolist() == (np.diff(off) * k).tolist()
    assert int(bf.emitted.sum()) < int(bn.emitted.sum()) / 20


def test_errors_map_to_reference_classes():
    sc = gm.SeedScheme(1)
    with pytest.raises(gm.InvalidWeightError):
        gm.sketch_csr(np.array([1, 2], np.uint32), np.array([1.0, -1.0]), np.array([0, 2]), 8, sc)
    with pytest.raises(gm.InvalidWeightError):
        gm.sketch_csr(np.array([1, 2], np.uint32), np.array([1.0, math.nan]), np.array([0, 2]), 8, sc)
    with pytest.raises(gm.EmptyVectorError):
        gm.sketch_csr(np.array([1, 2], np.uint32), np.array([1.0, 1.0]), np.array([0, 2, 2]), 8, sc)
    with pytest.raises(gm.InvalidParameterError):
        gm.sketch_csr(np.array([1], np.uint32), np.array([1.0]), np.array([0, 1]), (1 << 24) + 1, sc)
    with pytest.raises(gm.EmptyVectorError):
        gm.sketch_fast(gm.WeightedVector({}), gm.GenerationParams(k=4, scheme=sc))
    with pytest.raises(gm.InconsistentWeightError):
        gm.sketch_pairs(np.array([1, 2, 1], np.uint64), np.array([0.5, 1.0, 0.75]), 4, sc)
    with pytest.raises(gm.InvalidWeightError):
        gm.sketch_elements(np.array([1, 2], np.uint32), np.array([1.0, 0.0]), 8, sc)
    with pytest.raises(gm.MismatchedSketchError):
        gm.merge([])
    with pytest.raises(gm.InvalidParameterError):  # 32-bit s for 64-bit ids
        gm.sketch_csr_host(np.array([1 << 40], np.uint64), np.array([1.0]), np.array([0, 1]), 8, sc, s32=True)
    with pytest.raises(gm.InvalidParameterError):
        gm.estimate_cardinality_batch(gm.sketch_csr(np.array([1], np.uint32), np.array([1.0]), np.array([0, 1]), 1, sc))
    # the library recovers after a data error
    sk = gm.sketch_fast(gm.WeightedVector({1: 1.0}), gm.GenerationParams(k=4, scheme=sc))
    assert sk.s == (1, 1, 1, 1)


def test_device_register_sum_is_fsum():
    """gm_cardinality: exactly rounded sums (math.fsum) and (k-1)/sum."""
    rng = np.random.default_rng(21)
    rows = [rng.exponential(1e-3, 1024),
            np.exp(rng.uniform(-700, 700, 1024)),                  # 600 decades in one sum
            np.concatenate([[1.0], np.full(1023, 2.0**-60)]),      # ties and sticky bits
            np.concatenate([[2.0**53], np.ones(1023)]),
            np.full(1024, 5e-324),                                 # subnormals
            np.zeros(1024),
            rng.random(1024) * np.where(rng.random(1024) < 0.5, 1e-200, 1e200)]
    y = torch.from_numpy(np.stack(rows)).cuda()
    sums = torch.empty(len(rows), dtype=torch.float64, device="cuda")
    card = torch.empty_like(sums)
    assert gm._lib.load().gm_cardinality(y.data_ptr(), len(rows), 1024, sums.data_ptr(), card.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream) == 0
    got = sums.cpu().tolist()
    for r, g in zip(rows, got):
        assert g == math.fsum(r.tolist())
    ids, w, off, k, seed = workloads.config2(n_vectors=64)
    b = gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed))
    c = gm.estimate_cardinality_batch(b).cpu().tolist()
    assert c == [gm.estimate_cardinality(sk).value for sk in b.to_sketches()]


def _first_offenders(ids, w):
    """stream_update's rules, item by item (stream.py:58-78)."""
    seen = {}
    bad = conf = -1
    for i, (e, x) in enumerate(zip(ids.tolist(), w.tolist())):
        if bad < 0 and not (math.isfinite(x) and x > 0 and x >= 1e-300):
            bad = i
        if e in seen:
            if conf < 0 and seen[e] != x:
                conf = i
        else:
            seen[e] = x
    return bad, conf, seen


def test_device_stream_checks_match_item_by_item_rules():
    rng = np.random.default_rng(11)
    for trial in range(6):
        n = 20000
        ids = rng.integers(0, 3000, n).astype(np.uint64)
        ids[::997] = U64  # the table's empty-key value is a legal id
        key_w = rng.exponential(1.0, 3000) + 0.01
        w = np.where(ids == U64, 2.5, key_w[np.minimum(ids, 2999).astype(np.int64)])
        if trial % 3 == 1:
            w[rng.integers(100, n)] *= 1.5  # an inconsistent reappearance (or a first occurrence)
        if trial % 3 == 2:
            w[rng.integers(100, n)] = -1.0
        bad, conf, seen = _first_offenders(ids, w)
        dev_ids = torch.from_numpy(ids.view(np.int64)).cuda()
        dev_w = torch.from_numpy(w).cuda()
        ui, uw = torch.empty_like(dev_ids), torch.empty_like(dev_w)
        out = np.zeros(3, np.int64)
        rc = gm._lib.load().gm_check_pairs(dev_ids.data_ptr(), 64, dev_w.data_ptr(), 64, n, out[0:].ctypes.data,
                                           out[1:].ctypes.data, ui.data_ptr(), uw.data_ptr(), out[2:].ctypes.data,
                                           torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        assert (int(out[0]), int(out[1])) == (bad, conf)
        got = dict(zip(ui[: out[2]].cpu().numpy().view(np.uint64).tolist(), uw[: out[2]].cpu().tolist()))
        assert got == seen  # first occurrences, with their weights


def test_sketch_pairs_config4_prefix_bit_exact():
    ids, w, k, seed = workloads.config4(n_pairs=1_000_000, n_keys=10**6)
    sk = gm.sketch_pairs(ids, w, k, gm.SeedScheme(seed))
    rc, yo, so, _, _ = O.sketch_stream(ids, w.astype(np.float64), k, seed)
    assert rc == 0
    assert np.array_equal(np.array(sk.s, np.uint64), so) and list(sk.y) == yo.tolist()
    _, first_idx, inv = np.unique(ids, return_index=True, return_inverse=True)
    rep = np.nonzero(first_idx[inv] < np.arange(ids.size))[0]
    i = int(rep[len(rep) // 2])
    bad = w.copy()
    bad[i] *= 2  # a repeated id comes back with another weight
    with pytest.raises(gm.InconsistentWeightError, match=f"item {i}:"):
        gm.sketch_pairs(ids, bad, k, gm.SeedScheme(seed))


def test_stream_state_api():
    sc = gm.SeedScheme(77)
    st = gm.StreamSketchState(2, sc)
    gm.stream_update(st, (4, 1.5))
    assert st.unset_count == 0 and st.prune_enabled
    assert gm.stream_finalize(st).s == (4, 4)
    st = gm.StreamSketchState(3, sc)
    with pytest.raises(gm.IncompleteSketchError) as ei:
        gm.stream_finalize(st)
    assert ei.value.unset_registers == [0, 1, 2]
    st = gm.StreamSketchState(4, sc)
    gm.stream_update(st, (1, 0.5))
    with pytest.raises(gm.InconsistentWeightError):
        gm.stream_update(st, (1, 0.75))


@pytest.mark.parametrize("seed", [3, 11, 29])
def test_accumulate_light_then_heavy_flush(seed):
    """a stream whose first flush holds a few light items
    and whose next flush holds many heavy ones.  The second flush's tau comes
    from the heavy items alone and lies far below the light registers; every
    register above it must stay open until the heavy arrivals below it are
    folded in.  Compared with the oracle's one-item-at-a-time stream."""
    rng = np.random.default_rng(seed)
    k = 512
    light = rng.choice(1 << 40, 40, replace=False).astype(np.uint64) + 1
    heavy = rng.choice(1 << 40, 70_000, replace=False).astype(np.uint64) + (1 << 41)
    wl = rng.uniform(1e-4, 1e-3, light.size)
    wh = rng.uniform(10.0, 100.0, heavy.size)
    st = gm.StreamSketchState(k, gm.SeedScheme(seed))
    for e, x in zip(light.tolist(), wl.tolist()):
        gm.stream_update(st, (e, x))
    assert st.unset_count >= 0  # observing the state flushes the light items alone
    for e, x in zip(heavy.tolist(), wh.tolist()):
        gm.stream_update(st, (e, x))
    sk = gm.stream_finalize(st)
    ids = np.concatenate([light, heavy])
    w = np.concatenate([wl, wh])
    rc, yo, so, _, _ = O.sketch_stream(ids, w, k, seed)
    assert rc == 0
    assert_regs(sk.y, np.array(sk.s, np.uint64), yo, so)
    # and the device call directly: a complete light sketch, heavy items folded in
    y, s, _ = gm.sketch_elements(light, wl, 64, gm.SeedScheme(seed), exhaustive=True)
    gm.sketch_elements(heavy, wh, 64, gm.SeedScheme(seed), into=(y, s))
    rc, yo, so, _, _ = O.sketch_stream(ids, w, 64, seed)
    assert_regs(y.cpu().numpy(), s.cpu().numpy().view(np.uint64), yo, so)


def test_nccl_exchange_world1():
    """The C ABI's NCCL register exchange (gm_comm.cuh) on one rank: both
    protocols leave a sketch unchanged; the communicator is created and
    destroyed through the C ABI (the N > 1 protocol is covered on CPU by
    tests/test_multirank_gloo.py)."""
    import ctypes
    from paper_2302_05176_b200 import _device, _lib
    L = _lib.load()
    uid = (ctypes.c_char * L.gm_comm_id_bytes())()
    _device.call("gm_comm_unique_id", ctypes.addressof(uid))
    comm = ctypes.c_void_p()
    _device.call("gm_comm_init", ctypes.addressof(uid), 1, 0, ctypes.byref(comm))
    ids, w, k, seed = workloads.config4(n_pairs=300_000, n_keys=10**5)
    y, s, _ = gm.sketch_elements(ids, w, 512, gm.SeedScheme(seed))
    for fn in ("gm_allreduce_min_registers", "gm_allgather_merge_registers"):
        y2, s2 = y.clone(), s.clone()
        _device.call(fn, comm, y2.data_ptr(), s2.data_ptr(), 512, _device.stream_ptr())
        torch.cuda.synchronize()
        assert torch.equal(y2, y) and torch.equal(s2, s)
    _device.call("gm_comm_destroy", comm)


def test_workspace_lifecycle():
    """Scratch is per (device, stream); gm_release_stream frees one set and
    gm_finalize all of them; calls after either re-create what they need."""
    from paper_2302_05176_b200 import _device, _lib
    L = _lib.load()
    st = torch.cuda.Stream()
    ids, w, off, k, seed = workloads.config2(n_vectors=8)
    with torch.cuda.stream(st):
        a = gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed))
    n0 = L.gm_workspace_count()
    assert n0 >= 1
    _device.call("gm_release_stream", st.cuda_stream)
    assert L.gm_workspace_count() == n0 - 1
    _device.call("gm_finalize")
    assert L.gm_workspace_count() == 0
    b = gm.sketch_csr(ids, w, off, k, gm.SeedScheme(seed))
    assert torch.equal(a.y, b.y) and torch.equal(a.s, b.s)


def test_rand_int_between_any_range():
    """rand_int_between over ranges beyond 2**16, up to 2**64 (randgen.py:122-143)."""
    sc = gm.SeedScheme(5)
    for lo, hi, e, z in [(0, (1 << 20) - 1, 3, 1), (10, 10 + (1 << 40), 7, 9), (0, (1 << 64) - 1, 11, 2),
                         (-5, 5, -1, 3), (1, (1 << 63) + 12345, 1 << 70, 1 << 65)]:
        # the oracle draws the offset in [0, m) (m = 2**64 wraps in its u64 arithmetic: checked by range only)
        want = lo + O.rand_int_between(sc.perm_seed, e & U64, z & U64, 0, hi - lo) if hi - lo < U64 else None
        got = gm.rand_int_between(sc, e, z, lo, hi)
        assert lo <= got <= hi
        if want is not None:
            assert got == want


def test_service_exchanges_byte_identical():
    """The reference service's sketch and estimator routes (service/app.py:74-118)
    served by the CUDA engine (paper_2302_05176_b200.service): every recorded
    exchange of the reference's own app (tests/golden/make_service_golden.py)
    -- vector sketches (fast, naive, salted, a 5,000-entry vector that runs
    grid-wide), stream sketches, merges, estimators and the 400 errors --
    gives the same status and the same response bytes."""
    from fastapi.testclient import TestClient

    from paper_2302_05176_b200.service import create_app
    client = TestClient(create_app())
    for ex in load_json("service_exchanges.json"):
        r = client.get(ex["path"]) if ex["method"] == "GET" else client.post(ex["path"], json=ex["request"])
        assert r.status_code == ex["status"], (ex["path"], r.text[:200])
        assert r.text == ex["body"], (ex["path"], r.text[:200], ex["body"][:200])


def test_element_queue_state_on_device_matches_reference_queues():
    """ElementQueueState / next_order_statistic on the device (gm_queue_advance_batch)
    against the reference's full queues (tests/golden/rng_kats.json): bit-identical
    times and servers; QueueExhaustedError after k.  And advance_queues over many
    queues at once against the oracle's _run_queue."""
    for q in load_json("rng_kats.json")["queues"]:
        sc = gm.SeedScheme(q["seed"])
        st = gm.ElementQueueState(q["element"], float.fromhex(q["weight"]) if isinstance(q["weight"], str)
                                  else q["weight"], q["k"])
        got = [gm.next_order_statistic(st, sc) for _ in range(q["k"])]
        assert [t for t, _ in got] == hexs(q["times"]).tolist()
        assert [s for _, s in got] == list(q["servers"])
        assert st.exhausted and sorted(st.perm.tolist()) == list(range(1, q["k"] + 1))
        with pytest.raises(gm.QueueExhaustedError):
            gm.next_order_statistic(st, sc)
    sc = gm.SeedScheme(17)
    k = 300
    states = [gm.ElementQueueState(e, 0.1 + e / 7.0, k) for e in range(1, 65)]
    t1, s1 = gm.advance_queues(states, sc, 100)
    t2, s2 = gm.advance_queues(states, sc, 200)
    t, s = np.concatenate([t1, t2], axis=1), np.concatenate([s1, s2], axis=1)
    for i, e in enumerate(range(1, 65)):
        to, so = O.run_queue_full(17, sc.stream_salt, e, 0.1 + e / 7.0, k)
        assert t[i].tobytes() == to.tobytes() and s[i].tolist() == so.tolist()


@pytest.mark.parametrize("k", [65537, 100_003, 262_144])
def test_k_beyond_65536(k):
    """k > 65536 (the reference accepts any k, sketch.py:139-157): the grid-wide
    kernels with 64-bit Fisher-Yates words and exact 64-bit draws, through the
    batch, drop-in, naive and stream entry points, against the oracle."""
    rng = np.random.default_rng(k)
    n = 3000
    ids = rng.choice(1 << 40, n, replace=False).astype(np.uint64) + 1
    w = rng.exponential(1.0, n) + 0.01
    sc = gm.SeedScheme(k % 97)
    order = np.argsort(ids)
    rc, yo, so, _ = O.sketch_fast(ids[order], w[order], k, k % 97)
    assert rc == 0
    b = gm.sketch_csr(ids, w, np.array([0, n]), k, sc)
    assert_regs(b.y.cpu().numpy()[0], b.s.cpu().numpy().view(np.uint64)[0], yo, so)
    if k < 200_000:
        v = gm.WeightedVector(dict(zip(ids[:200].tolist(), w[:200].tolist())))
        sk = gm.sketch_fast(v, gm.GenerationParams(k=k, scheme=sc))
        o2 = np.argsort(ids[:200])
        rc, y2, s2, _ = O.sketch_fast(ids[:200][o2], w[:200][o2], k, k % 97)
        assert list(sk.y) == y2.tolist() and np.array_equal(np.array(sk.s, np.uint64), s2)
        small = gm.WeightedVector({int(e): float(x) for e, x in zip(ids[:3], w[:3])})
        nk, em = gm.sketch_naive_counted(small, gm.GenerationParams(k=k, scheme=sc))
        rc, y3, s3, _ = O.sketch_naive(np.sort(ids[:3]), w[:3][np.argsort(ids[:3])], k, k % 97)
        assert list(nk.y) == y3.tolist() and np.array_equal(np.array(nk.s, np.uint64), s3) and em == 3 * k
    rep = np.concatenate([ids, ids[:500]])
    wr = np.concatenate([w, w[:500]])
    y4, s4, _ = gm.sketch_elements(rep, wr, k, sc)
    rc, y5, s5, _, _ = O.sketch_stream(rep, wr, k, k % 97)
    assert rc == 0
    assert_regs(y4.cpu().numpy(), s4.cpu().numpy().view(np.uint64), y5, s5)


# ---------------------------------------------------------------- arithmetic
def test_branch_free_divide_equals_ieee_divide():
    """ddiv_fast (the lane walkers' divide) == __ddiv_rn on its weight range."""
    from paper_2302_05176_b200 import _device
    counts = torch.zeros(2, dtype=torch.int64, device="cuda")
    _device.call("gm_arith_check", 50_000_000, 0x5EED, counts.data_ptr(), _device.stream_ptr())
    bad_div, bad_log = counts.tolist()
    assert bad_div == 0, f"{bad_div} divides differ from IEEE"
    assert bad_log == 0, f"{bad_log} logs more than 1 ulp from CUDA's"


def test_device_log_is_glibc_log():
    """The device log (gm_glibc_log.cuh) == glibc's log (math.log in the
    reference) bit for bit: 1e8 keyed uniforms of the sketch's own formula,
    plus uniforms with few significant bits, the near-1 interval and its
    edges."""
    from paper_2302_05176_b200 import _device
    chunk = 20_000_000
    x = torch.empty(chunk, dtype=torch.float64, device="cuda")
    out = torch.empty_like(x)
    for c in range(5):
        u, want = O.log_uniforms(0xC0FFEE, c * chunk, chunk)
        x.copy_(torch.from_numpy(u))
        _device.call("gm_log_batch", x.data_ptr(), chunk, out.data_ptr(), _device.stream_ptr())
        got = out.cpu().numpy()
        bad = np.nonzero(got.view(np.int64) != want.view(np.int64))[0]
        assert bad.size == 0, f"chunk {c}: {bad.size} logs differ, first u={u[bad[0]].hex()}"
    rng = np.random.default_rng(21)
    v = rng.integers(0, 1 << 53, 400_000, dtype=np.uint64) >> rng.integers(0, 53, 400_000).astype(np.uint64)
    u = v.astype(np.float64) * 2.0**-53 + 2.0**-54
    near = 0.93 + rng.random(400_000) * 0.14
    edges = np.array([1.0, 1 - 2.0**-53, 0.5, 2.0**-54, 0.6875, 1.375, 1 - 2.0**-9, 1 - 2.0**-4,
                      np.nextafter(1 - 2.0**-4, 0), 1 + 0x109 * 2.0**-12, np.nextafter(1 + 0x109 * 2.0**-12, 0)])
    u = np.concatenate([u, near, edges])
    x = torch.from_numpy(u).cuda()
    out = torch.empty_like(x)
    _device.call("gm_log_batch", x.data_ptr(), x.numel(), out.data_ptr(), _device.stream_ptr())
    got = out.cpu().numpy()
    want = np.array([math.log(a) for a in u])
    assert got.tobytes() == want.tobytes()


_SCHEDULE_SCRIPT = r"""
import sys, json
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2302_05176_b200 as gm
from paper_2302_05176_b200 import workloads
ids, w, k, seed = workloads.config4(n_pairs=2_000_000, n_keys=10**7)
rng = np.random.default_rng(5)
w5 = rng.lognormal(0.0, 2.0, 3_000_000).astype(np.float32)
ids5 = np.arange(w5.size, dtype=np.uint32)
out = {}
for name, (i, ww, kk) in {"c4": (ids, w, k), "c5": (ids5, w5, 8192)}.items():
    y, s, em = gm.sketch_elements(i, ww, kk, gm.SeedScheme(seed))
    out[name] = [y.cpu().numpy().tobytes().hex(), s.cpu().numpy().tobytes().hex()]
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [
    {},                                                  # default schedule
    {"GM_ELEM_TAU_SCALE": "0.25"},                       # first walk fails, the list is re-walked / rebuilt
    {"GM_ELEM_TAU_SCALE": "0.25", "GM_ELEM_R": "1.0"},   # list bound = tau: every failed pass streams again
    {"GM_ELEM_TAU_SCALE": "0.5", "GM_ELEM_R": "64"},     # a wide list, several re-walks of it
    {"GM_ELEM_FUSED": "1"},                              # fused light kernel only (overflow fallback path)
])
def test_elements_schedules_agree_with_oracle(env):
    """Every K2 schedule -- first walk at tau or at the list bound, re-walks
    of the survivor list, streaming the input again, the fused kernel --
    gives the oracle's sketch bit for bit (s) on a config-4 Zipf prefix and a
    config-5 prefix.  The knobs are read once per process, hence the
    subprocess."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _SCHEDULE_SCRIPT, root], capture_output=True, text=True,
                         env={**os.environ, **env}, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    ids, w, k, seed = workloads.config4(n_pairs=2_000_000, n_keys=10**7)
    rng = np.random.default_rng(5)
    w5 = rng.lognormal(0.0, 2.0, 3_000_000).astype(np.float32)
    ids5 = np.arange(w5.size, dtype=np.uint64)
    for name, (i, ww, kk) in {"c4": (ids, w, k), "c5": (ids5, w5, 8192)}.items():
        y = np.frombuffer(bytes.fromhex(out[name][0]), np.float64)
        s = np.frombuffer(bytes.fromhex(out[name][1]), np.uint64)
        rc, yo, so, _, _ = O.sketch_stream(i, ww.astype(np.float64), kk, seed)
        assert rc == 0
        assert_regs(y, s, yo, so)


def test_device_sketches_serialise_to_reference_records():
    """End to end through the wire format: sketch_fast on the device (exact-y
    finalize) and merge, serialised with sketch_to_json, give byte-for-byte the
    records the reference wrote for the same inputs (tests/golden/wire_records.json),
    so device-built sketches interoperate with the reference's CLI and service files."""
    cases = load_json("sketch_cases.json")["vectors"]
    for rec in load_json("wire_records.json"):
        if "case" in rec:
            c = cases[rec["case"]]
            ids, w = vector_case(c)
            v = gm.WeightedVector({int(e): float(x) for e, x in zip(ids, w)})
            sk = gm.sketch_fast(v, gm.GenerationParams(k=c["k"], scheme=gm.SeedScheme(c["seed"])))
        else:
            m = rec["merge"]
            p = gm.GenerationParams(k=m["k"], scheme=gm.SeedScheme(m["seed"]))
            a = gm.WeightedVector({e: float.fromhex(x) for e, x in m["a"]})
            b = gm.WeightedVector({e: float.fromhex(x) for e, x in m["b"]})
            sk = gm.merge([gm.sketch_fast(a, p), gm.sketch_fast(b, p)])
        assert gm.sketch_to_json(sk) == rec["record"]


def test_empty_element_set_is_incomplete():
    """No elements leave every register unset: IncompleteSketchError, as
    stream_finalize raises for an empty stream (stream.py:132-134); folded
    into an existing complete sketch (accumulate) an empty set is a no-op."""
    with pytest.raises(gm.IncompleteSketchError):
        gm.sketch_elements(np.zeros(0, np.uint32), np.zeros(0, np.float32), 64, gm.SeedScheme(1))
    y, s, _ = gm.sketch_elements(np.arange(1, 500, dtype=np.uint32), np.ones(499, np.float32), 64, gm.SeedScheme(1))
    y2, s2 = y.clone(), s.clone()
    gm.sketch_elements(np.zeros(0, np.uint32), np.zeros(0, np.float32), 64, gm.SeedScheme(1), into=(y2, s2))
    assert torch.equal(y, y2) and torch.equal(s, s2)


@pytest.mark.parametrize("bad", [0.0, -1.0, float("nan"), float("inf"), -0.0])
@pytest.mark.parametrize("id_dtype", [np.uint32, np.uint64])
def test_elements_bad_weight_anywhere_raises(bad, id_dtype):
    """A weight that is not finite and > 0 anywhere in a large element set
    (the vectorised filter path, where u32-id weights are validated only on
    elements the filter keeps) raises InvalidWeightError (stream.py:63-66)."""
    n = 1 << 20
    rng = np.random.default_rng(17)
    w = rng.exponential(1.0, n).astype(np.float32) + np.float32(1e-3)
    ids = np.arange(n, dtype=id_dtype) * 7 + 1
    w[654_321] = np.float32(bad)
    with pytest.raises(gm.InvalidWeightError):
        gm.sketch_elements(ids, w, 1024, gm.SeedScheme(3))


@pytest.mark.parametrize("n,k,nd", [(200_000, 4096, 50), (500_000, 8192, 2000), (100_000, 64, 100_000),
                                    (300_000, 4096, 300)])
def test_elements_streams_where_nearly_everything_is_kept(n, k, nd):
    """K2 filter with few distinct heavy keys (every occurrence passes the
    first-arrival test): whole warps keep all eight of their elements in one
    iteration, more than the per-warp staging area holds -- the grouped
    staging path -- and streams of all-distinct ids with k small."""
    rng = np.random.default_rng(n + k)
    keys = rng.choice(1 << 62, size=nd, replace=False).astype(np.uint64) + np.uint64(1)
    kw = rng.uniform(0.5, 2.0, size=nd).astype(np.float32)
    idx = rng.integers(0, nd, size=n)
    ids, w = keys[idx], kw[idx]
    y, s, _ = gm.sketch_elements(ids, w, k, gm.SeedScheme(11))
    rc, yo, so, _, _ = O.sketch_stream(ids, w.astype(np.float64), k, 11)
    assert rc == 0
    assert_regs(y.cpu().numpy(), s.cpu().numpy().view(np.uint64), yo, so)


@pytest.mark.parametrize("n", [1, 3, 100, 1000, 5000])
@pytest.mark.parametrize("k", [1, 2, 64, 4096])
def test_elements_small_sets_with_repeats(n, k):
    """Small element sets (the sample covers every item, runs shorter than a
    block, the scalar filter path) with repeated ids of equal weight and ids
    near 2**64, against the oracle's stream sketch (repeats are no-ops)."""
    rng = np.random.default_rng(1000 * n + k)
    base = rng.integers(0, 1 << 63, size=max(1, n // 2), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    base[0] = np.uint64((1 << 64) - 1)
    wb = rng.lognormal(0.0, 1.0, base.size).astype(np.float32)
    pick = rng.integers(0, base.size, size=n)
    ids, w = base[pick], wb[pick]
    y, s, _ = gm.sketch_elements(ids, w, k, gm.SeedScheme(77))
    rc, yo, so, _, _ = O.sketch_stream(ids, w.astype(np.float64), k, 77)
    assert rc == 0
    assert_regs(y.cpu().numpy(), s.cpu().numpy().view(np.uint64), yo, so)


_ASYNC_SCRIPT = r"""
import sys, json
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2302_05176_b200 as gm
from paper_2302_05176_b200 import workloads
ids4, w4, k4, seed = workloads.config4(n_pairs=1_000_000, n_keys=10**6)
rng = np.random.default_rng(9)
w5 = rng.lognormal(0.0, 2.0, 2_000_000).astype(np.float32)
ids5 = np.arange(w5.size, dtype=np.uint32)
sets = [(ids4, w4), (ids5, w5), (ids4[:5000], w4[:5000]), (ids5[:300], w5[:300])]
out = gm.sketch_elements_many(sets, 2048, gm.SeedScheme(seed))
print(json.dumps([[y.cpu().numpy().tobytes().hex(), s.cpu().numpy().tobytes().hex()] for y, s in out]))
"""


@pytest.mark.parametrize("env", [{}, {"GM_ELEM_TAU_SCALE": "0.1"}])
def test_elements_many_async_equals_sync(env):
    """sketch_elements_many (gm_sketch_elements_async, one pass at the list
    bound per set, no host sync between sets) equals the oracle per set; with
    the first tau scaled down tenfold the one-pass sketches come back
    incomplete and are finished by the synchronous accumulate call."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _ASYNC_SCRIPT, root], capture_output=True, text=True,
                         env={**os.environ, **env}, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    ids4, w4, k4, seed = workloads.config4(n_pairs=1_000_000, n_keys=10**6)
    rng = np.random.default_rng(9)
    w5 = rng.lognormal(0.0, 2.0, 2_000_000).astype(np.float32)
    ids5 = np.arange(w5.size, dtype=np.uint64)
    sets = [(ids4, w4), (ids5, w5), (ids4[:5000], w4[:5000]), (ids5[:300], w5[:300])]
    for (i, w), (yh, sh) in zip(sets, out):
        rc, yo, so, _, _ = O.sketch_stream(i, w.astype(np.float64), 2048, seed)
        assert rc == 0
        assert_regs(np.frombuffer(bytes.fromhex(yh), np.float64), np.frombuffer(bytes.fromhex(sh), np.uint64), yo, so)
