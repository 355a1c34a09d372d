"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed):
  rng_kats.json       uniform_open / rand_int_between / fingerprint / derive_seed
                      KATs and full-queue runs (randgen.py:64-207)
  sketch_cases.json   small vectors -> sketch_naive / sketch_fast / sketch_stream
                      (y as float.hex, s, emitted) and merge cases (estimate.py:103)
  bench_golden.json   test_bench.py:67-82 golden (seed 2024, k=16)
  config1.npz         BASELINE config 1 (ids 0..9999, w = 1 - default_rng(1).random,
                      k=256, seed 1) via sketch_stream (ids include 0)
  config2_sample.npz  first 4 vectors of the config-2 generator via sketch_fast
  wire_records.json   sketch_to_json records (sketch.py:325-339) of the first 8
                      sketch_cases vectors' sketch_fast sketches and of one merge

Only the wire records:  python tests/golden/make_golden.py wire
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import gmsketch as G  # noqa: E402  (the reference)
from gmsketch.randgen import _run_queue, rand_int_between  # noqa: E402

from paper_2302_05176_b200 import workloads  # noqa: E402  (seeded input generators)


def rng_kats():
    rng = random.Random(0xC0FFEE)
    uni = []
    for _ in range(400):
        seed = rng.getrandbits(64)
        e = rng.choice([0, 1, 2, rng.getrandbits(32), rng.getrandbits(64), (1 << 64) - 1])
        z = rng.randrange(1, 9000)
        uni.append([seed, e, z, G.uniform_open(G.SeedScheme(seed), e, z).hex()])
    # pinned SURVEY Appendix B values
    for z in (1, 2, 3):
        uni.append([1, 1, z, G.uniform_open(G.SeedScheme(1), 1, z).hex()])
    ints = []
    for _ in range(400):
        seed = rng.getrandbits(64)
        e = rng.getrandbits(64)
        z = rng.randrange(1, 9000)
        lo = rng.randrange(0, 9000)
        hi = lo + rng.choice([0, 1, 5, 255, 1023, 8191, 65535, rng.getrandbits(40)])
        sc = G.SeedScheme(seed)
        ints.append([sc.perm_seed, e, z, lo, hi, rand_int_between(sc, e, z, lo, hi)])
    fps = []
    for seed, salt in [(1, G.randgen.DEFAULT_STREAM_SALT), (0, 0), (2024, 5), ((1 << 64) - 1, 7)]:
        sc = G.SeedScheme(seed, salt)
        fps.append([seed, salt, sc.fingerprint, sc.perm_seed])
    derive = [[m, t, G.derive_seed(m, t)] for m, t in [(42, 0), (42, 999), (0xACCE97ED, 3), (8080, 1)]]
    queues = []
    for seed, e, w, k in [(1, 5, 1.0, 8), (0x123456789ABCDEF0, 9, 0.31, 16), (77, 0, 2.5, 64),
                          (2024, (1 << 64) - 1, 1e-3, 33), (5, 123456789, 7.0, 256)]:
        sc = G.SeedScheme(seed)
        t = [0.0] * k
        s = [0] * k
        perm = G.randgen.LazyPermutation()
        _run_queue(sc.global_seed, sc.perm_seed, e, w, k, 0, k, 0.0, perm, t, s)
        queues.append({"seed": seed, "element": e, "weight": w.hex(), "k": k,
                       "times": [x.hex() for x in t], "servers": s})
    return {"uniform_open": uni, "rand_int_between": ints, "fingerprint": fps,
            "derive_seed": derive, "queues": queues}


def sk_json(sk, emitted=None):
    d = {"s": list(sk.s), "y": [v.hex() for v in sk.y], "fingerprint": sk.fingerprint}
    if emitted is not None:
        d["emitted"] = emitted
    return d


def sketch_cases():
    rng = random.Random(20240601)
    cases = []
    shapes = [(1, 1), (1, 3), (1, 64), (2, 16), (7, 16), (8, 8), (40, 96), (300, 16),
              (300, 96), (1000, 256), (50, 1), (5, 1024), (2000, 64)]
    for n, k in shapes:
        entries = {}
        while len(entries) < n:
            entries[rng.randrange(1, 10**6)] = rng.random() + 1e-9
        v = G.WeightedVector(entries)
        seed = rng.getrandbits(64)
        p = G.GenerationParams(k=k, scheme=G.SeedScheme(seed))
        fast, em_fast = G.sketch_fast_counted(v, p)
        case = {"n": n, "k": k, "seed": seed,
                "ids": [e for e, _ in v.items()], "w": [w.hex() for _, w in v.items()],
                "fast": sk_json(fast, em_fast)}
        if n * k <= 30000:
            naive, em_naive = G.sketch_naive_counted(v, p)
            assert naive == fast
            case["naive_emitted"] = em_naive
        cases.append(case)
    # heavy-tailed weights (Pareto) to exercise deep queues
    for n, k in [(200, 512), (30, 512)]:
        entries = {}
        while len(entries) < n:
            entries[rng.randrange(1, 1 << 32)] = 1.0 + rng.paretovariate(1.5)
        v = G.WeightedVector(entries)
        seed = rng.getrandbits(64)
        p = G.GenerationParams(k=k, scheme=G.SeedScheme(seed))
        fast, em_fast = G.sketch_fast_counted(v, p)
        cases.append({"n": n, "k": k, "seed": seed, "ids": [e for e, _ in v.items()],
                      "w": [w.hex() for _, w in v.items()], "fast": sk_json(fast, em_fast)})
    # streams with duplicates, id 0 and u64 ids (stream.py accepts any id)
    streams = []
    for n, k in [(9, 4), (60, 24), (500, 128), (3000, 256)]:
        base = {}
        while len(base) < n:
            e = rng.choice([0, rng.randrange(1, 10**5), rng.getrandbits(64)])
            base[e] = rng.random() + 1e-9
        items = list(base.items())
        items += [items[rng.randrange(len(items))] for _ in range(n // 2 + 1)]
        rng.shuffle(items)
        seed = rng.getrandbits(64)
        st = G.StreamSketchState(k, G.SeedScheme(seed))
        for it in items:
            G.stream_update(st, it)
        sk = G.stream_finalize(st)
        streams.append({"k": k, "seed": seed, "ids": [e for e, _ in items],
                        "w": [w.hex() for _, w in items], "sketch": sk_json(sk, st.emitted)})
    # merge cases (partition law, test_estimate.py:174-199)
    merges = []
    for k in (8, 48, 256):
        entries = {i: rng.random() + 1e-9 for i in range(1, 301)}
        items = list(entries.items())
        rng.shuffle(items)
        cuts = sorted(rng.sample(range(1, 300), 3))
        parts = [dict(items[:cuts[0]]), dict(items[cuts[0]:cuts[1]]), dict(items[cuts[1]:cuts[2]]),
                 dict(items[cuts[2]:])]
        seed = rng.getrandbits(64)
        p = G.GenerationParams(k=k, scheme=G.SeedScheme(seed))
        sks = [G.sketch_fast(G.WeightedVector(d), p) for d in parts]
        merged = G.merge(sks)
        assert merged == G.sketch_fast(G.WeightedVector(entries), p)
        merges.append({"k": k, "seed": seed, "parts": [sk_json(s) for s in sks],
                       "merged": sk_json(merged)})
    return {"vectors": cases, "streams": streams, "merges": merges}


def bench_golden():
    vectors = [{1: 0.50, 2: 0.25, 3: 1.00}, {2: 0.25, 3: 1.00, 4: 0.75}, {5: 2.00}]
    params = G.GenerationParams(k=16, scheme=G.SeedScheme(2024))
    sks = [G.sketch_fast(G.WeightedVector(v), params) for v in vectors]
    sim = G.estimate_jaccard_p(sks[0], sks[1])
    card = G.estimate_cardinality(sks[2])
    return {"seed": 2024, "k": 16, "vectors": [[[e, w] for e, w in v.items()] for v in vectors],
            "sketches": [sk_json(s) for s in sks], "matches": sim.matches, "jaccard": sim.value,
            "cardinality": card.value.hex()}


def config1():
    ids, w, k, seed = workloads.config1()
    sk = G.sketch_stream(zip(ids.tolist(), w.tolist()), k, G.SeedScheme(seed))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), ids=ids, w=w, k=k, seed=seed,
                        y=np.array(sk.y, np.float64), s=np.array(sk.s, np.uint64))


def config2_sample():
    ids, w, offsets, k, seed = workloads.config2(n_vectors=4)
    ys, ss, ems = [], [], []
    for v in range(4):
        lo, hi = offsets[v], offsets[v + 1]
        vec = G.WeightedVector({int(e): float(x) for e, x in zip(ids[lo:hi], w[lo:hi])})
        sk, em = G.sketch_fast_counted(vec, G.GenerationParams(k=k, scheme=G.SeedScheme(seed)))
        ys.append(sk.y)
        ss.append(sk.s)
        ems.append(em)
    np.savez_compressed(os.path.join(HERE, "config2_sample.npz"), ids=ids, w=w, offsets=offsets,
                        k=k, seed=seed, y=np.array(ys, np.float64), s=np.array(ss, np.uint64),
                        emitted=np.array(ems, np.int64))


def wire_records():
    """The reference's own serialisation of sketches built from the
    sketch_cases inputs (bit-exact hex floats)."""
    with open(os.path.join(HERE, "sketch_cases.json")) as f:
        cases = json.load(f)["vectors"]
    out = []
    sks = []
    for c in cases[:8]:
        v = G.WeightedVector({e: float.fromhex(w) for e, w in zip(c["ids"], c["w"])})
        sk = G.sketch_fast(v, G.GenerationParams(k=c["k"], scheme=G.SeedScheme(c["seed"])))
        out.append({"case": cases.index(c), "record": G.sketch_to_json(sk)})
        sks.append(sk)
    # a merge of two sketches of the same k and scheme (estimate.py:103-125)
    rng = random.Random(7)
    a = G.WeightedVector({rng.randrange(1, 10**6): rng.random() + 1e-9 for _ in range(50)})
    b = G.WeightedVector({rng.randrange(1, 10**6): rng.random() + 1e-9 for _ in range(70)})
    p = G.GenerationParams(k=32, scheme=G.SeedScheme(99))
    m = G.merge([G.sketch_fast(a, p), G.sketch_fast(b, p)])
    out.append({"merge": {"a": [[e, w.hex()] for e, w in a.items()], "b": [[e, w.hex()] for e, w in b.items()],
                          "k": 32, "seed": 99}, "record": G.sketch_to_json(m)})
    return out


if __name__ == "__main__":
    if sys.argv[1:] == ["wire"]:
        with open(os.path.join(HERE, "wire_records.json"), "w") as f:
            json.dump(wire_records(), f, indent=0)
        print("wire records written")
        sys.exit(0)
    with open(os.path.join(HERE, "rng_kats.json"), "w") as f:
        json.dump(rng_kats(), f)
    with open(os.path.join(HERE, "sketch_cases.json"), "w") as f:
        json.dump(sketch_cases(), f)
    with open(os.path.join(HERE, "bench_golden.json"), "w") as f:
        json.dump(bench_golden(), f, indent=1)
    with open(os.path.join(HERE, "wire_records.json"), "w") as f:
        json.dump(wire_records(), f, indent=0)
    config1()
    config2_sample()
    print("golden fixtures written to", HERE)
