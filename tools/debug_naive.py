"""Debug: naive (exhaustive) sketches of the golden vector cases on the device against the fixtures (GPU box)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05176_b200 as gm
from tests.golden_io import load_json, vector_case
cases = [c for c in load_json("sketch_cases.json")["vectors"] if c["n"] * c["k"] <= 300_000]
for case in cases:
    ids, w = vector_case(case)
    v = gm.WeightedVector({int(e): float(x) for e, x in zip(ids, w)})
    try:
        sk, em = gm.sketch_naive_counted(v, gm.GenerationParams(k=case["k"], scheme=gm.SeedScheme(case["seed"])))
        print("ok", case["n"], case["k"], em)
    except Exception as e:
        print("FAIL", case["n"], case["k"], repr(e))
