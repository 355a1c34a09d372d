"""Loaders for the committed golden fixtures (tests/golden/, generated from
the reference by tests/golden/make_golden.py)."""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_npz(name: str):
    return dict(np.load(os.path.join(GOLDEN, name)))


def hexs(values) -> np.ndarray:
    return np.array([float.fromhex(v) for v in values], dtype=np.float64)


def vector_case(case):
    ids = np.array(case["ids"], dtype=np.uint64)
    w = hexs(case["w"])
    return ids, w


def sketch_arrays(d):
    return hexs(d["y"]), np.array([int(x) & 0xFFFFFFFFFFFFFFFF for x in d["s"]], dtype=np.uint64)
