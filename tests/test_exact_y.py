"""Exact-y finalize (gm_exact_y, host code in libgmsketch_b200.so) against the
reference's own sketches: given the reference's winners s, the re-derived
registers y equal the reference's bit for bit.  Host logic only (no device
work), so these run without a GPU."""

import numpy as np
import pytest

import paper_2302_05176_b200 as gm
from tests.golden_io import hexs, load_json, load_npz, sketch_arrays, vector_case

U64 = (1 << 64) - 1


def test_vector_cases_bit_exact():
    for case in load_json("sketch_cases.json")["vectors"]:
        ids, w = vector_case(case)
        wy, ws = sketch_arrays(case["fast"])
        y = np.zeros(case["k"])
        gm.exact_y_host(ids, w, np.array([0, ids.size]), case["k"], gm.SeedScheme(case["seed"]), ws, y)
        assert y.tobytes() == wy.tobytes()


def test_stream_cases_bit_exact():
    for case in load_json("sketch_cases.json")["streams"]:
        ids = np.array([int(e) & U64 for e in case["ids"]], dtype=np.uint64)
        w = hexs(case["w"])
        wy, ws = sketch_arrays(case["sketch"])
        y = np.zeros(case["k"])
        gm.exact_y_host(ids, w, np.array([0, ids.size]), case["k"], gm.SeedScheme(case["seed"]), ws, y)
        assert y.tobytes() == wy.tobytes()


def test_config2_sample_batch_bit_exact():
    g = load_npz("config2_sample.npz")
    y = np.zeros_like(g["y"])
    gm.exact_y_host(g["ids"], g["w"], g["offsets"], int(g["k"]), gm.SeedScheme(int(g["seed"])), g["s"], y, threads=4)
    assert y.tobytes() == g["y"].tobytes()


def test_bench_golden_bit_exact():
    g = load_json("bench_golden.json")
    for vec, want in zip(g["vectors"], g["sketches"]):
        ids = np.array([e for e, _ in vec], dtype=np.uint64)
        w = np.array([x for _, x in vec], dtype=np.float64)
        wy, ws = sketch_arrays(want)
        y = np.zeros(16)
        gm.exact_y_host(ids, w, np.array([0, ids.size]), 16, gm.SeedScheme(2024), ws, y)
        assert y.tobytes() == wy.tobytes()


def test_foreign_winner_is_rejected():
    case = load_json("sketch_cases.json")["vectors"][0]
    ids, w = vector_case(case)
    _, ws = sketch_arrays(case["fast"])
    ws = ws.copy()
    ws[0] = int(ids.max()) + 12345  # not an element of the vector
    with pytest.raises(gm.MismatchedSketchError):
        gm.exact_y_host(ids, w, np.array([0, ids.size]), case["k"], gm.SeedScheme(case["seed"]), ws,
                        np.zeros(case["k"]))


def test_element_queue_state_validation():
    """ElementQueueState validates its weight like the reference (randgen.py:218-229)
    (the emissions themselves run on the device: tests/test_gpu_parity.py)."""
    with pytest.raises(gm.InvalidWeightError):
        gm.ElementQueueState(1, 0.0, 4)
    with pytest.raises(gm.InvalidWeightError):
        gm.ElementQueueState(1, 1e-301, 4)
    st = gm.ElementQueueState(3, 0.5, 8)
    assert st.z == 0 and not st.exhausted and st.perm.tolist() == list(range(1, 9))
