"""The draw-log form of the lane walker's Fisher-Yates state (K1, k <= 1024;
csrc/gm_csr.cuh: lane_step_log, log_trace) restated in Python and checked
against the reference's LazyPermutation semantics (randgen.py:146-155 and the
swap in _run_queue, randgen.py:200-204): the server of step z is the content
of the drawn position before the swap.  CPU only: this pins the ALGORITHM the
kernel implements (the kernel itself is checked against the oracle on the
GPU, tests/test_gpu_parity.py::test_draw_log_lanes_traces_and_handovers)."""

import random

import pytest


def servers_lazy_permutation(k, draws):
    """Reference semantics: perm[z-1], perm[j-1] swapped, server = perm[z-1] after the swap."""
    perm = {}
    out = []
    for z, j in enumerate(draws, start=1):
        zi, ji = z - 1, j - 1
        a, b = perm.get(zi, zi + 1), perm.get(ji, ji + 1)
        perm[zi], perm[ji] = b, a
        out.append(perm[zi])
    return out, perm


def log_trace(log, pos, n):
    """log[i] = 0-based position drawn at step i + 1; content of `pos` after the first n steps (value - 1)."""
    for i in range(n - 1, -1, -1):
        if log[i] == pos:
            pos = i
    return pos


def servers_draw_log(k, draws):
    bitmap = [False] * k
    log = []
    out = []
    traces = 0
    for z, j in enumerate(draws, start=1):
        zi, ji = z - 1, j - 1
        if bitmap[ji]:
            traces += 1
            v = log_trace(log, ji, zi)
        else:
            v = ji
        bitmap[ji] = True
        log.append(ji)
        out.append(v + 1)
    return out, log, traces


@pytest.mark.parametrize("k", [1, 2, 3, 8, 40, 300, 1024])
def test_draw_log_equals_lazy_permutation(k):
    rng = random.Random(k)
    for _ in range(200 if k <= 40 else 40):
        depth = rng.randint(1, min(k, 64))
        draws = [rng.randint(z, k) for z in range(1, depth + 1)]
        want, perm = servers_lazy_permutation(k, draws)
        got, log, _ = servers_draw_log(k, draws)
        assert got == want
        # hand-over to the warp walker: the dense array rebuilt from the log
        # (every logged position >= z0 traced over the whole log) is the
        # reference permutation's live part
        z0 = depth
        dense = {p: log_trace(log, p, z0) + 1 for p in log if p >= z0}
        live = {p: v for p, v in perm.items() if p >= z0 and v != p + 1}
        assert {p: v for p, v in dense.items() if v != p + 1} == live


def test_full_queue_is_a_permutation_and_traces_happen():
    k = 64
    rng = random.Random(5)
    draws = [rng.randint(z, k) for z in range(1, k + 1)]
    want, _ = servers_lazy_permutation(k, draws)
    got, _, traces = servers_draw_log(k, draws)
    assert got == want and sorted(got) == list(range(1, k + 1))
    assert traces > 0  # repeated draws are frequent at depth ~ k
