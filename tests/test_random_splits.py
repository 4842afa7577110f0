"""Random strided-group splits (the test-only SV_PLAN_CHUNKS override; any split is
a valid schedule because stages on different qubits commute, G18 / P:3080-3084).
CPU: the planner accepts exactly the splits whose groups fit the tile's processed
slots, and every accepted plan processes each qubit once per transform.  GPU: a few
random splits, every amplitude against the oracle (tools/soak_wht_gpu.py runs many)."""
import os
import sys

import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from soak_wht_gpu import random_split  # noqa: E402

TILE = {sv.SV_C64: 13, sv.SV_C128: 12}


def test_planner_accepts_random_splits(monkeypatch):
    rng = np.random.default_rng(5)
    accepted = 0
    for _ in range(150):
        dt = sv.SV_C64 if rng.random() < 0.6 else sv.SV_C128
        n = int(rng.integers(17, 30))
        split = random_split(rng, n - TILE[dt])
        monkeypatch.setenv("SV_PLAN_CHUNKS", split)
        lens = [int(t.rstrip("of")) for t in split.split(",")]
        assert sum(lens) == n - TILE[dt]
        try:
            steps = sv.sv_plan_wht(n, 1, dt, 1, True)
        except sv.SvError as e:
            assert "a group holds" in str(e), (split, str(e))
            continue
        accepted += 1
        assert len(steps) >= len(lens) + 1, (split, steps)
    assert accepted >= 100


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(10))
def test_random_split_matches_oracle(case, monkeypatch):
    from tests.test_parity_gpu import assert_close, ctx_with, rand_state

    rng = np.random.default_rng(1000 + case)
    dt = sv.SV_C64 if case % 3 else sv.SV_C128
    n = int(rng.integers(17, 22))
    k = int(rng.integers(1, 3))
    while True:
        split = random_split(rng, n - TILE[dt])
        monkeypatch.setenv("SV_PLAN_CHUNKS", split)
        try:
            sv.sv_plan_wht(n, 1, dt, k, True)
            break
        except sv.SvError:
            continue
    a = rand_state(n, dt)
    marked = orc.marked_from_seed(n, 37, 11 + case)
    with ctx_with(a, dt) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        got = sv.sv_get_amplitudes(c)
    assert_close(got, orc.iterate(a.copy(), marked, k, orc.WHT), dt, f"split {split} n={n}", n=n, k=k)
