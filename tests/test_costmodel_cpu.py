"""The product's analytical model (paper_quant_ph_9804039_b200/costmodel.py)
vs the oracle's literal Eqs. 2-9 (oracle/cost_model.py, pinned in
test_oracle_cost_model.py), and consistency of the B200 refit with the
library's schedules (host-only: sv_plan_wht / sv_plan_gates)."""
import numpy as np
import pytest

from oracle import cost_model as O
from paper_quant_ph_9804039_b200 import costmodel as C
from tests import circuits as CI


def as_dict(mp):
    return dict(t_op2=mp.t_op2, t_op3=mp.t_op3, t_t=mp.t_t, t_lat=mp.t_lat, t_b=mp.t_b, t_lr=mp.t_lr, q=mp.q)


def test_presets_are_fig9():
    assert as_dict(C.T3E) == O.T3E
    assert as_dict(C.SP2) == O.SP2


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("s", [2, 3])
def test_equations_match_oracle(seed, s):
    rng = np.random.default_rng(seed)
    mp = C.T3E if seed % 2 else C.SP2
    om = as_dict(mp)
    steps = []
    for _ in range(int(rng.integers(1, 6))):
        n_b = int(rng.integers(6, 14))
        n_l = int(rng.integers(0, n_b - 2))
        n_c = int(rng.integers(0, n_l + 1))
        steps.append((int(rng.integers(0, 5000)), n_b, n_l, n_c))
    psteps = [C.Step(*st) for st in steps]
    n_p = int(rng.integers(0, 3))
    rel = dict(rel=1e-12, abs=0)
    assert C.eq6_seqdyn(psteps, s, mp) == pytest.approx(O.t_seqdyn(steps, s, om), **rel)
    assert C.eq7_par(psteps, n_p, s, mp) == pytest.approx(O.t_par(steps, n_p, s, om), **rel)
    assert C.eq8_pardec(psteps, n_p, s, mp) == pytest.approx(O.t_pardec(steps, n_p, s, om), **rel)
    assert C.eq9_seqdec(psteps, s, mp) == pytest.approx(O.t_seqdec(steps, s, om), **rel)
    l, n_b, n_l, n_c = steps[0]
    assert C.eq2_reorg(n_l, n_b, n_c, s, mp) == pytest.approx(O.t_reorg(n_l, n_b, n_c, s, om), **rel)
    assert C.eq5_seqflat(l, n_b, s, mp) == pytest.approx(O.t_seqflat(l, n_b, s, om), **rel)
    assert C.eq3_dec(l, mp) == pytest.approx(O.t_dec(l, om), **rel)


def test_b200_refit_in_paper_terms():
    # with one bandwidth class, the schedule prediction is Eq. 4 with
    # l = passes, n_b = n, n_l = 0 (flat store) and t_op = 4 q / BW
    prm = C.B200Params(bw_pass={"default": 6.0e12}, t_launch=0.0)
    n, k = 30, 8
    pred = C.predict_wht(n, 1, 0, k, prm)
    mp = prm.as_machine_params(0)
    eq = C.eq7_par([C.Step(pred["passes"], n, 0, 0)], 0, 2, mp)
    assert pred["t"] == pytest.approx(eq, rel=1e-12)
    assert pred["passes"] == 4 * k + 1  # 2(p - 1) per iteration (p = 3 groups) + the unfused last visit


def test_b200_predictions_behave():
    prm = C.B200Params()
    t8 = C.predict_wht(32, 1, 0, 8, prm)["t"]
    t16 = C.predict_wht(32, 1, 0, 16, prm)["t"]
    assert t16 == pytest.approx(2 * t8, rel=0.05)
    # strong scaling over NVLink: more GPUs, less time, efficiency <= 1
    t1 = C.predict_wht(32, 1, 0, 16, prm)["t"]
    for P in (2, 4, 8):
        tP = C.predict_wht(32, P, 0, 16, prm)
        assert tP["swaps"] == 2 * 16 and tP["t"] < t1
        assert C.scaling_efficiency(t1, tP["t"], P) <= 1.05
    m = C.predict_mean(28, 1, 0, 64, prm)
    assert m["passes"] == 65
    # gates: a pass is at least its HBM round trip, and grows with its op count
    g1 = C.predict_gates(26, 1, 0, CI.circuit([CI.record(q, CI.H) for q in range(26)]), prm)
    # 41 layers of H fuse into one op per qubit on the host, H^41 = H: same ops,
    # same relayouts, same cost (an even count fuses to a diagonal op, cheaper) ...
    g40 = C.predict_gates(26, 1, 0, CI.circuit([CI.record(q, CI.H) for q in range(26)] * 41), prm)
    assert g1["passes"] == 3 and g40["t"] == pytest.approx(g1["t"])
    # ... while a chain of controlled gates does not fuse and costs compute
    chain = CI.circuit([CI.record(q, CI.H, [(q + 1) % 26]) for q in range(26)] * 40)
    assert C.predict_gates(26, 1, 0, chain, prm)["t"] > g1["t"]
