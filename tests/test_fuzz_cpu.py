"""Property-based tests (hypothesis): random sizes, marked
sets, iteration counts, seeds, shard counts and planner splits, CPU only.

* The oracle against the general-start closed form (
  exact up to rounding): a_M^(k), a_U^(k) from the Gaussian start, every
  amplitude, both diffusions, M = 0 .. N.
* The product's host planner (sv_plan_wht, with random SV_PLAN_CHUNKS splits
  and O / F0 roles on one GPU, random P on the sharded path), executed pass by
  pass on numpy shards (tests/plan_exec.py), against the oracle's (D O)^k --
  every schedule the planner can emit must be a valid factorisation of the
  iteration (stages commute across qubits, G18)."""
import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_quant_ph_9804039_b200 as sv
from oracle import closed_form as cf
from oracle import oracle as orc
from tests.plan_exec import execute

SETTINGS = dict(deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])


@settings(max_examples=60, **SETTINGS)
@given(n=st.integers(1, 10), mfrac=st.floats(0.0, 1.0), k=st.integers(0, 9), seed=st.integers(0, 2 ** 31 - 1),
       mean=st.booleans())
def test_oracle_matches_general_closed_form(n, mfrac, k, seed, mean):
    N = 1 << n
    m = int(round(mfrac * N))
    a0 = orc.init_gaussian(n, seed)
    marked = orc.marked_from_seed(n, m, seed)
    got = orc.iterate(a0.copy(), marked, k, orc.MEAN if mean else orc.WHT)
    ref = cf.general_state(a0, marked, k)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.sqrt(k)) * 10


@st.composite
def plan_case(draw):
    world = draw(st.sampled_from([1, 1, 2, 4, 8]))
    g = world.bit_length() - 1
    n = draw(st.integers(14, 20) if g == 0 else st.integers(13 + 2 * g, min(13 + 2 * g + 3, 21)))
    env = {}
    if world == 1 and draw(st.booleans()):
        rest = n - 13
        parts = []
        while rest > 0:
            p = draw(st.integers(1, min(10, rest)))
            parts.append(p)
            rest -= p
        tags = [""] * len(parts)
        roles = draw(st.sampled_from(["none", "o", "f", "of"]))
        if len(parts) >= 2 or roles in ("o", "f"):
            idx = draw(st.permutations(list(range(len(parts)))))
            if "o" in roles:
                tags[idx[0]] = "o"
            if "f" in roles and len(parts) >= 2:
                tags[idx[-1]] = "f"
            elif "f" in roles and tags[idx[0]] == "":
                tags[idx[0]] = "f"
        env["SV_PLAN_CHUNKS"] = ",".join(f"{p}{t}" for p, t in zip(parts, tags))
    if world > 1 and draw(st.booleans()):
        nl = n - g
        take_max = min(13 - 3 - g, max(nl - g - 13, 0))
        env["SV_PLAN_L1"] = str(g + draw(st.integers(0, take_max)))
    k = draw(st.integers(0, 3))
    m = draw(st.integers(0, 40))
    seed = draw(st.integers(0, 10 ** 6))
    return n, world, k, m, seed, env


@settings(max_examples=40, **SETTINGS)
@given(case=plan_case())
def test_planner_schedules_execute_to_oracle(case):
    n, world, k, m, seed, env = case
    old = {key: os.environ.get(key) for key in ("SV_PLAN_CHUNKS", "SV_PLAN_L1")}
    try:
        for key in old:
            os.environ.pop(key, None)
        os.environ.update(env)
        plan = sv.sv_plan_wht(n, world, sv.SV_C64, k, True)
    finally:
        for key, v in old.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v
    rng = np.random.default_rng(seed)
    N = 1 << n
    a0 = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    a0 /= np.linalg.norm(a0)
    marked = orc.marked_from_seed(n, min(m, N), seed)
    got = np.concatenate(execute(plan, np.split(a0.copy(), world), n, marked))
    ref = orc.iterate(a0.copy(), marked, k, orc.WHT)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12, err_msg=str(case))
    # every transform runs each qubit's stage exactly once (on every rank): 2 n k stage visits
    visits = sum(bin(st_["proc_mask"]).count("1") * (st_["pre"] + st_["post"]) for st_ in plan if st_["kind"] == 0)
    assert visits == 2 * n * k
