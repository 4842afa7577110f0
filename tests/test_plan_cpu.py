"""The product's WHT schedule (host planner in libsv.so), executed step by step
on numpy shards, equals the oracle's (D O)^k -- P = 1, 2, 4, 8 (CPU only)."""
import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests.plan_exec import execute

rng = np.random.default_rng(7)


@pytest.mark.parametrize("n,world,dtype", [(14, 1, sv.SV_C64), (16, 1, sv.SV_C128), (20, 1, sv.SV_C64),
                                           (24, 1, sv.SV_C64), (16, 2, sv.SV_C128), (18, 4, sv.SV_C64),
                                           (19, 8, sv.SV_C64), (20, 8, sv.SV_C128), (17, 2, sv.SV_C64)])
def test_schedule_equals_oracle(n, world, dtype):
    T = 13 if dtype == sv.SV_C64 else 12
    g = world.bit_length() - 1
    if world > 1 and n - 2 * g < T:
        pytest.skip("shard too small")
    N = 1 << n
    a0 = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    a0 /= np.linalg.norm(a0)
    marked = orc.marked_from_seed(n, 5, n)
    k = 2
    plan = sv.sv_plan_wht(n, world, dtype, k, True)
    shards = np.split(a0.copy(), world)
    got = np.concatenate(execute(plan, shards, n, marked))
    ref = orc.iterate(a0.copy(), marked, k, orc.WHT)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
    # a lone diffusion
    plan = sv.sv_plan_wht(n, world, dtype, 0, False)
    got = np.concatenate(execute(plan, np.split(a0.copy(), world), n, marked))
    np.testing.assert_allclose(got, orc.diffuse_wht(a0.copy()), rtol=0, atol=1e-12)
