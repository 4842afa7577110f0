"""GPU parity of every WHT tile-kernel variant the benches launch
(tests/variant_cases.py; coverage checked on the CPU by tests/test_variants.py):
each case runs the library with a planner override that gives a small state
the large configs' group shapes, and compares every amplitude with the oracle
(or_iterate / or_iterate_noisy / or_iterate_decoherent: the literal
per-operation contraction + renormalisation)."""
import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests.test_parity_gpu import assert_close, ctx_with, rand_state
from tests.test_variants import variants
from tests.variant_cases import CASES, DECOHERENT, IDEAL, NOISY

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_variant_case_matches_oracle(case, monkeypatch):
    cid, n, world, fl, k, sigma, rate, seed, env = case
    for key, v in env.items():
        monkeypatch.setenv(key, v)
    dtype = sv.SV_C64
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, 37, seed)
    with ctx_with(a, dtype, world=world) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_profile(c, True)
        if fl == IDEAL:
            sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        elif fl == NOISY:
            sv.sv_iterate_noisy(c, k, sigma, seed, 0)
        else:
            surv = sv.sv_iterate_decoherent(c, k, sigma, rate, seed, 0)
        launches, _ = sv.sv_profile_read(c, sv.SV_K_WHT_TILE)
        got = sv.sv_get_amplitudes(c)
    # the case launched what the host description says it launches
    desc = sv.sv_debug_wht_variants(n, world, dtype, fl, k, sigma, rate, seed, True)
    sub = sum(1 for v in desc if v[0] == 3)  # supertile passes: three sub-pass variants per launch
    assert sub % 3 == 0 and launches == len(desc) - sub + sub // 3
    assert variants(n, world, fl, k, sigma, rate, seed, env)
    if fl == IDEAL:
        ref = orc.iterate(a.copy(), marked, k, orc.WHT)
    elif fl == NOISY:
        ref = orc.iterate_noisy(a.copy(), marked, k, sigma, seed, 0)
    else:
        ref, surv_ref = orc.iterate_decoherent(a.copy(), marked, k, sigma, rate, seed, 0)
        np.testing.assert_allclose(surv, surv_ref, rtol=2e-6, atol=0)
    assert_close(got, ref, dtype, cid, n=n, k=k)
