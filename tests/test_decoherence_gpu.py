"""GPU parity of the decoherent Grover iteration (reading
G22) against the oracle, which applies the contraction and the global
renormalisation after EVERY laser operation literally as the paper describes;
the library folds the per-operation factors into per-qubit 2x2 matrices and
one renormalisation per iteration (the same linear map up to rounding)."""
import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests.test_parity_gpu import DT, DT_IDS, assert_close, ctx_with, rand_state

pytestmark = pytest.mark.gpu

SURV_RTOL = {sv.SV_C128: 1e-12, sv.SV_C64: 2e-6}


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,m,k,sigma,rate", [(4, 1, 3, 0.0, 0.05), (11, 3, 3, 0.05, 0.02), (14, 2, 2, 0.0, 0.01),
                                              (17, 5, 3, 0.05, 0.03), (21, 9, 2, 0.02, 0.01), (24, 1, 2, 0.0, 0.005)])
def test_decoherent_matches_oracle(dtype, n, m, k, sigma, rate):
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, m, n)
    seed, t0 = 77 + n, 4
    with ctx_with(a, dtype) as c:
        sv.sv_set_marked(c, marked)
        surv = sv.sv_iterate_decoherent(c, k, sigma, rate, seed, t0)
        got = sv.sv_get_amplitudes(c)
    ref, surv_ref = orc.iterate_decoherent(a.copy(), marked, k, sigma, rate, seed, t0)
    assert_close(got, ref, dtype, f"decoherent n={n}", n=n, k=k)
    np.testing.assert_allclose(surv, surv_ref, rtol=SURV_RTOL[dtype], atol=0)
    assert abs(float(np.sum(np.abs(got.astype(np.complex128)) ** 2)) - 1.0) < (1e-12 if dtype == sv.SV_C128 else 1e-5)


def test_decoherent_rate0_equals_noisy():
    n, dtype = 19, sv.SV_C128
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, 4, 3)
    with ctx_with(a, dtype) as c:
        sv.sv_set_marked(c, marked)
        surv = sv.sv_iterate_decoherent(c, 3, 0.05, 0.0, 8, 0)
        got = sv.sv_get_amplitudes(c)
    np.testing.assert_allclose(surv, 1.0, atol=1e-12)
    assert_close(got, orc.iterate_noisy(a.copy(), marked, 3, 0.05, 8, 0), dtype, "rate 0", n=n, k=3)


@pytest.mark.parametrize("world", [2, 8])
def test_decoherent_emulated_sharding(world):
    n, dtype = 20, sv.SV_C64
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, 6, 2)
    with ctx_with(a, dtype, world=world) as c:
        sv.sv_set_marked(c, marked)
        surv = sv.sv_iterate_decoherent(c, 2, 0.03, 0.02, 5, 1)
        got = sv.sv_get_amplitudes(c)
    ref, surv_ref = orc.iterate_decoherent(a.copy(), marked, 2, 0.03, 0.02, 5, 1)
    assert_close(got, ref, dtype, "decoherent sharded", n=n, k=2)
    np.testing.assert_allclose(surv, surv_ref, rtol=SURV_RTOL[dtype])


def test_decoherent_errors():
    with sv.sv_init(14, 0, sv.SV_C64) as c:
        with pytest.raises(sv.SvError):
            sv.sv_iterate_decoherent(c, 1, 0.0, 0.1, 1)  # no marked set
        sv.sv_set_marked(c, [3])
        for bad in ((1, 0.0, 1.0), (1, 0.0, -0.1), (-1, 0.0, 0.1)):
            with pytest.raises(sv.SvError):
                sv.sv_iterate_decoherent(c, bad[0], bad[1], bad[2], 1)
        assert sv.sv_iterate_decoherent(c, 0, 0.0, 0.1, 1).size == 0



def test_decoherent_full_size_n28_k1():
    """c3d's launch configuration at its full size (n = 28, sigma = 0.01, rate =
    1e-3, the bench's seed), one iteration, every amplitude and the survival
    probability vs or_iterate_decoherent (literal per-operation contraction and
    renormalisation)."""
    n, dtype, sigma, rate, seed = 28, sv.SV_C64, 0.01, 1e-3, 3
    marked = sv.sv_marked_from_seed(n, 1, seed)
    with sv.sv_init(n, seed, dtype, sv.SV_INIT_UNIFORM) as c:
        sv.sv_set_marked(c, marked)
        surv = sv.sv_iterate_decoherent(c, 1, sigma, rate, seed, 0)
        got = sv.sv_get_amplitudes(c)
    ref, surv_ref = orc.iterate_decoherent(orc.init_uniform(n), marked, 1, sigma, rate, seed, 0)
    assert_close(got, ref, dtype, "decoherent n=28 k=1", n=n, k=1)
    np.testing.assert_allclose(surv, surv_ref, rtol=SURV_RTOL[dtype], atol=0)
