"""GPU parity of the noisy Grover iteration (operational
angle errors, readings G19/G20) against the CPU oracle's or_iterate_noisy.
Same tolerances as tests/test_parity_gpu.py."""
import math

import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests.test_parity_gpu import DT, DT_IDS, assert_close, ctx_with, rand_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,m,k,sigma", [(5, 2, 3, 0.1), (12, 3, 4, 0.05), (14, 1, 3, 0.02), (17, 9, 2, 0.1),
                                         (20, 4, 3, 0.01), (23, 30, 2, 0.05), (25, 1, 2, 0.3)])
def test_noisy_iterate_matches_oracle(dtype, n, m, k, sigma):
    """One-CTA kernel (n <= T), and the fused tile schedule: the angle-error
    stages, with pre / post coefficient halves on every fused pass."""
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, m, n)
    seed, t0 = 1234 + n, 7
    with ctx_with(a, dtype) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate_noisy(c, k, sigma, seed, t0)
        got = sv.sv_get_amplitudes(c)
        nrm = sv.sv_norm2(c)
    ref = orc.iterate_noisy(a.copy(), marked, k, sigma, seed, t0)
    assert_close(got, ref, dtype, f"noisy n={n}", n=n, k=k)
    assert abs(nrm - orc.norm_sq(ref)) < (1e-12 if dtype == sv.SV_C128 else 1e-5)  # sv_norm2
    assert abs(float(np.sum(np.abs(got.astype(np.complex128)) ** 2)) - 1.0) < (1e-12 if dtype == sv.SV_C128 else 1e-5)


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
def test_noisy_sigma0_equals_ideal(dtype):
    n, m, k = 22, 4, 3
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, m, 1)
    with ctx_with(a, dtype) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate_noisy(c, k, 0.0, 5)
        noisy0 = sv.sv_get_amplitudes(c)
    ref = orc.iterate(a.copy(), marked, k, orc.WHT)
    assert_close(noisy0, ref, dtype, "sigma=0", n=n, k=k)


@pytest.mark.parametrize("fused", [True, False], ids=["fused-xchg", "alltoall"])
@pytest.mark.parametrize("n,world", [(19, 4), (20, 8), (17, 2)])
def test_noisy_emulated_sharding(n, world, fused):
    """Angle errors follow the LOGICAL qubit through the qubit swaps."""
    dtype = sv.SV_C64
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, 6, n)
    with ctx_with(a, dtype, world=world) as c:
        sv.sv_set_exchange(c, fused)
        sv.sv_set_marked(c, marked)
        sv.sv_iterate_noisy(c, 3, 0.05, 99, 0)
        got = sv.sv_get_amplitudes(c)
    ref = orc.iterate_noisy(a.copy(), marked, 3, 0.05, 99, 0)
    assert_close(got, ref, dtype, "noisy sharded", n=n, k=3)


def test_noisy_split_calls_and_errors():
    n, dtype = 18, sv.SV_C128
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, 3, 2)
    with ctx_with(a, dtype) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate_noisy(c, 2, 0.1, 3, 0)
        sv.sv_iterate_noisy(c, 3, 0.1, 3, 2)
        got = sv.sv_get_amplitudes(c)
        with pytest.raises(sv.SvError):
            sv.sv_iterate_noisy(c, -1, 0.1, 3, 0)
        with pytest.raises(sv.SvError):
            sv.sv_iterate_noisy(c, 1, -0.5, 3, 0)
    ref = orc.iterate_noisy(a.copy(), marked, 5, 0.1, 3, 0)
    assert_close(got, ref, dtype, "split", n=n, k=5)



def test_noisy_full_size_n28_k1():
    """c3n's launch configuration at its full size (n = 28, the bench's sigma =
    0.01 and seed), one iteration, every amplitude vs or_iterate_noisy."""
    n, dtype, sigma, seed = 28, sv.SV_C64, 0.01, 3
    marked = sv.sv_marked_from_seed(n, 1, seed)
    a = orc.init_uniform(n)
    with sv.sv_init(n, seed, dtype, sv.SV_INIT_UNIFORM) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate_noisy(c, 1, sigma, seed, 0)
        got = sv.sv_get_amplitudes(c)
    ref = orc.iterate_noisy(a, marked, 1, sigma, seed, 0)
    del a
    assert_close(got, ref, dtype, "noisy n=28 k=1", n=n, k=1)
