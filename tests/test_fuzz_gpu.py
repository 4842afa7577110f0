"""Property-based GPU parity (hypothesis: "random (n <= 12,
M, k, seed) parity", widened here to n <= 21 and to emulated sharding): the
library through the C ABI against the oracle, every amplitude, on random
sizes, dtypes, diffusions, marked sets, iteration counts, shard counts and
Gaussian seeds.  Tolerances as tests/test_parity_gpu.py."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_quant_ph_9804039_b200 as sv
from oracle import oracle as orc
from tests.test_parity_gpu import assert_close

pytestmark = pytest.mark.gpu


@st.composite
def case(draw):
    dtype = draw(st.sampled_from([sv.SV_C64, sv.SV_C128]))
    T = 13 if dtype == sv.SV_C64 else 12
    world = draw(st.sampled_from([1, 1, 1, 2, 4, 8]))
    g = world.bit_length() - 1
    lo = 1 if world == 1 else T + 2 * g
    n = draw(st.integers(lo, max(lo, 21)))
    N = 1 << n
    m = draw(st.integers(0, min(N, 64)))
    k = draw(st.integers(0, 6))
    diff = draw(st.sampled_from([sv.SV_DIFFUSE_WHT, sv.SV_DIFFUSE_MEAN]))
    seed = draw(st.integers(0, 10 ** 6))
    return dtype, world, n, m, k, diff, seed


@settings(max_examples=40, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])
@given(c=case())
def test_random_configs_match_oracle(c):
    dtype, world, n, m, k, diff, seed = c
    marked = orc.marked_from_seed(n, m, seed)
    a0 = orc.init_gaussian(n, seed, round_to_c64=(dtype == sv.SV_C64))
    with sv.sv_init(n, seed, dtype, sv.SV_INIT_GAUSSIAN, world=world) as ctx:
        sv.sv_set_marked(ctx, marked)
        sv.sv_iterate(ctx, k, diff)
        got = sv.sv_get_amplitudes(ctx)
    ref = orc.iterate(a0.copy(), marked, k, orc.WHT if diff == sv.SV_DIFFUSE_WHT else orc.MEAN)
    assert_close(got, ref, dtype, f"fuzz {c}", n=n, k=max(k, 1))
