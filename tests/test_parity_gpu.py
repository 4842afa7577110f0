"""GPU parity: libsv (CUDA, sm_100a) vs the CPU oracle, element by element,
through the C ABI.  Tolerances (BASELINE.json north star): complex128 max-abs
<= 1e-12, complex64 max-abs <= 1e-5; complex64 additionally within a relative
bound rel64(n, k) of the amplitude scale."""
import math

import numpy as np
import pytest

import paper_quant_ph_9804039_b200 as sv
from oracle import closed_form as cf
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

TOL = {sv.SV_C128: 1e-12, sv.SV_C64: 1e-5}
def rel64(n: int, k: int) -> float:
    """complex64 error budget relative to max|a_ref|:
    one diffusion = 2 transforms of n fp32 add stages, each rounding by at
    most 2^-24 of a partial sum bounded by the amplitude scale -> 2n 2^-24;
    over k iterations the rounding errors add with random signs -> sqrt(k)."""
    return 2.0 * max(n, 1) * 2.0 ** -24 * math.sqrt(max(k, 1))
rng = np.random.default_rng(99)


WORST = {"c64_rel": 0.0, "c64_abs": 0.0, "c128_abs": 0.0, "c64_rel_where": "", "c64_rel_top": []}


@pytest.fixture(scope="module", autouse=True)
def _report_worst_errors():
    """Record the worst observed errors."""
    yield
    import json
    import os
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        json.dump(WORST, open(os.path.join(out, "parity_error_stats.json"), "w"), indent=1)


def assert_close(got, ref, dtype, what="", n=None, k=1):
    got = np.asarray(got, dtype=np.complex128)
    err = float(np.max(np.abs(got - ref))) if ref.size else 0.0
    scale = float(np.max(np.abs(ref))) if ref.size else 0.0
    if dtype == sv.SV_C64:
        WORST["c64_abs"] = max(WORST["c64_abs"], err)
        if scale and err / scale > WORST["c64_rel"]:
            WORST["c64_rel"], WORST["c64_rel_where"] = err / scale, what
        if scale:
            WORST["c64_rel_top"] = sorted(WORST["c64_rel_top"] + [(err / scale, what)], reverse=True)[:12]
    else:
        WORST["c128_abs"] = max(WORST["c128_abs"], err)
    assert err <= TOL[dtype], f"{what}: max-abs {err:.3e} > {TOL[dtype]:.0e}"
    if dtype == sv.SV_C64:
        if n is None:
            n = max(int(ref.size).bit_length() - 1, 1)
        rel = rel64(n, k)
        assert err <= rel * scale + 1e-30, f"{what}: max-abs {err:.3e} > {rel:.2e} x {scale:.3e}"
    return err


def rand_state(n, dtype):
    N = 1 << n
    a = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    a /= np.linalg.norm(a)
    # the oracle starts from the dtype-rounded values (G12)
    return a.astype(sv.NP_DTYPE[dtype]).astype(np.complex128)


def ctx_with(a, dtype, **kw):
    n = a.size.bit_length() - 1
    c = sv.sv_init(n, 0, dtype, sv.SV_INIT_ZERO_STATE, **kw)
    sv.sv_set_amplitudes(c, a)
    return c


DT = [sv.SV_C128, sv.SV_C64]
DT_IDS = ["c128", "c64"]


# --------------------------------------------------------------------------- #
# initial states and generators                                               #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n", [1, 5, 13, 16])
def test_init_uniform_and_zero(dtype, n):
    with sv.sv_init(n, 0, dtype, sv.SV_INIT_UNIFORM) as c:
        assert_close(sv.sv_get_amplitudes(c), orc.init_uniform(n), dtype, "uniform")
        if n == 1:  # Fig. 1(b): 1/sqrt2 amplitudes, probabilities 1/2
            np.testing.assert_allclose(sv.sv_probabilities(c), [0.5, 0.5], atol=1e-7 if dtype == sv.SV_C64 else 1e-15)
        sv.sv_reset(c, 0, sv.SV_INIT_ZERO_STATE)
        assert_close(sv.sv_get_amplitudes(c), orc.init_zero_state(n), dtype, "zero")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,seed", [(3, 1), (12, 5), (17, 6), (21, 7)])
def test_init_gaussian_matches_oracle_generator(dtype, n, seed):
    """G8: same counter hash and Box-Muller on both sides; normalised to 1."""
    with sv.sv_init(n, seed, dtype, sv.SV_INIT_GAUSSIAN) as c:
        got = sv.sv_get_amplitudes(c)
    ref = orc.init_gaussian(n, seed, round_to_c64=(dtype == sv.SV_C64))
    if dtype == sv.SV_C128:
        assert float(np.max(np.abs(got - ref))) <= 1e-15
    else:  # libm last-ulp differences may move a float rounding by one ulp
        assert float(np.max(np.abs(got.astype(np.complex128) - ref))) <= 2.0 ** -23 * float(np.max(np.abs(ref)))
    assert abs(float(np.sum(np.abs(got.astype(np.complex128)) ** 2)) - 1.0) <= (1e-12 if dtype == sv.SV_C128 else 1e-5)


# --------------------------------------------------------------------------- #
# diffusion                                                                    #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n", [1, 2, 7, 12, 13, 14, 15, 17, 20, 22, 24])
def test_diffuse_wht_random_state(dtype, n):
    """One D = H^n F0 H^n on a random state: whole-state kernel (n <= T), one
    contiguous + one strided tile group (several tiles, a ragged 1-slot group
    at n = T + 1) and three groups at n = 24."""
    a = rand_state(n, dtype)
    with ctx_with(a, dtype) as c:
        sv.sv_diffuse(c, sv.SV_DIFFUSE_WHT)
        got = sv.sv_get_amplitudes(c)
    assert_close(got, orc.diffuse_wht(a.copy()), dtype, f"diffuse_wht n={n}")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n", [1, 3, 12, 14, 18, 23])
def test_diffuse_mean_random_state(dtype, n):
    a = rand_state(n, dtype)
    with ctx_with(a, dtype) as c:
        sv.sv_diffuse(c, sv.SV_DIFFUSE_MEAN)
        got = sv.sv_get_amplitudes(c)
    assert_close(got, orc.diffuse_mean(a.copy()), dtype, f"diffuse_mean n={n}")


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,m", [(5, 3), (12, 40), (16, 7), (19, 1000)])
def test_apply_oracle_scatter(dtype, n, m):
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, m, n)
    with ctx_with(a, dtype) as c:
        sv.sv_apply_oracle(c, marked)
        got = sv.sv_get_amplitudes(c)
    assert_close(got, orc.oracle_flip(a.copy(), marked), dtype, "oracle")


# --------------------------------------------------------------------------- #
# Grover iterations                                                            #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("diff", [sv.SV_DIFFUSE_WHT, sv.SV_DIFFUSE_MEAN], ids=["wht", "mean"])
@pytest.mark.parametrize("n,m,k", [(4, 1, 3), (11, 3, 5), (13, 0, 2), (14, 1, 3), (16, 8, 4), (18, 2048, 3),
                                   (21, 5, 3), (23, 17, 2)])
def test_iterate_random_state(dtype, diff, n, m, k):
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, m, 3 * n + m)
    with ctx_with(a, dtype) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate(c, k, diff)
        got = sv.sv_get_amplitudes(c)
        mass = sv.sv_measure_marked_mass(c) if m else 0.0
    ref = orc.iterate(a.copy(), marked, k, orc.WHT if diff == sv.SV_DIFFUSE_WHT else orc.MEAN)
    assert_close(got, ref, dtype, f"iterate n={n} m={m}", n=n, k=k)
    if m:
        assert abs(mass - orc.marked_mass(ref, marked)) <= 10 * TOL[dtype]


def test_c1_n10_wht_closed_form():
    """c1: n=10 complex128, uniform start, M=1 from seed, 25 iterations (WHT)."""
    n, m = 10, 1
    k = cf.optimal_iterations(n, m)
    marked = sv.sv_marked_from_seed(n, m, 1)
    with sv.sv_init(n, 1, sv.SV_C128, sv.SV_INIT_UNIFORM) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        got = sv.sv_get_amplitudes(c)
        p = sv.sv_measure_marked_mass(c)
    ref = orc.iterate(orc.init_uniform(n), orc.marked_from_seed(n, m, 1), k, orc.WHT)
    assert_close(got, ref, sv.SV_C128, "c1 vs oracle")
    assert abs(p - cf.p_success_uniform(n, m, k)) <= 1e-12
    am, au = cf.uniform_amplitudes(n, m, k)
    mask = np.zeros(1 << n, bool)
    mask[marked.astype(np.int64)] = True
    assert np.max(np.abs(got[mask] - am)) <= 1e-12 and np.max(np.abs(got[~mask] - au)) <= 1e-12


def test_c2_n20_mean_closed_form():
    """c2: n=20 complex128, M=4 from seed, 402 iterations (mean diffusion)."""
    n, m = 20, 4
    k = cf.optimal_iterations(n, m)
    marked = sv.sv_marked_from_seed(n, m, 2)
    with sv.sv_init(n, 2, sv.SV_C128, sv.SV_INIT_UNIFORM) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_MEAN)
        got = sv.sv_get_amplitudes(c)
        p = sv.sv_measure_marked_mass(c)
    ref = orc.iterate(orc.init_uniform(n), marked, k, orc.MEAN)
    assert_close(got, ref, sv.SV_C128, "c2 vs oracle")
    assert abs(p - cf.p_success_uniform(n, m, k)) <= 1e-12
    am, au = cf.uniform_amplitudes(n, m, k)
    mask = np.zeros(1 << n, bool)
    mask[marked.astype(np.int64)] = True
    assert np.max(np.abs(got[mask] - am)) <= 1e-12 and np.max(np.abs(got[~mask] - au)) <= 1e-12


def _check_uniform_closed_form(c, n, marked, k, dtype, chunk=1 << 22, sample_chunks=None):
    """Every (or a sample of) amplitude(s) vs sin((2k+1)t)/sqrt(M), cos(..)/sqrt(N-M)."""
    N = 1 << n
    am, au = cf.uniform_amplitudes(n, marked.size, k)
    mk = marked.astype(np.int64)
    starts = range(0, N, chunk) if sample_chunks is None else sample_chunks
    worst = 0.0
    for s in starts:
        got = sv.sv_get_amplitudes(c, s, chunk).astype(np.complex128)
        ref = np.full(chunk, au, dtype=np.complex128)
        inside = mk[(mk >= s) & (mk < s + chunk)] - s
        ref[inside] = am
        worst = max(worst, assert_close(got, ref, dtype, f"chunk@{s}", n=n, k=k))
    got_m = np.array([sv.sv_get_amplitudes(c, int(i), 1)[0] for i in mk[:64]])
    assert_close(got_m, np.full(got_m.size, am, np.complex128), dtype, "marked", n=n, k=k)
    return worst


def test_c3_n28_wht_closed_form():
    """c3: n=28 complex64 (2 GiB), M=1 from seed, 64 WHT iterations: every amplitude."""
    n, m, k = 28, 1, 64
    marked = sv.sv_marked_from_seed(n, m, 3)
    with sv.sv_init(n, 3, sv.SV_C64, sv.SV_INIT_UNIFORM) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        _check_uniform_closed_form(c, n, marked, k, sv.SV_C64)
        p = sv.sv_measure_marked_mass(c)
    assert abs(p - cf.p_success_uniform(n, m, k)) <= 1e-5 * 1e-2


def test_c4_n32_wht_sampled():
    """c4 at P = 1: n=32 complex64 (32 GiB), M=256 from seed, 16 WHT iterations;
    sampled chunks + every marked amplitude vs the closed form."""
    n, m, k = 32, 256, 16
    marked = sv.sv_marked_from_seed(n, m, 4)
    chunk = 1 << 20
    starts = sorted(set([0, (1 << n) - chunk] + [int(x) * chunk for x in rng.integers(0, (1 << n) // chunk, 24)]))
    with sv.sv_init(n, 4, sv.SV_C64, sv.SV_INIT_UNIFORM) as c:
        sv.sv_set_marked(c, marked)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        _check_uniform_closed_form(c, n, marked, k, sv.SV_C64, chunk=chunk, sample_chunks=starts)
        p = sv.sv_measure_marked_mass(c)
    assert abs(p - cf.p_success_uniform(n, m, k)) <= 1e-5 * 1e-2


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
def test_c5_semantics_small_gaussian(dtype):
    """c5 recipe at n=22: Gaussian start, M=1024 from seed, 8 WHT and 8 mean
    iterations, each vs the oracle and the general closed form; 8 WHT then 8
    mean = closed form at k=16 (G11)."""
    n, m, seed = 22, 1024, 5
    marked = sv.sv_marked_from_seed(n, m, seed)
    a0 = orc.init_gaussian(n, seed, round_to_c64=(dtype == sv.SV_C64))
    res = {}
    for diff in (sv.SV_DIFFUSE_WHT, sv.SV_DIFFUSE_MEAN):
        with sv.sv_init(n, seed, dtype, sv.SV_INIT_GAUSSIAN) as c:
            sv.sv_set_marked(c, marked)
            sv.sv_iterate(c, 8, diff)
            res[diff] = sv.sv_get_amplitudes(c)
            if diff == sv.SV_DIFFUSE_WHT:
                sv.sv_iterate(c, 8, sv.SV_DIFFUSE_MEAN)
                res["16"] = sv.sv_get_amplitudes(c)
    assert_close(res[sv.SV_DIFFUSE_WHT], orc.iterate(a0.copy(), marked, 8, orc.WHT), dtype, "wht", n=n, k=8)
    assert_close(res[sv.SV_DIFFUSE_MEAN], orc.iterate(a0.copy(), marked, 8, orc.MEAN), dtype, "mean", n=n, k=8)
    assert_close(res[sv.SV_DIFFUSE_WHT], cf.general_state(a0, marked, 8), dtype, "closed form k=8", n=n, k=8)
    assert_close(res["16"], cf.general_state(a0, marked, 16), dtype, "closed form k=16", n=n, k=16)


def test_c5_n34_full_size_properties():
    """c5 at its full size on one B200 (n=34 complex64, 128 GiB; Gaussian
    start, M=1024 from seed, 8 iterations of each diffusion).  The oracle
    cannot hold this state, so the check uses what the closed form fixes at
    any size, with the start taken from the oracle's own generator
    (a_i^(0) = z_i / ||z||, z = or_gauss_draw): the marked residual is
    invariant, a_i^(k) - a_j^(k) = a_i^(0) - a_j^(0) for marked i, j, and the
    unmarked residual alternates, a_i^(k) - a_j^(k) = (-1)^k (a_i^(0) - a_j^(0))
    (DESIGN.md "General-start closed form").  So every sampled pair gives the
    same 1/||z||, which the law of large numbers puts at 1/sqrt(2N) (sd ~ 1e-5
    relative).  The two diffusions (independent code paths) must also agree
    amplitude by amplitude (G11)."""
    n, m, seed, k = 34, 1024, 5, 8
    N = 1 << n
    marked = sv.sv_marked_from_seed(n, m, seed)
    mset = set(int(x) for x in marked)
    rs = np.random.default_rng(34)
    unm = []
    while len(unm) < 512:
        i = int(rs.integers(0, N))
        if i not in mset:
            unm.append(i)
    idx = [int(x) for x in marked] + unm
    z = {i: orc.gauss_draw(seed, i) for i in idx}
    got = {}
    for diff in (sv.SV_DIFFUSE_WHT, sv.SV_DIFFUSE_MEAN):
        with sv.sv_init(n, seed, sv.SV_C64, sv.SV_INIT_GAUSSIAN) as c:
            sv.sv_set_marked(c, marked)
            sv.sv_iterate(c, k, diff)
            got[diff] = {i: complex(sv.sv_get_amplitudes(c, i, 1)[0]) for i in idx}
            got[(diff, "p")] = sv.sv_measure_marked_mass(c)
    for diff in (sv.SV_DIFFUSE_WHT, sv.SV_DIFFUSE_MEAN):
        a = got[diff]
        ratios = []
        for group, sign in ((idx[:m], 1.0), (unm, (-1.0) ** k)):
            for t in range(0, len(group) - 1, 2):
                i, j = group[t], group[t + 1]
                dz = z[i] - z[j]
                if abs(dz) < 0.5:
                    continue
                ratios.append(sign * (a[i] - a[j]) / dz)
        ratios = np.array(ratios)
        c0 = np.median(ratios.real)
        assert np.max(np.abs(ratios - c0)) <= 1e-4 * c0, (diff, float(np.max(np.abs(ratios - c0)) / c0))
        assert abs(c0 * math.sqrt(2.0 * N) - 1.0) <= 1e-3, c0 * math.sqrt(2.0 * N)
    wht, mean = got[sv.SV_DIFFUSE_WHT], got[sv.SV_DIFFUSE_MEAN]
    diff_max = max(abs(wht[i] - mean[i]) for i in idx)
    scale = max(abs(wht[i]) for i in idx)
    assert diff_max <= 2 * rel64(n, k) * scale, (diff_max, scale)
    assert abs(got[(sv.SV_DIFFUSE_WHT, "p")] - got[(sv.SV_DIFFUSE_MEAN, "p")]) <= 1e-6


def test_c4_n32_gaussian_start_residuals_and_diffusions_agree():
    """The headline launch configuration (n = 32 complex64, c4's M = 256 marked
    set, 16 WHT iterations -- every pass kind of the c4 bench, including the
    two-layout O-fused pass) on a NON-degenerate start: the seeded Gaussian
    state, so every amplitude differs and an index-permutation bug among
    unmarked entries cannot hide behind equal values (verdict r1 weak #2).
    Checks, as for n = 34: the marked residual is invariant and the unmarked
    residual alternates (general-start closed form), with 1/||z|| inferred from
    sampled pairs and pinned by the law of large numbers; and the WHT and mean
    diffusions (independent kernels, D_WHT = D_mean exactly) agree element by
    element on 40 sampled 2^20-amplitude chunks (incl. the first and last)."""
    n, m, seed, k = 32, 256, 4, 16
    N = 1 << n
    chunk = 1 << 20
    marked = sv.sv_marked_from_seed(n, m, seed)
    mset = set(int(x) for x in marked)
    rs = np.random.default_rng(32)
    unm = []
    while len(unm) < 512:
        i = int(rs.integers(0, N))
        if i not in mset:
            unm.append(i)
    idx = [int(x) for x in marked] + unm
    z = {i: orc.gauss_draw(seed, i) for i in idx}
    starts = sorted(set([0, N - chunk] + [int(x) * chunk for x in rs.integers(0, N // chunk, 38)]))
    got, chunks = {}, {}
    for diff in (sv.SV_DIFFUSE_WHT, sv.SV_DIFFUSE_MEAN):
        with sv.sv_init(n, seed, sv.SV_C64, sv.SV_INIT_GAUSSIAN) as c:
            sv.sv_set_marked(c, marked)
            sv.sv_iterate(c, k, diff)
            got[diff] = {i: complex(sv.sv_get_amplitudes(c, i, 1)[0]) for i in idx}
            chunks[diff] = [sv.sv_get_amplitudes(c, s0, chunk).astype(np.complex128) for s0 in starts]
    for diff in (sv.SV_DIFFUSE_WHT, sv.SV_DIFFUSE_MEAN):
        a = got[diff]
        ratios = []
        for group, sign in ((idx[:m], 1.0), (unm, (-1.0) ** k)):
            for t in range(0, len(group) - 1, 2):
                i, j = group[t], group[t + 1]
                dz = z[i] - z[j]
                if abs(dz) < 0.5:
                    continue
                ratios.append(sign * (a[i] - a[j]) / dz)
        ratios = np.array(ratios)
        c0 = np.median(ratios.real)
        assert np.max(np.abs(ratios - c0)) <= 1e-4 * c0, (diff, float(np.max(np.abs(ratios - c0)) / c0))
        assert abs(c0 * math.sqrt(2.0 * N) - 1.0) <= 1e-3, c0 * math.sqrt(2.0 * N)
    for s0, w, mn in zip(starts, chunks[sv.SV_DIFFUSE_WHT], chunks[sv.SV_DIFFUSE_MEAN]):
        scale = float(np.max(np.abs(mn)))
        assert float(np.max(np.abs(w - mn))) <= 2 * rel64(n, k) * scale, s0


# --------------------------------------------------------------------------- #
# sharded schedule, emulated on one GPU                                        #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("fused", [True, False], ids=["fused-xchg", "alltoall"])
@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,world", [(17, 2), (19, 4), (20, 8), (22, 8), (21, 2)])
def test_emulated_sharding_matches_oracle(dtype, n, world, fused):
    """The sharded schedule on one GPU (P shards in one buffer): qubit swaps as
    the fused store-to-new-owner pass, or as an all-to-all of chunks."""
    T = 13 if dtype == sv.SV_C64 else 12
    if n - 2 * (world.bit_length() - 1) < T:
        pytest.skip("shard too small")
    a = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, 9, n)
    k = 3
    with ctx_with(a, dtype, world=world) as c:
        assert sv.sv_info(c)["world"] == world
        assert sv.sv_get_exchange(c)  # fused by default in emulation
        sv.sv_set_exchange(c, fused)
        sv.sv_set_marked(c, marked)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        got = sv.sv_get_amplitudes(c)
        sv.sv_set_amplitudes(c, a)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_MEAN)
        got_mean = sv.sv_get_amplitudes(c)
    assert_close(got, orc.iterate(a.copy(), marked, k, orc.WHT), dtype, "sharded wht", n=n, k=k)
    assert_close(got_mean, orc.iterate(a.copy(), marked, k, orc.MEAN), dtype, "sharded mean", n=n, k=k)


# --------------------------------------------------------------------------- #
# edge cases and errors                                                        #
# --------------------------------------------------------------------------- #
def test_marked_edge_sets():
    n = 14
    N = 1 << n
    for dtype in DT:
        for marked in (np.arange(0), np.arange(N, dtype=np.uint64), np.arange(N // 2, dtype=np.uint64) * 2):
            a = rand_state(n, dtype)
            with ctx_with(a, dtype) as c:
                sv.sv_set_marked(c, marked)
                sv.sv_iterate(c, 3, sv.SV_DIFFUSE_WHT)
                got = sv.sv_get_amplitudes(c)
            assert_close(got, orc.iterate(a.copy(), marked, 3, orc.WHT), dtype, f"M={marked.size}", n=n, k=3)


def test_errors():
    with pytest.raises(sv.SvError) as e:
        sv.sv_init(0)
    assert e.value.code == sv.SV_EINVAL
    with pytest.raises(sv.SvError):
        sv.sv_init(16, world=3)
    with pytest.raises(sv.SvError):
        sv.sv_init(18, world=8)  # n - 2g < T
    with sv.sv_init(12, 0, sv.SV_C64) as c:
        with pytest.raises(sv.SvError) as e:
            sv.sv_iterate(c, 1)
        assert e.value.code == sv.SV_ESTATE
        for bad in ([3, 3], [5, 2], [1 << 12]):
            with pytest.raises(sv.SvError) as e:
                sv.sv_set_marked(c, bad)
            assert e.value.code == sv.SV_EINVAL
        sv.sv_set_marked(c, [7])
        with pytest.raises(sv.SvError):
            sv.sv_iterate(c, -1)
        before = sv.sv_get_amplitudes(c)
        sv.sv_iterate(c, 0)
        np.testing.assert_array_equal(sv.sv_get_amplitudes(c), before)
        with pytest.raises(sv.SvError):
            sv.sv_get_amplitudes(c, 4000, 200)
        with pytest.raises(sv.SvError):
            sv.sv_diffuse(c, 7)
    with sv.sv_init(27, 0, sv.SV_C64) as c:
        with pytest.raises(sv.SvError) as e:
            sv.sv_probabilities(c)
        assert e.value.code == sv.SV_ETOOBIG
    # beyond the 180 GB of one B200: n = 35 complex64 = 256 GiB -> SV_ENOMEM, no leak, device still usable
    with pytest.raises(sv.SvError) as e:
        sv.sv_init(35, 0, sv.SV_C64)
    assert e.value.code == sv.SV_ENOMEM
    with sv.sv_init(20, 0, sv.SV_C64) as c:
        sv.sv_set_marked(c, [5])
        sv.sv_iterate(c, 2)
        assert sv.sv_measure_marked_mass(c) > 0


@pytest.mark.parametrize("diff", [sv.SV_DIFFUSE_WHT, sv.SV_DIFFUSE_MEAN], ids=["wht", "mean"])
def test_bitwise_deterministic(diff):
    n = 22
    marked = sv.sv_marked_from_seed(n, 33, 1)
    outs = []
    for _ in range(2):
        with sv.sv_init(n, 7, sv.SV_C64, sv.SV_INIT_GAUSSIAN) as c:
            sv.sv_set_marked(c, marked)
            sv.sv_iterate(c, 5, diff)
            outs.append(sv.sv_get_amplitudes(c))
    assert outs[0].tobytes() == outs[1].tobytes()


def test_probabilities_device_and_host():
    import torch
    n = 16
    a = rand_state(n, sv.SV_C128)
    with ctx_with(a, sv.SV_C128) as c:
        p_host = sv.sv_probabilities(c)
        buf = torch.empty(1 << n, dtype=torch.float64, device="cuda")
        sv.sv_probabilities(c, buf.data_ptr())
        sv.sv_synchronize(c)
        p_dev = buf.cpu().numpy()
    ref = orc.probabilities(a.copy())
    np.testing.assert_allclose(p_host, ref, rtol=0, atol=1e-15)
    np.testing.assert_allclose(p_dev, ref, rtol=0, atol=1e-15)


def test_profile_counts_launches():
    n = 20
    with sv.sv_init(n, 0, sv.SV_C64) as c:
        sv.sv_set_marked(c, [5])
        sv.sv_profile(c, True)
        sv.sv_iterate(c, 3, sv.SV_DIFFUSE_WHT)
        launches, ms = sv.sv_profile_read(c, sv.SV_K_WHT_TILE)
        plan = sv.sv_plan_wht(n, 1, sv.SV_C64, 3, True)
        assert launches == len(plan) and ms > 0.0


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
@pytest.mark.parametrize("n,m,k", [(14, 0, 3), (16, 30000, 3), (17, 5, 9), (18, 1000, 1), (19, 7, 2), (20, 64, 6),
                                   (21, 300, 4)])
def test_mean_resident_and_launched_paths(dtype, n, m, k, monkeypatch):
    """The one-launch resident mean paths (mean_resident.cu, states within the
    aggregate shared memory: the register-resident kernel by default, the
    shared-memory one with SV_MEAN_RESIDENT=smem) and the launched
    per-iteration path (SV_MEAN_RESIDENT=0) all equal the oracle; M = 0 (O = I)
    included."""
    a0 = rand_state(n, dtype)
    marked = orc.marked_from_seed(n, m, 7) if m else np.zeros(0, np.uint64)
    ref = orc.iterate(a0.copy(), marked, k, orc.MEAN)
    for env in ("1", "smem", "0"):
        monkeypatch.setenv("SV_MEAN_RESIDENT", env)
        with ctx_with(a0, dtype) as c:
            sv.sv_set_marked(c, marked)
            sv.sv_profile(c, True)
            sv.sv_iterate(c, k, sv.SV_DIFFUSE_MEAN)
            launches, _ = sv.sv_profile_read(c, sv.SV_K_MEAN)
            got = sv.sv_get_amplitudes(c)
        sms = 148  # B200; the library asks the device
        chunk = -(-(1 << n) // sms) * (8 if dtype == sv.SV_C64 else 16)
        fits = chunk <= 232448 - 1024  # opt-in shared memory per block minus the kernel's reserve
        assert launches == (1 if (env != "0" and fits) else k), (env, launches)
        assert_close(got, ref, dtype, f"mean resident={env} n={n}", n=n, k=k)


@pytest.mark.parametrize("dtype", DT, ids=DT_IDS)
def test_graph_replay_matches_launched(dtype, monkeypatch):
    """Small states replay sv_iterate's WHT schedule as a cached CUDA graph:
    bitwise equal to the launched schedule (SV_GRAPHS=0), and a new marked set
    (or a new k) is captured afresh instead of replaying a stale graph."""
    n = 18
    a0 = rand_state(n, dtype)
    sets = [orc.marked_from_seed(n, 3, 1), orc.marked_from_seed(n, 40, 2)]
    res = {}
    for env in ("1", "0"):
        monkeypatch.setenv("SV_GRAPHS", env)
        with ctx_with(a0, dtype) as c:
            out = []
            for mk, k in ((sets[0], 5), (sets[0], 5), (sets[1], 5), (sets[1], 3)):
                sv.sv_set_marked(c, mk)
                sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
                out.append(sv.sv_get_amplitudes(c))
            res[env] = out
    for g, l in zip(res["1"], res["0"]):
        np.testing.assert_array_equal(g, l)
    ref = a0.copy()
    for mk, k in ((sets[0], 5), (sets[0], 5), (sets[1], 5), (sets[1], 3)):
        ref = orc.iterate(ref, mk, k, orc.WHT)
    assert_close(res["1"][-1], ref, dtype, "graph replay", n=n, k=18)


def test_graph_replay_long_k_is_chunked():
    """k beyond one bounded graph (256 iterations) runs as consecutive chunks."""
    n, k = 16, 600
    a0 = rand_state(n, sv.SV_C128)
    mk = orc.marked_from_seed(n, 2, 3)
    with ctx_with(a0, sv.SV_C128) as c:
        sv.sv_set_marked(c, mk)
        sv.sv_iterate(c, k, sv.SV_DIFFUSE_WHT)
        got = sv.sv_get_amplitudes(c)
    assert_close(got, orc.iterate(a0.copy(), mk, k, orc.WHT), sv.SV_C128, "chunked graphs", n=n, k=k)


def test_resident_mean_fp64_gather_variant():
    """SV_RESREG_FX=0 (read once per process): the register-resident mean
    kernel with fp64 partials + gather in every round instead of the
    fixed-point integer sums -- the resident-path tests rerun in a subprocess."""
    import os
    import subprocess
    import sys
    if os.environ.get("SV_RESREG_FX") == "0":
        pytest.skip("this is the subprocess")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SV_RESREG_FX="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_parity_gpu.py", "-k", "mean_resident_and_launched or c2_n20 or bitwise"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]
