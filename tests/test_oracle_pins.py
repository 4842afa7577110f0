"""Pins of the CPU oracle against what the paper and mathematics fix.

Every function in oracle/ is checked against something other than itself:
paper figures (golden files), library routines (scipy's Sylvester Hadamard,
numpy Kronecker products / matrix powers), exact closed forms, exact special
cases and invariants.  CPU only (-m "not gpu").
"""
import ctypes
import math
import os

import numpy as np
import pytest
import scipy.linalg

from oracle import closed_form as cf
from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
rng = np.random.default_rng(20240417)


def crandn(N):
    return np.ascontiguousarray(rng.standard_normal(N) + 1j * rng.standard_normal(N))


# --------------------------------------------------------------------------- #
# Paper figures                                                                #
# --------------------------------------------------------------------------- #
def test_fig1_qubit_states_golden():
    """Fig. 1(a)/(b): |0> and the 1-qubit superposition."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "fig1_qubit_states.txt")) if l.strip() and l[0] != "#"]
    a_zero = orc.init_zero_state(1)
    a_sup = orc.init_uniform(1)  # H|0>
    for panel, n, idx, re, im, p in rows:
        a = a_zero if panel == "a" else a_sup
        idx = int(idx)
        assert a[idx] == pytest.approx(complex(float(re), float(im)), abs=1e-16)
        assert orc.probabilities(a)[idx] == pytest.approx(float(p), abs=4e-16)  # (2^-1/2)^2 rounds to 0.5+ulp
    # probabilities sum to one
    assert orc.probabilities(a_sup).sum() == pytest.approx(1.0, abs=1e-15)


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_fig3_pair_transform_is_kron_operator(n):
    """Fig. 3 / section 2.1: a 2x2 on bit q acts on the V/2 pairs
    differing only in bit q.  Independent construction: the VxV matrix of the
    gate (section 1.3) I_{2^{n-q-1}} (x) U (x) I_{2^q} with numpy.kron."""
    for q in range(n):
        U = crandn(4).reshape(2, 2)
        a = crandn(1 << n)
        G = np.kron(np.kron(np.eye(1 << (n - q - 1)), U), np.eye(1 << q))
        got = orc.apply_2x2(a.copy(), q, U[0, 0], U[0, 1], U[1, 0], U[1, 1])
        np.testing.assert_allclose(got, G @ a, rtol=0, atol=1e-13)


def test_fig3_four_state_example_pairs_lsb():
    """Fig. 3 on a four-element vector: the LSB transform pairs (a0,a1), (a2,a3);
    the transform on bit 1 pairs (a0,a2), (a1,a3) -- checked by which entries
    an arbitrary 2x2 mixes."""
    a = np.array([1, 0, 0, 0], dtype=np.complex128)
    out = orc.apply_2x2(a.copy(), 0, 2, 3, 5, 7)  # [w x; y z] = [2 3; 5 7]
    np.testing.assert_array_equal(out, [2, 5, 0, 0])
    out = orc.apply_2x2(a.copy(), 1, 2, 3, 5, 7)
    np.testing.assert_array_equal(out, [2, 0, 5, 0])


# --------------------------------------------------------------------------- #
# Walsh-Hadamard transform                                                     #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("n", range(1, 11))
def test_wht_equals_sylvester_hadamard(n):
    """Unnormalised W = Sylvester Hadamard matrix (scipy.linalg.hadamard)."""
    a = crandn(1 << n)
    W = scipy.linalg.hadamard(1 << n).astype(np.float64)
    np.testing.assert_allclose(orc.wht(a.copy()), W @ a, rtol=0, atol=1e-11 * (1 << n))


@pytest.mark.parametrize("n", range(0, 7))
def test_dense_kron_hadamard_is_normalised_sylvester(n):
    K = orc.dense_hadamard(n)
    W = scipy.linalg.hadamard(1 << n).astype(np.float64) if n else np.ones((1, 1))
    np.testing.assert_allclose(K, W / math.sqrt(1 << n), rtol=0, atol=1e-14)
    np.testing.assert_allclose(K @ K, np.eye(1 << n), rtol=0, atol=1e-13)  # H^n involution


@pytest.mark.parametrize("n", [1, 4, 9, 14])
def test_wht_twice_is_N_identity(n):
    a = crandn(1 << n)
    b = orc.wht(orc.wht(a.copy()))
    np.testing.assert_allclose(b, a * (1 << n), rtol=0, atol=1e-10 * (1 << n))


# --------------------------------------------------------------------------- #
# Diffusion                                                                    #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("n", [1, 2, 3, 6, 10, 13])
def test_diffusions_equal_dense_reflection(n):
    """D = H^n F0 H^n = 2|s><s| - I; both independent code paths (WHT butterflies,
    mean reduction) equal the dense reflection, hence each other (G2)."""
    N = 1 << n
    a = crandn(N)
    if n <= 6:
        K = orc.dense_hadamard(n)
        F0 = -np.eye(N)
        F0[0, 0] = 1.0
        D = 2.0 * np.full((N, N), 1.0 / N) - np.eye(N)
        np.testing.assert_allclose(K @ F0 @ K, D, rtol=0, atol=1e-13)
        ref = D @ a
    else:
        ref = 2.0 * a.mean() - a  # numpy mean as the library routine
    np.testing.assert_allclose(orc.diffuse_wht(a.copy()), ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(orc.diffuse_mean(a.copy()), ref, rtol=0, atol=1e-12)


def test_diffusion_invariants():
    """D^2 = I, D|s> = |s>, O^2 = I, D preserves sum_i a_i."""
    n = 9
    a = crandn(1 << n)
    marked = orc.marked_from_seed(n, 7, 3)
    np.testing.assert_allclose(orc.diffuse_wht(orc.diffuse_wht(a.copy())), a, atol=1e-13)
    s = orc.init_uniform(n)
    np.testing.assert_allclose(orc.diffuse_mean(s.copy()), s, atol=1e-16)
    np.testing.assert_allclose(orc.diffuse_wht(s.copy()), s, atol=1e-15)
    np.testing.assert_array_equal(orc.oracle_flip(orc.oracle_flip(a.copy(), marked), marked), a)
    assert orc.state_sum(orc.diffuse_wht(a.copy())) == pytest.approx(a.sum(), abs=1e-12)


def test_state_sum_matches_math_fsum():
    a = crandn(1 << 16)
    s = orc.state_sum(a)
    assert s.real == pytest.approx(math.fsum(a.real), abs=1e-13)
    assert s.imag == pytest.approx(math.fsum(a.imag), abs=1e-13)


# --------------------------------------------------------------------------- #
# The Grover iteration                                                         #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("n,m", [(1, 1), (2, 1), (3, 2), (4, 3), (5, 1), (6, 9), (6, 0), (6, 64)])
def test_iterate_equals_dense_matrix_power(n, m):
    """(D O)^k a with dense numpy matrices (section 1.3's VxV transformation)."""
    N = 1 << n
    a0 = crandn(N)
    a0 /= np.linalg.norm(a0)
    marked = orc.marked_from_seed(n, m, 11 + n)
    O = np.eye(N)
    O[marked, marked] = -1.0
    D = 2.0 * np.full((N, N), 1.0 / N) - np.eye(N)
    G = D @ O
    for k in (0, 1, 2, 5, 11):
        ref = np.linalg.matrix_power(G, k) @ a0
        for diff in (orc.WHT, orc.MEAN):
            got = orc.iterate(a0.copy(), marked, k, diff)
            np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)


def test_c1_closed_form():
    """c1: n=10, M=1, k=floor(pi/4 sqrt N)=25, WHT diffusion: sin^2((2k+1)theta)."""
    n, m = 10, 1
    k = cf.optimal_iterations(n, m)
    assert k == 25
    marked = orc.marked_from_seed(n, m, 1)
    a = orc.iterate(orc.init_uniform(n), marked, k, orc.WHT)
    am, au = cf.uniform_amplitudes(n, m, k)
    is_m = np.zeros(1 << n, bool)
    is_m[marked.astype(np.int64)] = True
    np.testing.assert_allclose(a[is_m], am, rtol=0, atol=1e-13)
    np.testing.assert_allclose(a[~is_m], au, rtol=0, atol=1e-13)
    assert orc.marked_mass(a, marked) == pytest.approx(cf.p_success_uniform(n, m, k), abs=1e-13)
    assert cf.p_success_uniform(n, m, k) == pytest.approx(0.9994612447444079, abs=1e-15)


@pytest.mark.parametrize("diffusion,k", [(orc.MEAN, None), (orc.WHT, 3)])
def test_c2_closed_form(diffusion, k):
    """c2: n=20, M=4, k=402 (mean); the WHT variant at k=3 (runtime bound)."""
    n, m = 20, 4
    if k is None:
        k = cf.optimal_iterations(n, m)
        assert k == 402
    marked = orc.marked_from_seed(n, m, 2)
    assert len(set(marked.tolist())) == 4
    a = orc.iterate(orc.init_uniform(n), marked, k, diffusion)
    am, au = cf.uniform_amplitudes(n, m, k)
    is_m = np.zeros(1 << n, bool)
    is_m[marked.astype(np.int64)] = True
    np.testing.assert_allclose(a[is_m], am, rtol=0, atol=1e-12)
    np.testing.assert_allclose(a[~is_m], au, rtol=0, atol=1e-12)
    assert abs(orc.norm_sq(a) - 1.0) <= 1e-9


def test_exact_special_cases():
    """N=4, M=1, k=1 gives P=1 (theta=pi/6); M=N/4, k=1 gives P=1; M=N/2 gives
    P=1/2 for every k.  Here every intermediate is an exact binary fraction."""
    for diff in (orc.WHT, orc.MEAN):
        for mk in range(4):
            a = orc.iterate(orc.init_uniform(2), np.array([mk], np.uint64), 1, diff)
            assert orc.marked_mass(a, np.array([mk], np.uint64)) == pytest.approx(1.0, abs=1e-15)
        for n in range(2, 6):
            marked = orc.marked_from_seed(n, (1 << n) // 4, 5)
            a = orc.iterate(orc.init_uniform(n), marked, 1, diff)
            assert orc.marked_mass(a, marked) == pytest.approx(1.0, abs=1e-14)
        n = 6
        marked = orc.marked_from_seed(n, 32, 9)
        a = orc.init_uniform(n)
        for k in range(8):
            assert orc.marked_mass(a, marked) == pytest.approx(0.5, abs=1e-14)
            orc.iterate(a, marked, 1, diff)


@pytest.mark.parametrize("n,m,seed", [(8, 1, 1), (10, 5, 2), (12, 37, 3), (9, 0, 4), (9, 512, 5), (11, 1024, 6)])
def test_general_start_closed_form(n, m, seed):
    """Gaussian start (G8): every amplitude and the marked mass vs the closed form."""
    a0 = orc.init_gaussian(n, seed)
    marked = orc.marked_from_seed(n, m, seed)
    for k in (1, 2, 7, 20):
        for diff in (orc.WHT, orc.MEAN):
            got = orc.iterate(a0.copy(), marked, k, diff)
            np.testing.assert_allclose(got, cf.general_state(a0, marked, k), rtol=0, atol=1e-12)
            assert orc.marked_mass(got, marked) == pytest.approx(cf.general_marked_mass(a0, marked, k), abs=1e-12)
            assert abs(orc.norm_sq(got) - 1.0) < 1e-12


def test_closed_form_uniform_is_general_special_case():
    n, m, k = 12, 3, 17
    a0 = orc.init_uniform(n)
    marked = orc.marked_from_seed(n, m, 1)
    am, au = cf.uniform_amplitudes(n, m, k)
    st = cf.general_state(a0, marked, k)
    is_m = np.zeros(1 << n, bool)
    is_m[marked.astype(np.int64)] = True
    np.testing.assert_allclose(st[is_m], am, atol=1e-15)
    np.testing.assert_allclose(st[~is_m], au, atol=1e-15)


def test_pinned_closed_form_values():
    """The c1-c4 values of SURVEY.md 8(c) (sin^2((2k+1)theta) at the BJ configs)."""
    assert cf.p_success_uniform(10, 1, 25) == pytest.approx(0.9994612447444079, abs=1e-15)
    assert cf.p_success_uniform(20, 4, 402) == pytest.approx(0.99999783822585953, abs=1e-15)
    assert cf.p_success_uniform(28, 1, 64) == pytest.approx(6.1991274918609562e-05, rel=1e-12)
    assert cf.p_success_uniform(32, 256, 16) == pytest.approx(6.4908055049548032e-05, rel=1e-12)
    assert cf.uniform_amplitudes(28, 1, 64)[1] == pytest.approx(6.1033264510787869e-05, rel=1e-12)


# --------------------------------------------------------------------------- #
# Seeded generators                                                            #
# --------------------------------------------------------------------------- #
def test_splitmix64_reference_vector():
    vals = [l.strip() for l in open(os.path.join(GOLDEN, "splitmix64_vectors.txt")) if l.strip() and l[0] != "#"]
    seed = int(vals[0].split()[1])
    st = ctypes.c_uint64(seed)
    got = [orc.lib().or_splitmix64_next(ctypes.byref(st)) for _ in range(5)]
    assert got == [int(v) for v in vals[1:]]


@pytest.mark.parametrize("n", [1, 2, 3, 7, 12, 16])
def test_perm_is_bijection(n):
    img = {orc.perm(n, 77, x) for x in range(1 << n)}
    assert img == set(range(1 << n))


def test_marked_set_sorted_distinct_in_range():
    for n, m in [(10, 1), (20, 4), (28, 1), (32, 256), (34, 1024), (12, 4096)]:
        mk = orc.marked_from_seed(n, m, n)
        assert mk.size == m
        assert np.all(np.diff(mk.astype(np.float64)) > 0) if m > 1 else True
        assert int(mk.max()) < (1 << n)
    with pytest.raises(ValueError):
        orc.marked_from_seed(3, 9, 0)


def test_gaussian_draws_are_standard_normal():
    """Box-Muller from the counter hash: re, im ~ iid N(0,1) (G8) -- moments
    within 6 sigma over 2^16 draws."""
    n = 16
    z = np.array([orc.gauss_draw(123, i) for i in range(1 << n)])
    N = z.size
    for x in (z.real, z.imag):
        assert abs(x.mean()) < 6 / math.sqrt(N)
        assert abs(x.var() - 1.0) < 6 * math.sqrt(2.0 / N)
    assert abs(np.mean(z.real * z.imag)) < 6 / math.sqrt(N)
    a = orc.init_gaussian(12, 5)
    assert orc.norm_sq(a) == pytest.approx(1.0, abs=1e-14)
    a32 = orc.init_gaussian(12, 5, round_to_c64=True)
    np.testing.assert_array_equal(a32, a.astype(np.complex64).astype(np.complex128))


# --------------------------------------------------------------------------- #
# Emulated sharding (section 3.1 / Fig. 8 / Eq. 2)                              #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("n,g", [(2, 1), (6, 1), (8, 2), (9, 3), (12, 3), (6, 3)])
def test_sharded_wht_equals_wht(n, g):
    a = crandn(1 << n)
    np.testing.assert_allclose(orc.wht_sharded(a.copy(), g), orc.wht(a.copy()), rtol=0, atol=1e-11 * (1 << n))


@pytest.mark.parametrize("n,g", [(6, 1), (8, 2), (9, 3), (10, 3)])
def test_reorganisation_moves_fraction_one_minus_inv_p(n, g):
    """Fig. 8: a block whose owner is unchanged stays ("do
    nothing"); Eq. 2 moves s^{n_l} - s^{n_l-n_c} blocks, i.e. the
    fraction 1 - 1/P when all g parallel bits change.  Track every element."""
    N, P = 1 << n, 1 << g
    Nl = N // P
    a = np.arange(N, dtype=np.float64).astype(np.complex128)
    b = orc.reorganize(a.copy(), g)
    pos = np.empty(N, dtype=np.int64)
    pos[b.real.astype(np.int64)] = np.arange(N)
    src = np.arange(N)
    owner_before, owner_after = src // Nl, pos // Nl
    moved = int(np.sum(owner_before != owner_after))
    assert moved == N - N // P
    # new owner = old top-g local bits; new top-g local bits = old owner
    local = src % Nl
    assert np.array_equal(owner_after, local >> (n - 2 * g))
    assert np.array_equal((pos % Nl) >> (n - 2 * g), owner_before)
    assert np.array_equal(pos % (Nl >> g), src % (Nl >> g))
    # unchanged owner => unchanged position ("do nothing")
    stay = owner_before == owner_after
    assert np.array_equal(pos[stay], src[stay])
    # applied twice it is the identity
    np.testing.assert_array_equal(orc.reorganize(b.copy(), g), a)


# --------------------------------------------------------------------------- #
# Seeded measurement (NEXT-3, reading G21)                                     #
# --------------------------------------------------------------------------- #
def test_sample_fig1_superposition_and_basis_state():
    """Fig. 1(b): the 1-qubit superposition measures 0 or 1 with probability
    1/2 each -> index 0 exactly when u < 1/2; a basis state
    always measures its own index."""
    shots = 4096
    idx, _ = orc.sample(orc.init_uniform(1), shots, 3)
    u = np.array([orc.sample_uniform(3, s) for s in range(shots)])
    np.testing.assert_array_equal(idx, (u >= 0.5).astype(np.uint64))
    assert abs(idx.mean() - 0.5) < 6 * 0.5 / math.sqrt(shots)
    a = np.zeros(1 << 7, np.complex128)
    a[77] = 1j
    idx, _ = orc.sample(a, 100, 1)
    assert set(idx.tolist()) == {77}


def test_sample_is_numpy_inverse_cdf():
    """Inverse CDF with numpy's cumsum + searchsorted (library routines)."""
    n, shots, seed = 9, 20000, 11
    a = crandn(1 << n)
    a /= np.linalg.norm(a)
    idx, cdf = orc.sample(a, shots, seed)
    p = np.abs(a) ** 2
    c = np.cumsum(p)
    np.testing.assert_allclose(cdf, c, rtol=0, atol=1e-14)
    u = np.array([orc.sample_uniform(seed, s) for s in range(shots)])
    ref = np.searchsorted(c, u * c[-1], side="right")
    bad = np.nonzero(idx != ref)[0]
    for s in bad:  # only a rounding-level boundary may differ
        assert abs(c[min(idx[s], ref[s])] - u[s] * c[-1]) < 1e-14
    # frequencies follow |a|^2 (chi-square, 6-sigma bound on the statistic)
    counts = np.bincount(idx.astype(np.int64), minlength=1 << n)
    expected = p * shots
    chi2 = np.sum((counts - expected) ** 2 / expected)
    dof = (1 << n) - 1
    assert chi2 < dof + 6 * math.sqrt(2 * dof)


def test_sample_grover_state_finds_the_marked_index():
    n, m = 10, 1
    marked = orc.marked_from_seed(n, m, 1)
    a = orc.iterate(orc.init_uniform(n), marked, cf.optimal_iterations(n, m), orc.WHT)
    idx, _ = orc.sample(a, 10000, 2)
    assert np.mean(idx == marked[0]) > 0.998  # P_success = 0.99946


# --------------------------------------------------------------------------- #
# Decoherence step (NEXT-2, reading G22)                                       #
# --------------------------------------------------------------------------- #
@pytest.mark.parametrize("n", [1, 2, 4])
def test_decoherent_iteration_equals_dense_brute_force(n):
    """Every laser op as a dense matrix: the 2x2 on qubit q (numpy.kron), the
    contraction diag(1, sqrt(1-r)) on the drawn site, then division by the
    norm; survival = product of the pre-renormalisation sums.  n = 1 is
    SPEC's example: the sum after a contraction is |alpha|^2 + (1-r)|beta|^2."""
    N = 1 << n
    sigma, rate, seed, t0, k = 0.1, 0.05, 21, 3, 2
    a0 = crandn(N)
    a0 /= np.linalg.norm(a0)
    marked = orc.marked_from_seed(n, max(1, N // 4), 2)
    O = np.eye(N)
    O[marked, marked] = -1.0

    def on_qubit(U, q):
        return np.kron(np.kron(np.eye(1 << (n - q - 1)), U), np.eye(1 << q))

    ref = a0.copy()
    surv_ref = []
    for t in range(t0, t0 + k):
        ref = O @ ref
        surv = 1.0
        for w in (0, 1):
            if w == 1:
                ref = -ref
                ref[0] = -ref[0]
            for q in range(n):
                phi = math.pi / 4 + orc.noise_delta(seed, t, w, q, sigma)
                ref = on_qubit(np.array([[math.cos(phi), math.sin(phi)], [math.sin(phi), -math.cos(phi)]]), q) @ ref
                s = orc.decay_site(n, seed, t, w, q)
                ref = on_qubit(np.diag([1.0, math.sqrt(1 - rate)]), s) @ ref
                nrm = float(np.sum(np.abs(ref) ** 2))
                surv *= nrm
                ref = ref / math.sqrt(nrm)
        surv_ref.append(surv)
    got, surv = orc.iterate_decoherent(a0.copy(), marked, k, sigma, rate, seed, t0)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(surv, surv_ref, rtol=1e-12)


def test_decoherence_single_qubit_survival_closed_form():
    """contraction of |1> by sqrt(1-r) on alpha|0> + beta|1> leaves
    sum |alpha|^2 + (1-r)|beta|^2.  With sigma = 0 and M = 0 the first laser op
    maps |0> to the superposition (Fig. 1(b)): sum = 1/2 + (1-r)/2."""
    r = 0.3
    a = orc.init_zero_state(1)
    _, surv = orc.iterate_decoherent(a, np.zeros(0, np.uint64), 1, 0.0, r, 1)
    # op 1: H|0> = (1,1)/sqrt2 -> contraction -> 1/2 + (1-r)/2
    s1 = 0.5 + (1 - r) / 2
    # op 2 acts on the renormalised (1, sqrt(1-r))/sqrt(s1 * 2) after F0 and H
    v = np.array([1.0, math.sqrt(1 - r)]) / math.sqrt(2 * s1)
    v = np.array([v[0], -v[1]])
    h = np.array([[1, 1], [1, -1]]) / math.sqrt(2)
    v = h @ v
    s2 = v[0] ** 2 + (1 - r) * v[1] ** 2
    assert surv[0] == pytest.approx(s1 * s2, rel=1e-14)


def test_decoherence_rate0_is_noisy_iteration_and_norm_is_kept():
    n = 11
    a0 = orc.init_gaussian(n, 4)
    marked = orc.marked_from_seed(n, 3, 4)
    got, surv = orc.iterate_decoherent(a0.copy(), marked, 4, 0.05, 0.0, 9, 2)
    np.testing.assert_allclose(got, orc.iterate_noisy(a0.copy(), marked, 4, 0.05, 9, 2), rtol=0, atol=1e-13)
    np.testing.assert_allclose(surv, 1.0, atol=1e-13)
    got, surv = orc.iterate_decoherent(a0.copy(), marked, 4, 0.05, 0.02, 9, 2)
    assert orc.norm_sq(got) == pytest.approx(1.0, abs=1e-12)
    assert np.all((surv > 0) & (surv < 1))
    _, surv2 = orc.iterate_decoherent(a0.copy(), marked, 4, 0.05, 0.04, 9, 2)
    assert np.all(surv2 < surv)
    sites = {orc.decay_site(n, 9, t, w, q) for t in range(20) for w in (0, 1) for q in range(n)}
    assert sites == set(range(n))


# --------------------------------------------------------------------------- #
# Operational angle errors (NEXT-1, readings G19/G20)                          #
# --------------------------------------------------------------------------- #
def test_noisy_sigma0_is_ideal_grover():
    """sigma = 0: U(pi/4) is the normalised Hadamard, so the noisy iteration
    is the ideal one (closed form)."""
    n, m, k = 10, 1, 25
    marked = orc.marked_from_seed(n, m, 1)
    a = orc.iterate_noisy(orc.init_uniform(n), marked, k, 0.0, 7)
    np.testing.assert_allclose(a, orc.iterate(orc.init_uniform(n), marked, k, orc.WHT), rtol=0, atol=1e-13)
    assert orc.marked_mass(a, marked) == pytest.approx(cf.p_success_uniform(n, m, k), abs=1e-13)


@pytest.mark.parametrize("n", [1, 3, 5])
def test_noisy_iteration_equals_dense_kron_product(n):
    """Each noisy transform is the Kronecker product of its n per-qubit 2x2s
    (qubit q = bit q: kron order q = n-1 ... 0), built with numpy.kron."""
    N = 1 << n
    sigma, seed, t0, k = 0.2, 99, 5, 3
    a0 = crandn(N)
    a0 /= np.linalg.norm(a0)
    marked = orc.marked_from_seed(n, max(1, N // 3), 4)
    O = np.eye(N)
    O[marked, marked] = -1.0
    F0 = -np.eye(N)
    F0[0, 0] = 1.0

    def transform(t, w):
        M = np.ones((1, 1))
        for q in reversed(range(n)):
            phi = math.pi / 4 + orc.noise_delta(seed, t, w, q, sigma)
            U = np.array([[math.cos(phi), math.sin(phi)], [math.sin(phi), -math.cos(phi)]])
            M = np.kron(M, U)
        return M

    ref = a0.copy()
    for t in range(t0, t0 + k):
        ref = transform(t, 1) @ F0 @ transform(t, 0) @ O @ ref
    got = orc.iterate_noisy(a0.copy(), marked, k, sigma, seed, t0)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)


def test_noisy_unitary_deterministic_and_noise_statistics():
    n = 12
    a0 = orc.init_gaussian(n, 3)
    marked = orc.marked_from_seed(n, 5, 3)
    a = orc.iterate_noisy(a0.copy(), marked, 6, 0.3, 11)
    assert orc.norm_sq(a) == pytest.approx(1.0, abs=1e-12)
    np.testing.assert_array_equal(orc.iterate_noisy(a0.copy(), marked, 6, 0.3, 11), a)
    # splitting the iterations across calls with t0 gives the same state
    b = orc.iterate_noisy(a0.copy(), marked, 2, 0.3, 11, 0)
    orc.iterate_noisy(b, marked, 4, 0.3, 11, 2)
    np.testing.assert_array_equal(b, a)
    z = np.array([orc.noise_delta(5, t, w, q, 1.0) for t in range(256) for w in (0, 1) for q in range(64)])
    assert abs(z.mean()) < 6 / math.sqrt(z.size) and abs(z.var() - 1) < 6 * math.sqrt(2 / z.size)
    # more angle error -> further from the ideal state (monotone in expectation)
    ideal = orc.iterate(a0.copy(), marked, 6, orc.WHT)
    d = [np.mean([np.linalg.norm(orc.iterate_noisy(a0.copy(), marked, 6, s, sd) - ideal) for sd in range(8)])
         for s in (1e-3, 1e-2, 1e-1)]
    assert d[0] < d[1] < d[2]


def test_snapshot_format_fig1(tmp_path):
    """SPEC's snapshot format written by the oracle: Fig. 1(a)'s |0>
    and Fig. 1(b)'s uniform superposition."""
    p = tmp_path / "s.txt"
    assert orc.write_snapshot(orc.init_zero_state(3), str(p)) == 1
    assert p.read_text() == "s=2 M=3\n0 1 0\n"
    assert orc.write_snapshot(orc.init_uniform(1), str(p)) == 2
    assert p.read_text() == "s=2 M=1\n0 0.70710678118654757 0\n1 0.70710678118654757 0\n"
    s, m, amps = orc.read_snapshot(str(p))
    assert (s, m) == (2, 1) and amps == {0: 2 ** -0.5, 1: 2 ** -0.5}
