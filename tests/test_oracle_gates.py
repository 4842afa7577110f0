"""Pins of the NEXT-4 gate oracle (or_apply_gates, or_apply_gates_sharded)
against what the paper and mathematics fix -- never against the oracle itself:

  * section 2.1: a gate is a V x V matrix that is "simply 2x2 or
    4x4 matrices replicated many times" -> the dense matrix built by numpy
    Kronecker products I (x) M (x) I, with controls as the projector sum
    (I - Pi) + Pi (I (x) M (x) I), must equal the pair loop (n <= 6, random
    circuits, random controls);
  * Fig. 3: the 2x2 on the low bit pairs (a0, a1), (a2, a3);
  * textbook circuits with closed forms: the QFT equals sqrt(N) ifft, CNOT /
    Toffoli are the basis permutations of their truth tables, XYZ = iI,
    Grover written as gates reaches sin^2((2k+1) theta) (G1) with the
    (-1)^k global phase of D_circuit = -(2|s><s| - I);
  * unitarity (norm preserved) and inverse circuits (U^dagger in reverse
    order) returning the start state;
  * the sharded replica (Fig. 8 reorganisations, section 3.1) equals the plain
    one, and counts the reorganisations the schedule implies.
"""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from tests import circuits as C


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return a / np.linalg.norm(a)


def dense_gate(n, g):
    """V x V matrix of one gate by Kronecker products (qubit q = bit q, so the
    factor order is [qubit n-1, ..., qubit 0])."""
    t = int(g["target"])
    M = C.matrix_of(g)
    U = np.kron(np.kron(np.eye(1 << (n - 1 - t)), M), np.eye(1 << t))
    cm = int(g["controls"])
    if cm == 0:
        return U
    idx = np.arange(1 << n)
    Pi = np.diag(((idx & cm) == cm).astype(float))
    return (np.eye(1 << n) - Pi) + Pi @ U


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (3, 2), (4, 3), (5, 4), (6, 5)])
def test_gates_equal_dense_kronecker(n, seed):
    gates = C.random_circuit(n, 24, seed, max_controls=min(3, n - 1))
    a0 = rand_state(n, 100 + seed)
    U = np.eye(1 << n, dtype=complex)
    for g in gates:
        U = dense_gate(n, g) @ U
    got = orc.apply_gates(a0.copy(), gates)
    np.testing.assert_allclose(got, U @ a0, atol=1e-13, rtol=0)


def test_fig3_low_bit_pairs():
    # Fig. 3: [w x; y z] on qubit 0 of a 4-element vector acts on (a0,a1), (a2,a3)
    w, x, y, z = 2.0, 3.0, 5.0, 7.0
    g = C.circuit([C.record(0, np.array([[w, x], [y, z]]))])
    a = np.array([1.0, 10.0, 100.0, 1000.0], dtype=complex)
    got = orc.apply_gates(a.copy(), g)
    np.testing.assert_array_equal(got, [w * 1 + x * 10, y * 1 + z * 10, w * 100 + x * 1000, y * 100 + z * 1000])


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 10])
def test_qft_equals_fft(n):
    a0 = rand_state(n, 7 + n)
    got = orc.apply_gates(a0.copy(), C.qft_circuit(n))
    ref = np.fft.ifft(a0) * math.sqrt(1 << n)  # sum_x a_x e^{+2 pi i x y / N} / sqrt(N)
    np.testing.assert_allclose(got, ref, atol=1e-12, rtol=0)


def test_cnot_toffoli_truth_tables():
    n = 4
    for x in range(1 << n):
        a = np.zeros(1 << n, complex)
        a[x] = 1
        got = orc.apply_gates(a.copy(), C.circuit([C.record(2, C.X, [0])]))
        y = x ^ (4 if x & 1 else 0)
        assert np.argmax(np.abs(got)) == y and abs(got[y] - 1) == 0
        got = orc.apply_gates(a.copy(), C.circuit([C.record(3, C.X, [0, 1])]))
        y = x ^ (8 if (x & 3) == 3 else 0)
        assert np.argmax(np.abs(got)) == y and abs(got[y] - 1) == 0


def test_pauli_algebra_xyz_is_i():
    n = 3
    a0 = rand_state(n, 3)
    for q in range(n):
        got = orc.apply_gates(a0.copy(), C.circuit([C.record(q, C.Z), C.record(q, C.Y), C.record(q, C.X)]))
        np.testing.assert_allclose(got, 1j * a0, atol=1e-15, rtol=0)


@pytest.mark.parametrize("n,k", [(2, 1), (4, 3), (6, 6), (8, 12)])
def test_grover_as_gates_closed_form(n, k):
    N = 1 << n
    marked = (0x5A5A >> 1) % N
    a = np.zeros(N, complex)
    a[0] = 1
    got = orc.apply_gates(a, C.grover_circuit(n, marked, k))
    th = math.asin(math.sqrt(1.0 / N))
    sign = (-1) ** k
    am = sign * math.sin((2 * k + 1) * th)
    au = sign * math.cos((2 * k + 1) * th) / math.sqrt(N - 1)
    ref = np.full(N, au, complex)
    ref[marked] = am
    np.testing.assert_allclose(got, ref, atol=1e-12, rtol=0)


def test_unitarity_and_inverse_circuit():
    n = 9
    gates = C.random_circuit(n, 60, 11, max_controls=3)
    a0 = rand_state(n, 12)
    a = orc.apply_gates(a0.copy(), gates)
    assert abs(np.vdot(a, a).real - 1.0) < 1e-13
    inv = gates[::-1].copy()
    for i in range(inv.size):
        M = C.matrix_of(inv[i]).conj().T
        inv[i] = C.record(int(inv[i]["target"]), M, [q for q in range(n) if (int(inv[i]["controls"]) >> q) & 1])
    back = orc.apply_gates(a, inv)
    np.testing.assert_allclose(back, a0, atol=1e-13, rtol=0)


def test_invalid_gates_rejected():
    a = rand_state(3, 0)
    for rec in (C.record(3, C.X), C.record(-1, C.X), C.record(1, C.X, [1]), C.record(0, C.X, [5])):
        with pytest.raises(ValueError):
            orc.apply_gates(a.copy(), C.circuit([rec]))


@pytest.mark.parametrize("n,g", [(6, 1), (8, 2), (9, 3), (12, 3)])
def test_sharded_replica_equals_plain(n, g):
    gates = C.random_circuit(n, 80, n * 10 + g, max_controls=3)
    a0 = rand_state(n, 5)
    ref = orc.apply_gates(a0.copy(), gates)
    a = a0.copy()
    reorgs = orc.apply_gates_sharded(a, gates, g)
    np.testing.assert_allclose(a, ref, atol=1e-12, rtol=0)
    # the schedule's reorganisation count: a swap whenever a target sits on
    # the current parallel set (positions >= n - g), plus one restore
    nl, swapped, cnt = n - g, False, 0
    for gt in gates:
        t = int(gt["target"])
        top = (t >= nl) if not swapped else (nl - g <= t < nl)
        if top:
            swapped, cnt = not swapped, cnt + 1
    assert reorgs == cnt + (1 if swapped else 0)
