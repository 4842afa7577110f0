"""Seeded gate-circuit INPUTS for the NEXT-4 tests (and bench.py's gate workload).

Holds none of the method's arithmetic: it only writes gate records (target,
control mask, 2x2 matrix) in the 80-byte layout shared by the oracle's
or_gate and the library's sv_gate.  Matrices are the textbook 2x2s (H, X, Y,
Z, phase) and seeded random unitaries; the circuits are the textbook QFT and a
Grover iteration written as gates, plus seeded random circuits.  Both the
oracle and the CUDA path consume these records; neither is imported here.
"""
from __future__ import annotations

import math

import numpy as np

GATE_DTYPE = np.dtype([("target", "<i4"), ("reserved", "<i4"), ("controls", "<u8"), ("m", "<f8", (8,))])

S2 = 1.0 / math.sqrt(2.0)
H = np.array([[S2, S2], [S2, -S2]], dtype=np.complex128)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
I2 = np.eye(2, dtype=np.complex128)


def phase(theta: float) -> np.ndarray:
    return np.array([[1, 0], [0, np.exp(1j * theta)]], dtype=np.complex128)


def random_unitary(rng: np.random.Generator) -> np.ndarray:
    """Haar-ish 2x2 unitary: QR of a complex Gaussian matrix with phase fix."""
    z = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    return q * (d / np.abs(d))


def record(target: int, m: np.ndarray, controls=()) -> np.ndarray:
    g = np.zeros((), GATE_DTYPE)
    g["target"] = target
    cm = 0
    for c in controls:
        cm |= 1 << int(c)
    g["controls"] = cm
    m = np.asarray(m, dtype=np.complex128)
    g["m"] = [m[0, 0].real, m[0, 0].imag, m[0, 1].real, m[0, 1].imag,
              m[1, 0].real, m[1, 0].imag, m[1, 1].real, m[1, 1].imag]
    return g


def circuit(records) -> np.ndarray:
    return np.array(list(records), dtype=GATE_DTYPE)


def matrix_of(g) -> np.ndarray:
    m = g["m"]
    return np.array([[m[0] + 1j * m[1], m[2] + 1j * m[3]], [m[4] + 1j * m[5], m[6] + 1j * m[7]]])


def random_circuit(n: int, count: int, seed: int, max_controls: int = 2, qubits=None,
                   p_control: float = 0.5) -> np.ndarray:
    """count gates: random target (from `qubits`, default all), each with
    probability p_control 1..max_controls random distinct controls, random
    unitary matrix."""
    rng = np.random.default_rng(seed)
    qs = list(range(n)) if qubits is None else list(qubits)
    out = []
    for _ in range(count):
        t = int(rng.choice(qs))
        ctr = []
        if max_controls > 0 and n > 1 and rng.random() < p_control:
            others = [q for q in range(n) if q != t]
            k = int(rng.integers(1, min(max_controls, len(others)) + 1))
            ctr = [int(c) for c in rng.choice(others, size=k, replace=False)]
        out.append(record(t, random_unitary(rng), ctr))
    return circuit(out)


def qft_circuit(n: int) -> np.ndarray:
    """Textbook QFT on n qubits (qubit q = bit q): for j = n-1 .. 0: H on j,
    then controlled-phase(pi / 2^(j-k)) on j controlled by each k < j; then the
    bit reversal as 3 CNOTs per swapped pair.  Maps |x> to
    N^{-1/2} sum_y exp(2 pi i x y / N) |y>."""
    out = []
    for j in range(n - 1, -1, -1):
        out.append(record(j, H))
        for k in range(j - 1, -1, -1):
            out.append(record(j, phase(math.pi / (1 << (j - k))), [k]))
    for a in range(n // 2):
        b = n - 1 - a
        out += [record(b, X, [a]), record(a, X, [b]), record(b, X, [a])]
    return circuit(out)


def multi_controlled_z(n: int) -> list:
    """Z on qubit 0 controlled by all others: -1 on |1...1> only."""
    return [record(0, Z, list(range(1, n)))]


def grover_circuit(n: int, marked: int, k: int, prepare: bool = True) -> np.ndarray:
    """k Grover iterations as gates (optionally after H^n |0>):
    O = X^{~m} C^{n-1}Z X^{~m} (phase -1 on |m>),
    D = H^n X^n C^{n-1}Z X^n H^n (= I - 2|s><s| = -(2|s><s| - I))."""
    out = []
    if prepare:
        out += [record(q, H) for q in range(n)]
    flip = [q for q in range(n) if not (marked >> q) & 1]
    for _ in range(k):
        out += [record(q, X) for q in flip]
        out += multi_controlled_z(n)
        out += [record(q, X) for q in flip]
        out += [record(q, H) for q in range(n)]
        out += [record(q, X) for q in range(n)]
        out += multi_controlled_z(n)
        out += [record(q, X) for q in range(n)]
        out += [record(q, H) for q in range(n)]
    return circuit(out)


def structured_circuit(n: int, count: int, seed: int, max_controls: int = 2) -> np.ndarray:
    """Gates drawn from the special shapes the engine treats specially and
    the general case: X (NOT), Y (anti-diagonal), Z / S / T / phase(theta)
    (phase: w = 1), diag(e^{ia}, e^{ib}), H and random unitaries, each with
    0..max_controls random controls."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        t = int(rng.integers(0, n))
        kind = int(rng.integers(0, 8))
        if kind == 0:
            m = X
        elif kind == 1:
            m = Y
        elif kind == 2:
            m = Z
        elif kind == 3:
            m = phase(float(rng.uniform(-math.pi, math.pi)))
        elif kind == 4:
            a, b = rng.uniform(-math.pi, math.pi, 2)
            m = np.diag([np.exp(1j * a), np.exp(1j * b)])
        elif kind == 5:
            a, b = rng.uniform(-math.pi, math.pi, 2)
            m = np.array([[0, np.exp(1j * a)], [np.exp(1j * b), 0]])
        elif kind == 6:
            m = H
        else:
            m = random_unitary(rng)
        ctr = []
        if max_controls > 0 and n > 1:
            k = int(rng.integers(0, min(max_controls, n - 1) + 1))
            others = [q for q in range(n) if q != t]
            ctr = [int(c) for c in rng.choice(others, size=k, replace=False)]
        out.append(record(t, m, ctr))
    return circuit(out)


def layered_circuit(n: int, layers: int, seed: int) -> np.ndarray:
    """Hardware-efficient-ansatz-like layers: a random unitary on every qubit,
    then a CZ (controlled-Z) chain q -> q+1."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(layers):
        out += [record(q, random_unitary(rng)) for q in range(n)]
        out += [record(q + 1, Z, [q]) for q in range(n - 1)]
    return circuit(out)
