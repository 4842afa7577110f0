"""Exact closed forms of the Grover iteration a^(k) = (D O)^k a^(0).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).

The paper cites quantum search only ([Grov96], section 1.5: "runs
in O(sqrt N) time for N items"); the iteration is fixed by BASELINE.json's
north star (G1 in DESIGN.md): O = I - 2 sum_{m in M} |m><m|,
D = 2|s><s| - I with |s> = H^n|0> = 2^{-n/2} (1,...,1).

Two-dimensional reduction (textbook; verified against the plain simulator and
against dense matrix powers in tests/test_oracle_pins.py):
  U = complement of M,  mu_M = mean_M a^(0),  mu_U = mean_U a^(0),
  alpha_0 = sqrt(M) mu_M,  beta_0 = sqrt(N-M) mu_U,  sin(theta) = sqrt(M/N)
  alpha_k = sin(2k theta) beta_0 + cos(2k theta) alpha_0
  beta_k  = cos(2k theta) beta_0 - sin(2k theta) alpha_0
  i in M: a_i^(k) = alpha_k / sqrt(M) + (a_i^(0) - mu_M)         (residual invariant)
  i in U: a_i^(k) = beta_k / sqrt(N-M) + (-1)^k (a_i^(0) - mu_U) (residual alternates)
  marked mass = |alpha_k|^2 + sum_M |a_i^(0) - mu_M|^2
Uniform start: a_marked = sin((2k+1) theta)/sqrt(M), a_unmarked =
cos((2k+1) theta)/sqrt(N-M), P_success = sin^2((2k+1) theta) (north star).
The edges M = 0 and M = N are handled explicitly (an empty set has no mean).
"""
from __future__ import annotations

import math

import numpy as np


def theta(n: int, m: int) -> float:
    """sin(theta) = sqrt(M/N)."""
    return math.asin(math.sqrt(m / float(1 << n)))


def optimal_iterations(n: int, m: int) -> int:
    """floor(pi/4 sqrt(N/M)) -- the c1/c2 iteration counts (G9)."""
    return int(math.floor(math.pi / 4.0 * math.sqrt((1 << n) / m)))


def p_success_uniform(n: int, m: int, k: int) -> float:
    """P_success(k) = sin^2((2k+1) theta) for the uniform start."""
    return math.sin((2 * k + 1) * theta(n, m)) ** 2


def uniform_amplitudes(n: int, m: int, k: int) -> tuple[float, float]:
    """(a_marked, a_unmarked) after k iterations from |s>; nan for an empty set."""
    N = 1 << n
    t = theta(n, m)
    am = math.sin((2 * k + 1) * t) / math.sqrt(m) if m > 0 else float("nan")
    au = math.cos((2 * k + 1) * t) / math.sqrt(N - m) if m < N else float("nan")
    return am, au


class GeneralParams:
    """Scalars of the general-start closed form, from O(N) sums of a^(0)."""

    def __init__(self, n: int, m: int, sum_all: complex, sum_marked: complex, k: int):
        N = 1 << n
        self.n, self.m, self.k, self.N = n, m, k, N
        t = theta(n, m)
        self.mu_M = sum_marked / m if m > 0 else 0.0
        self.mu_U = (sum_all - sum_marked) / (N - m) if m < N else 0.0
        alpha0 = math.sqrt(m) * self.mu_M
        beta0 = math.sqrt(N - m) * self.mu_U
        c, s = math.cos(2 * k * t), math.sin(2 * k * t)
        self.alpha_k = s * beta0 + c * alpha0
        self.beta_k = c * beta0 - s * alpha0
        self.sign = -1.0 if (k % 2) else 1.0

    def marked_amp(self, a0_i: complex) -> complex:
        return self.alpha_k / math.sqrt(self.m) + (a0_i - self.mu_M)

    def unmarked_amp(self, a0_i: complex) -> complex:
        return self.beta_k / math.sqrt(self.N - self.m) + self.sign * (a0_i - self.mu_U)


def general_state(a0: np.ndarray, marked: np.ndarray, k: int) -> np.ndarray:
    """Every amplitude of (D O)^k a0 via the closed form (vectorised over i)."""
    N = a0.size
    n = N.bit_length() - 1
    marked = np.asarray(marked, dtype=np.int64)
    is_m = np.zeros(N, dtype=bool)
    is_m[marked] = True
    m = int(is_m.sum())
    gp = GeneralParams(n, m, complex(a0.sum()), complex(a0[is_m].sum()) if m else 0j, k)
    out = np.empty_like(a0)
    if m:
        out[is_m] = gp.alpha_k / math.sqrt(m) + (a0[is_m] - gp.mu_M)
    if m < N:
        out[~is_m] = gp.beta_k / math.sqrt(N - m) + gp.sign * (a0[~is_m] - gp.mu_U)
    return out


def general_marked_mass(a0: np.ndarray, marked: np.ndarray, k: int) -> float:
    N = a0.size
    n = N.bit_length() - 1
    marked = np.asarray(marked, dtype=np.int64)
    m = marked.size
    if m == 0:
        return 0.0
    gp = GeneralParams(n, m, complex(a0.sum()), complex(a0[marked].sum()), k)
    resid = a0[marked] - gp.mu_M
    return abs(gp.alpha_k) ** 2 + float(np.sum(np.abs(resid) ** 2))
