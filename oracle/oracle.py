"""ctypes binding of the plain C oracle (oracle/sv_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product path
(paper_quant_ph_9804039_b200) never imports this module, and this module never
imports the product.

Each wrapper names the C function it calls; the C file cites the paper passage
(P:NNNN = line of /root/reference/PAPER.md) each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

WHT = 0
MEAN = 1


def build(force: bool = False) -> str:
    """Compile sv_oracle.c with gcc (plain -O2, single thread, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _C128(ctypes.Structure):
    """Layout- and ABI-compatible with C99 double _Complex (SysV: two SSE eightbytes)."""
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, i32, dp, vp = ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
        L.or_splitmix64_next.argtypes = [ctypes.POINTER(u64)]
        L.or_splitmix64_next.restype = u64
        L.or_hash64.argtypes = [u64]
        L.or_hash64.restype = u64
        L.or_perm.argtypes = [i32, u64, u64]
        L.or_perm.restype = u64
        L.or_marked_from_seed.argtypes = [i32, u64, u64, vp]
        L.or_marked_from_seed.restype = i32
        L.or_init_uniform.argtypes = [i32, vp]
        L.or_init_zero_state.argtypes = [i32, vp]
        L.or_init_gaussian.argtypes = [i32, u64, i32, vp]
        L.or_gauss_key.argtypes = [u64]
        L.or_gauss_key.restype = u64
        L.or_gauss_draw.argtypes = [u64, u64, dp, dp]
        L.or_oracle_flip.argtypes = [vp, vp, u64]
        L.or_apply_2x2.argtypes = [i32, vp, i32] + [_C128] * 4
        L.or_wht.argtypes = [i32, vp]
        L.or_f0_scaled.argtypes = [i32, vp]
        L.or_diffuse_wht.argtypes = [i32, vp]
        L.or_diffuse_mean.argtypes = [i32, vp]
        L.or_sum.argtypes = [i32, vp]
        L.or_sum.restype = _C128
        L.or_iterate.argtypes = [i32, vp, vp, u64, i32, i32]
        L.or_probabilities.argtypes = [i32, vp, vp]
        L.or_marked_mass.argtypes = [vp, vp, u64]
        L.or_marked_mass.restype = ctypes.c_double
        L.or_norm_sq.argtypes = [i32, vp]
        L.or_norm_sq.restype = ctypes.c_double
        L.or_dense_hadamard.argtypes = [i32, vp]
        L.or_dense_hadamard.restype = i32
        L.or_noise_delta.argtypes = [u64, u64, i32, i32, ctypes.c_double]
        L.or_noise_delta.restype = ctypes.c_double
        L.or_noisy_transform.argtypes = [i32, vp, u64, u64, i32, ctypes.c_double]
        L.or_f0.argtypes = [i32, vp]
        L.or_iterate_noisy.argtypes = [i32, vp, vp, u64, i32, ctypes.c_double, u64, u64]
        L.or_decay_site.argtypes = [i32, u64, u64, i32, i32]
        L.or_decay_site.restype = i32
        L.or_iterate_decoherent.argtypes = [i32, vp, vp, u64, i32, ctypes.c_double, ctypes.c_double, u64, u64, vp]
        L.or_sample_uniform.argtypes = [u64, u64]
        L.or_sample_uniform.restype = ctypes.c_double
        L.or_sample.argtypes = [i32, vp, u64, u64, vp, vp]
        L.or_reorganize.argtypes = [i32, i32, vp, vp]
        L.or_wht_sharded.argtypes = [i32, i32, vp]
        L.or_wht_sharded.restype = i32
        L.or_apply_controlled_2x2.argtypes = [i32, vp, i32, u64] + [_C128] * 4
        L.or_apply_gates.argtypes = [i32, vp, vp, u64]
        L.or_apply_gates.restype = i32
        L.or_apply_gates_sharded.argtypes = [i32, i32, vp, u64, vp]
        L.or_apply_gates_sharded.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _state(a: np.ndarray) -> np.ndarray:
    assert a.dtype == np.complex128 and a.flags["C_CONTIGUOUS"], "oracle works in complex128"
    return a


def _nbits(a: np.ndarray) -> int:
    n = int(a.size).bit_length() - 1
    assert a.size == 1 << n
    return n


# ---- seeded generators (G6, G8) --------------------------------------------
def hash64(x: int) -> int:
    return int(lib().or_hash64(x))


def perm(n: int, seed: int, x: int) -> int:
    return int(lib().or_perm(n, seed, x))


def marked_from_seed(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty(m, dtype=np.uint64)
    rc = lib().or_marked_from_seed(n, m, seed, _ptr(out))
    if rc != 0:
        raise ValueError("m > 2^n")
    return out


# ---- initial states ----------------------------------------------------------
def init_uniform(n: int) -> np.ndarray:
    a = np.empty(1 << n, dtype=np.complex128)
    lib().or_init_uniform(n, _ptr(a))
    return a


def init_zero_state(n: int) -> np.ndarray:
    a = np.empty(1 << n, dtype=np.complex128)
    lib().or_init_zero_state(n, _ptr(a))
    return a


def init_gaussian(n: int, seed: int, round_to_c64: bool = False) -> np.ndarray:
    a = np.empty(1 << n, dtype=np.complex128)
    lib().or_init_gaussian(n, seed, 1 if round_to_c64 else 0, _ptr(a))
    return a


def gauss_draw(seed: int, i: int) -> complex:
    key = lib().or_gauss_key(seed)
    re, im = ctypes.c_double(), ctypes.c_double()
    lib().or_gauss_draw(key, i, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


# ---- the iteration -----------------------------------------------------------
def oracle_flip(a: np.ndarray, marked: np.ndarray) -> np.ndarray:
    marked = np.ascontiguousarray(marked, dtype=np.uint64)
    lib().or_oracle_flip(_ptr(_state(a)), _ptr(marked), marked.size)
    return a


def apply_2x2(a: np.ndarray, q: int, w: complex, x: complex, y: complex, z: complex) -> np.ndarray:
    lib().or_apply_2x2(_nbits(a), _ptr(_state(a)), q, *(_C128(v.real, v.imag) for v in map(complex, (w, x, y, z))))
    return a


def wht(a: np.ndarray) -> np.ndarray:
    lib().or_wht(_nbits(a), _ptr(_state(a)))
    return a


def f0_scaled(a: np.ndarray) -> np.ndarray:
    lib().or_f0_scaled(_nbits(a), _ptr(_state(a)))
    return a


def diffuse_wht(a: np.ndarray) -> np.ndarray:
    lib().or_diffuse_wht(_nbits(a), _ptr(_state(a)))
    return a


def diffuse_mean(a: np.ndarray) -> np.ndarray:
    lib().or_diffuse_mean(_nbits(a), _ptr(_state(a)))
    return a


def state_sum(a: np.ndarray) -> complex:
    r = lib().or_sum(_nbits(a), _ptr(_state(a)))
    return complex(r.re, r.im)


def iterate(a: np.ndarray, marked: np.ndarray, k: int, diffusion: int) -> np.ndarray:
    marked = np.ascontiguousarray(marked, dtype=np.uint64)
    lib().or_iterate(_nbits(a), _ptr(_state(a)), _ptr(marked), marked.size, k, diffusion)
    return a


# ---- readouts ---------------------------------------------------------------
def probabilities(a: np.ndarray) -> np.ndarray:
    p = np.empty(a.size, dtype=np.float64)
    lib().or_probabilities(_nbits(a), _ptr(_state(a)), _ptr(p))
    return p


def marked_mass(a: np.ndarray, marked: np.ndarray) -> float:
    marked = np.ascontiguousarray(marked, dtype=np.uint64)
    return float(lib().or_marked_mass(_ptr(_state(a)), _ptr(marked), marked.size))


def decay_site(n: int, seed: int, t: int, w: int, q: int) -> int:
    return int(lib().or_decay_site(n, seed, t, w, q))


def iterate_decoherent(a: np.ndarray, marked: np.ndarray, k: int, sigma: float, rate: float, seed: int,
                       t0: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """k iterations with angle errors and the decoherence step after every
    laser operation (readings G19, G20, G22); returns (state, survival[k])."""
    marked = np.ascontiguousarray(marked, dtype=np.uint64)
    surv = np.empty(k, dtype=np.float64)
    lib().or_iterate_decoherent(_nbits(a), _ptr(_state(a)), _ptr(marked), marked.size, k, sigma, rate, seed, t0,
                                _ptr(surv) if k else None)
    return a, surv


def sample_uniform(seed: int, s: int) -> float:
    return float(lib().or_sample_uniform(seed, s))


def sample(a: np.ndarray, shots: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Seeded whole-register measurement (G21): (indices, inclusive CDF)."""
    out = np.empty(shots, dtype=np.uint64)
    cdf = np.empty(a.size, dtype=np.float64)
    lib().or_sample(_nbits(a), _ptr(_state(a)), shots, seed, _ptr(out), _ptr(cdf))
    return out, cdf


def norm_sq(a: np.ndarray) -> float:
    return float(lib().or_norm_sq(_nbits(a), _ptr(_state(a))))


# ---- brute force / emulated sharding -------------------------------------------
def dense_hadamard(n: int) -> np.ndarray:
    K = np.empty((1 << n, 1 << n), dtype=np.float64)
    if lib().or_dense_hadamard(n, _ptr(K)) != 0:
        raise ValueError("n > 8")
    return K


def wht_sharded(a: np.ndarray, g: int) -> np.ndarray:
    if lib().or_wht_sharded(_nbits(a), g, _ptr(_state(a))) != 0:
        raise ValueError("need 2g <= n")
    return a


def reorganize(a: np.ndarray, g: int) -> np.ndarray:
    """One Fig. 8 reorganisation of the concatenated shards of a (in place)."""
    n = _nbits(_state(a))
    P, Nl = 1 << g, a.size >> g
    ptrs = (ctypes.c_void_p * P)(*[a.ctypes.data + r * Nl * a.itemsize for r in range(P)])
    tmp = np.empty_like(a)
    lib().or_reorganize(n, g, ptrs, _ptr(tmp))
    return a


# ---- operational angle errors (NEXT-1; readings G19, G20) ----------------------
def noise_delta(seed: int, t: int, w: int, q: int, sigma: float) -> float:
    return float(lib().or_noise_delta(seed, t, w, q, sigma))


def noisy_transform(a: np.ndarray, seed: int, t: int, w: int, sigma: float) -> np.ndarray:
    lib().or_noisy_transform(_nbits(a), _ptr(_state(a)), seed, t, w, sigma)
    return a


def f0(a: np.ndarray) -> np.ndarray:
    lib().or_f0(_nbits(a), _ptr(_state(a)))
    return a


def iterate_noisy(a: np.ndarray, marked: np.ndarray, k: int, sigma: float, seed: int, t0: int = 0) -> np.ndarray:
    marked = np.ascontiguousarray(marked, dtype=np.uint64)
    lib().or_iterate_noisy(_nbits(a), _ptr(_state(a)), _ptr(marked), marked.size, k, sigma, seed, t0)
    return a


# --------------------------------------------------------------------------- #
# NEXT-4: gate circuits (or_apply_gates; section 2.1, Fig. 3)     #
# --------------------------------------------------------------------------- #
# Layout of or_gate (80 bytes): int32 target, int32 reserved, uint64 controls,
# double m[8] = w, x, y, z as (re, im) pairs of [w x; y z].
GATE_DTYPE = np.dtype([("target", "<i4"), ("reserved", "<i4"), ("controls", "<u8"), ("m", "<f8", (8,))])


def _gates(gates) -> np.ndarray:
    g = np.ascontiguousarray(gates, dtype=GATE_DTYPE)
    assert g.dtype.itemsize == 80
    return g


def apply_controlled_2x2(a: np.ndarray, q: int, controls: int, w, x, y, z) -> np.ndarray:
    lib().or_apply_controlled_2x2(_nbits(a), _ptr(_state(a)), q, controls,
                                  *(_C128(v.real, v.imag) for v in map(complex, (w, x, y, z))))
    return a


def apply_gates(a: np.ndarray, gates) -> np.ndarray:
    """or_apply_gates: the gates in order on the full vector (raises on an invalid gate)."""
    g = _gates(gates)
    if lib().or_apply_gates(_nbits(a), _ptr(_state(a)), _ptr(g), g.size) != 0:
        raise ValueError("invalid gate (target/control out of range or control == target)")
    return a


def apply_gates_sharded(a: np.ndarray, gates, g_bits: int) -> int:
    """or_apply_gates_sharded: the same circuit over 2^g shards with Fig. 8
    reorganisations; returns the reorganisation count."""
    g = _gates(gates)
    r = lib().or_apply_gates_sharded(_nbits(a), g_bits, _ptr(g), g.size, _ptr(_state(a)))
    if r < 0:
        raise ValueError("invalid gate or g")
    return r


def write_snapshot(a: np.ndarray, path: str) -> int:
    """SPEC's debug/oracle snapshot: header "s=<s> M=<M>" (s = 2 basis
    states per QU-bit, M = QU-bits), then "<index> <re> <im>" with 17
    significant digits for every nonzero amplitude in index order.  Plain
    Python (no C); returns the number of amplitude lines."""
    n = _nbits(a)
    lines = 0
    with open(path, "w") as f:
        f.write(f"s=2 M={n}\n")
        for i, v in enumerate(a):
            if v.real == 0.0 and v.imag == 0.0:
                continue
            f.write(f"{i} {float(v.real):.17g} {float(v.imag):.17g}\n")
            lines += 1
    return lines


def read_snapshot(path: str) -> tuple[int, int, dict]:
    """(s, M, {index: complex}) of a snapshot file."""
    with open(path) as f:
        head = f.readline().split()
        s = int(head[0].split("=")[1])
        m = int(head[1].split("=")[1])
        amps = {}
        for line in f:
            i, re, im = line.split()
            amps[int(i)] = complex(float(re), float(im))
    return s, m, amps
