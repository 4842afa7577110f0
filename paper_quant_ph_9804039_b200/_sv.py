"""Thin ctypes binding of include/sv.h (argument marshalling only).

Every function here has the name of the C entry point it calls; all device
work runs in libsv.so's CUDA kernels.  There is no CPU fallback: if libsv.so
is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# SV_LIB may point at an alternative build of the same library (A/B tuning).
LIB_PATH = os.environ.get("SV_LIB") or os.path.join(_PKG, "libsv.so")

SV_OK, SV_EINVAL, SV_ENOMEM, SV_ECUDA, SV_ENCCL, SV_ESTATE, SV_ETOOBIG = 0, -1, -2, -3, -4, -5, -6
SV_C64, SV_C128 = 0, 1
SV_INIT_UNIFORM, SV_INIT_GAUSSIAN, SV_INIT_ZERO_STATE = 0, 1, 2
SV_DIFFUSE_WHT, SV_DIFFUSE_MEAN = 0, 1
(SV_K_WHT_TILE, SV_K_WHT_WHOLE, SV_K_MEAN, SV_K_REDUCE, SV_K_INIT, SV_K_ORACLE, SV_K_READOUT,
 SV_K_EXCHANGE, SV_K_ALLREDUCE, SV_K_GATE_TILE, SV_K_SCALE, SV_K_COUNT) = range(12)
KERNEL_KIND_NAMES = ["wht_tile", "wht_whole", "mean", "reduce", "init", "oracle", "readout", "exchange", "allreduce",
                     "gate_tile", "scale"]
# sv_gate (80 bytes): int32 target, int32 reserved, uint64 controls, double m[8] = [w x; y z] as (re, im)
GATE_DTYPE = np.dtype([("target", "<i4"), ("reserved", "<i4"), ("controls", "<u8"), ("m", "<f8", (8,))])

NP_DTYPE = {SV_C64: np.complex64, SV_C128: np.complex128}


class SvError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn} -> {code}: {msg}")
        self.code = code


class sv_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("nccl_id", ctypes.c_void_p),
                ("device", ctypes.c_int), ("stream", ctypes.c_void_p)]


class sv_plan_step(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("pre", ctypes.c_int), ("mid", ctypes.c_int), ("post", ctypes.c_int),
                ("in_recv", ctypes.c_int), ("tile_bits", ctypes.c_int), ("tile_mask", ctypes.c_uint64),
                ("proc_mask", ctypes.c_uint64)]


class sv_tile_variant(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("u", ctypes.c_int), ("pre", ctypes.c_int), ("mid", ctypes.c_int),
                ("post", ctypes.c_int), ("noisy", ctypes.c_int), ("xchg", ctypes.c_int)]


class sv_gate_plan_step(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("tile_bits", ctypes.c_int), ("tile_mask", ctypes.c_uint64),
                ("proc_mask", ctypes.c_uint64), ("first", ctypes.c_uint64), ("count", ctypes.c_uint64),
                ("ops", ctypes.c_uint64), ("lin_ops", ctypes.c_uint64)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python paper_quant_ph_9804039_b200/build.py` "
                      "(no CPU fallback exists)")
lib = ctypes.CDLL(LIB_PATH)

_u64, _i32, _vp, _dp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
_ctxp = ctypes.c_void_p
_SIGS = {
    "sv_init": ([ctypes.POINTER(_ctxp), _i32, _u64, _i32, _i32, ctypes.POINTER(sv_dist)], _i32),
    "sv_reset": ([_ctxp, _u64, _i32], _i32),
    "sv_set_marked": ([_ctxp, _vp, _u64], _i32),
    "sv_apply_oracle": ([_ctxp, _vp, _u64], _i32),
    "sv_diffuse": ([_ctxp, _i32], _i32),
    "sv_iterate": ([_ctxp, _i32, _i32], _i32),
    "sv_iterate_noisy": ([_ctxp, _i32, ctypes.c_double, _u64, _u64], _i32),
    "sv_iterate_decoherent": ([_ctxp, _i32, ctypes.c_double, ctypes.c_double, _u64, _u64, _vp], _i32),
    "sv_probabilities": ([_ctxp, _vp, _u64, _i32], _i32),
    "sv_measure_marked_mass": ([_ctxp, _dp], _i32),
    "sv_norm2": ([_ctxp, _dp], _i32),
    "sv_sample": ([_ctxp, _u64, _u64, _vp, _i32], _i32),
    "sv_get_amplitudes": ([_ctxp, _vp, _u64, _u64], _i32),
    "sv_set_amplitudes": ([_ctxp, _vp, _u64, _u64], _i32),
    "sv_marked_from_seed": ([_i32, _u64, _u64, _vp], _i32),
    "sv_info": ([_ctxp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                 ctypes.POINTER(_u64), ctypes.POINTER(_i32)], _i32),
    "sv_synchronize": ([_ctxp], _i32),
    "sv_comm_info": ([_ctxp, ctypes.POINTER(_i32), ctypes.POINTER(_i32)], _i32),
    "sv_attach": ([_ctxp, _vp, _u64], _i32),
    "sv_snapshot": ([_ctxp, ctypes.c_char_p, ctypes.POINTER(_u64)], _i32),
    "sv_set_exchange": ([_ctxp, _i32], _i32),
    "sv_get_exchange": ([_ctxp, ctypes.POINTER(_i32)], _i32),
    "sv_nccl_unique_id": ([_vp, ctypes.c_size_t], _i32),
    "sv_plan_wht": ([_i32, _i32, _i32, _i32, _i32, ctypes.POINTER(sv_plan_step), _i32, ctypes.POINTER(_i32)], _i32),
    "sv_debug_wht_variants": ([_i32, _i32, _i32, _i32, _i32, ctypes.c_double, ctypes.c_double, _u64, _i32,
                               ctypes.POINTER(sv_tile_variant), _i32, ctypes.POINTER(_i32)], _i32),
    "sv_apply_gates": ([_ctxp, _vp, _u64], _i32),
    "sv_plan_gates": ([_i32, _i32, _i32, _vp, _u64, ctypes.POINTER(sv_gate_plan_step), _i32, ctypes.POINTER(_i32),
                       _vp], _i32),
    "sv_debug_gate_relayouts": ([_i32, _i32, _i32, _vp, _u64, _vp, _i32, ctypes.POINTER(_i32)], _i32),
    "sv_debug_gate_jit": ([_i32, _i32, _vp, _u64, _i32, ctypes.POINTER(_u64), ctypes.POINTER(_u64), _dp], _i32),
    "sv_profile": ([_ctxp, _i32], _i32),
    "sv_profile_read": ([_ctxp, _i32, ctypes.POINTER(_u64), _dp], _i32),
    "sv_profile_timeline": ([_ctxp, _vp, _vp, _u64, ctypes.POINTER(_u64)], _i32),
    "sv_free": ([_ctxp], None),
    "sv_last_error": ([], ctypes.c_char_p),
    "sv_debug_tile_layout": ([_i32, _i32, _i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32)], _i32),
    "sv_debug_tile_owner": ([_i32, _i32, _i32], _i32),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def _check(rc: int, fn: str) -> None:
    if rc != SV_OK:
        raise SvError(rc, fn, lib.sv_last_error().decode())


def _u64_array(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


class Ctx:
    """Owns one sv_ctx* (freed on close / garbage collection)."""

    def __init__(self, ptr: int, n: int, dtype: int):
        self.ptr = ctypes.c_void_p(ptr)
        self.n = n
        self.dtype = dtype

    def close(self):
        if self.ptr:
            lib.sv_free(self.ptr)
            self.ptr = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def sv_init(n: int, seed: int = 0, dtype: int = SV_C64, init: int = SV_INIT_UNIFORM, rank: int = 0, world: int = 1,
            nccl_id: bytes | None = None, device: int = 0, stream: int | None = None) -> Ctx:
    out = ctypes.c_void_p()
    dist = None
    idbuf = None
    if world > 1 or stream is not None or device != 0 or nccl_id is not None:
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        dist = sv_dist(rank, world, ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None, device,
                       stream if stream else None)
    _check(lib.sv_init(ctypes.byref(out), n, seed, dtype, init, ctypes.byref(dist) if dist else None), "sv_init")
    return Ctx(out.value, n, dtype)


def sv_reset(ctx: Ctx, seed: int = 0, init: int = SV_INIT_UNIFORM) -> None:
    _check(lib.sv_reset(ctx.ptr, seed, init), "sv_reset")


def sv_set_marked(ctx: Ctx, marked) -> None:
    m = _u64_array(marked)
    _check(lib.sv_set_marked(ctx.ptr, m.ctypes.data if m.size else None, m.size), "sv_set_marked")


def sv_apply_oracle(ctx: Ctx, marked) -> None:
    m = _u64_array(marked)
    _check(lib.sv_apply_oracle(ctx.ptr, m.ctypes.data if m.size else None, m.size), "sv_apply_oracle")


def sv_diffuse(ctx: Ctx, diffusion: int = SV_DIFFUSE_WHT) -> None:
    _check(lib.sv_diffuse(ctx.ptr, diffusion), "sv_diffuse")


def sv_iterate(ctx: Ctx, k: int, diffusion: int = SV_DIFFUSE_WHT) -> None:
    _check(lib.sv_iterate(ctx.ptr, k, diffusion), "sv_iterate")


def sv_iterate_noisy(ctx: Ctx, k: int, sigma: float, seed: int, t0: int = 0) -> None:
    _check(lib.sv_iterate_noisy(ctx.ptr, k, sigma, seed, t0), "sv_iterate_noisy")


def sv_iterate_decoherent(ctx: Ctx, k: int, sigma: float, rate: float, seed: int, t0: int = 0) -> np.ndarray:
    """k iterations with angle errors + the decoherence step (G22); returns survival[k]."""
    surv = np.zeros(max(k, 1), dtype=np.float64)
    _check(lib.sv_iterate_decoherent(ctx.ptr, k, sigma, rate, seed, t0, surv.ctypes.data), "sv_iterate_decoherent")
    return surv[:k]


def sv_info(ctx: Ctx) -> dict:
    n, w, r, dt = _i32(), _i32(), _i32(), _i32()
    ll = _u64()
    _check(lib.sv_info(ctx.ptr, ctypes.byref(n), ctypes.byref(w), ctypes.byref(r), ctypes.byref(ll),
                       ctypes.byref(dt)), "sv_info")
    return {"n": n.value, "world": w.value, "rank": r.value, "local_len": ll.value, "dtype": dt.value}


def sv_probabilities(ctx: Ctx, out_device_ptr: int | None = None, length: int | None = None) -> np.ndarray | None:
    """Host path returns a float64 array; device path writes to out_device_ptr."""
    ll = sv_info(ctx)["local_len"] if length is None else length
    if out_device_ptr is not None:
        _check(lib.sv_probabilities(ctx.ptr, out_device_ptr, ll, 1), "sv_probabilities")
        return None
    p = np.empty(ll, dtype=np.float64)
    _check(lib.sv_probabilities(ctx.ptr, p.ctypes.data, ll, 0), "sv_probabilities")
    return p


def sv_sample(ctx: Ctx, shots: int, seed: int, out_device_ptr: int | None = None) -> np.ndarray | None:
    """Seeded whole-register measurement (G21): `shots` global indices."""
    if out_device_ptr is not None:
        _check(lib.sv_sample(ctx.ptr, shots, seed, out_device_ptr, 1), "sv_sample")
        return None
    out = np.empty(shots, dtype=np.uint64)
    _check(lib.sv_sample(ctx.ptr, shots, seed, out.ctypes.data if shots else None, 0), "sv_sample")
    return out


def sv_measure_marked_mass(ctx: Ctx) -> float:
    v = ctypes.c_double()
    _check(lib.sv_measure_marked_mass(ctx.ptr, ctypes.byref(v)), "sv_measure_marked_mass")
    return v.value


def sv_norm2(ctx: Ctx) -> float:
    """sum |a|^2 over the whole register (fp64, all ranks)."""
    v = ctypes.c_double()
    _check(lib.sv_norm2(ctx.ptr, ctypes.byref(v)), "sv_norm2")
    return v.value


def sv_get_amplitudes(ctx: Ctx, offset: int = 0, count: int | None = None) -> np.ndarray:
    if count is None:
        count = sv_info(ctx)["local_len"] - offset
    out = np.empty(count, dtype=NP_DTYPE[ctx.dtype])
    _check(lib.sv_get_amplitudes(ctx.ptr, out.ctypes.data, offset, count), "sv_get_amplitudes")
    return out


def sv_set_amplitudes(ctx: Ctx, values: np.ndarray, offset: int = 0) -> None:
    v = np.ascontiguousarray(values, dtype=NP_DTYPE[ctx.dtype])
    _check(lib.sv_set_amplitudes(ctx.ptr, v.ctypes.data, offset, v.size), "sv_set_amplitudes")


def sv_marked_from_seed(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty(m, dtype=np.uint64)
    _check(lib.sv_marked_from_seed(n, m, seed, out.ctypes.data if m else None), "sv_marked_from_seed")
    return out


def sv_set_exchange(ctx: Ctx, fused: bool) -> None:
    _check(lib.sv_set_exchange(ctx.ptr, int(fused)), "sv_set_exchange")


def sv_get_exchange(ctx: Ctx) -> bool:
    v = _i32()
    _check(lib.sv_get_exchange(ctx.ptr, ctypes.byref(v)), "sv_get_exchange")
    return bool(v.value)


def sv_comm_info(ctx: Ctx) -> dict:
    """The context's NCCL communicator: {"nranks": 0, "rank": -1} without one."""
    nr, ur = _i32(), _i32()
    _check(lib.sv_comm_info(ctx.ptr, ctypes.byref(nr), ctypes.byref(ur)), "sv_comm_info")
    return {"nranks": nr.value, "rank": ur.value}


def sv_attach(ctx: Ctx, dev_ptr: int, nbytes: int) -> None:
    """Compute in place in a caller-owned device buffer (e.g. tensor.data_ptr()); the caller keeps ownership."""
    _check(lib.sv_attach(ctx.ptr, dev_ptr, nbytes), "sv_attach")


def sv_snapshot(ctx: Ctx, path: str) -> int:
    """SPEC's text snapshot (header "s=2 M=<n>", "<index> <re> <im>" per nonzero amplitude); returns the line count."""
    w = _u64()
    _check(lib.sv_snapshot(ctx.ptr, os.fsencode(path), ctypes.byref(w)), "sv_snapshot")
    return w.value


def sv_synchronize(ctx: Ctx) -> None:
    _check(lib.sv_synchronize(ctx.ptr), "sv_synchronize")


def sv_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.sv_nccl_unique_id(buf, 128), "sv_nccl_unique_id")
    return buf.raw


def sv_plan_wht(n: int, world: int, dtype: int, k: int, with_oracle: bool) -> list[dict]:
    cnt = _i32()
    _check(lib.sv_plan_wht(n, world, dtype, k, int(with_oracle), None, 0, ctypes.byref(cnt)), "sv_plan_wht")
    arr = (sv_plan_step * max(cnt.value, 1))()
    _check(lib.sv_plan_wht(n, world, dtype, k, int(with_oracle), arr, cnt.value, ctypes.byref(cnt)), "sv_plan_wht")
    return [{f: getattr(arr[i], f) for f, _ in sv_plan_step._fields_} for i in range(cnt.value)]


def sv_debug_wht_variants(n: int, world: int, dtype: int, flavour: int, k: int, sigma: float = 0.0,
                          rate: float = 0.0, seed: int = 0, fused: bool = True) -> list[tuple]:
    """Kernel variants (family, u, pre, mid, post, noisy, xchg) one call launches, in order (host only)."""
    cnt = _i32()
    args = (n, world, dtype, flavour, k, sigma, rate, seed, int(fused))
    _check(lib.sv_debug_wht_variants(*args, None, 0, ctypes.byref(cnt)), "sv_debug_wht_variants")
    arr = (sv_tile_variant * max(cnt.value, 1))()
    _check(lib.sv_debug_wht_variants(*args, arr, cnt.value, ctypes.byref(cnt)), "sv_debug_wht_variants")
    return [tuple(getattr(arr[i], f) for f, _ in sv_tile_variant._fields_) for i in range(cnt.value)]


def _gates(gates) -> np.ndarray:
    g = np.ascontiguousarray(gates, dtype=GATE_DTYPE)
    assert g.dtype.itemsize == 80
    return g


def sv_apply_gates(ctx: Ctx, gates) -> None:
    g = _gates(gates)
    _check(lib.sv_apply_gates(ctx.ptr, g.ctypes.data if g.size else None, g.size), "sv_apply_gates")


def sv_plan_gates(n: int, world: int, dtype: int, gates) -> tuple[list[dict], np.ndarray]:
    g = _gates(gates)
    gp = g.ctypes.data if g.size else None
    cnt = _i32()
    _check(lib.sv_plan_gates(n, world, dtype, gp, g.size, None, 0, ctypes.byref(cnt), None), "sv_plan_gates")
    arr = (sv_gate_plan_step * max(cnt.value, 1))()
    order = np.zeros(max(g.size, 1), dtype=np.uint64)
    _check(lib.sv_plan_gates(n, world, dtype, gp, g.size, arr, cnt.value, ctypes.byref(cnt), order.ctypes.data),
           "sv_plan_gates")
    steps = [{f: getattr(arr[i], f) for f, _ in sv_gate_plan_step._fields_} for i in range(cnt.value)]
    return steps, order[:g.size]


def sv_debug_gate_relayouts(n: int, world: int, dtype: int, gates) -> np.ndarray:
    g = _gates(gates)
    ns = ctypes.c_int()
    _check(lib.sv_debug_gate_relayouts(n, world, dtype, g.ctypes.data if len(g) else None, len(g), None, 0,
                                       ctypes.byref(ns)), "sv_debug_gate_relayouts")
    out = np.zeros(max(ns.value, 1), dtype=np.uint64)
    _check(lib.sv_debug_gate_relayouts(n, world, dtype, g.ctypes.data if len(g) else None, len(g), out.ctypes.data,
                                       ns.value, ctypes.byref(ns)), "sv_debug_gate_relayouts")
    return out[:ns.value]


def sv_debug_gate_jit(n: int = 0, dtype: int = SV_C64, gates=None, compile: int = 0) -> dict:
    """Gate-engine JIT: compile=1 compiles every pass kernel of a circuit (host only); always returns
    the launch-side counters (kernels compiled and loaded, NVRTC seconds)."""
    g = _gates(gates if gates is not None else np.zeros(0, dtype=GATE_DTYPE))
    p, c, t = _u64(), _u64(), ctypes.c_double()
    _check(lib.sv_debug_gate_jit(n, dtype, g.ctypes.data if g.size else None, g.size, int(compile), ctypes.byref(p),
                                 ctypes.byref(c), ctypes.byref(t)), "sv_debug_gate_jit")
    return {"passes": p.value, "compiles": c.value, "compile_seconds": t.value}


def sv_profile(ctx: Ctx, enable: bool) -> None:
    _check(lib.sv_profile(ctx.ptr, int(enable)), "sv_profile")


def sv_profile_read(ctx: Ctx, kind: int) -> tuple[int, float]:
    n = _u64()
    ms = ctypes.c_double()
    _check(lib.sv_profile_read(ctx.ptr, kind, ctypes.byref(n), ctypes.byref(ms)), "sv_profile_read")
    return n.value, ms.value


def sv_profile_timeline(ctx: Ctx) -> list[tuple[int, float]]:
    cnt = _u64()
    _check(lib.sv_profile_timeline(ctx.ptr, None, None, 0, ctypes.byref(cnt)), "sv_profile_timeline")
    kinds = np.zeros(max(cnt.value, 1), dtype=np.int32)
    ms = np.zeros(max(cnt.value, 1), dtype=np.float64)
    _check(lib.sv_profile_timeline(ctx.ptr, kinds.ctypes.data, ms.ctypes.data, cnt.value, ctypes.byref(cnt)),
           "sv_profile_timeline")
    return [(int(kinds[i]), float(ms[i])) for i in range(cnt.value)]


def sv_free(ctx: Ctx) -> None:
    ctx.close()


def sv_last_error() -> str:
    return lib.sv_last_error().decode()
