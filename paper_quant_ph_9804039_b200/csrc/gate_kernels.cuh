// gate_kernels.cuh -- device side of the gate-circuit tile pass (SURVEY 8(f)
// NEXT-4): op records, the 2x2 / phase-polynomial op code, the op-program
// interpreter kernels.  Included by gates.cu (nvcc) and by the pass-specialised
// kernels gate_jit.cpp compiles at run time with NVRTC (device code only).
#pragma once
#include "wht_kernels.cuh"

namespace sv {

// Coefficients per op record: w, x, y, z as (re, im); complex64 records add
// the pairs (-w.im, w.im), (-x.im, x.im), (-y.im, y.im), (-z.im, z.im) so the
// packed FFMA2 form reads them as 64-bit uniform operands (no per-pair
// re-assembly).
template <typename R>
constexpr int kNM = sizeof(R) == 4 ? 16 : 8;

template <typename R>
struct alignas(16) GOp {
    R m[kNM<R>];             // w, x, y, z as (re, im) [+ complex64: the (-im, im) pairs]
    unsigned int ph;         // register layout (0 = A, 1 = B, 2 = C) | kind << 8
    unsigned int ri;         // register index of the target tile bit (whole kernel: target slot)
    unsigned int jm;         // controls that are register bits of ph (register-index space)
    unsigned int tm;         // controls that are thread bits of ph (tile-element space)
    unsigned long long fm;   // controls outside the tile (local index space; whole kernel: all controls)
};

// Matrix shape, decided on the host from the exact coefficients: the same
// [w x; y z] product with the zero terms (and unit factors) skipped, so the
// result is identical to the general formula up to the rounding of the
// skipped exact zeros / ones.
enum GateKind : unsigned int {
    GK_GENERAL = 0,   // [w x; y z]
    GK_DIAG = 1,      // x = y = 0: (w u, z v)
    GK_PHASE = 2,     // x = y = 0, w = 1: (u, z v)
    GK_ANTI = 3,      // w = z = 0: (x v, y u)
    GK_SWAP = 4,      // w = z = 0, x = y = 1 (NOT): (v, u)
    GK_LINPHASE = 5,  // merged run of phase gates on one target, <= 1 control each (below)
    GK_DIAGT = 6,     // diagonal gate whose target is a THREAD bit of the current layout:
                      // every amplitude of the thread gets w (bit 0) or z (bit 1); ri = target tile bit
};

// GK_LINPHASE: the product of phase gates diag(1, z_g) on one target t, each
// with at most one control c_g, multiplies amplitude i by
//   prod_g z_g^(b_t(i) b_cg(i))  =  [b_t(i)] F(thread, tile) R(register bits),
// a phase that factorises over the control bits (degree-2 phase polynomial,
// as in the QFT).  The host merges a run of such gates (diagonal gates
// commute) into ONE op; it needs no relayout (its target need not be a
// register bit) and costs ~40 complex multiplies per thread instead of one
// dispatched op per gate.  The op record is followed by `tm` entry records:
// m[0], m[1] = z; ri = where the control lives (LP_*); jm = its register
// index / tile bit / slot.  The op's own ri/jm say where the TARGET lives
// (LP_REG with register index, or LP_THR with tile bit).
enum LinWhere : unsigned int { LP_REG = 0, LP_THR = 1, LP_FREE = 2, LP_CONST = 3 };

// (u, v) <- (w u + x v, y u + z v), complex.
#ifndef SV_GATE_PACKED
#define SV_GATE_PACKED 1
#endif
template <typename E, typename R>
__device__ __forceinline__ void cmat(E &u, E &v, const R (&m)[kNM<R>]) {
#if SV_GATE_PACKED
    if constexpr (sizeof(R) == 4) {  // complex64: packed (re, im) FMUL2 / FFMA2, 8 instead of 16 per pair
        const float2 a = u, b = v;
        const float2 as = make_float2(a.y, a.x), bs = make_float2(b.y, b.x);
        float2 t = __fmul2_rn(make_float2(m[0], m[0]), a);
        t = __ffma2_rn(make_float2(m[8], m[9]), as, t);
        t = __ffma2_rn(make_float2(m[2], m[2]), b, t);
        u = __ffma2_rn(make_float2(m[10], m[11]), bs, t);
        t = __fmul2_rn(make_float2(m[4], m[4]), a);
        t = __ffma2_rn(make_float2(m[12], m[13]), as, t);
        t = __ffma2_rn(make_float2(m[6], m[6]), b, t);
        v = __ffma2_rn(make_float2(m[14], m[15]), bs, t);
        return;
    }
#endif
    const E a = u, b = v;
    u.x = m[0] * a.x - m[1] * a.y + m[2] * b.x - m[3] * b.y;
    u.y = m[0] * a.y + m[1] * a.x + m[2] * b.y + m[3] * b.x;
    v.x = m[4] * a.x - m[5] * a.y + m[6] * b.x - m[7] * b.y;
    v.y = m[4] * a.y + m[5] * a.x + m[6] * b.y + m[7] * b.x;
}

// c <- (re, im) * c, complex
template <typename E, typename R>
__device__ __forceinline__ void cscale(E &c, R re, R im) {
    const E a = c;
    c.x = re * a.x - im * a.y;
    c.y = re * a.y + im * a.x;
}

// complex64: c <- coefficient q of the record times c, packed: (re, re) * c
// + (-im, im) * swap(c)
template <int Q>
__device__ __forceinline__ float2 cscale_p(const float2 c, const float (&m)[16]) {
    const float2 t = __fmul2_rn(make_float2(m[2 * Q], m[2 * Q]), c);
    return __ffma2_rn(make_float2(m[8 + 2 * Q], m[9 + 2 * Q]), make_float2(c.y, c.x), t);
}

template <unsigned int K, typename E, typename R>
__device__ __forceinline__ void cmat_k(E &u, E &v, const R (&m)[kNM<R>]) {
#if SV_GATE_PACKED
    if constexpr (sizeof(R) == 4 && K != GK_GENERAL && K != GK_SWAP) {
        if constexpr (K == GK_DIAG) {
            u = cscale_p<0>(u, m);
            v = cscale_p<3>(v, m);
        } else if constexpr (K == GK_PHASE) {
            v = cscale_p<3>(v, m);
        } else {  // GK_ANTI
            const float2 a = u;
            u = cscale_p<1>(v, m);
            v = cscale_p<2>(a, m);
        }
        return;
    }
#endif
    if constexpr (K == GK_GENERAL) {
        cmat(u, v, m);
    } else if constexpr (K == GK_DIAG) {
        cscale(u, m[0], m[1]);
        cscale(v, m[6], m[7]);
    } else if constexpr (K == GK_PHASE) {
        cscale(v, m[6], m[7]);
    } else if constexpr (K == GK_ANTI) {
        const E a = u, b = v;
        u.x = m[2] * b.x - m[3] * b.y;
        u.y = m[2] * b.y + m[3] * b.x;
        v.x = m[4] * a.x - m[5] * a.y;
        v.y = m[4] * a.y + m[5] * a.x;
    } else {
        const E a = u;
        u = v;
        v = a;
    }
}

template <int I, unsigned int K, int NR, typename E, typename R>
__device__ __forceinline__ void gate_apply(E (&x)[NR], const R (&m)[kNM<R>], unsigned int jm) {
#pragma unroll
    for (int j = 0; j < NR; ++j)
        if (!(j & (1 << I)))
            if (((unsigned int)j & jm) == jm) cmat_k<K>(x[j], x[j | (1 << I)], m);
}

#ifndef SV_GATE_KINDS
#define SV_GATE_KINDS 2  // 2: all shapes; 1: general + phase; 0: general only (smaller code)
#endif
template <int I, int NR, typename E, typename R>
__device__ __forceinline__ void gate_apply_kind(E (&x)[NR], const R (&m)[kNM<R>], unsigned int jm, unsigned int kind) {
#if SV_GATE_KINDS >= 2
    switch (kind) {
        case GK_DIAG: gate_apply<I, GK_DIAG>(x, m, jm); break;
        case GK_PHASE: gate_apply<I, GK_PHASE>(x, m, jm); break;
        case GK_ANTI: gate_apply<I, GK_ANTI>(x, m, jm); break;
        case GK_SWAP: gate_apply<I, GK_SWAP>(x, m, jm); break;
        default: gate_apply<I, GK_GENERAL>(x, m, jm); break;
    }
#elif SV_GATE_KINDS == 1
    if (kind == GK_PHASE) gate_apply<I, GK_PHASE>(x, m, jm);
    else gate_apply<I, GK_GENERAL>(x, m, jm);
#else
    (void)kind;
    gate_apply<I, GK_GENERAL>(x, m, jm);
#endif
}

template <class L, typename E, typename R>
__device__ __forceinline__ void gate_dispatch(E (&x)[L::NR], const R (&m)[kNM<R>], unsigned int ri, unsigned int jm,
                                              unsigned int kind) {
    switch (ri) {
        case 0: gate_apply_kind<0>(x, m, jm, kind); break;
        case 1: gate_apply_kind<1>(x, m, jm, kind); break;
        case 2: gate_apply_kind<2>(x, m, jm, kind); break;
        case 3: gate_apply_kind<3>(x, m, jm, kind); break;
        default:
            if constexpr (L::kRB > 4) gate_apply_kind<(L::kRB > 4 ? 4 : 0)>(x, m, jm, kind);
            break;
    }
}

template <class L, typename E>
__device__ __forceinline__ void relayout_dyn(E (&x)[L::NR], E *sm, int tid, unsigned int from, unsigned int to) {
    if constexpr (L::kNPH == 2) {  // two-layout family: A <-> B only
        if (from == 0 && to == 1) relayout<L, 0, 1>(x, sm, tid);
        else if (from == 1 && to == 0) relayout<L, 1, 0>(x, sm, tid);
        return;
    } else {
        switch (from * 3 + to) {
            case 1: relayout<L, 0, 1>(x, sm, tid); break;
            case 2: relayout<L, 0, 2>(x, sm, tid); break;
            case 3: relayout<L, 1, 0>(x, sm, tid); break;
            case 5: relayout<L, 1, 2>(x, sm, tid); break;
            case 6: relayout<L, 2, 0>(x, sm, tid); break;
            case 7: relayout<L, 2, 1>(x, sm, tid); break;
            default: break;
        }
    }
}

// Op-program reads: GLB = the program in global memory (read-only path);
// else it is a __grid_constant__ kernel parameter (constant bank).
template <bool GLB, typename T>
__device__ __forceinline__ T ldop(const T *q) {
    if constexpr (GLB) return __ldg(q);
    else return *q;
}

template <bool GLB, typename R>
__device__ __forceinline__ void load_op(const GOp<R> *op, R (&m)[kNM<R>], unsigned int &ph, unsigned int &ri,
                                        unsigned int &jm, unsigned int &tm, unsigned long long &fm) {
#pragma unroll
    for (int e = 0; e < kNM<R>; ++e) m[e] = ldop<GLB>(&op->m[e]);
    ph = ldop<GLB>(&op->ph);
    ri = ldop<GLB>(&op->ri);
    jm = ldop<GLB>(&op->jm);
    tm = ldop<GLB>(&op->tm);
    fm = ldop<GLB>(&op->fm);
}

template <typename E, typename R>
__device__ __forceinline__ void cmul_by(E &a, R br, R bi) {
    const E t = a;
    a.x = t.x * br - t.y * bi;
    a.y = t.x * bi + t.y * br;
}
template <typename E>
__device__ __forceinline__ E cprod(const E &a, const E &b) {
#if SV_GATE_PACKED
    if constexpr (sizeof(a.x) == 4) {  // complex64: (b.re, b.re) * a + (-b.im, b.im) * swap(a)
        const float2 t = __fmul2_rn(make_float2(b.x, b.x), a);
        return __ffma2_rn(make_float2(-b.y, b.y), make_float2(a.y, a.x), t);
    }
#endif
    E r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}

template <class L, bool GLB, typename E, typename R>
__device__ __forceinline__ void apply_linphase(E (&x)[L::NR], const GOp<R> *ent, unsigned int cnt, unsigned int tcls,
                                               unsigned int tbit, unsigned int et, unsigned long long base,
                                               unsigned int nthr) {
    constexpr int RB = L::kRB, LO = RB < 3 ? RB : 3, HI = RB - LO;
    // entries: [0, RB) per-register-bit factors, [RB, RB + nthr) thread-bit
    // factors, then the tile-uniform free-slot / constant factors -- those are
    // the same for the whole CTA, so the lanes of a warp take them in
    // parallel and combine them in a fixed tree (every lane gets lane 0's
    // product: identical, deterministic)
    const unsigned int lane = threadIdx.x & 31u;
    E F;
    F.x = (R)1;
    F.y = (R)0;
    if constexpr (!GLB) {
        // program in the constant bank: lane-varying entry indices would
        // serialise the constant cache, so every lane walks the entries with
        // uniform loads and multiplies them in entry order (identical in all lanes)
        for (unsigned int e = RB + nthr; e < cnt; ++e) {
            const unsigned int w = ldop<GLB>(&ent[e].ri), bit = ldop<GLB>(&ent[e].jm);
            if (w == LP_CONST || ((base >> bit) & 1ull)) cmul_by(F, ldop<GLB>(&ent[e].m[0]), ldop<GLB>(&ent[e].m[1]));
        }
    } else {
    for (unsigned int e = RB + nthr + lane; e < cnt; e += 32u) {
        const unsigned int w = ldop<GLB>(&ent[e].ri), bit = ldop<GLB>(&ent[e].jm);
        if (w == LP_CONST || ((base >> bit) & 1ull)) cmul_by(F, ldop<GLB>(&ent[e].m[0]), ldop<GLB>(&ent[e].m[1]));
    }
    if (cnt > RB + nthr) {  // any tile-uniform entries: every lane needs the full product
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            E t;
            t.x = __shfl_down_sync(0xffffffffu, F.x, o);
            t.y = __shfl_down_sync(0xffffffffu, F.y, o);
            if (lane + o < 32u) F = cprod(F, t);
        }
        F.x = __shfl_sync(0xffffffffu, F.x, 0);
        F.y = __shfl_sync(0xffffffffu, F.y, 0);
    }
    }
    if (tcls == LP_THR && !((et >> tbit) & 1u)) return;  // target bit 0 for all of this thread's amplitudes
    E P[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) { P[i].x = ldop<GLB>(&ent[i].m[0]); P[i].y = ldop<GLB>(&ent[i].m[1]); }
    for (unsigned int e = RB; e < RB + nthr; ++e)
        if ((et >> ldop<GLB>(&ent[e].jm)) & 1u) cmul_by(F, ldop<GLB>(&ent[e].m[0]), ldop<GLB>(&ent[e].m[1]));
    // factor of register index j = F * prod_{i in bits(j)} P[i]: tables over
    // the low LO and the high HI register bits
    E lo[1 << LO], hi[1 << HI];
    lo[0].x = (R)1;
    lo[0].y = (R)0;
#pragma unroll
    for (int j = 1; j < (1 << LO); ++j) lo[j] = cprod(lo[j & (j - 1)], (j & 1) ? P[0] : ((j & 2) ? P[1] : P[RB > 2 ? 2 : 0]));
    hi[0] = F;
#pragma unroll
    for (int j = 1; j < (1 << HI); ++j) hi[j] = cprod(hi[j & (j - 1)], (j & 1) ? P[LO < RB ? LO : 0] : P[LO + 1 < RB ? LO + 1 : 0]);
#pragma unroll
    for (int j = 0; j < L::NR; ++j)
        if (tcls != LP_REG || ((j >> tbit) & 1)) {
            const E f = cprod(lo[j & ((1 << LO) - 1)], hi[j >> LO]);
            x[j] = cprod(x[j], f);
        }
}

// The pass's op program on one tile held in registers (layout A on entry);
// returns the layout the tile is left in.
template <class L, bool LIN, bool GLB, typename E, typename R>
__device__ __forceinline__ unsigned int run_gate_ops(E (&x)[L::NR], E *sm, int tid, unsigned long long base,
                                                     const GOp<R> *__restrict__ ops, int nops) {
    const unsigned int eth[3] = {L::ethr(0, tid), L::ethr(1, tid), L::ethr(2, tid)};
    unsigned int cur = 0;
    for (int k = 0; k < nops; ++k) {
        R m[kNM<R>];
        unsigned int ph, ri, jm, tm;
        unsigned long long fm;
        load_op<GLB>(ops + k, m, ph, ri, jm, tm, fm);
        const unsigned int kind = ph >> 8;
        ph &= 0xffu;
        if (ph != cur) {
            relayout_dyn<L>(x, sm, tid, cur, ph);
            cur = ph;
        }
        const unsigned int et = cur == 0 ? eth[0] : (cur == 1 ? eth[1] : eth[2]);
        if constexpr (LIN) {  // passes holding merged phase runs get their own instantiation
            if (kind == GK_LINPHASE) {  // tm entry records follow
                apply_linphase<L, GLB>(x, ops + k + 1, tm, ri, jm, et, base, (unsigned int)fm);
                k += (int)tm;
                continue;
            }
        }
        if (kind == GK_DIAGT) {  // diagonal, target on a thread bit: no relayout needed
            if ((et & tm) == tm && (base & fm) == fm) {
                const bool one = (et >> ri) & 1u;
                const R fr = one ? m[6] : m[0], fi = one ? m[7] : m[1];
                if (!(fr == (R)1 && fi == (R)0)) {
#if SV_GATE_PACKED
                    if constexpr (sizeof(R) == 4) {  // packed: (fr, fr) * x + (-fi, fi) * swap(x)
                        const float2 pr = make_float2(fr, fr), pi = make_float2(-fi, fi);
#pragma unroll
                        for (int j = 0; j < L::NR; ++j)
                            if (((unsigned int)j & jm) == jm)
                                x[j] = __ffma2_rn(pi, make_float2(x[j].y, x[j].x), __fmul2_rn(pr, x[j]));
                        continue;
                    }
#endif
#pragma unroll
                    for (int j = 0; j < L::NR; ++j)
                        if (((unsigned int)j & jm) == jm) cmul_by(x[j], fr, fi);
                }
            }
            continue;
        }
        if ((et & tm) == tm && (base & fm) == fm) gate_dispatch<L>(x, m, ri, jm, kind);
    }
    return cur;
}

template <class L, bool XCHG, typename E>
__device__ __forceinline__ void gate_tile_store(const E (&x)[L::NR], unsigned int cur, const KParams &p,
                                                unsigned long long base, int tid, E *const *s_dst) {
    E *gout = reinterpret_cast<E *>(p.out) + base;
    if (cur == 0) pass_store<L, 0, XCHG>(x, gout, base, p, tid, s_dst);
    else if (cur == 1 || L::kNPH == 2) pass_store<L, 1, XCHG>(x, gout, base, p, tid, s_dst);
    else pass_store<L, (L::kNPH > 2 ? 2 : 1), XCHG>(x, gout, base, p, tid, s_dst);
}

template <class L, bool XCHG, bool LIN, bool GLB, typename E, typename R>
__device__ __forceinline__ void gate_tile_body(const KParams &p, const GOp<R> *ops, int nops) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E *sm = reinterpret_cast<E *>(smem_raw);
    __shared__ E *s_dst[XCHG ? 8 : 1];
    if constexpr (XCHG) load_xdst(p, threadIdx.x, s_dst);
    const int tid = threadIdx.x;
    const unsigned long long base = tile_base(blockIdx.x, p);
    E x[L::NR];
    global_load<L, 0>(x, reinterpret_cast<const E *>(p.in) + base, p, tid);
    const unsigned int cur = run_gate_ops<L, LIN, GLB>(x, sm, tid, base, ops, nops);
    gate_tile_store<L, XCHG>(x, cur, p, base, tid, s_dst);
}

// The register-layout family of a gate pass: the three-layout Layout (16-B
// accesses) or, for complex64 strided passes whose non-diagonal targets start
// at tile bit 3 or 4 (the WHT's rule), the two-layout Layout2 (one relayout per
// A <-> B round trip, 8-B accesses; gates.cu gate_pass_l2).
template <typename E, int TB, int RB, bool L2>
struct GateLayout {
    using T = Layout<E, TB, RB>;
};
template <int TB, int RB>
struct GateLayout<float2, TB, RB, true> {
    using T = Layout2<TB, RB>;
};

// One CTA per tile; the op program in global memory.
template <typename E, int TB, int RB, bool XCHG, bool LIN, bool L2 = false>
__global__ void __launch_bounds__(1 << (TB - RB), (TB - RB <= 7) ? 4 : 2)
    gate_tile_kernel(const KParams p, const GOp<typename RealOf<E>::T> *__restrict__ ops, int nops) {
    gate_tile_body<typename GateLayout<E, TB, RB, L2>::T, XCHG, LIN, true, E>(p, ops, nops);
}

// The same with the op program as a kernel parameter (constant bank: uniform
// loads, no global round trip per op) -- passes of up to kParamOps records.
constexpr size_t kParamProgBytes = 24576;
template <typename R>
struct GProg {
    GOp<R> op[kParamProgBytes / sizeof(GOp<R>)];
};
template <typename E, int TB, int RB, bool XCHG, bool LIN, bool L2 = false>
__global__ void __launch_bounds__(1 << (TB - RB), (TB - RB <= 7) ? 4 : 2)
    gate_tile_kernel_p(const KParams p, const __grid_constant__ GProg<typename RealOf<E>::T> prog, int nops) {
    gate_tile_body<typename GateLayout<E, TB, RB, L2>::T, XCHG, LIN, false, E>(p, prog.op, nops);
}

// Whole state (n <= T) in one CTA: every gate as a V/2-pair loop over shared
// memory, one barrier per gate.
template <typename E>
__global__ void __launch_bounds__(512) gate_whole_kernel(E *a, int n, const GOp<typename RealOf<E>::T> *ops,
                                                         int nops) {
    using R = typename RealOf<E>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E *s = reinterpret_cast<E *>(smem_raw);
    const unsigned int N = 1u << n, tid = threadIdx.x, nt = blockDim.x;
    for (unsigned int i = tid; i < N; i += nt) s[i] = a[i];
    __syncthreads();
    for (int k = 0; k < nops; ++k) {
        R m[kNM<R>];
        unsigned int ph, q, jm, tm;
        unsigned long long cm;
        load_op<true>(ops + k, m, ph, q, jm, tm, cm);
        const unsigned int kind = ph >> 8;
        const unsigned int bit = 1u << q;
        for (unsigned int pr = tid; pr < N / 2; pr += nt) {
            const unsigned int i = ((pr >> q) << (q + 1)) | (pr & (bit - 1));
            if ((i & (unsigned int)cm) == (unsigned int)cm) {
                switch (kind) {
                    case GK_DIAG: cmat_k<GK_DIAG>(s[i], s[i | bit], m); break;
                    case GK_PHASE: cmat_k<GK_PHASE>(s[i], s[i | bit], m); break;
                    case GK_ANTI: cmat_k<GK_ANTI>(s[i], s[i | bit], m); break;
                    case GK_SWAP: cmat_k<GK_SWAP>(s[i], s[i | bit], m); break;
                    default: cmat_k<GK_GENERAL>(s[i], s[i | bit], m); break;
                }
            }
        }
        __syncthreads();
    }
    for (unsigned int i = tid; i < N; i += nt) a[i] = s[i];
}

}  // namespace sv
