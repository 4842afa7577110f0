// gates.cu -- gate-circuit tile pass: every gate of a
// planned pass (gate_plan.cpp) applied to a 2^T-amplitude tile on-chip, one
// HBM read + write per pass.
//
// What it computes: for each gate, Fig. 3's general 2x2 [w x; y z]
// on the pairs (a_i, a_{i | 2^t}) with bit t of i clear and all
// control bits of i set ("a 2x2 transformation on a vector of size V, is a
// sequence of V/2 independent 2x2 transformations"; G23 for the
// controls).
//
// How (B200 design): the tile machinery of the
// WHT pass (wht_kernels.cuh): 256 threads, 2^R amplitudes per thread in
// registers, three register layouts A/B/C that together cover the T tile
// bits, XOR-swizzled shared-memory relayouts with one barrier each, 128-bit
// coalesced global accesses in layout A.  A gate on tile bit b runs in a
// layout where b is a register bit (complex 2x2 on register pairs, no
// shared-memory traffic); the host orders the pass's ops to minimise
// relayouts (commuting gates only).  A control bit is a register-index
// predicate (register bit), a thread predicate (thread bit), or a tile
// predicate (slot outside the tile); controls on rank bits are decided per
// rank on the host.  The op program lives in device memory and is read with
// uniform (broadcast) loads.
#include <cuda_runtime.h>

#include <string.h>

#include <algorithm>
#include <complex>
#include <memory>

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
    else if (cur == 1) pass_store<L, 1, XCHG>(x, gout, base, p, tid, s_dst);
    else pass_store<L, 2, XCHG>(x, gout, base, p, tid, s_dst);
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

// One CTA per tile; the op program in global memory.
template <typename E, int TB, int RB, bool XCHG, bool LIN>
__global__ void __launch_bounds__(1 << (TB - RB), (TB - RB <= 7) ? 4 : 2)
    gate_tile_kernel(const KParams p, const GOp<typename RealOf<E>::T> *__restrict__ ops, int nops) {
    gate_tile_body<Layout<E, TB, RB>, XCHG, LIN, true, E>(p, ops, nops);
}

// The same with the op program as a kernel parameter (constant bank: uniform
// loads, no global round trip per op) -- passes of up to kParamOps records.
constexpr size_t kParamProgBytes = 24576;
template <typename R>
struct GProg {
    GOp<R> op[kParamProgBytes / sizeof(GOp<R>)];
};
template <typename E, int TB, int RB, bool XCHG, bool LIN>
__global__ void __launch_bounds__(1 << (TB - RB), (TB - RB <= 7) ? 4 : 2)
    gate_tile_kernel_p(const KParams p, const __grid_constant__ GProg<typename RealOf<E>::T> prog, int nops) {
    gate_tile_body<Layout<E, TB, RB>, XCHG, LIN, false, E>(p, prog.op, nops);
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

// ------------------------------------------------------------------------- //
// Host: op programs                                                          //
// ------------------------------------------------------------------------- //
namespace {

unsigned int gate_kind(const sv_gate &g) {
    const double *m = g.m;
    const bool offzero = m[2] == 0.0 && m[3] == 0.0 && m[4] == 0.0 && m[5] == 0.0;
    const bool diagzero = m[0] == 0.0 && m[1] == 0.0 && m[6] == 0.0 && m[7] == 0.0;
    if (offzero) return (m[0] == 1.0 && m[1] == 0.0) ? GK_PHASE : GK_DIAG;
    if (diagzero) return (m[2] == 1.0 && m[3] == 0.0 && m[4] == 1.0 && m[5] == 0.0) ? GK_SWAP : GK_ANTI;
    return GK_GENERAL;
}

template <typename R>
GOp<R> op_coefs(const sv_gate &g) {
    GOp<R> o{};
    for (int e = 0; e < 8; ++e) o.m[e] = (R)g.m[e];
    if constexpr (kNM<R> == 16)
        for (int q = 0; q < 4; ++q) {
            o.m[8 + 2 * q] = -(R)g.m[2 * q + 1];
            o.m[9 + 2 * q] = (R)g.m[2 * q + 1];
        }
    o.ph = gate_kind(g) << 8;
    return o;
}

// Program of one tile pass for the three-layout family L: tile bits, the
// layout schedule and the per-op predicates.
template <class L, typename R>
void build_tile_ops(const GatePassArgs &a, std::vector<GOp<R>> &out) {
    int slot2bit[64];
    for (int i = 0; i < 64; ++i) slot2bit[i] = -1;
    int b = 0;
    for (int sl = 0; sl < 64; ++sl)
        if ((a.tile_mask >> sl) & 1) slot2bit[sl] = b++;
    struct LinEntry {
        int where;   // 0 tile bit, 1 free slot, 2 none
        int bit;     // tile bit / slot
        double zr, zi;
        sv_gate src;           // the original gate (a short run is emitted gate by gate)
        unsigned int tc;
        unsigned long long fm;
    };
    struct Pend {
        sv_gate g;           // the gate (matrix possibly fused with later ones); for a merged phase
                             // run: diag(1, 1) with the union of the controls (commutation proxy)
        int bt;              // target tile bit
        unsigned int tc;     // controls on tile bits (tile-element space)
        unsigned long long fm;
        std::vector<LinEntry> lin;  // non-empty: a merged run of phase gates (GK_LINPHASE)
    };
    std::vector<Pend> pend;
    for (uint64_t k = 0; k < a.count; ++k) {
        const sv_gate &g = a.gates[a.order[k]];
        const int pt = gate_phys(g.target, a.nl, a.g, a.swapped);
        SV_CHECK(slot2bit[pt] >= 0, SV_EINVAL, "internal: gate target outside its pass tile");
        Pend pd{g, slot2bit[pt], 0u, 0ull, {}};
        bool live = true;
        for (int q = 0; q < a.n; ++q) {
            if (!((g.controls >> q) & 1ull)) continue;
            const int pq = gate_phys(q, a.nl, a.g, a.swapped);
            if (pq >= a.nl && !a.emulated) {  // rank bit of a real rank
                if (!((a.rank >> (pq - a.nl)) & 1)) live = false;
            } else if (slot2bit[pq] >= 0) {
                pd.tc |= 1u << slot2bit[pq];
            } else {
                pd.fm |= 1ull << pq;
            }
        }
        if (!live) continue;
        // Phase gates diag(1, z) with at most one (live) control are merged
        // into a run on their target (GK_LINPHASE) when only commuting ops lie
        // between -- checked before the 2x2 fusion below.
        const bool phase1 = gate_kind(g) == GK_PHASE && __builtin_popcount(pd.tc) + __builtin_popcountll(pd.fm) <= 1;
        if (phase1) {
            LinEntry le{2, 0, g.m[6], g.m[7], g, pd.tc, pd.fm};
            if (pd.tc) { le.where = 0; le.bit = __builtin_ctz(pd.tc); }
            else if (pd.fm) { le.where = 1; le.bit = __builtin_ctzll(pd.fm); }
            bool merged = false;
            CommuteSet between;
            for (size_t i = pend.size(); i-- > 0;) {
                Pend &e = pend[i];
                if (!e.lin.empty() && e.bt == pd.bt && between.commutes(g)) {
                    e.lin.push_back(le);
                    e.g.controls |= g.controls;
                    merged = true;
                    break;
                }
                between.add(e.g);
                if (!between.commutes(g)) break;
            }
            if (merged) continue;
            pd.lin.push_back(le);
            pd.g.m[6] = 1.0;  // proxy: diagonal, support = target + controls
            pd.g.m[7] = 0.0;
            pend.push_back(pd);
            continue;
        }
        // Fusion: a gate with the same target and controls as an earlier op
        // of this pass, with only commuting ops in between, is multiplied
        // into it (host fp64 2x2 product M_later * M_earlier).
        bool fused = false;
        CommuteSet between;
        for (size_t i = pend.size(); i-- > 0;) {
            sv_gate &e = pend[i].g;
            if (pend[i].lin.empty() && e.target == g.target && e.controls == g.controls && between.commutes(g)) {
                double r[8];
                for (int rr = 0; rr < 2; ++rr)
                    for (int cc = 0; cc < 2; ++cc) {
                        double re = 0.0, im = 0.0;
                        for (int kk = 0; kk < 2; ++kk) {
                            const double ar = g.m[2 * (2 * rr + kk)], ai = g.m[2 * (2 * rr + kk) + 1];
                            const double br = e.m[2 * (2 * kk + cc)], bi = e.m[2 * (2 * kk + cc) + 1];
                            re += ar * br - ai * bi;
                            im += ar * bi + ai * br;
                        }
                        r[2 * (2 * rr + cc)] = re;
                        r[2 * (2 * rr + cc) + 1] = im;
                    }
                for (int t = 0; t < 8; ++t) e.m[t] = r[t];
                fused = true;
                break;
            }
            between.add(e);
            if (!between.commutes(g)) break;
        }
        if (!fused) pend.push_back(pd);
    }
    // A merged phase run pays ~40 complex multiplies per thread for its
    // factor tables: runs of fewer than kMinLinRun gates go back to one op
    // per gate (all diagonal: they commute, so their order is free).
    constexpr size_t kMinLinRun = 4;
    {
        std::vector<Pend> expanded;
        for (Pend &pd : pend) {
            if (pd.lin.empty() || pd.lin.size() >= kMinLinRun) {
                expanded.push_back(std::move(pd));
                continue;
            }
            for (const LinEntry &le : pd.lin) expanded.push_back(Pend{le.src, pd.bt, le.tc, le.fm, {}});
        }
        pend.swap(expanded);
    }
    // Layout schedule: in the current layout run every ready op (commutes
    // with all earlier pending ops) whose target is a register bit; when none
    // is left, move to the layout that runs the most ready ops next.
    auto ready_in = [&](int ph, std::vector<size_t> *take) {
        CommuteSet skipped;
        int cnt = 0;
        for (size_t i = 0; i < pend.size(); ++i) {
            // a merged phase run or a diagonal gate needs no register target: it runs in any layout
            if (skipped.commutes(pend[i].g) &&
                (!pend[i].lin.empty() || gate_diag(pend[i].g) || L::is_reg(ph, pend[i].bt))) {
                ++cnt;
                if (take) take->push_back(i);
            } else {
                skipped.add(pend[i].g);
            }
        }
        return cnt;
    };
    int cur = 0;
    std::vector<size_t> take;
    while (!pend.empty()) {
        take.clear();
        ready_in(cur, &take);
        if (take.empty()) {
            int best = -1, bc = -1;
            for (int ph = 0; ph < 3; ++ph) {
                if (ph == cur) continue;
                const int c = ready_in(ph, nullptr);
                if (c > bc) { bc = c; best = ph; }
            }
            SV_CHECK(bc > 0, SV_EINVAL, "internal: gate layout schedule stuck");
            cur = best;
            continue;
        }
        std::vector<char> used(pend.size(), 0);
        for (size_t i : take) {
            const Pend &pd = pend[i];
            if (!pd.lin.empty()) {
                GOp<R> o{};
                o.ph = (GK_LINPHASE << 8) | (unsigned int)cur;
                o.ri = LP_THR;
                o.jm = (unsigned int)pd.bt;
                for (int r = 0; r < L::kRB; ++r)
                    if (L::reg_bit(cur, r) == pd.bt) { o.ri = LP_REG; o.jm = (unsigned int)r; }
                // host fp64 products: per register bit of this layout, per
                // thread tile bit, per free slot, and the constant factor
                std::complex<double> preg[16], pthr[16], pconst(1.0, 0.0);
                std::vector<std::pair<int, std::complex<double>>> pfree;
                for (int r = 0; r < 16; ++r) { preg[r] = 1.0; pthr[r] = 1.0; }
                for (const LinEntry &le : pd.lin) {
                    const std::complex<double> z(le.zr, le.zi);
                    if (le.where == 2) { pconst *= z; continue; }
                    if (le.where == 1) {
                        bool found = false;
                        for (auto &f : pfree)
                            if (f.first == le.bit) { f.second *= z; found = true; }
                        if (!found) pfree.push_back({le.bit, z});
                        continue;
                    }
                    int reg = -1;
                    for (int r = 0; r < L::kRB; ++r)
                        if (L::reg_bit(cur, r) == le.bit) reg = r;
                    if (reg >= 0) preg[reg] *= z;
                    else pthr[le.bit] *= z;
                }
                std::vector<GOp<R>> ent;
                auto rec = [&](unsigned int w, unsigned int bit, std::complex<double> z) {
                    GOp<R> e{};
                    e.m[0] = (R)z.real();
                    e.m[1] = (R)z.imag();
                    e.ri = w;
                    e.jm = bit;
                    ent.push_back(e);
                };
                for (int r = 0; r < L::kRB; ++r) rec(LP_REG, (unsigned int)r, preg[r]);
                for (int t = 0; t < L::kTB; ++t)
                    if (pthr[t] != std::complex<double>(1.0, 0.0)) rec(LP_THR, (unsigned int)t, pthr[t]);
                o.fm = ent.size() - (size_t)L::kRB;  // thread-bit entries come first
                if (pconst != std::complex<double>(1.0, 0.0)) rec(LP_CONST, 0u, pconst);
                for (auto &f : pfree) rec(LP_FREE, (unsigned int)f.first, f.second);
                o.tm = (unsigned int)ent.size();
                out.push_back(o);
                out.insert(out.end(), ent.begin(), ent.end());
                used[i] = 1;
                continue;
            }
            GOp<R> o = op_coefs<R>(pd.g);
            o.ph |= (unsigned int)cur;
            o.ri = 0;
            bool treg = false;
            for (int r = 0; r < L::kRB; ++r)
                if (L::reg_bit(cur, r) == pd.bt) { o.ri = (unsigned int)r; treg = true; }
            if (!treg) {  // only diagonal gates are scheduled off a register target
                SV_CHECK(gate_diag(pd.g), SV_EINVAL, "internal: non-diagonal gate without a register target");
                o.ph = (GK_DIAGT << 8) | (unsigned int)cur;
                o.ri = (unsigned int)pd.bt;
            }
            o.jm = 0;
            o.tm = 0;
            for (int tbit = 0; tbit < L::kTB; ++tbit) {
                if (!((pd.tc >> tbit) & 1u)) continue;
                bool reg = false;
                for (int r = 0; r < L::kRB; ++r)
                    if (L::reg_bit(cur, r) == tbit) { o.jm |= 1u << r; reg = true; }
                if (!reg) o.tm |= 1u << tbit;
            }
            o.fm = pd.fm;
            out.push_back(o);
            used[i] = 1;
        }
        std::vector<Pend> rest;
        for (size_t i = 0; i < pend.size(); ++i)
            if (!used[i]) rest.push_back(pend[i]);
        pend.swap(rest);
    }
}

template <typename R>
size_t append_ops(const std::vector<GOp<R>> &ops, std::vector<unsigned char> &prog) {
    const size_t off = prog.size();
    prog.resize(off + ops.size() * sizeof(GOp<R>));
    if (!ops.empty()) memcpy(prog.data() + off, ops.data(), ops.size() * sizeof(GOp<R>));
    return ops.size();
}

// SV_GATE_PARAM_OPS=0: always read the op program from global memory (A/B).
inline bool gate_param_ops() {
    static const int mode = [] {
        const char *e = getenv("SV_GATE_PARAM_OPS");
        return e ? atoi(e) : 1;
    }();
    return mode != 0;
}

template <typename E, int TB, int RB>
void launch_tile_gates(const GatePassArgs &a, const void *dev_ops, const void *host_ops, uint64_t nops, bool lin,
                       cudaStream_t s) {
    using L = Layout<E, TB, RB>;
    using R = typename RealOf<E>::T;
    KParams kp{};
    kp.in = a.in;
    kp.out = a.out;
    kp.xchg = a.xchg_nl > 0 ? 1 : 0;
    if (kp.xchg) {
        SV_CHECK(a.xchg_g >= 1 && a.xchg_g <= 3 && a.xchg_nl - a.xchg_g >= 1, SV_EINVAL,
                 "internal: fused exchange supports 2..8 ranks");
        kp.xnl = a.xchg_nl;
        kp.xg = a.xchg_g;
        kp.xrank = a.xchg_rank;
        for (int i = 0; i < 8; ++i) kp.xdst[i] = i < (1 << a.xchg_g) ? a.xchg_dst[i] : nullptr;
    }
    int b = 0, f = 0;
    kp.free_mask = 0;
    for (int sl = 0; sl < a.total_bits; ++sl) {
        if ((a.tile_mask >> sl) & 1) {
            SV_CHECK(b < 16, SV_EINVAL, "internal: tile too large");
            kp.slot[b++] = (signed char)sl;
        } else {
            kp.free_mask |= 1ull << sl;
            ++f;
        }
    }
    SV_CHECK(b == TB, SV_EINVAL, "internal: gate tile mask does not have T slots");
    kp_set_free_runs(kp);
    SV_CHECK(nops <= 0x7fffffffull, SV_EINVAL, "too many gates in one pass");
    const unsigned long long ntiles = 1ull << f;
    SV_CHECK(ntiles <= 0x7fffffffull, SV_EINVAL, "too many tiles for one launch");
    const int smem = (1 << TB) * (int)sizeof(E);
    static bool attr = false;
    if (!attr) {
        for (auto f : {gate_tile_kernel<E, TB, RB, true, true>, gate_tile_kernel<E, TB, RB, false, true>,
                       gate_tile_kernel<E, TB, RB, true, false>, gate_tile_kernel<E, TB, RB, false, false>})
            SV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (auto f : {gate_tile_kernel_p<E, TB, RB, true, true>, gate_tile_kernel_p<E, TB, RB, false, true>,
                       gate_tile_kernel_p<E, TB, RB, true, false>, gate_tile_kernel_p<E, TB, RB, false, false>})
            SV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    constexpr uint64_t cap = sizeof(GProg<R>) / sizeof(GOp<R>);
    if (host_ops != nullptr && nops <= cap && gate_param_ops()) {
        auto prog = std::make_unique<GProg<R>>();
        memcpy(prog->op, host_ops, nops * sizeof(GOp<R>));
        auto fn = lin ? (kp.xchg ? gate_tile_kernel_p<E, TB, RB, true, true> : gate_tile_kernel_p<E, TB, RB, false, true>)
                      : (kp.xchg ? gate_tile_kernel_p<E, TB, RB, true, false> : gate_tile_kernel_p<E, TB, RB, false, false>);
        fn<<<(unsigned int)ntiles, L::NT, smem, s>>>(kp, *prog, (int)nops);
    } else {
        auto fn = lin ? (kp.xchg ? gate_tile_kernel<E, TB, RB, true, true> : gate_tile_kernel<E, TB, RB, false, true>)
                      : (kp.xchg ? gate_tile_kernel<E, TB, RB, true, false> : gate_tile_kernel<E, TB, RB, false, false>);
        fn<<<(unsigned int)ntiles, L::NT, smem, s>>>(kp, reinterpret_cast<const GOp<R> *>(dev_ops), (int)nops);
    }
    SV_CUDA(cudaGetLastError());
}

template <typename E>
void whole_ops(const GatePassArgs &a, std::vector<GOp<typename RealOf<E>::T>> &ops) {
    using R = typename RealOf<E>::T;
    for (uint64_t k = 0; k < a.count; ++k) {
        const sv_gate &g = a.gates[a.order[k]];
        GOp<R> o = op_coefs<R>(g);
        o.ri = (unsigned int)g.target;
        o.fm = g.controls;
        ops.push_back(o);
    }
}

template <typename E>
void launch_whole_gates(const GatePassArgs &a, const void *dev_ops, uint64_t nops, cudaStream_t s) {
    using R = typename RealOf<E>::T;
    if (nops == 0) return;
    SV_CHECK(nops <= 0x7fffffffull, SV_EINVAL, "too many gates");
    const unsigned int N = 1u << a.n;
    const int threads = N >= 1024 ? 512 : (N / 2 >= 32 ? (int)(N / 2) : 32);
    const int smem = (int)(N * sizeof(E));
    SV_CUDA(cudaFuncSetAttribute(gate_whole_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    gate_whole_kernel<E><<<1, threads, smem, s>>>(reinterpret_cast<E *>(a.in), a.n,
                                                   reinterpret_cast<const GOp<R> *>(dev_ops), (int)nops);
    SV_CUDA(cudaGetLastError());
}

}  // namespace

uint64_t build_gate_ops(sv_dtype dt, const GatePassArgs &a, bool whole, std::vector<unsigned char> &prog,
                        bool *has_lin) {
    // every op record is 16-byte aligned inside the program
    prog.resize((prog.size() + 15) & ~(size_t)15);
    auto lin_in = [](const auto &ops) {
        for (const auto &o : ops)
            if ((o.ph >> 8) == GK_LINPHASE) return true;
        return false;
    };
    if (dt == SV_C64) {
        std::vector<GOp<float>> ops;
        if (whole) whole_ops<float2>(a, ops);
        else build_tile_ops<Layout<float2, kGateTileBitsC64, kRegBitsC64>, float>(a, ops);
        if (has_lin) *has_lin = lin_in(ops);
        return append_ops(ops, prog);
    }
    std::vector<GOp<double>> ops;
    if (whole) whole_ops<double2>(a, ops);
    else build_tile_ops<Layout<double2, kTileBitsC128, kRegBitsC128>, double>(a, ops);
    if (has_lin) *has_lin = lin_in(ops);
    return append_ops(ops, prog);
}

template <typename R>
static uint64_t relayouts_of(const std::vector<GOp<R>> &ops) {
    uint64_t r = 0;
    unsigned int cur = 0;
    for (size_t k = 0; k < ops.size(); ++k) {  // as the kernel's op loop walks the program
        const unsigned int ph = ops[k].ph & 0xffu, kind = ops[k].ph >> 8;
        if (ph != cur) {
            ++r;
            cur = ph;
        }
        if (kind == GK_LINPHASE) k += ops[k].tm;  // its entry records
    }
    return r;
}

uint64_t count_gate_relayouts(sv_dtype dt, const GatePassArgs &a) {
    if (dt == SV_C64) {
        std::vector<GOp<float>> ops;
        build_tile_ops<Layout<float2, kGateTileBitsC64, kRegBitsC64>, float>(a, ops);
        return relayouts_of(ops);
    }
    std::vector<GOp<double>> ops;
    build_tile_ops<Layout<double2, kTileBitsC128, kRegBitsC128>, double>(a, ops);
    return relayouts_of(ops);
}

void launch_gate_pass(sv_dtype dt, const GatePassArgs &a, const void *dev_ops, const void *host_ops, uint64_t nops,
                      bool has_lin, cudaStream_t s) {
    if (dt == SV_C64) launch_tile_gates<float2, kGateTileBitsC64, kRegBitsC64>(a, dev_ops, host_ops, nops, has_lin, s);
    else launch_tile_gates<double2, kTileBitsC128, kRegBitsC128>(a, dev_ops, host_ops, nops, has_lin, s);
}

void launch_gate_whole(sv_dtype dt, const GatePassArgs &a, const void *dev_ops, uint64_t nops, cudaStream_t s) {
    if (dt == SV_C64) launch_whole_gates<float2>(a, dev_ops, nops, s);
    else launch_whole_gates<double2>(a, dev_ops, nops, s);
}

}  // namespace sv
