// wht_kernels.cuh -- fused multi-stage Walsh-Hadamard tile pass (sm_100a):
// layouts, device helpers, kernels and launch templates.  Instantiated by
// wht.cu (ideal stages) and wht_noisy.cu (angle-error stages, NEXT-1).
//
// What it computes: for one group of qubits (slots), every butterfly stage
//   (x, y) -> (x + y, x - y)  on index pairs that differ only in that bit,
// i.e. Fig. 3's 2x2 transformation with w = x = y = 1, z = -1,
// applied as "a sequence of V/2 independent 2x2 transformations" per qubit
// (section 2.1).  Optionally an elementwise op between two
// stage sets of the same group: the phase oracle O (negate marked entries,
// G3) or F0 = 2|0><0| - I with the exact 2^{-n} scale (G2, G5).
//
// How (B200 design):
//  * A tile is 2^T amplitudes whose local indices differ only in T slots
//    (the group's processed slots + the lowest unprocessed slots, so every
//    tile row is a >= 64 B contiguous run).  One CTA = one tile; 256 threads
//    hold 2^R amplitudes each in registers.
//  * The T tile bits are covered by three register layouts A, B, C; each runs
//    its R butterfly stages in registers.  Layout changes go through one
//    swizzled shared-memory tile (one __syncthreads each: every thread writes
//    exactly the slots it read in the previous layout).
//  * Layout A owns tile bit 0 and the top tile bits, so HBM is touched with
//    coalesced 128-bit loads (512 contiguous bytes per warp instruction on a
//    contiguous tile).  No tensor cores: the path is add/sub only (<= 1.75
//    FLOP/B), memory-bound.
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>

#include "sv_internal.h"
#else
#include "sv_consts.h"  // runtime-compiled kernels (gate_jit.cpp): device code only
#endif

#ifndef SV_2LAYOUT_MAX_U
#define SV_2LAYOUT_MAX_U 4  // strided c64 tiles with U in [3, this] use the two-layout family
#endif

#ifndef SV_TILE_MIN_BLOCKS
#define SV_TILE_MIN_BLOCKS 2
#endif

namespace sv {

template <typename E> struct RealOf;
template <> struct RealOf<float2> { using T = float; };
template <> struct RealOf<double2> { using T = double; };

// ------------------------------------------------------------------------- //
// Register / shared-memory layouts of a 2^TB tile with 2^RB amps per thread  //
// ------------------------------------------------------------------------- //
template <typename E, int TB, int RB>
struct Layout {
    static constexpr int VE = (sizeof(E) == 8) ? 2 : 1;   // amplitudes per 16 B
    static constexpr int NT = 1 << (TB - RB);             // threads
    static constexpr int NR = 1 << RB;                    // amplitudes per thread
    static constexpr int kTB = TB, kRB = RB;
    static constexpr int kNPH = 3;                        // register layouts A, B, C
    // complex64: tile bit 0 is a register bit in EVERY layout, so each thread
    // always holds adjacent pairs (e, e|1) = 16 bytes -> every shared and
    // global access is 128-bit; the other RB-1 register bits cover 3(RB-1)
    // tile bits.  complex128: one amplitude is already 16 bytes.
    static_assert(VE == 2 ? (TB >= 2 * RB - 1 && TB <= 3 * RB - 2) : (TB >= 2 * RB && TB <= 3 * RB),
                  "three layouts must cover the tile");
    static_assert(TB - RB >= 5, "need at least one warp");

    // i-th register bit (ascending) of layout ph (0 = A, 1 = B, 2 = C).
    __host__ __device__ static constexpr int reg_bit(int ph, int i) {
        return VE == 2 ? (i == 0 ? 0 : ph == 0 ? TB - RB + i : ph == 1 ? i : TB - 2 * RB + 1 + i)
                       : (ph == 0 ? TB - RB + i : ph == 1 ? i : TB - 2 * RB + i);
    }
    __host__ __device__ static constexpr bool is_reg(int ph, int b) {
        bool r = false;
        for (int i = 0; i < RB; ++i) r = r || (reg_bit(ph, i) == b);
        return r;
    }
    // i-th thread bit (ascending) of layout ph: the tile bits that are not
    // register bits.  Lane = thread bits 0..4.
    __host__ __device__ static constexpr int thr_bit(int ph, int i) {
        int c = 0;
        for (int b = 0; b < TB; ++b)
            if (!is_reg(ph, b)) {
                if (c == i) return b;
                ++c;
            }
        return -1;
    }
    // Each tile bit's stage runs in exactly one layout: A and B are disjoint;
    // C runs only the bits B does not have.
    __host__ __device__ static constexpr bool owns(int ph, int b) {
        return ph == 0 ? is_reg(0, b) : ph == 1 ? (is_reg(1, b) && !is_reg(0, b)) : (is_reg(2, b) && !is_reg(1, b) && !is_reg(0, b));
    }
    // XOR swizzle of the shared-memory index (linear over GF(2)): makes the
    // 8-lane (16 B) / 16-lane (8 B) wavefronts of every layout bank-conflict
    // free -- checked exhaustively by tests/test_layouts.py via sv_debug.
    __host__ __device__ static constexpr uint32_t swz(uint32_t e) {
        return VE == 2 ? (e ^ (((e >> RB) & 7u) << 1)) : (e ^ ((e >> RB) & 7u));
    }
    __host__ __device__ static constexpr uint32_t ereg(int ph, int j) {
        uint32_t e = 0;
        for (int i = 0; i < RB; ++i)
            if ((j >> i) & 1) e |= 1u << reg_bit(ph, i);
        return e;
    }
    __host__ __device__ static constexpr uint32_t ethr(int ph, uint32_t t) {
        uint32_t e = 0;
        for (int i = 0; i < TB - RB; ++i)
            if ((t >> i) & 1) e |= 1u << thr_bit(ph, i);
        return e;
    }
};

// Two-layout family for STRIDED complex64 tiles (processed tile bits [U, TB)
// with U >= 3, i.e. at most 10 processed bits): A holds the top RB tile bits,
// B the RB bits below them; the carry bits 0..2 are never register bits, so
// every access moves one 8-byte amplitude.  A fused strided pass then needs 2
// shared-memory relayouts instead of 4 (an unfused one 1 instead of 2); when
// U >= TB - RB every processed bit is in A and no relayout is needed at all.
template <int TB, int RB>
struct Layout2 {
    static constexpr int VE = 1;               // element-granular (8 B) accesses
    static constexpr int NT = 1 << (TB - RB);
    static constexpr int NR = 1 << RB;
    static constexpr int kTB = TB, kRB = RB;
    static constexpr int kNPH = 2;             // register layouts A, B
    static_assert(TB - 2 * RB >= 3, "carry bits 0..2 must stay outside both layouts");
    __host__ __device__ static constexpr int reg_bit(int ph, int i) {
        return ph == 0 ? TB - RB + i : TB - 2 * RB + i;
    }
    __host__ __device__ static constexpr bool is_reg(int ph, int b) {
        return ph == 0 ? (b >= TB - RB && b < TB) : (b >= TB - 2 * RB && b < TB - RB);
    }
    __host__ __device__ static constexpr int thr_bit(int ph, int i) {
        int c = 0;
        for (int b = 0; b < TB; ++b)
            if (!is_reg(ph, b)) {
                if (c == i) return b;
                ++c;
            }
        return -1;
    }
    __host__ __device__ static constexpr bool owns(int ph, int b) { return ph <= 1 && is_reg(ph, b); }
    // B's half-warp lanes are tile bits {0,1,2,TB-RB}: fold bit TB-RB into bit 3
    __host__ __device__ static constexpr uint32_t swz(uint32_t e) { return e ^ (((e >> (TB - RB)) & 1u) << 3); }
    __host__ __device__ static constexpr uint32_t ereg(int ph, int j) {
        uint32_t e = 0;
        for (int i = 0; i < RB; ++i)
            if ((j >> i) & 1) e |= 1u << reg_bit(ph, i);
        return e;
    }
    __host__ __device__ static constexpr uint32_t ethr(int ph, uint32_t t) {
        uint32_t e = 0;
        for (int i = 0; i < TB - RB; ++i)
            if ((t >> i) & 1) e |= 1u << thr_bit(ph, i);
        return e;
    }
};

struct KParams {
    const void *in;
    void *out;
    const unsigned long long *marked;
    unsigned long long n_marked;
    const unsigned int *tilemap;   // bit t: contiguous tile t holds a marked index
    double f0_scale;
    int mid;
    int has_origin;
    unsigned int proc;       // processed tile bits
    unsigned long long free_mask;  // slots not in the tile; tile id bits scatter into them
    // the free slots as runs of consecutive slots (host-built, kp_set_free_runs):
    // tile id bits [off, off + len) land at slots [start, start + len); nruns = 0:
    // more than kMaxRuns runs -> bit-by-bit scatter
    int nruns;
    unsigned char run_start[8], run_len[8];
    signed char slot[16];          // tile bit -> slot
    // fused qubit-swap exchange (global_store_xchg): 0 = plain store
    int xchg, xnl, xg, xrank;      // local index bits, rank bits, own rank (-1: emulated)
    void *xdst[8];                 // destination buffer of each rank
    const double *scale_in;        // != nullptr: multiply the loaded tile by *scale_in (renormalisation)
    double *sumsq;                 // != nullptr: write the tile's fp64 sum |a|^2 (after the pass) to sumsq[tile]
};

// The general-2x2 flavour (NEXT-1/2) carries its per-pass coefficients as
// kernel parameters: per half (0 = before the op, 1 = after) and tile bit,
// [w x; y z] row-major.  The ideal flavour's parameter block stays small
// (measured on B200: the 1 KiB coefficient block in every launch's
// parameters cost the contiguous c4 pass ~10%).
// NOISY: 0 = ideal butterflies; 1 = general real 2x2 per stage (angle
// errors with decoherence contractions, G19/G22); 2 = angle errors only:
// U(phi) = c [[1, t], [t, -1]] with t = tan(phi), the per-stage factors c
// multiplied once into the loaded tile (pass_scale) -- 2 packed FMAs per
// butterfly instead of 4.
template <int NOISY>
struct KParamsT : KParams {
    double coef[2][16][4];
    double pass_scale;
    // the same, rounded to fp32 on the host (complex64 kernels: the device
    // conversions were ~90-150 F2F per thread per tile on the conversion pipe;
    // host rounding is the same round-to-nearest, so results are unchanged)
    float coeff[2][16][4];
    float pass_scalef;
};
template <>
struct KParamsT<0> : KParams {};

// Publish the exchange destinations in shared memory (constant indices only:
// a runtime-indexed kernel-parameter array would be copied to local memory).
template <typename E>
__device__ __forceinline__ void load_xdst(const KParams &p, int tid, E **s_dst) {
    if (p.xchg) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (tid == i) s_dst[i] = reinterpret_cast<E *>(p.xdst[i]);
    }
}

template <typename E>
__device__ __forceinline__ void bfly(E &x, E &y) {
    E t = x;
    x.x = t.x + y.x;
    x.y = t.y + y.y;
    y.x = t.x - y.x;
    y.y = t.y - y.y;
}

// complex64: one packed FADD2 for the sum and one for the difference
// (sm_100a add/sub.rn.f32x2; per-lane IEEE fp32, identical to two FADDs).
template <>
__device__ __forceinline__ void bfly<float2>(float2 &x, float2 &y) {
    unsigned long long a = *reinterpret_cast<unsigned long long *>(&x);
    unsigned long long b = *reinterpret_cast<unsigned long long *>(&y);
    unsigned long long s, d;
    asm("add.rn.f32x2 %0, %2, %3;\n\tsub.rn.f32x2 %1, %2, %3;" : "=l"(s), "=l"(d) : "l"(a), "l"(b));
    x = *reinterpret_cast<float2 *>(&s);
    y = *reinterpret_cast<float2 *>(&d);
}

// General real 2x2 stage (Fig. 3's [w x; y z]):
// (u, v) -> (w u + x v, y u + z v).  Angle errors (G19) use
// [[cos, sin], [sin, -cos]]; with decoherence (G22) the per-qubit matrix also
// carries the contractions of the laser operations around it.
template <typename E>
__device__ __forceinline__ void bfly_gen(E &x, E &y, const double *m) {
    using R = decltype(E{}.x);
    const R w = (R)m[0], xx = (R)m[1], yy = (R)m[2], z = (R)m[3];
    E t = x;
    x.x = w * t.x + xx * y.x;
    x.y = w * t.y + xx * y.y;
    y.x = yy * t.x + z * y.x;
    y.y = yy * t.y + z * y.y;
}

template <>
__device__ __forceinline__ void bfly_gen<float2>(float2 &x, float2 &y, const double *m) {
    const float w = (float)m[0], xx = (float)m[1], yy = (float)m[2], z = (float)m[3];
    const float2 W = make_float2(w, w), X = make_float2(xx, xx), Y = make_float2(yy, yy), Z = make_float2(z, z);
    const unsigned long long a = *reinterpret_cast<unsigned long long *>(&x);
    const unsigned long long b = *reinterpret_cast<unsigned long long *>(&y);
    const unsigned long long w2 = *reinterpret_cast<const unsigned long long *>(&W);
    const unsigned long long x2 = *reinterpret_cast<const unsigned long long *>(&X);
    const unsigned long long y2 = *reinterpret_cast<const unsigned long long *>(&Y);
    const unsigned long long z2 = *reinterpret_cast<const unsigned long long *>(&Z);
    unsigned long long t, u;
    asm("mul.rn.f32x2 %0, %2, %4;\n\t"
        "fma.rn.f32x2 %0, %3, %5, %0;\n\t"
        "mul.rn.f32x2 %1, %2, %6;\n\t"
        "fma.rn.f32x2 %1, %3, %7, %1;"
        : "=&l"(t), "=&l"(u) : "l"(a), "l"(b), "l"(w2), "l"(x2), "l"(y2), "l"(z2));
    x = *reinterpret_cast<float2 *>(&t);
    y = *reinterpret_cast<float2 *>(&u);
}

// complex64 with fp32 coefficients (KParamsT::coeff)
__device__ __forceinline__ void bfly_gen(float2 &x, float2 &y, const float *m) {
    const float2 W = make_float2(m[0], m[0]), X = make_float2(m[1], m[1]), Y = make_float2(m[2], m[2]),
                 Z = make_float2(m[3], m[3]);
    const unsigned long long a = *reinterpret_cast<unsigned long long *>(&x);
    const unsigned long long b = *reinterpret_cast<unsigned long long *>(&y);
    const unsigned long long w2 = *reinterpret_cast<const unsigned long long *>(&W);
    const unsigned long long x2 = *reinterpret_cast<const unsigned long long *>(&X);
    const unsigned long long y2 = *reinterpret_cast<const unsigned long long *>(&Y);
    const unsigned long long z2 = *reinterpret_cast<const unsigned long long *>(&Z);
    unsigned long long t, u;
    asm("mul.rn.f32x2 %0, %2, %4;\n\t"
        "fma.rn.f32x2 %0, %3, %5, %0;\n\t"
        "mul.rn.f32x2 %1, %2, %6;\n\t"
        "fma.rn.f32x2 %1, %3, %7, %1;"
        : "=&l"(t), "=&l"(u) : "l"(a), "l"(b), "l"(w2), "l"(x2), "l"(y2), "l"(z2));
    x = *reinterpret_cast<float2 *>(&t);
    y = *reinterpret_cast<float2 *>(&u);
}

// Angle-error butterfly without its factor c: (u, v) -> (u + t v, t u - v).
template <typename E>
__device__ __forceinline__ void bfly_tan(E &x, E &y, double td) {
    using R = decltype(E{}.x);
    const R t = (R)td;
    const E a = x;
    x.x = a.x + t * y.x;
    x.y = a.y + t * y.y;
    y.x = t * a.x - y.x;
    y.y = t * a.y - y.y;
}

__device__ __forceinline__ void bfly_tan(float2 &x, float2 &y, float t) {
    const float2 T = make_float2(t, t), a = x, b = y;
    x = __ffma2_rn(T, b, a);                          // u = t b + a
    y = __ffma2_rn(T, a, make_float2(-b.x, -b.y));    // v = t a - b
}

template <>
__device__ __forceinline__ void bfly_tan<float2>(float2 &x, float2 &y, double td) {
    const float t = (float)td;
    const float2 T = make_float2(t, t), a = x, b = y;
    // intrinsics (not inline asm) so ptxas folds the negation of b into the
    // FFMA2 operand instead of a LOP3 per butterfly
    x = __ffma2_rn(T, b, a);                          // u = t b + a
    y = __ffma2_rn(T, a, make_float2(-b.x, -b.y));    // v = t a - b
}

template <typename E, typename R>
__device__ __forceinline__ void scale(E &x, R s) {
    x.x *= s;
    x.y *= s;
}

template <>
__device__ __forceinline__ void scale<float2, float>(float2 &x, float s) {
    unsigned long long a = *reinterpret_cast<unsigned long long *>(&x), r;
    float2 ss = make_float2(s, s);
    unsigned long long b = *reinterpret_cast<unsigned long long *>(&ss);
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    x = *reinterpret_cast<float2 *>(&r);
}

// Stages of layout PH.  The processed tile bits are always [U, TB): the
// unprocessed slots of a tile are its lowest ones (plan.cpp make_group), so
// U is a template parameter and the unrolled stage code has no branches.
template <class L, int PH, int U, int NOISY, int HALF, typename E>
__device__ __forceinline__ void run_stages(E (&x)[L::NR], const KParamsT<NOISY> &p) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        if (i < L::kRB) {
            const int b = L::reg_bit(PH, i);
            if (L::owns(PH, b) && b >= U) {
#pragma unroll
                for (int j = 0; j < L::NR; ++j)
                    if (!(j & (1 << i))) {
                        constexpr bool F32 = sizeof(E) == 8;  // complex64: the host-rounded fp32 coefficients
                        if constexpr (NOISY == 2 && F32)
                            bfly_tan(x[j], x[j | (1 << i)], p.coeff[HALF][b][0]);
                        else if constexpr (NOISY == 2)
                            bfly_tan(x[j], x[j | (1 << i)], p.coef[HALF][b][0]);
                        else if constexpr (NOISY == 1 && F32)
                            bfly_gen(x[j], x[j | (1 << i)], p.coeff[HALF][b]);
                        else if constexpr (NOISY == 1)
                            bfly_gen(x[j], x[j | (1 << i)], p.coef[HALF][b]);
                        else
                            bfly(x[j], x[j | (1 << i)]);
                    }
            }
        }
    }
}

// Read this thread's amplitudes of layout PR from the swizzled smem tile
// (sr = swizzled thread part of the index).
template <class L, int PR, typename E>
__device__ __forceinline__ void smem_read(E (&x)[L::NR], const E *sm, uint32_t sr) {
    if constexpr (L::VE == 2) {
#pragma unroll
        for (int v = 0; v < L::NR / 2; ++v) {
            float4 q = *reinterpret_cast<const float4 *>(&sm[sr ^ L::swz(L::ereg(PR, 2 * v))]);
            x[2 * v].x = q.x; x[2 * v].y = q.y; x[2 * v + 1].x = q.z; x[2 * v + 1].y = q.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < L::NR; ++j) x[j] = sm[sr ^ L::swz(L::ereg(PR, j))];
    }
}

// Shared-memory layout change PW -> PR.  One barrier: each thread writes the
// positions it read in the previous change (or, for the first write, nobody
// has read yet), so no write can race a pending read.
template <class L, int PW, int PR, typename E>
__device__ __forceinline__ void relayout(E (&x)[L::NR], E *sm, int tid) {
    const uint32_t sw = L::swz(L::ethr(PW, tid));
    const uint32_t sr = L::swz(L::ethr(PR, tid));
    if constexpr (L::VE == 2) {
#pragma unroll
        for (int v = 0; v < L::NR / 2; ++v) {
            float4 q;
            q.x = x[2 * v].x; q.y = x[2 * v].y; q.z = x[2 * v + 1].x; q.w = x[2 * v + 1].y;
            *reinterpret_cast<float4 *>(&sm[sw ^ L::swz(L::ereg(PW, 2 * v))]) = q;
        }
    } else {
#pragma unroll
        for (int j = 0; j < L::NR; ++j) sm[sw ^ L::swz(L::ereg(PW, j))] = x[j];
    }
    __syncthreads();
    smem_read<L, PR>(x, sm, sr);
}

// Streaming 128-bit global load.  Every amplitude is read exactly once per
// pass, so L1 allocation only costs: SV_LD_MODE 0 = default (ld.global),
// 1 = ld.global.cg (L2 only), 2 = ld.global.nc.L1::no_allocate.
#ifndef SV_LD_MODE
#define SV_LD_MODE 1
#endif
#ifndef SV_L2_PF_V4
#define SV_L2_PF_V4 0  // A/B: 256 = the L2::256B prefetch-size hint on the 128-bit loads as well
#endif
__device__ __forceinline__ float4 ld_stream(const float4 *p) {
#if SV_LD_MODE == 1 && SV_L2_PF_V4 == 256
    float4 r;
    asm volatile("ld.global.cg.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
#elif SV_LD_MODE == 1
    return __ldcg(p);
#elif SV_LD_MODE == 2
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
#else
    return *p;
#endif
}

// Element-granular load (strided two-layout tiles, complex128 tiles).
// SV_L2_PF (complex64): 0 = plain ld.global.cg; 128 / 256 = with the
// L2::128B / L2::256B prefetch-size hint, so an L2 miss on a 64-B (128-B)
// row also brings in the adjacent row -- the next tile id's, which a
// co-resident CTA reads next (tile id bit 0 sits at the lowest free slot).
#ifndef SV_L2_PF
#define SV_L2_PF 256  // measured on B200 (c4): strided passes -0.6 %, 128B no change
#endif
template <typename E>
__device__ __forceinline__ E ld_elem(const E *p) { return __ldcg(p); }
template <>
__device__ __forceinline__ float2 ld_elem<float2>(const float2 *p) {
#if SV_L2_PF == 128
    float2 r;
    asm volatile("ld.global.cg.L2::128B.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
#elif SV_L2_PF == 256
    float2 r;
    asm volatile("ld.global.cg.L2::256B.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
#else
    return __ldcg(p);
#endif
}

// Global offset (elements) of tile element e under the pass's slot map.
// CONTIG: the tile is slots [0, T) (the contiguous group): offsets are
// compile-time functions of the thread and register bits, no slot map.
template <class L, int PH, bool CONTIG = false>
__device__ __forceinline__ unsigned long long goff_thr(const KParams &p, int tid) {
    if constexpr (CONTIG) return (unsigned long long)L::ethr(PH, (uint32_t)tid);
    // The slot loads are unconditional (uniform LDCU); a thread-dependent
    // branch around them made ptxas emit per-thread predicated LDCs through
    // the indexed constant cache at every CTA start (measured on B200: +11%
    // on the contiguous c4 pass, whose CTAs are short-lived).
    unsigned long long o = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (i < (L::kTB - L::kRB)) {
            const unsigned long long stride = 1ull << p.slot[L::thr_bit(PH, i)];
            o += (unsigned long long)((tid >> i) & 1) * stride;
        }
    return o;
}

template <class L, int PH, bool CONTIG = false, typename E>
__device__ __forceinline__ void global_load(E (&x)[L::NR], const E *g, const KParams &p, int tid) {
    const unsigned long long t = goff_thr<L, PH, CONTIG>(p, tid);
    unsigned long long st[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (i < L::kRB) st[i] = CONTIG ? (1ull << L::reg_bit(PH, i)) : (1ull << p.slot[L::reg_bit(PH, i)]);
    if constexpr (L::VE == 2) {
#pragma unroll
        for (int v = 0; v < L::NR / 2; ++v) {
            unsigned long long o = t;
#pragma unroll
            for (int i = 1; i < 16; ++i)
                if (i < L::kRB && (((2 * v) >> i) & 1)) o += st[i];
            float4 q = ld_stream(reinterpret_cast<const float4 *>(g + o));
            x[2 * v].x = q.x; x[2 * v].y = q.y; x[2 * v + 1].x = q.z; x[2 * v + 1].y = q.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < L::NR; ++j) {
            unsigned long long o = t;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < L::kRB && ((j >> i) & 1)) o += st[i];
            x[j] = ld_elem(g + o);  // one element (8 B c64 / 16 B c128), L2 only
        }
    }
}

template <class L, int PH, bool CONTIG = false, typename E>
__device__ __forceinline__ void global_store(const E (&x)[L::NR], E *g, const KParams &p, int tid) {
    const unsigned long long t = goff_thr<L, PH, CONTIG>(p, tid);
    unsigned long long st[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (i < L::kRB) st[i] = CONTIG ? (1ull << L::reg_bit(PH, i)) : (1ull << p.slot[L::reg_bit(PH, i)]);
    if constexpr (L::VE == 2) {
#pragma unroll
        for (int v = 0; v < L::NR / 2; ++v) {
            unsigned long long o = t;
#pragma unroll
            for (int i = 1; i < 16; ++i)
                if (i < L::kRB && (((2 * v) >> i) & 1)) o += st[i];
            float4 q;
            q.x = x[2 * v].x; q.y = x[2 * v].y; q.z = x[2 * v + 1].x; q.w = x[2 * v + 1].y;
            *reinterpret_cast<float4 *>(g + o) = q;
        }
    } else {
#pragma unroll
        for (int j = 0; j < L::NR; ++j) {
            unsigned long long o = t;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < L::kRB && ((j >> i) & 1)) o += st[i];
            g[o] = x[j];
        }
    }
}

// Store that IS the qubit-swap exchange (the paper's reorganisation, Fig. 8,
// P:4631-4646, fused into the pass that precedes it): element with local
// index i of rank r belongs to rank j = i's top-g local bits and lands in
// rank j's destination buffer at r*B + (i mod B), B = N_l / P.  dst[j] is a
// peer pointer (NVLink, CUDA IPC) on a real multi-GPU run, or rank j's shard
// of the one buffer in single-GPU emulation (rank r = launched index >> nl).
template <class L, int PH, typename E>
__device__ __forceinline__ void global_store_xchg(const E (&x)[L::NR], unsigned long long base, const KParams &p,
                                                  int tid, E *const *sdst) {
    const unsigned long long t = base + goff_thr<L, PH>(p, tid);
    unsigned long long st[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (i < L::kRB) st[i] = 1ull << p.slot[L::reg_bit(PH, i)];
    const unsigned long long nlm = (1ull << p.xnl) - 1ull;
    const unsigned long long bm = (1ull << (p.xnl - p.xg)) - 1ull;
    const unsigned long long pm = (1ull << p.xg) - 1ull;
    auto dst = [&](unsigned long long idx) {
        const unsigned long long loc = idx & nlm;
        const unsigned long long r = p.xrank >= 0 ? (unsigned long long)p.xrank : (idx >> p.xnl);
        return sdst[(loc >> (p.xnl - p.xg)) & pm] + (r << (p.xnl - p.xg)) + (loc & bm);
    };
    if constexpr (L::VE == 2) {
#pragma unroll
        for (int v = 0; v < L::NR / 2; ++v) {
            unsigned long long o = t;
#pragma unroll
            for (int i = 1; i < 16; ++i)
                if (i < L::kRB && (((2 * v) >> i) & 1)) o += st[i];
            float4 q;
            q.x = x[2 * v].x; q.y = x[2 * v].y; q.z = x[2 * v + 1].x; q.w = x[2 * v + 1].y;
            *reinterpret_cast<float4 *>(dst(o)) = q;  // pair (e, e|1) never straddles ranks
        }
    } else {
#pragma unroll
        for (int j = 0; j < L::NR; ++j) {
            unsigned long long o = t;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < L::kRB && ((j >> i) & 1)) o += st[i];
            *dst(o) = x[j];
        }
    }
}

// Final store of a pass: plain (in place / to the next pass's buffer) or
// through the exchange.  XCHG is a template parameter so the plain passes
// carry no exchange code at all (measured on B200: a runtime branch here cost
// 10% on every c4 pass).
template <class L, int PH, bool XCHG, bool CONTIG = false, typename E>
__device__ __forceinline__ void pass_store(const E (&x)[L::NR], E *gout, unsigned long long base, const KParams &p,
                                           int tid, E *const *sdst) {
    if constexpr (XCHG) {
        __syncthreads();  // sdst published
        global_store_xchg<L, PH>(x, base, p, tid, sdst);
    } else {
        global_store<L, PH, CONTIG>(x, gout, p, tid);
    }
}

// Elementwise op between the two stage sets, in register layout PH.
template <class L, int PH, typename E>
__device__ __forceinline__ void mid_op(E (&x)[L::NR], const KParams &p, unsigned long long base, int tid,
                                       unsigned long long mlo, unsigned long long mcnt) {
    using R = typename RealOf<E>::T;
    if (p.mid == MID_F0) {
        // F0 = 2|0><0| - I with the 2^{-n} scale of the two unnormalised
        // transforms (G2, G5): -2^{-n} x everywhere, +2^{-n} x at index 0.
        const R s = (R)(-p.f0_scale);
#pragma unroll
        for (int j = 0; j < L::NR; ++j) scale(x[j], s);
        if (p.has_origin && base == 0 && tid == 0) { x[0].x = -x[0].x; x[0].y = -x[0].y; }
    } else if (p.mid == MID_ORACLE) {
        // O: negate marked amplitudes (G3).  Keys are (tile id << 16 | tile
        // element e), e = the marked index's tile-slot bits (host-built).
        for (unsigned long long r = 0; r < mcnt; ++r) {
            const uint32_t e = (uint32_t)(p.marked[mlo + r] & 0xFFFFull);
            uint32_t t = 0, jj = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < (L::kTB - L::kRB)) t |= ((e >> L::thr_bit(PH, i)) & 1u) << i;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < L::kRB) jj |= ((e >> L::reg_bit(PH, i)) & 1u) << i;
            if ((int)t == tid) {
#pragma unroll
                for (int j = 0; j < L::NR; ++j)
                    if ((uint32_t)j == jj) { x[j].x = -x[j].x; x[j].y = -x[j].y; }
            }
        }
    }
}

// Renormalisation folded into the load (decoherence, G22): x *= s.
template <typename E, int NR>
__device__ __forceinline__ void apply_scale(E (&x)[NR], double s) {
    using R = decltype(E{}.x);
#pragma unroll
    for (int j = 0; j < NR; ++j) scale(x[j], (R)s);
}

// x *= s with an fp32 factor (complex64, host-rounded pass_scalef)
template <int NR>
__device__ __forceinline__ void apply_scalef(float2 (&x)[NR], float s) {
#pragma unroll
    for (int j = 0; j < NR; ++j) scale(x[j], s);
}

// Decoherence (G22): the fp64 sum |a|^2 of the tile as stored, in a fixed
// order (per thread in register order, warp xor tree, warps in order), into
// out[tile] -- the global sum of Eq. 3 then needs no extra read
// pass of the state (reduced by launch_sum_partials).
template <typename E, int NR>
__device__ __forceinline__ void tile_sumsq(const E (&x)[NR], double *out, unsigned long long tile, int tid) {
    __shared__ double s_w[32];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NR; ++j) s += (double)x[j].x * (double)x[j].x + (double)x[j].y * (double)x[j].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((tid & 31) == 0) s_w[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_w[w];
        out[tile] = t;
    }
}

// Tile base: scatter the tile id into the free slots (software pdep).  The
// free slots of a pass are a few runs of consecutive slots, so the scatter is
// one shift-mask-shift per run (the former bit-by-bit loop was a ~100-
// instruction dependent chain in front of every CTA's first load).
__device__ __forceinline__ unsigned long long tile_base_bits(unsigned long long tile, unsigned long long fm) {
    unsigned long long base = 0;
    while (fm) {
        const unsigned long long low = fm & (~fm + 1ull);
        if (tile & 1ull) base |= low;
        tile >>= 1;
        fm ^= low;
    }
    return base;
}
__device__ __forceinline__ unsigned long long tile_base(unsigned long long tile, const KParams &p) {
    if (p.nruns == 0) return tile_base_bits(tile, p.free_mask);
    unsigned long long base = 0;
    int off = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        if (r < p.nruns) {
            const int len = p.run_len[r];
            base |= ((tile >> off) & ((1ull << len) - 1ull)) << p.run_start[r];
            off += len;
        }
    }
    return base;
}

#ifndef __CUDACC_RTC__
// Host: the runs of a free-slot mask (<= 8, else nruns = 0).
inline void kp_set_free_runs(KParams &kp) {
    kp.nruns = 0;
    unsigned long long fm = kp.free_mask;
    int n = 0;
    for (int sl = 0; sl < 64;) {
        if (!((fm >> sl) & 1ull)) { ++sl; continue; }
        int len = 0;
        while (sl + len < 64 && ((fm >> (sl + len)) & 1ull)) ++len;
        if (n == 8) { kp.nruns = 0; return; }
        kp.run_start[n] = (unsigned char)sl;
        kp.run_len[n] = (unsigned char)len;
        ++n;
        sl += len;
    }
    kp.nruns = n;
}
#endif

// Oracle tiles: one bitmap word says whether this tile holds a marked index
// (rare); only then does thread 0 binary-search the sorted keys (tile id << 16
// | element) for this tile's range and publish it in shared memory.
__device__ __forceinline__ bool oracle_lookup(const KParams &p, unsigned long long tile, int tid,
                                              unsigned long long *s_mlo, unsigned long long *s_mcnt) {
    const bool has = (__ldg(&p.tilemap[tile >> 5]) >> (tile & 31)) & 1u;
    if (has && tid == 0) {
        const unsigned long long first = tile << 16;
        unsigned long long lo = 0, hi = p.n_marked;
        while (lo < hi) {
            unsigned long long md = (lo + hi) >> 1;
            if (p.marked[md] < first) lo = md + 1; else hi = md;
        }
        const unsigned long long a = lo;
        hi = p.n_marked;
        const unsigned long long end = first + (1ull << 16);
        while (lo < hi) {
            unsigned long long md = (lo + hi) >> 1;
            if (p.marked[md] < end) lo = md + 1; else hi = md;
        }
        *s_mlo = a;
        *s_mcnt = lo - a;
    }
    return has;
}

// Layout PH runs at least one processed stage (tile bits [U, TB)).
template <class L, int U>
__host__ __device__ constexpr bool layout_has_work(int ph) {
    bool w = false;
    for (int b = U; b < L::kTB; ++b) w = w || L::owns(ph, b);
    return w;
}

// Everything after the tile is in registers (layout A): stage sets, the
// elementwise op, relayouts through `sm`, and the global store.  Only the
// layouts that own a processed tile bit are visited (A always does: it holds
// the top tile bits), so a strided tile whose processed bits all live in A
// and C skips B and needs one relayout per stage set instead of two (U = 5..8),
// and one whose processed bits are all A register bits needs none (U >= 9).
template <class L, bool PRE, bool POST, int U, int NOISY, bool XCHG, typename E>
__device__ __forceinline__ void tile_body(E (&x)[L::NR], E *sm, const KParamsT<NOISY> &p, unsigned long long base, E *gout,
                                          int tid, E *const *sdst, bool has_marked, const unsigned long long *s_mlo,
                                          const unsigned long long *s_mcnt) {
    constexpr bool wB = layout_has_work<L, U>(1), wC = layout_has_work<L, U>(2);
    constexpr int kLast = wC ? 2 : (wB ? 1 : 0);   // last layout of a forward visit
    constexpr int kMid = wB ? 1 : 0;               // the layout before C
    if (PRE) {
        run_stages<L, 0, U, NOISY, 0>(x, p);
        if constexpr (wB) {
            relayout<L, 0, 1>(x, sm, tid);
            run_stages<L, 1, U, NOISY, 0>(x, p);
        }
        if constexpr (wC) {
            relayout<L, kMid, 2>(x, sm, tid);
            run_stages<L, 2, U, NOISY, 0>(x, p);
        }
        if constexpr (kLast == 0) {
            if (has_marked) __syncthreads();  // s_mlo / s_mcnt (no relayout barrier on this path)
        }
        if (p.mid == MID_F0 || has_marked) mid_op<L, kLast>(x, p, base, tid, *s_mlo, *s_mcnt);
        if (POST) {
            run_stages<L, kLast, U, NOISY, 1>(x, p);
            if constexpr (wC) {
                relayout<L, 2, kMid>(x, sm, tid);
                run_stages<L, kMid, U, NOISY, 1>(x, p);
            }
            if constexpr (wB) {
                relayout<L, 1, 0>(x, sm, tid);
                run_stages<L, 0, U, NOISY, 1>(x, p);
            }
            pass_store<L, 0, XCHG, (U == 0)>(x, gout, base, p, tid, sdst);
        } else {
            pass_store<L, kLast, XCHG, (U == 0)>(x, gout, base, p, tid, sdst);
        }
    } else {
        if (has_marked) __syncthreads();  // s_mlo / s_mcnt (uniform branch)
        if (p.mid == MID_F0 || has_marked) mid_op<L, 0>(x, p, base, tid, *s_mlo, *s_mcnt);
        if (POST) {
            run_stages<L, 0, U, NOISY, 1>(x, p);
            if constexpr (wB) {
                relayout<L, 0, 1>(x, sm, tid);
                run_stages<L, 1, U, NOISY, 1>(x, p);
            }
            if constexpr (wC) {
                relayout<L, kMid, 2>(x, sm, tid);
                run_stages<L, 2, U, NOISY, 1>(x, p);
            }
            pass_store<L, kLast, XCHG, (U == 0)>(x, gout, base, p, tid, sdst);
        } else {
            pass_store<L, 0, XCHG, (U == 0)>(x, gout, base, p, tid, sdst);
        }
    }
}

// tile_body for the two-layout strided family (Layout2): A -> B stages,
// the op in B, B -> A stages; without processed bits in B it stays in A.
template <class L, bool PRE, bool POST, int U, int NOISY, bool XCHG, typename E>
__device__ __forceinline__ void tile_body2(E (&x)[L::NR], E *sm, const KParamsT<NOISY> &p, unsigned long long base, E *gout,
                                           int tid, E *const *sdst, bool has_marked, const unsigned long long *s_mlo,
                                           const unsigned long long *s_mcnt) {
    constexpr bool kNeedB = U < L::kTB - L::kRB;
    constexpr int kLast = kNeedB ? 1 : 0;
    if (PRE) {
        run_stages<L, 0, U, NOISY, 0>(x, p);
        if constexpr (kNeedB) {
            relayout<L, 0, 1>(x, sm, tid);
            run_stages<L, 1, U, NOISY, 0>(x, p);
        } else if (has_marked) {
            __syncthreads();  // s_mlo / s_mcnt (no relayout barrier on this path)
        }
        if (p.mid == MID_F0 || has_marked) mid_op<L, kLast>(x, p, base, tid, *s_mlo, *s_mcnt);
        if (POST) {
            run_stages<L, kLast, U, NOISY, 1>(x, p);
            if constexpr (kNeedB) {
                relayout<L, 1, 0>(x, sm, tid);
                run_stages<L, 0, U, NOISY, 1>(x, p);
            }
            pass_store<L, 0, XCHG>(x, gout, base, p, tid, sdst);
        } else {
            pass_store<L, kLast, XCHG>(x, gout, base, p, tid, sdst);
        }
    } else {
        if (has_marked) __syncthreads();
        if (p.mid == MID_F0 || has_marked) mid_op<L, 0>(x, p, base, tid, *s_mlo, *s_mcnt);
        if (POST) {
            run_stages<L, 0, U, NOISY, 1>(x, p);
            if constexpr (kNeedB) {
                relayout<L, 0, 1>(x, sm, tid);
                run_stages<L, 1, U, NOISY, 1>(x, p);
            }
        }
        pass_store<L, POST ? kLast : 0, XCHG>(x, gout, base, p, tid, sdst);
    }
}

// Strided complex64 tiles (U >= 3) with the two-layout family.
template <int TB, int RB, bool PRE, bool POST, int U, int NOISY, bool XCHG>
__global__ void __launch_bounds__(1 << (TB - RB), SV_TILE_MIN_BLOCKS) wht_tile2_kernel(const KParamsT<NOISY> p) {
    using L = Layout2<TB, RB>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *sm = reinterpret_cast<float2 *>(smem_raw);
    __shared__ unsigned long long s_mlo, s_mcnt;
    __shared__ float2 *s_dst[XCHG ? 8 : 1];
    if constexpr (XCHG) load_xdst(p, threadIdx.x, s_dst);
    const int tid = threadIdx.x;
    const unsigned long long base = tile_base(blockIdx.x, p);
    float2 x[L::NR];
    global_load<L, 0>(x, reinterpret_cast<const float2 *>(p.in) + base, p, tid);
    if constexpr (NOISY) {  // renormalisation (decoherence) rides only on the general-2x2 flavours
        if (p.scale_in) apply_scale(x, *p.scale_in);
    }
    if constexpr (NOISY == 2) apply_scalef(x, p.pass_scalef);  // the product of the pass's factors c
    const bool has_marked = (p.mid == MID_ORACLE) && oracle_lookup(p, blockIdx.x, tid, &s_mlo, &s_mcnt);
    tile_body2<L, PRE, POST, U, NOISY, XCHG>(x, sm, p, base, reinterpret_cast<float2 *>(p.out) + base, tid, s_dst, has_marked, &s_mlo,
                                &s_mcnt);
    if constexpr (NOISY) {
        if (p.sumsq) tile_sumsq(x, p.sumsq, blockIdx.x, tid);
    }
}

// One CTA per tile: 128-bit loads straight into registers (layout A).
template <typename E, int TB, int RB, bool PRE, bool POST, int U, int NOISY, bool XCHG>
__global__ void __launch_bounds__(1 << (TB - RB), (TB - RB >= 9) ? 1 : SV_TILE_MIN_BLOCKS) wht_tile_kernel(const KParamsT<NOISY> p) {
    using L = Layout<E, TB, RB>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E *sm = reinterpret_cast<E *>(smem_raw);
    __shared__ unsigned long long s_mlo, s_mcnt;
    __shared__ E *s_dst[XCHG ? 8 : 1];
    if constexpr (XCHG) load_xdst(p, threadIdx.x, s_dst);
    const int tid = threadIdx.x;
    // U == 0: the contiguous group, tile t = slots [0, T) at t * 2^T
    const unsigned long long base =
        (U == 0) ? ((unsigned long long)blockIdx.x << TB) : tile_base(blockIdx.x, p);
    E x[L::NR];
    global_load<L, 0, (U == 0)>(x, reinterpret_cast<const E *>(p.in) + base, p, tid);
    if constexpr (NOISY) {  // renormalisation (decoherence) rides only on the general-2x2 flavours
        if (p.scale_in) apply_scale(x, *p.scale_in);
    }
    if constexpr (NOISY == 2) {  // the product of the pass's factors c
        if constexpr (sizeof(E) == 8) apply_scalef(x, p.pass_scalef);
        else apply_scale(x, p.pass_scale);
    }
    const bool has_marked = (p.mid == MID_ORACLE) && oracle_lookup(p, blockIdx.x, tid, &s_mlo, &s_mcnt);
    tile_body<L, PRE, POST, U, NOISY, XCHG>(x, sm, p, base, reinterpret_cast<E *>(p.out) + base, tid, s_dst, has_marked, &s_mlo, &s_mcnt);
    if constexpr (NOISY) {
        if (p.sumsq) tile_sumsq(x, p.sumsq, blockIdx.x, tid);
    }
}

#ifndef __CUDACC_RTC__
template <typename E, int TB, int RB, bool PRE, bool POST, int U, int NOISY, bool XCHG>
static void launch_tile_x(const KParamsT<NOISY> &kp, unsigned long long ntiles, cudaStream_t s) {
    using L = Layout<E, TB, RB>;
    auto fn = wht_tile_kernel<E, TB, RB, PRE, POST, U, NOISY, XCHG>;
    // short-run strided c64 tiles (64-128 B runs): halve the relayouts with the
    // two-layout family; longer runs keep 16-byte accesses (measured on B200:
    // U = 3/4 passes 14-17% faster, U = 6 passes 9% slower with Layout2)
    if constexpr (sizeof(E) == 8 && U >= 3 && U <= SV_2LAYOUT_MAX_U)
        fn = wht_tile2_kernel<TB, RB, PRE, POST, U, NOISY, XCHG>;
    const int smem = (1 << TB) * (int)sizeof(E);
    static bool attr = false;
    if (!attr) {
        SV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    SV_CHECK(ntiles <= 0x7fffffffull, SV_EINVAL, "too many tiles for one launch");
    fn<<<(unsigned int)ntiles, L::NT, smem, s>>>(kp);
    SV_CUDA(cudaGetLastError());
}

template <typename E, int TB, int RB, bool PRE, bool POST, int U, int NOISY>
static void launch_tile_t(const KParamsT<NOISY> &kp, unsigned long long ntiles, cudaStream_t s) {
    if (kp.xchg) launch_tile_x<E, TB, RB, PRE, POST, U, NOISY, true>(kp, ntiles, s);
    else launch_tile_x<E, TB, RB, PRE, POST, U, NOISY, false>(kp, ntiles, s);
}

template <typename E, int TB, int RB, int U, int NOISY>
static void launch_tile_u(const KParamsT<NOISY> &kp, int pre, int post, int u, unsigned long long ntiles, cudaStream_t s) {
    if constexpr (U < TB) {
        if (u != U) return launch_tile_u<E, TB, RB, U + 1, NOISY>(kp, pre, post, u, ntiles, s);
        if (pre && post) launch_tile_t<E, TB, RB, true, true, U, NOISY>(kp, ntiles, s);
        else if (pre) launch_tile_t<E, TB, RB, true, false, U, NOISY>(kp, ntiles, s);
        else if (post) launch_tile_t<E, TB, RB, false, true, U, NOISY>(kp, ntiles, s);
        else SV_CHECK(false, SV_EINVAL, "internal: tile pass without stages");
    } else {
        SV_CHECK(false, SV_EINVAL, "internal: no processed tile bits");
    }
}

#endif  // __CUDACC_RTC__ (host launch templates)
}  // namespace sv

#ifndef __CUDACC_RTC__
namespace sv {
// wht.cu: kernel parameters of one tile pass (flavour 0/1/2, unprocessed bits, tile count).
int pack_tile_params(sv_dtype dt, const PassArgs &a, bool check_lookup, KParams &kp, KParamsT<1> &kc,
                     KParamsT<2> &ka, int *u_out, unsigned long long *ntiles);
// Both dtypes, one stage flavour (instantiated in wht.cu / wht_noisy.cu).
template <int NOISY>
void launch_tile_dispatch(sv_dtype dt, const KParamsT<NOISY> &kp, int pre, int post, int u, unsigned long long ntiles,
                          cudaStream_t s) {
    if (dt == SV_C64) launch_tile_u<float2, kTileBitsC64, kRegBitsC64, 0, NOISY>(kp, pre, post, u, ntiles, s);
    else launch_tile_u<double2, kTileBitsC128, kRegBitsC128, 0, NOISY>(kp, pre, post, u, ntiles, s);
}
extern template void launch_tile_dispatch<0>(sv_dtype, const KParamsT<0> &, int, int, int, unsigned long long,
                                                 cudaStream_t);
extern template void launch_tile_dispatch<1>(sv_dtype, const KParamsT<1> &, int, int, int, unsigned long long,
                                                cudaStream_t);
extern template void launch_tile_dispatch<2>(sv_dtype, const KParamsT<2> &, int, int, int, unsigned long long,
                                              cudaStream_t);
}  // namespace sv
#endif  // __CUDACC_RTC__
