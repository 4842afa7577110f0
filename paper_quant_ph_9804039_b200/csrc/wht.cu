// wht.cu -- host side of the WHT tile pass (parameter packing, dispatch), the
// ideal-stage instantiation, the whole-state kernel and layout introspection.
// The kernels themselves are in wht_kernels.cuh.
#include <cuda_runtime.h>

#include <type_traits>
#include <math.h>

#include "wht_kernels.cuh"

namespace sv {

template void launch_tile_dispatch<0>(sv_dtype, const KParamsT<0> &, int, int, int, unsigned long long,
                                          cudaStream_t);

// Kernel variant (template instantiation) a tile pass launches -- the same
// decisions as launch_wht_tile_pass, without a device (tests/test_variants.py
// maps every variant the benches launch to a parity test that runs it).
TileVariant describe_tile_pass(sv_dtype dt, const PassArgs &a) {
    TileVariant v;
    launch_wht_tile_pass(dt, a, nullptr, &v);
    return v;
}

// Kernel parameters of one tile pass (shared with the supertile pass,
// wht_super.cu): slot map, free-slot runs, op, exchange, coefficients of the
// general 2x2 (kc) and tan (ka) flavours.  Returns the stage flavour (0 ideal,
// 1 general 2x2, 2 tan form) and the unprocessed tile bits in *u.
int pack_tile_params(sv_dtype dt, const PassArgs &a, bool check_lookup, KParams &kp, KParamsT<1> &kc,
                     KParamsT<2> &ka, int *u_out, unsigned long long *ntiles) {
    const int TB = tile_bits(dt);
    kp = KParams{};
    kc = KParamsT<1>{};
    ka = KParamsT<2>{};
    kp.in = a.in;
    kp.out = a.out;
    kp.marked = reinterpret_cast<const unsigned long long *>(a.marked);
    kp.tilemap = a.tilemap;
    kp.n_marked = a.n_marked;
    kp.f0_scale = a.f0_scale;
    kp.mid = a.mid;
    kp.has_origin = a.has_origin;
    SV_CHECK(a.scale_in == nullptr || a.noisy, SV_EINVAL, "internal: scale_in needs the general-2x2 kernels");
    SV_CHECK(a.sumsq == nullptr || a.noisy, SV_EINVAL, "internal: sumsq needs the general-2x2 kernels");
    kp.scale_in = a.scale_in;
    kp.sumsq = a.sumsq;
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
    unsigned int proc = 0;
    kp.free_mask = 0;
    for (int sl = 0; sl < a.total_bits; ++sl) {
        if ((a.tile_mask >> sl) & 1) {
            SV_CHECK(b < 16, SV_EINVAL, "internal: tile too large");
            if ((a.proc_mask >> sl) & 1) proc |= 1u << b;
            if (a.noisy)
                for (int h = 0; h < 2; ++h)
                    for (int e = 0; e < 4; ++e) kc.coef[h][b][e] = a.coef[h][sl][e];
            kp.slot[b++] = (signed char)sl;
        } else {
            kp.free_mask |= 1ull << sl;
            ++f;
        }
    }
    SV_CHECK(b == TB, SV_EINVAL, "internal: tile mask does not have T slots");
    SV_CHECK(kp.slot[0] == 0, SV_EINVAL, "internal: tile must contain slot 0");
    kp_set_free_runs(kp);
    if (a.mid == MID_ORACLE && check_lookup)
        SV_CHECK(a.tilemap != nullptr && (a.n_marked == 0 || a.marked != nullptr), SV_EINVAL,
                 "internal: oracle pass without its tile lookup");
    kp.proc = proc;
    // processed tile bits must be [u, TB) (see run_stages)
    int u = 0;
    while (u < TB && !((proc >> u) & 1u)) ++u;
    SV_CHECK(u < TB && proc == (((1u << TB) - 1u) & ~((1u << u) - 1u)), SV_EINVAL,
             "internal: processed tile bits are not the top ones");
    // u == 0 kernels assume the contiguous tile (slots [0, T), tile t at t * 2^T)
    SV_CHECK(u != 0 || (a.tile_mask == (1ull << TB) - 1ull && kp.free_mask == ((~0ull >> (64 - a.total_bits)) & ~((1ull << TB) - 1ull))),
             SV_EINVAL, "internal: a fully processed tile must be the contiguous one");
    *u_out = u;
    *ntiles = 1ull << f;
    if (!a.noisy) return 0;
    // pure angle errors ([c s; s -c] on every processed bit, no decoherence
    // contraction) take the tan form: [[1, t], [t, -1]] and one factor c per bit
    bool tan_form = true;
    double pass_scale = 1.0;
    for (int bb = 0; bb < TB && tan_form; ++bb) {
        if (!((proc >> bb) & 1u)) continue;
        for (int h = 0; h < 2; ++h) {
            if ((h == 0 && !a.pre) || (h == 1 && !a.post)) continue;
            const double *m = kc.coef[h][bb];
            if (!(m[1] == m[2] && m[3] == -m[0] && fabs(m[0]) > 0.25)) { tan_form = false; break; }
            pass_scale *= m[0];
        }
    }
    static_cast<KParams &>(kc) = kp;
    static_cast<KParams &>(ka) = kp;
    for (int h = 0; h < 2; ++h)
        for (int bb = 0; bb < 16; ++bb) ka.coef[h][bb][0] = kc.coef[h][bb][0] != 0.0 ? kc.coef[h][bb][1] / kc.coef[h][bb][0] : 0.0;
    ka.pass_scale = pass_scale;
    for (int h = 0; h < 2; ++h)
        for (int bb = 0; bb < 16; ++bb)
            for (int e = 0; e < 4; ++e) {
                kc.coeff[h][bb][e] = (float)kc.coef[h][bb][e];
                ka.coeff[h][bb][e] = (float)ka.coef[h][bb][e];
            }
    kc.pass_scalef = 1.0f;  // (the general flavour carries no pass factor)
    ka.pass_scalef = (float)ka.pass_scale;
    return tan_form ? 2 : 1;
}

void launch_wht_tile_pass(sv_dtype dt, const PassArgs &a, cudaStream_t s, TileVariant *describe) {
    KParams kp;
    KParamsT<1> kc;
    KParamsT<2> ka;
    int u = 0;
    unsigned long long ntiles = 0;
    const int flavour = pack_tile_params(dt, a, describe == nullptr, kp, kc, ka, &u, &ntiles);
    if (describe) {
        describe->u = u;
        describe->pre = a.pre;
        describe->mid = a.mid;
        describe->post = a.post;
        describe->xchg = kp.xchg;
        // two-layout family: strided complex64 tiles with U in [3, SV_2LAYOUT_MAX_U] (launch_tile_x)
        describe->family = (dt == SV_C64 && u >= 3 && u <= SV_2LAYOUT_MAX_U) ? 2 : 1;
        describe->noisy = flavour;
        return;
    }
    if (flavour == 2) {
        launch_tile_dispatch<2>(dt, ka, a.pre, a.post, u, ntiles, s);
    } else if (flavour == 1) {
        launch_tile_dispatch<1>(dt, kc, a.pre, a.post, u, ntiles, s);
    } else {
        KParamsT<0> ki{};
        static_cast<KParams &>(ki) = kp;
        launch_tile_dispatch<0>(dt, ki, a.pre, a.post, u, ntiles, s);
    }
}

// ------------------------------------------------------------------------- //
// Whole state in one CTA (n <= T): k iterations without leaving shared memory //
// ------------------------------------------------------------------------- //
// coefs != nullptr: general 2x2 transforms (NEXT-1 angle errors, NEXT-2
// decoherence); coefs[((it*2 + w)*n + q)*4 + {0..3}] = [w x; y z] of qubit q
// in transform w of iteration it; F0 then carries no 2^{-n} (f0_scale = 1).
// survival != nullptr: renormalise after every iteration (G22) and record the
// pre-renormalisation sum |a|^2 of iteration it in survival[it].
// stages per round trip: 0 = per dtype (measured on B200, 25 iterations:
// complex128 n=10 / 12: 2 -> 102 / 316 us (1: 120 / 464, 3: 104 / 356,
// 4: 110 / 317); complex64 n=13: 3 -> 409 us (1: 526, 2: 424, 4: 572))
#ifndef SV_WHOLE_MAXR
#define SV_WHOLE_MAXR 0
#endif
template <typename E>
__global__ void __launch_bounds__(512) whole_state_kernel(E *a, int n, int k, int with_oracle, int diffusion,
                                                          const unsigned long long *marked,
                                                          unsigned long long m, double f0_scale,
                                                          const double *coefs, double *survival) {
    using R = typename RealOf<E>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E *s = reinterpret_cast<E *>(smem_raw);
    __shared__ double red[2 * 32];
    const unsigned int N = 1u << n, tid = threadIdx.x, nt = blockDim.x;
    for (unsigned int i = tid; i < N; i += nt) s[i] = a[i];
    __syncthreads();
    // Up to kMaxR stages (qubits q .. q + RR - 1) per shared-memory round trip
    // and barrier: each thread owns a group of 2^RR amplitudes differing in
    // those qubits, keeps them in registers and applies the RR stages in qubit
    // order -- the same pair operations in the same per-pair order as
    // stage-by-stage, so results are bit-identical.
    auto phase = [&](auto rr, int it, int w, int q) {
        constexpr int RR = decltype(rr)::value;
        constexpr unsigned int G = 1u << RR;
        const unsigned int lowm = (1u << q) - 1u;
        for (unsigned int pr = tid; pr < (N >> RR); pr += nt) {
            const unsigned int i0 = ((pr >> q) << (q + RR)) | (pr & lowm);
            E v[G];
#pragma unroll
            for (unsigned int g = 0; g < G; ++g) v[g] = s[i0 | (g << q)];
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const double *c = coefs ? coefs + ((size_t)(2 * it + w) * n + q + r) * 4 : nullptr;
#pragma unroll
                for (unsigned int g = 0; g < G; ++g)
                    if (!(g & (1u << r))) {
                        if (c) bfly_gen(v[g], v[g | (1u << r)], c);
                        else bfly(v[g], v[g | (1u << r)]);
                    }
            }
#pragma unroll
            for (unsigned int g = 0; g < G; ++g) s[i0 | (g << q)] = v[g];
        }
        __syncthreads();
    };
    auto transform = [&](int it, int w) {
        for (int q = 0; q < n;) {
            // as many stages as keep >= 256 threads busy (N / 2^rr groups), at most 4
            constexpr int kMaxR = SV_WHOLE_MAXR > 0 ? SV_WHOLE_MAXR : (sizeof(E) == 8 ? 3 : 2);
            int rr = n - q >= kMaxR ? kMaxR : n - q;
            while (rr > 1 && (N >> rr) < 256u) --rr;
            switch (rr) {
                case 4: phase(std::integral_constant<int, 4>{}, it, w, q); break;
                case 3: phase(std::integral_constant<int, 3>{}, it, w, q); break;
                case 2: phase(std::integral_constant<int, 2>{}, it, w, q); break;
                default: phase(std::integral_constant<int, 1>{}, it, w, q); break;
            }
            q += rr;
        }
    };
    const int reps = k;
    for (int it = 0; it < reps; ++it) {
        if (with_oracle) {
            for (unsigned long long j = tid; j < m; j += nt) {
                E &v = s[marked[j]];
                v.x = -v.x;
                v.y = -v.y;
            }
            __syncthreads();
        }
        if (diffusion == SV_DIFFUSE_WHT) {
            transform(it, 0);
            for (unsigned int i = tid; i < N; i += nt) {
                const R sc = (R)(i == 0 ? f0_scale : -f0_scale);
                s[i].x *= sc;
                s[i].y *= sc;
            }
            __syncthreads();
            transform(it, 1);
            if (survival) {  // fixed-order block sum of |a|^2, then scale to norm 1
                double sq = 0.0, dummy = 0.0;
                for (unsigned int i = tid; i < N; i += nt)
                    sq += (double)s[i].x * (double)s[i].x + (double)s[i].y * (double)s[i].y;
                for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
                if ((tid & 31) == 0) red[2 * (tid >> 5)] = sq;
                __syncthreads();
                double tot = 0.0;
                for (unsigned int w = 0; w < nt / 32; ++w) tot += red[2 * w];
                (void)dummy;
                if (tid == 0) survival[it] = tot;
                const R inv = (R)(1.0 / sqrt(tot));
                for (unsigned int i = tid; i < N; i += nt) { s[i].x *= inv; s[i].y *= inv; }
                __syncthreads();
            }
        } else {
            // fixed-order block reduction in fp64 (deterministic)
            double re = 0.0, im = 0.0;
            for (unsigned int i = tid; i < N; i += nt) { re += (double)s[i].x; im += (double)s[i].y; }
            for (int o = 16; o > 0; o >>= 1) {
                re += __shfl_xor_sync(0xffffffffu, re, o);
                im += __shfl_xor_sync(0xffffffffu, im, o);
            }
            if ((tid & 31) == 0) { red[2 * (tid >> 5)] = re; red[2 * (tid >> 5) + 1] = im; }
            __syncthreads();
            double mr = 0.0, mi = 0.0;
            for (unsigned int w = 0; w < nt / 32; ++w) { mr += red[2 * w]; mi += red[2 * w + 1]; }
            mr *= f0_scale;  // 1/N
            mi *= f0_scale;
            const R two_mr = (R)(2.0 * mr), two_mi = (R)(2.0 * mi);
            for (unsigned int i = tid; i < N; i += nt) { s[i].x = two_mr - s[i].x; s[i].y = two_mi - s[i].y; }
            __syncthreads();
        }
    }
    for (unsigned int i = tid; i < N; i += nt) a[i] = s[i];
}

// ------------------------------------------------------------------------- //
// Whole state in the REGISTERS of 2^LOGW warps (n = LOGR + 5 + LOGW): 2^LOGR //
// amplitudes per thread.  Layout A: index = tid * 2^LOGR + r -- the register //
// bits [0, LOGR) and the lane bits [LOGR, LOGR + 5) run in registers and by  //
// warp shuffles (the lane with the bit clear forms x + y, its partner        //
// y' - x' = a_i - a_j: the pair butterfly's two sums).  Layout B (one        //
// shared-memory relayout away): r = the top LOGR index bits, lane = the 5    //
// below, warp = the lowest LOGW -- the warp bits of A, [LOGR + 5, n), are    //
// register or lane bits there.  A transform visits A then B, the next one B  //
// then A (stages on different bits commute, G18), so each transform costs    //
// ONE relayout and barrier; F0 runs in B, O in A.  Round 2 widened it from 4 //
// warps (1 warp per SMSP: issue stalled on every dependency) to 8-16.        //
// ------------------------------------------------------------------------- //
template <typename E, typename R, bool GEN>
__device__ __forceinline__ void shfl_stage(E &x, int d, bool hi, const double *c) {
    E y;
    y.x = __shfl_xor_sync(0xffffffffu, x.x, d);
    y.y = __shfl_xor_sync(0xffffffffu, x.y, d);
    if constexpr (!GEN) {  // ideal butterfly: (a_i, a_j) -> (a_i + a_j, a_i - a_j)
        // one FMA by +-1 per component: lo lanes x + y, hi lanes y - x -- the
        // same single rounding as the add / subtract (bitwise identical), but
        // without computing both and selecting (2 adds + 4 selects per element)
        const R sg = hi ? (R)-1 : (R)1;
        x.x = fma(sg, x.x, y.x);
        x.y = fma(sg, x.y, y.y);
    } else {  // Fig. 3's [w x; y z]: a_i' = w a_i + x a_j, a_j' = y a_i + z a_j
        const R w = (R)c[0], xx = (R)c[1], yy = (R)c[2], z = (R)c[3];
        if (!hi) { x.x = w * x.x + xx * y.x; x.y = w * x.y + xx * y.y; }
        else { x.x = yy * y.x + z * x.x; x.y = yy * y.y + z * x.y; }
    }
}

template <typename E, int LOGR, int LOGW>
struct WR {
    static constexpr int NR = 1 << LOGR, NT = 32 << LOGW, n = LOGR + 5 + LOGW;
    static_assert(LOGW >= 2 && LOGW <= LOGR + 5, "layout B must hold A's warp bits in registers and lanes");
    // XOR swizzle of the shared-memory index: every quarter-warp (16-B
    // elements) / half-warp (8-B) access of both layouts is bank-conflict free
    // (brute-force checked for every instantiated (LOGR, LOGW))
    static constexpr uint32_t M = sizeof(E) == 16 ? 7u : 15u;
    static constexpr int S1 = (sizeof(E) == 8 && LOGR == 6 && LOGW == 2) ? 2 : 1;
    static constexpr int S2 = LOGR > LOGW ? LOGR : LOGW;
    __device__ static __forceinline__ uint32_t swz(uint32_t i) { return i ^ ((i >> S1) & M) ^ ((i >> S2) & M); }
    __device__ static __forceinline__ uint32_t idxA(int tid, int r) { return ((uint32_t)tid << LOGR) | (uint32_t)r; }
    __device__ static __forceinline__ uint32_t idxB(int tid, int r) {
        return ((uint32_t)r << (n - LOGR)) | ((uint32_t)(tid & 31) << (n - LOGR - 5)) | ((uint32_t)tid >> 5);
    }
};

// Stages of layout A: index bits [0, LOGR + 5).
template <typename E, int LOGR, int LOGW, bool GEN>
__device__ __forceinline__ void wr_stages_a(E (&x)[1 << LOGR], int lane, const double *cbase) {
    using R = typename RealOf<E>::T;
    constexpr int NR = 1 << LOGR;
#pragma unroll
    for (int q = 0; q < LOGR; ++q) {
#pragma unroll
        for (int j = 0; j < NR; ++j)
            if (!(j & (1 << q))) {
                if constexpr (GEN) bfly_gen(x[j], x[j | (1 << q)], cbase + 4 * q);
                else bfly(x[j], x[j | (1 << q)]);
            }
    }
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        const bool hi = (lane >> b) & 1;
#pragma unroll
        for (int j = 0; j < NR; ++j) shfl_stage<E, R, GEN>(x[j], 1 << b, hi, GEN ? cbase + 4 * (LOGR + b) : nullptr);
    }
}

// Stages of layout B: index bits [LOGR + 5, n) -- register bits at the top,
// lane bits below them.
template <typename E, int LOGR, int LOGW, bool GEN>
__device__ __forceinline__ void wr_stages_b(E (&x)[1 << LOGR], int lane, const double *cbase) {
    using R = typename RealOf<E>::T;
    constexpr int NR = 1 << LOGR, n = LOGR + 5 + LOGW;
#pragma unroll
    for (int t = LOGR + 5; t < n; ++t) {
        if (t >= n - LOGR) {
            const int q = t - (n - LOGR);
#pragma unroll
            for (int j = 0; j < NR; ++j)
                if (!(j & (1 << q))) {
                    if constexpr (GEN) bfly_gen(x[j], x[j | (1 << q)], cbase + 4 * t);
                    else bfly(x[j], x[j | (1 << q)]);
                }
        } else {
            const int b = t - (n - LOGR - 5);
            const bool hi = (lane >> b) & 1;
#pragma unroll
            for (int j = 0; j < NR; ++j) shfl_stage<E, R, GEN>(x[j], 1 << b, hi, GEN ? cbase + 4 * t : nullptr);
        }
    }
}

// Relayout A -> B (TO_B) or B -> A through the swizzled tile: each thread
// rewrites only the positions it read in the previous relayout, so one
// barrier per change suffices.
template <typename E, int LOGR, int LOGW, bool TO_B>
__device__ __forceinline__ void wr_relayout(E (&x)[1 << LOGR], E *s, int tid) {
    using W = WR<E, LOGR, LOGW>;
#pragma unroll
    for (int r = 0; r < W::NR; ++r) s[W::swz(TO_B ? W::idxA(tid, r) : W::idxB(tid, r))] = x[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < W::NR; ++r) x[r] = s[W::swz(TO_B ? W::idxB(tid, r) : W::idxA(tid, r))];
}

// fixed-order CTA sums: the thread's values in register order, a warp xor
// butterfly (every lane ends with bitwise the same value), the warps in order
template <int NW>
__device__ __forceinline__ void wr_cta_sum2(double re, double im, double &tre, double &tim, double *red, int tid) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if ((tid & 31) == 0) { red[2 * (tid >> 5)] = re; red[2 * (tid >> 5) + 1] = im; }
    __syncthreads();
    tre = 0.0;
    tim = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) { tre += red[2 * w]; tim += red[2 * w + 1]; }
    __syncthreads();  // red reused
}

template <typename E, int LOGR, int LOGW, bool GEN>
__global__ void __launch_bounds__(32 << LOGW) whole_reg_kernel(E *a, int k, int with_oracle, int diffusion,
                                                               const unsigned long long *marked, unsigned long long m,
                                                               double f0_scale, const double *coefs, double *survival) {
    using R = typename RealOf<E>::T;
    using W = WR<E, LOGR, LOGW>;
    constexpr int NR = W::NR, n = W::n;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E *s = reinterpret_cast<E *>(smem_raw);
    __shared__ double red[2 * (1 << LOGW)];
    const int tid = threadIdx.x, lane = tid & 31;
    __shared__ unsigned long long s_mk[64];  // the marked set, when it is small, read once
    E x[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) x[r] = a[W::idxA(tid, r)];
    const bool mk_smem = with_oracle && m <= 64;
    if (mk_smem && tid < (int)m) s_mk[tid] = marked[tid];
    __syncthreads();
    for (int it = 0; it < k; ++it) {
        if (with_oracle) {  // layout A
            for (unsigned long long j = 0; j < m; ++j) {
                const unsigned long long mk = mk_smem ? s_mk[j] : marked[j];
                if ((int)(mk >> LOGR) == tid) {
                    const int rr = (int)(mk & (NR - 1));
#pragma unroll
                    for (int r = 0; r < NR; ++r)
                        if (r == rr) { x[r].x = -x[r].x; x[r].y = -x[r].y; }
                }
            }
        }
        if (diffusion == SV_DIFFUSE_WHT) {
            const double *c1 = GEN ? coefs + (size_t)(2 * it) * n * 4 : nullptr;
            const double *c2 = GEN ? coefs + (size_t)(2 * it + 1) * n * 4 : nullptr;
            wr_stages_a<E, LOGR, LOGW, GEN>(x, lane, c1);
            wr_relayout<E, LOGR, LOGW, true>(x, s, tid);
            wr_stages_b<E, LOGR, LOGW, GEN>(x, lane, c1);
            // F0 = 2|0><0| - I with the 2^-n of the unnormalised transforms (G2, G5);
            // index 0 is thread 0's register 0 in both layouts
#pragma unroll
            for (int r = 0; r < NR; ++r) scale(x[r], (R)(-f0_scale));
            if (tid == 0) { x[0].x = -x[0].x; x[0].y = -x[0].y; }
            wr_stages_b<E, LOGR, LOGW, GEN>(x, lane, c2);
            wr_relayout<E, LOGR, LOGW, false>(x, s, tid);
            wr_stages_a<E, LOGR, LOGW, GEN>(x, lane, c2);
            if (survival) {  // renormalise (G22): sum |a|^2 in fixed order, record it, scale to norm 1
                double sq = 0.0;
#pragma unroll
                for (int r = 0; r < NR; ++r) sq += (double)x[r].x * (double)x[r].x + (double)x[r].y * (double)x[r].y;
                double tot, dummy;
                wr_cta_sum2<1 << LOGW>(sq, 0.0, tot, dummy, red, tid);
                if (tid == 0) survival[it] = tot;
                const R inv = (R)(1.0 / sqrt(tot));
#pragma unroll
                for (int r = 0; r < NR; ++r) { x[r].x *= inv; x[r].y *= inv; }
            }
        } else {  // inversion about the mean
            double re = 0.0, im = 0.0;
#pragma unroll
            for (int r = 0; r < NR; ++r) { re += (double)x[r].x; im += (double)x[r].y; }
            double mr, mi;
            wr_cta_sum2<1 << LOGW>(re, im, mr, mi, red, tid);
            const R two_mr = (R)(2.0 * mr * f0_scale), two_mi = (R)(2.0 * mi * f0_scale);
#pragma unroll
            for (int r = 0; r < NR; ++r) { x[r].x = two_mr - x[r].x; x[r].y = two_mi - x[r].y; }
        }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) a[W::idxA(tid, r)] = x[r];
}

template <typename E, int LOGR, int LOGW>
static void launch_whole_reg(E *state, int k, int with_oracle, int diffusion, const unsigned long long *mk,
                             uint64_t m, double f0, const double *coefs, double *survival, cudaStream_t s) {
    const int smem = (int)((1u << (LOGR + 5 + LOGW)) * sizeof(E));
    auto kern = coefs ? whole_reg_kernel<E, LOGR, LOGW, true> : whole_reg_kernel<E, LOGR, LOGW, false>;
    SV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, 32 << LOGW, smem, s>>>(state, k, with_oracle, diffusion, mk, m, f0, coefs, survival);
    SV_CUDA(cudaGetLastError());
}

// Warp bits of the register kernel per (dtype, n): SV_WHOLE_W=<LOGW> picks
// another instantiated split (tools/whole_state_bench.py).
static int whole_reg_logw(bool c64, int n) {
    static const int forced = [] {
        const char *e = getenv("SV_WHOLE_W");
        return e ? atoi(e) : 0;
    }();
    if (forced) return forced;
    // measured (profiles/r2_whole_state_bench.txt): 4 warps at n = 9, 8 up to
    // n = 12, 16 for complex64 n = 13
    (void)c64;
    return n <= 9 ? 2 : n <= 12 ? 3 : 4;
}

#ifndef SV_WHOLE_REG
#define SV_WHOLE_REG 1  // 0: every whole-state run on whole_state_kernel (A/B)
#endif

void launch_whole_state(sv_dtype dt, void *state, int n, int k, int with_oracle, int diffusion,
                        const uint64_t *marked, uint64_t m, cudaStream_t s, const double *coefs, double *survival) {
    const unsigned int N = 1u << n;
    if (SV_WHOLE_REG && n >= 9 && (dt == SV_C64 ? n <= 13 : n <= 12)) {  // the register-resident kernel
        const double f0r = coefs ? 1.0 : ldexp(1.0, -n);
        SV_CHECK(!coefs || diffusion == SV_DIFFUSE_WHT, SV_EINVAL, "internal: angle errors need the WHT diffusion");
        const auto mkr = reinterpret_cast<const unsigned long long *>(marked);
        const int w = whole_reg_logw(dt == SV_C64, n);
#define SV_WR(E, LR, LW) \
    if (n == LR + 5 + LW && w == LW) \
        return launch_whole_reg<E, LR, LW>(reinterpret_cast<E *>(state), k, with_oracle, diffusion, mkr, m, f0r, coefs, survival, s)
        if (dt == SV_C64) {
            SV_WR(float2, 2, 2); SV_WR(float2, 3, 2); SV_WR(float2, 2, 3); SV_WR(float2, 4, 2); SV_WR(float2, 3, 3);
            SV_WR(float2, 2, 4); SV_WR(float2, 5, 2); SV_WR(float2, 4, 3); SV_WR(float2, 3, 4); SV_WR(float2, 6, 2);
            SV_WR(float2, 5, 3); SV_WR(float2, 4, 4); SV_WR(float2, 0, 5);
        } else {
            SV_WR(double2, 2, 2); SV_WR(double2, 3, 2); SV_WR(double2, 2, 3); SV_WR(double2, 4, 2); SV_WR(double2, 3, 3);
            SV_WR(double2, 2, 4); SV_WR(double2, 4, 3); SV_WR(double2, 3, 4); SV_WR(double2, 1, 4);
            SV_WR(double2, 0, 5);
        }
#undef SV_WR
    }
    const int threads = N >= 1024 ? 512 : (N / 2 >= 32 ? (int)(N / 2) : 32);
    const double f0 = coefs ? 1.0 : ldexp(1.0, -n);
    SV_CHECK(!coefs || diffusion == SV_DIFFUSE_WHT, SV_EINVAL, "internal: angle errors need the WHT diffusion");
    const auto mk = reinterpret_cast<const unsigned long long *>(marked);
    if (dt == SV_C64) {
        const int smem = (int)(N * sizeof(float2));
        SV_CUDA(cudaFuncSetAttribute(whole_state_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        whole_state_kernel<float2>
            <<<1, threads, smem, s>>>((float2 *)state, n, k, with_oracle, diffusion, mk, m, f0, coefs, survival);
    } else {
        const int smem = (int)(N * sizeof(double2));
        SV_CUDA(cudaFuncSetAttribute(whole_state_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        whole_state_kernel<double2>
            <<<1, threads, smem, s>>>((double2 *)state, n, k, with_oracle, diffusion, mk, m, f0, coefs, survival);
    }
    SV_CUDA(cudaGetLastError());
}

// Host-side view of the tile layouts for tests/test_layouts.py (no device).
extern "C" int sv_debug_tile_layout(int dtype, int phase, int tid, int reg, int *tile_elem, int *smem_index) {
    if (phase < 0 || phase > 2) return -1;
    if (dtype == 2) {  // complex64 strided two-layout family
        using L = Layout2<kTileBitsC64, kRegBitsC64>;
        if (phase > 1 || tid < 0 || tid >= L::NT || reg < 0 || reg >= L::NR) return -1;
        const uint32_t e = L::ethr(phase, tid) | L::ereg(phase, reg);
        *tile_elem = (int)e;
        *smem_index = (int)L::swz(e);
        return 0;
    }
    if (dtype == SV_C64) {
        using L = Layout<float2, kTileBitsC64, kRegBitsC64>;
        if (tid < 0 || tid >= L::NT || reg < 0 || reg >= L::NR) return -1;
        const uint32_t e = L::ethr(phase, tid) | L::ereg(phase, reg);
        *tile_elem = (int)e;
        *smem_index = (int)L::swz(e);
        return 0;
    }
    using L = Layout<double2, kTileBitsC128, kRegBitsC128>;
    if (tid < 0 || tid >= L::NT || reg < 0 || reg >= L::NR) return -1;
    const uint32_t e = L::ethr(phase, tid) | L::ereg(phase, reg);
    *tile_elem = (int)e;
    *smem_index = (int)L::swz(e);
    return 0;
}

extern "C" int sv_debug_tile_owner(int dtype, int phase, int bit) {
    if (dtype == 2) return Layout2<kTileBitsC64, kRegBitsC64>::owns(phase, bit) ? 1 : 0;
    if (dtype == SV_C64) return Layout<float2, kTileBitsC64, kRegBitsC64>::owns(phase, bit) ? 1 : 0;
    return Layout<double2, kTileBitsC128, kRegBitsC128>::owns(phase, bit) ? 1 : 0;
}

}  // namespace sv
