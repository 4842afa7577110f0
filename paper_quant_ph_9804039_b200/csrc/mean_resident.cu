// mean_resident.cu -- all k Grover iterations with the mean diffusion in ONE
// persistent launch, for states that fit the GPU's aggregate shared memory
// (148 SMs x ~220 KiB: n <= 20 complex128 / 21 complex64, e.g. c2).
//
// Same arithmetic as mean.cu (north star; Eq. 3's accumulate-and-redistribute
// of a global sum):  b = O a,  a' = 2 mu - b,  mu = sum(b) / N.
// At c2's size a launched iteration is launch- and reduction-latency bound
// (~16 us for 33 MB of L2 traffic); here every block keeps its slice of the
// state in shared memory for the whole call, so an iteration is one pass
// over shared memory plus one grid barrier:
//   * block b owns elements [b C, min((b+1) C, N)), loaded once, stored once;
//   * per iteration: negate the block's marked elements (O), a_i <- 2 mu - a_i,
//     fp64 partial sums of the new (O a')_i -> one partial per block in global
//     memory -> grid barrier -> every block sums all partials in block order
//     (identical, deterministic totals everywhere; G14) -> next mu;
//   * the grid barrier is a generation counter (co-residency is guaranteed by
//     the cooperative launch).
// Single GPU only (sharded runs need the cross-rank allreduce between
// iterations, so they keep the launched path).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "sv_internal.h"

namespace sv {

constexpr int kResThreads = 1024;

__device__ __forceinline__ void grid_barrier(unsigned int *count, unsigned int *gen, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *vgen = gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// Block-wide fp64 (re, im) sum, result in thread 0 only (one barrier: the
// next write of red[2 w] comes after the grid barrier's own __syncthreads,
// which thread 0 reaches only after reading them).
__device__ __forceinline__ void block_sum_t0(double &re, double &im, double *red) {
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { red[2 * w] = re; red[2 * w + 1] = im; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0, m = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { r += red[2 * i]; m += red[2 * i + 1]; }
        re = r;
        im = m;
    }
}

// One published block total: the fp64 (re, im) partial and the epoch it
// belongs to (launch-unique: the host advances the base by k + 1 per launch,
// so a slot left over from an earlier call never matches).
struct alignas(32) ResSlot {
    double re, im;
    unsigned long long epoch;
    unsigned long long pad;
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

#ifndef SV_RES_SLOTS
#define SV_RES_SLOTS 0  // 1: all-gather slots (measured slower: 7.7 vs 5.1 us per iteration at c2), A/B
#endif

template <typename E>
__global__ void __launch_bounds__(kResThreads, 1)
    mean_resident_kernel(E *a, unsigned long long N, unsigned long long C, double inv_N,
                         const unsigned long long *marked, unsigned long long n_marked, int k, double *partials,
                         unsigned int *bar, ResSlot *slots, unsigned long long epoch0) {
    using R = decltype(E{}.x);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E *s = reinterpret_cast<E *>(smem_raw);
    __shared__ double red[66];
    __shared__ unsigned long long s_mlo, s_mcnt;
    __shared__ unsigned long long s_mk[256];  // this block's marked entries, when few (read every iteration)
    const unsigned long long lo = (unsigned long long)blockIdx.x * C;
    const unsigned long long hi = lo + C < N ? lo + C : N;
    const unsigned int len = (unsigned int)(hi > lo ? hi - lo : 0);
    const unsigned int nb = gridDim.x;
    if (threadIdx.x == 0) {  // this block's marked entries: marked[s_mlo .. s_mlo + s_mcnt)
        unsigned long long l = 0, h = n_marked;
        while (l < h) { const unsigned long long md = (l + h) >> 1; if (marked[md] < lo) l = md + 1; else h = md; }
        const unsigned long long first = l;
        h = n_marked;
        while (l < h) { const unsigned long long md = (l + h) >> 1; if (marked[md] < hi) l = md + 1; else h = md; }
        s_mlo = first;
        s_mcnt = l - first;
    }
    for (unsigned int i = threadIdx.x; i < len; i += blockDim.x) s[i] = __ldcg(a + lo + i);
    __syncthreads();
    const unsigned long long mlo = s_mlo, mcnt = s_mcnt;
    const bool mk_smem = mcnt <= 256;
    if (mk_smem && threadIdx.x < mcnt) s_mk[threadIdx.x] = marked[mlo + threadIdx.x];
    __syncthreads();
    // Negate this block's marked entries (O); returns the thread's share of
    // sum over them of the values BEFORE negation.
    auto negate_marked = [&](double &cr, double &ci) {
        cr = 0.0;
        ci = 0.0;
        for (unsigned long long j = threadIdx.x; j < mcnt; j += blockDim.x) {
            E &v = s[(mk_smem ? s_mk[j] : marked[mlo + j]) - lo];
            cr += (double)v.x;
            ci += (double)v.y;
            v.x = -v.x;
            v.y = -v.y;
        }
    };
    unsigned int parity_round = 0;  // rounds gathered so far (epoch offset)
    (void)parity_round;
    // Grid total of the per-block values (r, m): one partial per block, grid
    // barrier, then warp 0 sums the partials in a fixed order (lane-strided,
    // then a fixed shuffle tree) -- the same total in every block.
    auto grid_total = [&](double r, double m, int parity, double &tr, double &ti) {
        block_sum_t0(r, m, red);  // (thread 0 publishes it)
#if SV_RES_SLOTS
        // all-gather instead of a counter barrier: every block publishes its
        // total with a release store of the round's epoch, and warp 0 of every
        // block waits (acquire) on each slot's epoch before reading it -- no
        // single atomic that all blocks serialise on, no second wait for a
        // generation flip; the slots alternate by parity, so a slot is never
        // rewritten before every block has read it (the next write to it comes
        // after its owner has gathered the round in between, which needs every
        // block's publication of that round, i.e. after every block's read)
        const unsigned long long want = epoch0 + (unsigned long long)(parity_round++);
        ResSlot *sl = slots + (size_t)parity * nb;
        if (threadIdx.x == 0) {
            sl[blockIdx.x].re = r;
            sl[blockIdx.x].im = m;
            st_release_u64(&sl[blockIdx.x].epoch, want);
        }
        if (threadIdx.x < 32) {
            double R0 = 0.0, M0 = 0.0;
            for (unsigned int b = threadIdx.x; b < nb; b += 32) {
                while (ld_acquire_u64(&sl[b].epoch) != want) {
                }
                R0 += __ldcg(&sl[b].re);
                M0 += __ldcg(&sl[b].im);
            }
#else
        double *part = partials + (size_t)parity * 2 * nb;
        if (threadIdx.x == 0) { part[2 * blockIdx.x] = r; part[2 * blockIdx.x + 1] = m; }
        grid_barrier(bar, bar + 1, nb);
        if (threadIdx.x < 32) {
            double R0 = 0.0, M0 = 0.0;
            for (unsigned int b = threadIdx.x; b < nb; b += 32) { R0 += __ldcg(&part[2 * b]); M0 += __ldcg(&part[2 * b + 1]); }
#endif
            for (int o = 16; o > 0; o >>= 1) {
                R0 += __shfl_xor_sync(0xffffffffu, R0, o);
                M0 += __shfl_xor_sync(0xffffffffu, M0, o);
            }
            if (threadIdx.x == 0) { red[64] = R0; red[65] = M0; }
        }
        __syncthreads();
        tr = red[64];
        ti = red[65];
    };
    // first sum: of O a
    double cr, ci, r = 0.0, m = 0.0;
    for (unsigned int i = threadIdx.x; i < len; i += blockDim.x) { r += (double)s[i].x; m += (double)s[i].y; }
    __syncthreads();  // every element read before any is negated (another thread may own it)
    negate_marked(cr, ci);
    double tr, ti;
    grid_total(r - 2.0 * cr, m - 2.0 * ci, 0, tr, ti);
    // invariant at the top of an iteration: s holds O a and (tr, ti) = sum(O a)
    for (int it = 0; it < k; ++it) {
        const R two_mr = (R)(2.0 * tr * inv_N), two_mi = (R)(2.0 * ti * inv_N);
        r = 0.0;
        m = 0.0;
        for (unsigned int i = threadIdx.x; i < len; i += blockDim.x) {
            E v = s[i];
            v.x = two_mr - v.x;  // 2 mu - (O a)_i
            v.y = two_mi - v.y;
            s[i] = v;
            r += (double)v.x;
            m += (double)v.y;
        }
        if (it + 1 == k) break;
        __syncthreads();
        negate_marked(cr, ci);  // O of the next iteration: sum(O a') = sum(a') - 2 sum_marked(a')
        // (the negated entries are next read after grid_total's barriers)
        grid_total(r - 2.0 * cr, m - 2.0 * ci, (it + 1) & 1, tr, ti);
    }
    __syncthreads();
    for (unsigned int i = threadIdx.x; i < len; i += blockDim.x) a[lo + i] = s[i];
}

// Register-resident variant (round 2, the default where it fits: C <= NT x
// NPT).  Same iteration, held differently:
//   * thread tid keeps its NPT elements (block-local j * NT + tid) in
//     registers for the whole call -- an iteration touches no memory but one
//     partial per block (the shared-memory sweep above moved 226 KB of smem per
//     SM per iteration at c2, ~0.9 us);
//   * O is a per-thread sign mask built once (bit j: slot j is marked), so the
//     registers hold b = O a between iterations and one pass per iteration
//     computes a' = 2 mu - b, b' = O a' (a sign-bit flip) and the fp64 sums
//     of b' -- exactly sum(O a'), the next mu, with no separate marked pass;
//   * the block total is folded by warp 0 (a 5-level shuffle tree); the
//     per-iteration grid sums are exact fixed-point integer atomics (FX,
//     the default; see fx_total), the first rounds (and FX = false) publish
//     one 16-B fp64 partial, count in with ONE release-add on a monotonic
//     64-bit counter (zeroed before the launch; round r is complete at
//     (r + 1) x grid) and gather with all of a lane's partials in flight.
// Measured alternatives (tools/mean_resident_scan.py): flag-in-word
// all-gather polling, counter + flag-in-word partials, and a last-arriver
// broadcast into per-block lines were all slower (polling contention on L2).
// Partials alternate by round parity: a block writes round r + 2's partial
// only after round r + 1 completes, which every block reaches after gathering
// round r.
__device__ __forceinline__ void red_release_add_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr int kResRegMaxGrid = 160;  // blocks (one per SM; B200: 148)
__device__ __forceinline__ void red_relaxed_add_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Round-to-nearest-even of |x| < 2^51 to an integer with one fp64 add (the
// 1.5 * 2^52 magic number), and back: exact, no F2I / I2F.
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
__device__ __forceinline__ long long round_i64(double x, double &xd) {
    const double t = x + kMagic;
    xd = t - kMagic;  // the rounded value as a double (exact)
    return __double_as_longlong(t) - __double_as_longlong(kMagic);
}
__device__ __forceinline__ double i64_to_double(long long i) {  // |i| < 2^51
    return __longlong_as_double(i + __double_as_longlong(kMagic)) - kMagic;
}
constexpr int kAccWords = 64;  // uint64 per iteration slot of the fixed-point sums: 4 words, 128 B apart
__device__ __forceinline__ void ld_relaxed_v2_u64(const unsigned long long *p, unsigned long long &a,
                                                  unsigned long long &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
#ifndef SV_RESREG_TRACE
#define SV_RESREG_TRACE 0  // 1: clock64 phase sums per round, printed by 3 blocks (A/B builds only)
#endif

// x with its sign flipped when s (0 or 1) is set: a sign-bit XOR, exact.
__device__ __forceinline__ double flip_if(double x, unsigned int s) {
    return __hiloint2double(__double2hiint(x) ^ (int)(s << 31), __double2loint(x));
}
__device__ __forceinline__ float flip_if(float x, unsigned int s) {
    return __int_as_float(__float_as_int(x) ^ (int)(s << 31));
}

// FX: the per-iteration grid sums as exact fixed-point integer adds (see
// fx_total below); false: fp64 partials + gather for every round.
template <typename E, int NPT, int NT, bool FX>
__global__ void __launch_bounds__(NT, 1)
    mean_resreg_kernel(E *a, unsigned long long N, unsigned long long C, double inv_N,
                       const unsigned long long *marked, unsigned long long n_marked, int k, double2 *partials,
                       unsigned long long *ctr, unsigned long long *acc) {
    using R = decltype(E{}.x);
    __shared__ double red[66];
    __shared__ unsigned long long s_mlo, s_mcnt;
    __shared__ unsigned int s_mm[NT];  // per-thread marked-slot masks (built once)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned long long lo = (unsigned long long)blockIdx.x * C;
    const unsigned long long hi = lo + C < N ? lo + C : N;
    const unsigned int len = (unsigned int)(hi > lo ? hi - lo : 0);
    const unsigned int nb = gridDim.x;
    if (tid == 0) {  // this block's marked entries: marked[s_mlo .. s_mlo + s_mcnt)
        unsigned long long l = 0, h = n_marked;
        while (l < h) { const unsigned long long md = (l + h) >> 1; if (marked[md] < lo) l = md + 1; else h = md; }
        const unsigned long long first = l;
        h = n_marked;
        while (l < h) { const unsigned long long md = (l + h) >> 1; if (marked[md] < hi) l = md + 1; else h = md; }
        s_mlo = first;
        s_mcnt = l - first;
    }
    s_mm[tid] = 0u;
    __syncthreads();
    for (unsigned long long r = tid; r < s_mcnt; r += NT) {
        const unsigned int off = (unsigned int)(marked[s_mlo + r] - lo);
        atomicOr(&s_mm[off % NT], 1u << (off / NT));
    }
    __syncthreads();
    const unsigned int mmask = s_mm[tid];
    // slots j < nv hold elements (j * NT + tid < len); the rest are padding
    const int nv = len > (unsigned int)tid ? (int)((len - (unsigned int)tid + NT - 1) / NT) : 0;
    E v[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        if (j < nv) v[j] = __ldcg(a + lo + (unsigned int)j * NT + (unsigned int)tid);
        else { v[j].x = (R)0; v[j].y = (R)0; }
    }
#if SV_RESREG_TRACE
    long long tr_prev = clock64(), tr_sum[6] = {0, 0, 0, 0, 0, 0};
#endif
    // Grid total of the per-thread values: warp trees, warp 0 folds the warp
    // sums, publishes the block partial, waits for the round, then sums all
    // partials in block order (lane-strided + fixed tree): the same total in
    // every block.
    auto grid_total = [&](double r, double m, unsigned int round, double &tr, double &ti) {
#if SV_RESREG_TRACE
        const long long t_a = clock64();
        tr_sum[0] += t_a - tr_prev;  // compute since the last broadcast
#endif
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            r += __shfl_xor_sync(0xffffffffu, r, o);
            m += __shfl_xor_sync(0xffffffffu, m, o);
        }
        if (lane == 0) { red[2 * w] = r; red[2 * w + 1] = m; }
        __syncthreads();
#if SV_RESREG_TRACE
        const long long t_b = clock64();
        tr_sum[1] += t_b - t_a;  // warp trees + block barrier
#endif
        if (w == 0) {
            double R0 = lane < NT / 32 ? red[2 * lane] : 0.0, M0 = lane < NT / 32 ? red[2 * lane + 1] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                R0 += __shfl_xor_sync(0xffffffffu, R0, o);
                M0 += __shfl_xor_sync(0xffffffffu, M0, o);
            }
            double2 *part = partials + (size_t)(round & 1u) * nb;
            if (lane == 0) {
                part[blockIdx.x] = make_double2(R0, M0);
#if SV_RESREG_TRACE
                const long long t_0 = clock64();
#endif
                red_release_add_u64(ctr, 1ull);
#if SV_RESREG_TRACE
                const long long t_1 = clock64();
                tr_sum[3] += t_1 - t_0;  // fence + red issue
#endif
                const unsigned long long target = (unsigned long long)(round + 1u) * nb;
                while (ld_acquire_u64(ctr) < target) {
                }
#if SV_RESREG_TRACE
                tr_sum[4] += clock64() - t_1;  // wait until the round is complete
#endif
            }
            __syncwarp();
            // all of the lane's partials in flight at once (16-B loads, fixed order)
            constexpr int kPer = kResRegMaxGrid / 32;
            double2 q[kPer];
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const unsigned int b = (unsigned int)lane + 32u * i;
                q[i] = b < nb ? __ldcg(part + b) : make_double2(0.0, 0.0);
            }
            R0 = 0.0;
            M0 = 0.0;
#pragma unroll
            for (int i = 0; i < kPer; ++i) { R0 += q[i].x; M0 += q[i].y; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                R0 += __shfl_xor_sync(0xffffffffu, R0, o);
                M0 += __shfl_xor_sync(0xffffffffu, M0, o);
            }
            if (lane == 0) { red[64] = R0; red[65] = M0; }
        }
        __syncthreads();
        tr = red[64];
        ti = red[65];
#if SV_RESREG_TRACE
        tr_prev = clock64();
        tr_sum[2] += tr_prev - t_b;  // publish + wait + gather + broadcast
#endif
    };
    // b = O a and its sum (padding slots hold 0 and add nothing)
    double r = 0.0, m = 0.0;
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        const unsigned int sj = (mmask >> j) & 1u;
        v[j].x = flip_if(v[j].x, sj);
        v[j].y = flip_if(v[j].y, sj);
        r += (double)v[j].x;
        m += (double)v[j].y;
    }
    double tr, ti;
    unsigned int round = 0;
    grid_total(r, m, round++, tr, ti);
    // Fixed-point rounds (FX).  Every later sum is of b' = O a' over a subset
    // of the state, so |sum| <= sqrt(N) ||a|| (Cauchy-Schwarz; D and O are
    // unitary).  One more fp64 round gives ||a||^2; every block derives the
    // same scale 2^sh with 2 sqrt(N) ||a|| 2^sh < 2^51 and, per iteration,
    // adds its partial as two's-complement integers (a high word at 2^-sh and
    // a low word at 2^-(sh+44)), each with an arrival count in its low 8 bits
    // -- four relaxed 64-bit atomics into this iteration's own zeroed slot,
    // each word on its own 128-B line.  Integer adds commute, so the total is
    // the same bits in every block and run (deterministic, G14) and it is the
    // EXACT sum of the partials to 2^-(sh+44) ~ 1e-28 of sqrt(N) ||a||,
    // rounded to fp64 once (the fp64 gather rounds 148 times); count and data
    // share each word, so no fence and no gather: a block polls the four
    // words until every count reaches the grid size.
    int sh = 0;
    if constexpr (FX) {
        double q = 0.0;
#pragma unroll
        for (int j = 0; j < NPT; ++j)
            if (j < nv) q += (double)v[j].x * (double)v[j].x + (double)v[j].y * (double)v[j].y;
        double tq, tdummy;
        grid_total(q, 0.0, round++, tq, tdummy);
        int e = 0;
        frexp(2.0 * sqrt((double)N * tq) + 1e-300, &e);  // bound < 2^e
        sh = 51 - e;  // |partials|, |total| < 2^50: inside the magic-number rounding range
        sh = sh > 1000 ? 1000 : sh;
    }
    // invariant at the top of an iteration: v holds b = O a and (tr, ti) = sum(b)
    if constexpr (FX) {
        // Pipelined: sum(b') = sum_j s_j (2 mu - b_j) = 2 mu S - P with S = sum_j s_j
        // (s_j = -1 on marked slots, a block constant) and P = sum_j s_j b_j, which
        // is known BEFORE mu arrives -- so a block publishes its next partial the
        // moment it reads mu, and the element update plus the next P overlap the
        // round in flight.  (Exact algebra; the stored b' differ from the summed
        // values by their own rounding only.)
        // fold: warp trees -> smem -> warp 0 (valid in warp 0 only)
        auto fold = [&](double r, double m, double &R, double &M) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                r += __shfl_xor_sync(0xffffffffu, r, o);
                m += __shfl_xor_sync(0xffffffffu, m, o);
            }
            if (lane == 0) { red[2 * w] = r; red[2 * w + 1] = m; }
            __syncthreads();
            R = 0.0;
            M = 0.0;
            if (w == 0) {
                R = lane < NT / 32 ? red[2 * lane] : 0.0;
                M = lane < NT / 32 ? red[2 * lane + 1] : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    R += __shfl_xor_sync(0xffffffffu, R, o);
                    M += __shfl_xor_sync(0xffffffffu, M, o);
                }
            }
        };
        auto signed_sum = [&](double &pr, double &pi) {  // this thread's sum_j s_j v_j
            pr = 0.0;
            pi = 0.0;
#pragma unroll
            for (int j = 0; j < NPT; ++j)
                if (j < nv) {
                    const unsigned int sj = (mmask >> j) & 1u;
                    pr += (double)flip_if(v[j].x, sj);
                    pi += (double)flip_if(v[j].y, sj);
                }
        };
        double sc = 0.0;
#pragma unroll
        for (int j = 0; j < NPT; ++j)
            if (j < nv) sc += ((mmask >> j) & 1u) ? -1.0 : 1.0;
        const double up = ldexp(1.0, sh), dn = ldexp(1.0, -sh);  // exact powers of two (|sh| <= 1000)
        double S_blk, dummy, P_r, P_i, pr, pi;
        fold(sc, 0.0, S_blk, dummy);
        __syncthreads();  // red[] reused by the next fold
        signed_sum(pr, pi);
        fold(pr, pi, P_r, P_i);
#if SV_RESREG_TRACE
        long long tp[5] = {0, 0, 0, 0, 0}, tprev = clock64();
#endif
        for (int it = 0; it < k; ++it) {
            const R two_mr = (R)(2.0 * tr * inv_N), two_mi = (R)(2.0 * ti * inv_N);
            if (it + 1 == k) {  // the last a' = 2 mu - b is the result
#pragma unroll
                for (int j = 0; j < NPT; ++j) {
                    v[j].x = two_mr - v[j].x;
                    v[j].y = two_mi - v[j].y;
                }
                break;
            }
            unsigned long long *sl = acc + (size_t)kAccWords * (unsigned int)it;
#if SV_RESREG_TRACE
            long long tc = clock64();
            tp[0] += tc - tprev;  // barrier -> top
            tprev = tc;
#endif
            if (w == 0 && lane == 0) {
                // this block's sum of b' = O a', as the elements will hold it (2 mu in R)
                // (scalings by exact powers of two and magic-number roundings: ldexp and
                // F2I / I2F were ~800 cycles on this, the iteration's critical path)
                const double xr = ((double)two_mr * S_blk - P_r) * up, xi = ((double)two_mi * S_blk - P_i) * up;
                double hrd, hid;
                const long long hr = round_i64(xr, hrd), hi_ = round_i64(xi, hid);
                double unused;
                const long long lr = round_i64((xr - hrd) * 0x1p44, unused);
                const long long li = round_i64((xi - hid) * 0x1p44, unused);
                red_relaxed_add_u64(sl, ((unsigned long long)hr << 8) + 1ull);
                red_relaxed_add_u64(sl + 16, ((unsigned long long)hi_ << 8) + 1ull);
                red_relaxed_add_u64(sl + 32, ((unsigned long long)lr << 8) + 1ull);
                red_relaxed_add_u64(sl + 48, ((unsigned long long)li << 8) + 1ull);
            }
#if SV_RESREG_TRACE
            tc = clock64();
            tp[1] += tc - tprev;  // publish
            tprev = tc;
#endif
            // b' = O a',  a' = 2 mu - b; the next P = sum_j s_j b'_j = sum_j a'_j
            pr = 0.0;
            pi = 0.0;
#pragma unroll
            for (int j = 0; j < NPT; ++j) {
                const unsigned int sj = (mmask >> j) & 1u;
                const R ar = two_mr - v[j].x, ai = two_mi - v[j].y;
                if (j < nv) {
                    pr += (double)ar;
                    pi += (double)ai;
                }
                v[j].x = flip_if(ar, sj);
                v[j].y = flip_if(ai, sj);
            }
#if SV_RESREG_TRACE
            tc = clock64();
            tp[2] += tc - tprev;  // update
            tprev = tc;
#endif
            fold(pr, pi, P_r, P_i);  // P of the new b, for the next publication
#if SV_RESREG_TRACE
            tc = clock64();
            tp[3] += tc - tprev;  // fold
            tprev = tc;
#endif
            if (w == 0 && lane == 0) {
                unsigned long long w0, w1, w2, w3;
                do {
                    w0 = ld_relaxed_u64(sl);
                    w1 = ld_relaxed_u64(sl + 16);
                    w2 = ld_relaxed_u64(sl + 32);
                    w3 = ld_relaxed_u64(sl + 48);
                } while ((w0 & 0xffull) != nb || (w1 & 0xffull) != nb || (w2 & 0xffull) != nb ||
                         (w3 & 0xffull) != nb);
                // wrapped intermediate sums are harmless: the final integer fits
                red[64] = (i64_to_double((long long)w0 >> 8) + i64_to_double((long long)w2 >> 8) * 0x1p-44) * dn;
                red[65] = (i64_to_double((long long)w1 >> 8) + i64_to_double((long long)w3 >> 8) * 0x1p-44) * dn;
            }
            __syncthreads();
            tr = red[64];
            ti = red[65];
#if SV_RESREG_TRACE
            tc = clock64();
            tp[4] += tc - tprev;  // wait + barrier
            tprev = tc;
#endif
        }
#if SV_RESREG_TRACE
        if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == nb / 2 || blockIdx.x + 1 == nb))
            printf("resreg FX trace block %u iters %d: cycles/iter top %.0f publish %.0f update %.0f fold %.0f wait %.0f\n",
                   blockIdx.x, k - 1, (double)tp[0] / (k - 1), (double)tp[1] / (k - 1), (double)tp[2] / (k - 1),
                   (double)tp[3] / (k - 1), (double)tp[4] / (k - 1));
#endif
    } else {
        for (int it = 0; it < k; ++it) {
            const R two_mr = (R)(2.0 * tr * inv_N), two_mi = (R)(2.0 * ti * inv_N);
            if (it + 1 == k) {  // the last a' = 2 mu - b is the result
#pragma unroll
                for (int j = 0; j < NPT; ++j) {
                    v[j].x = two_mr - v[j].x;
                    v[j].y = two_mi - v[j].y;
                }
                break;
            }
            r = 0.0;
            m = 0.0;
#pragma unroll
            for (int j = 0; j < NPT; ++j) {
                const unsigned int sj = (mmask >> j) & 1u;
                v[j].x = flip_if(two_mr - v[j].x, sj);  // b' = O a',  a' = 2 mu - b
                v[j].y = flip_if(two_mi - v[j].y, sj);
                if (j < nv) {
                    r += (double)v[j].x;
                    m += (double)v[j].y;
                }
            }
            grid_total(r, m, round++, tr, ti);
        }
    }
#pragma unroll
    for (int j = 0; j < NPT; ++j)
        if (j < nv) a[lo + (unsigned int)j * NT + (unsigned int)tid] = v[j];
#if SV_RESREG_TRACE
    if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == nb / 2 || blockIdx.x + 1 == nb))
        printf("resreg trace block %u rounds %u: cycles/round compute %.0f reduce %.0f grid %.0f (fence+red %.0f "
               "wait %.0f)\n", blockIdx.x, round, (double)tr_sum[0] / round, (double)tr_sum[1] / round,
               (double)tr_sum[2] / round, (double)tr_sum[3] / round, (double)tr_sum[4] / round);
#endif
}

// Launch geometry: one wave of co-resident blocks, each holding C elements
// in shared memory; grid = 0 if the state does not fit.
static void resident_geometry(sv_dtype dt, uint64_t N, int &grid, uint64_t &C, int &smem, void *&fn) {
    int dev = 0, sms = 0, smem_max = 0;
    SV_CUDA(cudaGetDevice(&dev));
    SV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SV_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const size_t eb = elem_bytes(dt);
    const size_t budget = (size_t)smem_max - 1024;  // static shared + slack
    fn = dt == SV_C64 ? (void *)mean_resident_kernel<float2> : (void *)mean_resident_kernel<double2>;
    C = (N + sms - 1) / sms;
    grid = 0;
    smem = 0;
    if (C * eb > budget) return;
    smem = (int)(C * eb);
    SV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per = 0;
    SV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kResThreads, smem));
    const int g = (int)((N + C - 1) / C);
    if (per >= 1 && g <= per * sms) grid = g;
}

bool mean_resident_fits(sv_dtype dt, uint64_t N, size_t partials_cap) {
    int grid, smem;
    uint64_t C;
    void *fn;
    resident_geometry(dt, N, grid, C, smem, fn);
    return grid > 0 && (size_t)4 * grid <= partials_cap;
}

size_t mean_resident_slot_bytes(sv_dtype dt, uint64_t N) {
    int grid, smem;
    uint64_t C;
    void *fn;
    resident_geometry(dt, N, grid, C, smem, fn);
    return (size_t)2 * (size_t)(grid > 0 ? grid : 0) * sizeof(ResSlot);
}

// Register-resident configurations (threads NT, elements per thread NPT),
// the first with NT x NPT >= C is used.  Registers per thread are capped at
// 65536 / NT (ptxas -v: no spills in any of them).
struct ResRegCfg {
    int nt, npt;
    void *fn[2];  // [FX]
};
static const ResRegCfg *resreg_cfg(sv_dtype dt, uint64_t C) {
    static const ResRegCfg t64[] = {{512, 1, {(void *)mean_resreg_kernel<float2, 1, 512, false>, (void *)mean_resreg_kernel<float2, 1, 512, true>}},
                                    {512, 2, {(void *)mean_resreg_kernel<float2, 2, 512, false>, (void *)mean_resreg_kernel<float2, 2, 512, true>}},
                                    {512, 4, {(void *)mean_resreg_kernel<float2, 4, 512, false>, (void *)mean_resreg_kernel<float2, 4, 512, true>}},
                                    {512, 8, {(void *)mean_resreg_kernel<float2, 8, 512, false>, (void *)mean_resreg_kernel<float2, 8, 512, true>}},
                                    {512, 16, {(void *)mean_resreg_kernel<float2, 16, 512, false>, (void *)mean_resreg_kernel<float2, 16, 512, true>}},
                                    {512, 32, {(void *)mean_resreg_kernel<float2, 32, 512, false>, (void *)mean_resreg_kernel<float2, 32, 512, true>}}};
    static const ResRegCfg t128[] = {{512, 1, {(void *)mean_resreg_kernel<double2, 1, 512, false>, (void *)mean_resreg_kernel<double2, 1, 512, true>}},
                                     {512, 2, {(void *)mean_resreg_kernel<double2, 2, 512, false>, (void *)mean_resreg_kernel<double2, 2, 512, true>}},
                                     {512, 4, {(void *)mean_resreg_kernel<double2, 4, 512, false>, (void *)mean_resreg_kernel<double2, 4, 512, true>}},
                                     {512, 8, {(void *)mean_resreg_kernel<double2, 8, 512, false>, (void *)mean_resreg_kernel<double2, 8, 512, true>}},
                                     {512, 16, {(void *)mean_resreg_kernel<double2, 16, 512, false>, (void *)mean_resreg_kernel<double2, 16, 512, true>}}};
    const ResRegCfg *t = dt == SV_C64 ? t64 : t128;
    for (int i = 0; i < (dt == SV_C64 ? 6 : 5); ++i)
        if ((uint64_t)t[i].nt * t[i].npt >= C) return &t[i];
    return nullptr;
}

void launch_mean_resident(sv_dtype dt, void *a, uint64_t N, double inv_N, const uint64_t *marked, uint64_t m, int k,
                          double *partials, unsigned int *bar, void *slots, unsigned long long epoch0, bool regs,
                          void *acc, cudaStream_t s) {
    int grid, smem;
    uint64_t C;
    void *fn;
    resident_geometry(dt, N, grid, C, smem, fn);
    SV_CHECK(grid > 0 && k >= 1, SV_EINVAL, "internal: resident mean launch without a fitting geometry");
    unsigned long long Nl = N, Cl = C, ml = m;
    const unsigned long long *mk = reinterpret_cast<const unsigned long long *>(marked);
    const ResRegCfg *rc = regs ? resreg_cfg(dt, C) : nullptr;
    if (rc != nullptr) {
        int per = 0, dev = 0, sms = 0;
        static const int fx_env = [] {  // SV_RESREG_FX=0: fp64 partials + gather every round (A/B)
            const char *e = getenv("SV_RESREG_FX");
            return e ? atoi(e) : 1;
        }();
        const bool fx = fx_env != 0 && acc != nullptr;
        void *rfn = rc->fn[fx ? 1 : 0];
        SV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rfn, rc->nt, 0));
        SV_CUDA(cudaGetDevice(&dev));
        SV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (per >= 1 && grid <= per * sms && grid <= kResRegMaxGrid) {
            // the monotonic 64-bit arrival counter lives after the {count, generation} pair
            unsigned long long *ctr = reinterpret_cast<unsigned long long *>(bar + 2);
            SV_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s));
            double2 *part2 = reinterpret_cast<double2 *>(partials);
            unsigned long long *acc64 = reinterpret_cast<unsigned long long *>(acc);
            if (fx) SV_CUDA(cudaMemsetAsync(acc64, 0, kAccWords * sizeof(unsigned long long) * (size_t)k, s));
            void *args[] = {&a, &Nl, &Cl, &inv_N, &mk, &ml, &k, &part2, &ctr, &acc64};
            SV_CUDA(cudaLaunchCooperativeKernel(rfn, dim3(grid), dim3(rc->nt), args, 0, s));
            return;
        }
    }
    ResSlot *sl = reinterpret_cast<ResSlot *>(slots);
    void *args[] = {&a, &Nl, &Cl, &inv_N, &mk, &ml, &k, &partials, &bar, &sl, &epoch0};
    SV_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kResThreads), args, (size_t)smem, s));
}

}  // namespace sv
