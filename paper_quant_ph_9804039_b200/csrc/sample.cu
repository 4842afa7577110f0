// sample.cu -- seeded whole-register measurement on the device (SURVEY 8(f)
// NEXT-3).  "This measurement operation forces the state to one of the two
// values" with "the probability of each state ... the square of this complex
// amplitude".  Reading G21: shot s draws u_s from a counter hash
// and returns the smallest index whose inclusive cumulative probability
// exceeds u_s times the total.
//
// Device plan (five launches, fp64, fixed order => deterministic):
//   1. chunk_sum_kernel: one warp per 4096-amplitude chunk, 32 rows of 128
//      amplitudes; lane l of a row owns its 4 consecutive amplitudes 4l..4l+3
//      and sums them in order, the row sum is a fixed xor-butterfly over the
//      lanes, rows are accumulated in row order (HBM-bound read of the state,
//      32-64 contiguous bytes per lane); it also stores each row's
//      chunk-local exclusive running sum (32 doubles per chunk);
//   2. scan_partial / scan_offsets / scan_apply: exclusive prefix of the
//      chunk sums in a fixed order (segments of 8192 sums per block);
//   3. sample_kernel: one warp per shot, binary search over the chunk
//      prefixes, the row from the chunk's 32 row starts (prefix + row
//      running sum, one ballot), then rows from there in kernel 1's order
//      until the running sum passes the target; the crossing lane comes from
//      an inclusive warp scan of the lane sums, the amplitude from that
//      lane's 4 in order.
#include <cuda_runtime.h>

#include "sv_internal.h"

namespace sv {

constexpr int kSampChunk = 4096;        // amplitudes per chunk
#ifndef SV_SAMP_PER_LANE
#define SV_SAMP_PER_LANE 4
#endif
constexpr int kPerLane = SV_SAMP_PER_LANE;  // consecutive amplitudes per lane per row
constexpr int kRowLen = 32 * kPerLane;  // 128 amplitudes per row
constexpr int kRows = kSampChunk / kRowLen;
inline uint64_t sample_chunks_impl(uint64_t N) { return (N + kSampChunk - 1) / kSampChunk; }
#ifndef SV_SAMP_BATCH
#define SV_SAMP_BATCH 8  // rows per batch of loads in the chunk-sum sweep
#endif

__device__ __forceinline__ uint64_t smix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename E>
__device__ __forceinline__ double prob(const E *a, uint64_t i, uint64_t N) {
    if (i >= N) return 0.0;
    const E v = a[i];
    const double re = (double)v.x, im = (double)v.y;
    return __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
}

__device__ __forceinline__ double warp_xor_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// The lane's 4 probabilities of row r (fixed order), and their sum.
template <typename E>
__device__ __forceinline__ double lane_probs(const E *a, uint64_t i0, uint64_t N, double (&p)[kPerLane]) {
#pragma unroll
    for (int e = 0; e < kPerLane; ++e) p[e] = prob(a, i0 + e, N);
    double q = p[0];
#pragma unroll
    for (int e = 1; e < kPerLane; ++e) q = __dadd_rn(q, p[e]);
    return q;
}

// The same for a row lying entirely below N: vector loads, no guards.
__device__ __forceinline__ double lane_probs_full(const float2 *a, uint64_t i0, double (&p)[kPerLane]) {
#pragma unroll
    for (int h = 0; h < kPerLane / 2; ++h) {
        const float4 v = __ldcg(reinterpret_cast<const float4 *>(a + i0) + h);
        const double r0 = (double)v.x, i0d = (double)v.y, r1 = (double)v.z, i1 = (double)v.w;
        p[2 * h] = __dadd_rn(__dmul_rn(r0, r0), __dmul_rn(i0d, i0d));
        p[2 * h + 1] = __dadd_rn(__dmul_rn(r1, r1), __dmul_rn(i1, i1));
    }
    double q = p[0];
#pragma unroll
    for (int e = 1; e < kPerLane; ++e) q = __dadd_rn(q, p[e]);
    return q;
}
__device__ __forceinline__ double lane_probs_full(const double2 *a, uint64_t i0, double (&p)[kPerLane]) {
#pragma unroll
    for (int e = 0; e < kPerLane; ++e) {
        const double2 v = __ldcg(a + i0 + e);
        p[e] = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
    }
    double q = p[0];
#pragma unroll
    for (int e = 1; e < kPerLane; ++e) q = __dadd_rn(q, p[e]);
    return q;
}

template <typename E>
__global__ void __launch_bounds__(256) chunk_sum_kernel(const E *a, uint64_t N, double *sums, double *rowp,
                                                        uint64_t nchunks) {
    const int lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x / 32;
    static_assert(kRows == 32, "one row prefix per lane");
    for (uint64_t c = blockIdx.x * wpb + threadIdx.x / 32; c < nchunks; c += (uint64_t)gridDim.x * wpb) {
        double acc = 0.0, mine = 0.0;  // lane r: the chunk-local running sum before row r
        const uint64_t base = c * kSampChunk;
        if (base + kSampChunk <= N) {  // warp-uniform: the whole chunk is below N
            for (int r0 = 0; r0 < kRows; r0 += SV_SAMP_BATCH) {
                double q[SV_SAMP_BATCH];  // a batch of rows' loads in flight, then the same row order
#pragma unroll
                for (int r = 0; r < SV_SAMP_BATCH; ++r) {
                    double p[kPerLane];
                    q[r] = lane_probs_full(a, base + (r0 + r) * kRowLen + kPerLane * lane, p);
                }
#pragma unroll
                for (int r = 0; r < SV_SAMP_BATCH; ++r) {
                    if (lane == r0 + r) mine = acc;
                    acc = __dadd_rn(acc, warp_xor_sum(q[r]));
                }
            }
        } else {
            for (int r = 0; r < kRows; ++r) {
                double p[kPerLane];
                if (lane == r) mine = acc;
                acc = __dadd_rn(acc, warp_xor_sum(lane_probs(a, base + r * kRowLen + kPerLane * lane, N, p)));
            }
        }
        if (lane == 0) sums[c] = acc;
        rowp[c * kRows + lane] = mine;
    }
}

// In place: sums -> exclusive prefix; total -> *total (fixed order, three
// launches; round 1's single-block sequential scan of the 2^20 chunk sums of
// an n = 32 state took ~1.8 ms, a quarter of the prefix phase).  Segments of
// kScanSeg consecutive chunk sums, one 256-thread block each: thread t sums
// its kScanPer consecutive values in order; the thread totals are scanned in
// a fixed order (warp Hillis-Steele by shuffles, warp totals in order); the
// segment totals are scanned sequentially by one thread; the apply pass
// recomputes the same thread sums and writes every exclusive prefix.
constexpr int kScanPer = 32;
constexpr int kScanThreads = 256;
constexpr uint64_t kScanSeg = (uint64_t)kScanPer * kScanThreads;  // 8192 chunk sums per segment

uint64_t sample_scan_blocks(uint64_t N) { return (sample_chunks_impl(N) + kScanSeg - 1) / kScanSeg; }

// The thread's kScanPer values in order (0 beyond n).
__device__ __forceinline__ double scan_thread_sum(const double *sums, uint64_t lo, uint64_t n) {
    double s = 0.0;
    if (lo + kScanPer <= n) {
#pragma unroll
        for (int h = 0; h < kScanPer / 2; ++h) {
            const double2 v = __ldcg(reinterpret_cast<const double2 *>(sums + lo) + h);
            s = __dadd_rn(s, v.x);
            s = __dadd_rn(s, v.y);
        }
    } else {
        for (uint64_t i = lo; i < n; ++i) s = __dadd_rn(s, sums[i]);
    }
    return s;
}

// Exclusive prefix of v over the block's threads (fixed order) and the block total.
__device__ __forceinline__ double scan_block_exclusive(double v, double &total) {
    __shared__ double s_w[kScanThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = __dadd_rn(inc, u);
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    double woff = 0.0, tot = 0.0;
#pragma unroll
    for (int i = 0; i < kScanThreads / 32; ++i) {
        if (i == w) woff = tot;
        tot = __dadd_rn(tot, s_w[i]);
    }
    total = tot;
    double exc = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) exc = 0.0;
    return __dadd_rn(woff, exc);
}

__global__ void __launch_bounds__(kScanThreads) scan_partial_kernel(const double *sums, uint64_t n, double *bsum) {
    const uint64_t lo = blockIdx.x * kScanSeg + (uint64_t)threadIdx.x * kScanPer;
    double total;
    (void)scan_block_exclusive(scan_thread_sum(sums, lo, n), total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

// One thread: the segment totals -> exclusive offsets (in order), total.
__global__ void scan_offsets_kernel(double *bsum, uint64_t nb, double *total) {
    double run = 0.0;
    for (uint64_t b = 0; b < nb; ++b) {
        const double v = bsum[b];
        bsum[b] = run;
        run = __dadd_rn(run, v);
    }
    *total = run;
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(double *sums, uint64_t n, const double *boff) {
    const uint64_t lo = blockIdx.x * kScanSeg + (uint64_t)threadIdx.x * kScanPer;
    double total;
    const double exc = scan_block_exclusive(scan_thread_sum(sums, lo, n), total);
    double run = __dadd_rn(boff[blockIdx.x], exc);  // (each thread rewrites only the values it read)
    const uint64_t hi = lo + kScanPer < n ? lo + kScanPer : n;
    for (uint64_t i = lo; i < hi; ++i) {
        const double v = sums[i];
        sums[i] = run;
        run = __dadd_rn(run, v);
    }
}

// g = {global total, this rank's cumulative offset off_r, the next rank's
// off_{r+1}}: every rank computes the same running sums in the same order, so
// the windows [off_r, off_{r+1}) partition [0, total) exactly and each shot
// u * total is claimed by exactly one rank (the last rank also takes any
// target at or above its offset).  Unclaimed shots are written as 0 (the host
// then sums the lists over ranks).
__global__ void rank_window_kernel(const double *totals, int world, int rank, double *g) {
    double all = 0.0, off = 0.0, next = 0.0;
    for (int r = 0; r < world; ++r) {
        if (r == rank) off = all;
        all = __dadd_rn(all, totals[r]);
        if (r == rank) next = all;
    }
    g[0] = all;
    g[1] = off;
    g[2] = next;
}

template <typename E>
__global__ void __launch_bounds__(256) sample_kernel(const E *a, uint64_t N, const double *prefix, const double *rowp,
                                                     uint64_t nchunks,
                                                     const double *g, uint64_t key, uint64_t shots,
                                                     uint64_t index_base, int last_rank, uint64_t *out) {
    const int lane = threadIdx.x & 31;
    const uint64_t wpb = blockDim.x / 32;
    for (uint64_t s = blockIdx.x * wpb + threadIdx.x / 32; s < shots; s += (uint64_t)gridDim.x * wpb) {
        const double u = ((double)(smix64((key ^ s) + 0x9E3779B97F4A7C15ull) >> 11) + 0.5) * 0x1.0p-53;
        const double gt = __dmul_rn(u, g[0]);  // the shot's target on the global CDF
        if (gt < g[1] || (!last_rank && gt >= g[2])) {
            if (lane == 0) out[s] = 0;  // another rank's shot
            continue;
        }
        const double target = __dsub_rn(gt, g[1]);
        // last chunk whose exclusive prefix is <= target
        uint64_t lo = 0, hi = nchunks - 1;
        while (lo < hi) {
            const uint64_t md = (lo + hi + 1) >> 1;
            if (prefix[md] <= target) lo = md; else hi = md - 1;
        }
        const uint64_t base = lo * kSampChunk;
        // the row: the last whose start prefix[lo] + rowp[row] is <= target
        // (starts are nondecreasing; one 256-B load per shot instead of
        // walking the chunk's rows from the first)
        const double start = __dadd_rn(prefix[lo], __ldcg(rowp + lo * kRows + lane));
        const unsigned le = __ballot_sync(0xffffffffu, start <= target);
        const int r_first = le ? 31 - __clz(le) : 0;
        double run = __shfl_sync(0xffffffffu, start, r_first);
        uint64_t pick = (base + kSampChunk <= N ? base + kSampChunk : N) - 1;
        uint64_t last_nz = base + (uint64_t)r_first * kRowLen;
        for (int r = r_first; r < kRows; ++r) {
            const uint64_t i0 = base + r * kRowLen + kPerLane * lane;
            double p[kPerLane];
            const double q = base + kSampChunk <= N ? lane_probs_full(a, i0, p) : lane_probs(a, i0, N, p);
            const double row = warp_xor_sum(q);
            int lz = -1;  // the lane's last nonzero amplitude
#pragma unroll
            for (int e = 0; e < kPerLane; ++e)
                if (p[e] > 0.0) lz = e;
            const unsigned nzm = __ballot_sync(0xffffffffu, lz >= 0);
            if (nzm) {
                const int ll = 31 - __clz(nzm);
                const int lze = __shfl_sync(0xffffffffu, lz, ll);
                last_nz = base + r * kRowLen + kPerLane * ll + lze;
            }
            if (__dadd_rn(run, row) > target) {
                double inc = q;  // inclusive scan of the lane sums (fixed order)
                for (int o = 1; o < 32; o <<= 1) {
                    const double v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc = __dadd_rn(inc, v);
                }
                double exc = __shfl_up_sync(0xffffffffu, inc, 1);
                if (lane == 0) exc = 0.0;
                const unsigned m = __ballot_sync(0xffffffffu, __dadd_rn(run, inc) > target && q > 0.0);
                if (!m) {
                    pick = last_nz;
                    break;
                }
                const int L = __ffs(m) - 1;
                // that lane's amplitudes in order from its exclusive prefix
                int e_pick = -1;
                if (lane == L) {
                    double cum = __dadd_rn(run, exc);
                    for (int e = 0; e < kPerLane; ++e) {
                        cum = __dadd_rn(cum, p[e]);
                        if (cum > target && p[e] > 0.0) { e_pick = e; break; }
                    }
                    if (e_pick < 0) e_pick = lz;  // rounding: the lane's own last nonzero
                }
                e_pick = __shfl_sync(0xffffffffu, e_pick, L);
                pick = base + r * kRowLen + kPerLane * L + e_pick;
                break;
            }
            run = __dadd_rn(run, row);
            if (r == kRows - 1) pick = last_nz;  // rounding: target sits on the chunk's upper edge
        }
        if (lane == 0) out[s] = index_base + pick;
    }
}

uint64_t sample_chunks(uint64_t N) { return sample_chunks_impl(N); }

void launch_sample_prefix(sv_dtype dt, const void *a, uint64_t N, double *scratch, double *rank_total,
                          double *bscratch, double *rowp, cudaStream_t s) {
    const uint64_t nch = sample_chunks(N);
    const unsigned g1 = (unsigned)((nch + 7) / 8 < 148 * 64 ? (nch + 7) / 8 : 148 * 64);
    if (dt == SV_C64) chunk_sum_kernel<float2><<<g1, 256, 0, s>>>((const float2 *)a, N, scratch, rowp, nch);
    else chunk_sum_kernel<double2><<<g1, 256, 0, s>>>((const double2 *)a, N, scratch, rowp, nch);
    SV_CUDA(cudaGetLastError());
    const uint64_t nb = (nch + kScanSeg - 1) / kScanSeg;
    SV_CHECK(nb <= 0x7fffffffull, SV_EINVAL, "internal: too many scan segments");
    scan_partial_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(scratch, nch, bscratch);
    SV_CUDA(cudaGetLastError());
    scan_offsets_kernel<<<1, 1, 0, s>>>(bscratch, nb, rank_total);
    SV_CUDA(cudaGetLastError());
    scan_apply_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(scratch, nch, bscratch);
    SV_CUDA(cudaGetLastError());
}

void launch_sample_draw(sv_dtype dt, const void *a, uint64_t N, const double *scratch, const double *rowp,
                        const double *totals,
                        int world, int rank, double *g, uint64_t key, uint64_t shots, uint64_t index_base,
                        uint64_t *out, cudaStream_t s) {
    rank_window_kernel<<<1, 1, 0, s>>>(totals, world, rank, g);
    SV_CUDA(cudaGetLastError());
    if (shots == 0) return;
    const uint64_t nch = sample_chunks(N);
    const unsigned g3 = (unsigned)((shots + 7) / 8 < 148 * 64 ? (shots + 7) / 8 : 148 * 64);
    const int last = rank == world - 1 ? 1 : 0;
    if (dt == SV_C64)
        sample_kernel<float2><<<g3, 256, 0, s>>>((const float2 *)a, N, scratch, rowp, nch, g, key, shots, index_base, last,
                                                 out);
    else
        sample_kernel<double2><<<g3, 256, 0, s>>>((const double2 *)a, N, scratch, rowp, nch, g, key, shots, index_base,
                                                  last, out);
    SV_CUDA(cudaGetLastError());
}

}  // namespace sv
