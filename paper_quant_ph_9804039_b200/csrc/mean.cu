// mean.cu -- fused oracle flip + inversion about the mean (sm_100a).
//
// One Grover iteration with the mean diffusion (north star; D = 2|s><s| - I
// acts as a_i <- 2 mean(a) - a_i):
//     b_i  = (O a)_i        (negate marked entries, G3)
//     a_i' = 2 mu - b_i,    mu = (1/N) sum_i b_i
// The global sum is the paper's "accumulate and redistribute a sum from all
// the processors after every laser operation ... two messages" (Eq. 3,
// P:5248-5251).  Here the sum needed by iteration t+1, sum_i (O a')_i, is
// accumulated while iteration t writes a' -- one HBM read + one write per
// iteration.  Per-thread fp64 accumulation, warp shuffle -> block -> per-block
// partials -> the last block to finish sums the partials in a fixed order
// (deterministic: no floating-point atomics, G14).
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "reduce.cuh"
#include "sv_internal.h"

namespace sv {

#ifndef SV_MEAN_PER
#define SV_MEAN_PER 8
#endif
#ifndef SV_MEAN_PIPE
#define SV_MEAN_PIPE 1
#endif
#ifndef SV_MEAN_THREADS
#define SV_MEAN_THREADS 256
#endif
constexpr int kMeanThreads = SV_MEAN_THREADS;
constexpr int kMeanPer = SV_MEAN_PER;                          // 16-byte vectors per thread per chunk
constexpr unsigned long long kChunkVec = kMeanThreads * kMeanPer;  // 2048 vectors = 32 KiB

template <typename E> struct Vec;                 // one 16-byte vector
template <> struct Vec<float2> { using T = float4; static constexpr int VE = 2; };
template <> struct Vec<double2> { using T = double2; static constexpr int VE = 1; };

__device__ __forceinline__ bool is_marked(unsigned long long i, const unsigned long long *mk, unsigned long long n) {
    unsigned long long lo = 0, hi = n;
    while (lo < hi) {  // binary search in the sorted marked list
        unsigned long long md = (lo + hi) >> 1;
        unsigned long long v = mk[md];
        if (v == i) return true;
        if (v < i) lo = md + 1; else hi = md;
    }
    return false;
}

// The state is swept in 32 KiB chunks; block b takes chunks b, b + grid, ...
// so the whole GPU streams through one compact address window at a time
// (an earlier one-contiguous-range-per-block version lost 30 % at n = 34 to
// ~1200 concurrent far-apart streams).  A per-chunk bitmap (host-built)
// says whether a chunk holds a marked index; only those chunks look entries
// up.  Fixed grid + fixed chunk order => deterministic sums (G14).
template <typename E, bool WRITE>
__global__ void __launch_bounds__(kMeanThreads) mean_kernel(MeanArgs a) {
    using V = typename Vec<E>::T;
    using R = decltype(E{}.x);
    constexpr int VE = Vec<E>::VE;
    __shared__ double red[2 * (kMeanThreads / 32)];
    const unsigned long long nvec = a.N / VE;
    const unsigned long long nchunks = (nvec + kChunkVec - 1) / kChunkVec;
    const auto *mk = reinterpret_cast<const unsigned long long *>(a.marked);

    R two_mr = 0, two_mi = 0;
    if (WRITE) {
        const double mr = a.sum_in[0] * a.inv_total, mi = a.sum_in[1] * a.inv_total;
        two_mr = (R)(2.0 * mr);
        two_mi = (R)(2.0 * mi);
    }
    V *p = reinterpret_cast<V *>(a.a);
    double sr = 0.0, si = 0.0;
#if SV_MEAN_PIPE
    // software pipeline: the next chunk's loads are issued before this
    // chunk's stores (program order; the chunks are disjoint)
    V nxt[kMeanPer];
    if (blockIdx.x < nchunks) {
        const unsigned long long w0 = blockIdx.x * kChunkVec + threadIdx.x;
#pragma unroll
        for (int u = 0; u < kMeanPer; ++u) {
            const unsigned long long v = w0 + (unsigned long long)u * kMeanThreads;
            if (v < nvec) nxt[u] = __ldcg(p + v);
        }
    }
#endif
    for (unsigned long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const unsigned long long v0 = c * kChunkVec + threadIdx.x;
        V buf[kMeanPer];
#if SV_MEAN_PIPE
#pragma unroll
        for (int u = 0; u < kMeanPer; ++u) buf[u] = nxt[u];
        if (c + gridDim.x < nchunks) {
            const unsigned long long w0 = (c + gridDim.x) * kChunkVec + threadIdx.x;
#pragma unroll
            for (int u = 0; u < kMeanPer; ++u) {
                const unsigned long long v = w0 + (unsigned long long)u * kMeanThreads;
                if (v < nvec) nxt[u] = __ldcg(p + v);
            }
        }
#else
#pragma unroll
        for (int u = 0; u < kMeanPer; ++u) {
            const unsigned long long v = v0 + (unsigned long long)u * kMeanThreads;
            if (v < nvec) buf[u] = __ldcg(p + v);
        }
#endif
        const bool any = a.n_marked != 0 && ((__ldg(&a.chunkmap[c >> 5]) >> (c & 31)) & 1u);
#pragma unroll
        for (int u = 0; u < kMeanPer; ++u) {
            const unsigned long long v = v0 + (unsigned long long)u * kMeanThreads;
            if (v >= nvec) continue;
            E e[VE];
            if constexpr (VE == 2) {
                e[0].x = buf[u].x; e[0].y = buf[u].y;
                e[1].x = buf[u].z; e[1].y = buf[u].w;
            } else {
                e[0].x = buf[u].x; e[0].y = buf[u].y;
            }
#pragma unroll
            for (int q = 0; q < VE; ++q) {
                const bool m = any && is_marked(v * VE + q, mk, a.n_marked);
                if (m) { e[q].x = -e[q].x; e[q].y = -e[q].y; }   // O
                if (WRITE) {
                    e[q].x = two_mr - e[q].x;                       // 2 mu - (O a)_i
                    e[q].y = two_mi - e[q].y;
                    // contribution of (O a')_i to the next iteration's sum
                    sr += m ? -(double)e[q].x : (double)e[q].x;
                    si += m ? -(double)e[q].y : (double)e[q].y;
                } else {
                    sr += (double)e[q].x;
                    si += (double)e[q].y;
                }
            }
            if (WRITE) {
                if constexpr (VE == 2) {
                    buf[u].x = e[0].x; buf[u].y = e[0].y; buf[u].z = e[1].x; buf[u].w = e[1].y;
                } else {
                    buf[u].x = e[0].x; buf[u].y = e[0].y;
                }
                p[v] = buf[u];
            }
        }
    }
    block_sum2(sr, si, red);
    finalize(sr, si, a.partials, a.counter, a.sum_out, red);
}

// ------------------------------------------------------------------------- //
// Tile-per-CTA form (round 2, default): one CTA = one 64 KiB tile, 16 x
// 128-bit loads per thread issued at once, 2 CTAs per SM -- the access shape of
// the contiguous WHT tile pass, which streams the same 2 S bytes ~15 % faster
// than the persistent chunk sweep above (n = 34: 39.4 vs 46.3 ms).  Each CTA
// writes its fp64 (re, im) partial to tilepart[tile]; sum_pairs_kernel then
// sums the tile partials in tile order (contiguous segments per block, the
// last block sums the segments in block order): fixed order, deterministic.
// ------------------------------------------------------------------------- //
constexpr int kTilePer = 16;
constexpr int grid_cap_pairs = 4096;  // the partials capacity (sv_api.cu kMaxGrid)                                           // 16-byte vectors per thread
constexpr unsigned long long kTileVec = (unsigned long long)kMeanThreads * kTilePer;  // 64 KiB

bool mean_tile_mode() {
    static const bool on = [] {
        const char *e = getenv("SV_MEAN_TILE");
        return !(e && strcmp(e, "0") == 0);
    }();
    return on;
}

template <typename E, bool WRITE>
__global__ void __launch_bounds__(kMeanThreads, 2) mean_tile_kernel(MeanArgs a) {
    using V = typename Vec<E>::T;
    using R = decltype(E{}.x);
    constexpr int VE = Vec<E>::VE;
    __shared__ double red[2 * (kMeanThreads / 32)];
    const unsigned long long nvec = a.N / VE;
    const unsigned long long t = blockIdx.x;
    const unsigned long long v0 = t * kTileVec + threadIdx.x;
    V *p = reinterpret_cast<V *>(a.a);
    V buf[kTilePer];
#pragma unroll
    for (int u = 0; u < kTilePer; ++u) {
        const unsigned long long v = v0 + (unsigned long long)u * kMeanThreads;
        if (v < nvec) buf[u] = __ldcg(p + v);
    }
    R two_mr = 0, two_mi = 0;
    if (WRITE) {
        const double mr = a.sum_in[0] * a.inv_total, mi = a.sum_in[1] * a.inv_total;
        two_mr = (R)(2.0 * mr);
        two_mi = (R)(2.0 * mi);
    }
    const auto *mk = reinterpret_cast<const unsigned long long *>(a.marked);
    const bool any = a.n_marked != 0 && ((__ldg(&a.chunkmap[t >> 5]) >> (t & 31)) & 1u);
    double sr = 0.0, si = 0.0;
#pragma unroll
    for (int u = 0; u < kTilePer; ++u) {
        const unsigned long long v = v0 + (unsigned long long)u * kMeanThreads;
        if (v >= nvec) continue;
        E e[VE];
        if constexpr (VE == 2) {
            e[0].x = buf[u].x; e[0].y = buf[u].y;
            e[1].x = buf[u].z; e[1].y = buf[u].w;
        } else {
            e[0].x = buf[u].x; e[0].y = buf[u].y;
        }
#pragma unroll
        for (int q = 0; q < VE; ++q) {
            const bool m = any && is_marked(v * VE + q, mk, a.n_marked);
            if (m) { e[q].x = -e[q].x; e[q].y = -e[q].y; }   // O
            if (WRITE) {
                e[q].x = two_mr - e[q].x;                       // 2 mu - (O a)_i
                e[q].y = two_mi - e[q].y;
                sr += m ? -(double)e[q].x : (double)e[q].x;     // (O a')_i for the next sum
                si += m ? -(double)e[q].y : (double)e[q].y;
            } else {
                sr += (double)e[q].x;
                si += (double)e[q].y;
            }
        }
        if (WRITE) {
            if constexpr (VE == 2) {
                buf[u].x = e[0].x; buf[u].y = e[0].y; buf[u].z = e[1].x; buf[u].w = e[1].y;
            } else {
                buf[u].x = e[0].x; buf[u].y = e[0].y;
            }
            p[v] = buf[u];
        }
    }
    block_sum2(sr, si, red);
    if (threadIdx.x == 0) {
        a.tilepart[2 * t] = sr;
        a.tilepart[2 * t + 1] = si;
    }
}

// Fixed-order sum of `count` (re, im) pairs -> out[0..1].
__global__ void __launch_bounds__(kMeanThreads) sum_pairs_kernel(const double *in, unsigned long long count,
                                                                 double *partials, unsigned int *counter,
                                                                 double *out) {
    __shared__ double red[2 * (kMeanThreads / 32)];
    const unsigned long long per = (count + gridDim.x - 1) / gridDim.x;
    const unsigned long long lo = per * blockIdx.x, hi = lo + per < count ? lo + per : count;
    double r = 0.0, m = 0.0;
    for (unsigned long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        r += __ldcg(in + 2 * i);
        m += __ldcg(in + 2 * i + 1);
    }
    block_sum2(r, m, red);
    finalize(r, m, partials, counter, out, red);
}

uint64_t mean_tiles(uint64_t N, sv_dtype dt) {
    const uint64_t nvec = N * elem_bytes(dt) / 16;
    return (nvec + kTileVec - 1) / kTileVec;
}

uint64_t mean_chunk_elems(sv_dtype dt) { return (mean_tile_mode() ? kTileVec : kChunkVec) * (dt == SV_C64 ? 2 : 1); }


int mean_grid(uint64_t N, sv_dtype dt) {
    int dev = 0, sms = 148, per = 1;
    SV_CUDA(cudaGetDevice(&dev));
    SV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (dt == SV_C64)
        SV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mean_kernel<float2, true>, kMeanThreads, 0));
    else
        SV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mean_kernel<double2, true>, kMeanThreads, 0));
    uint64_t want = (uint64_t)sms * (uint64_t)(per > 0 ? per : 1);  // one full wave
    const uint64_t nvec = N * elem_bytes(dt) / 16;
    uint64_t cap = (nvec + kChunkVec - 1) / kChunkVec;             // >= 1 chunk per block
    if (cap < 1) cap = 1;
    return (int)(want < cap ? want : cap);
}

void launch_mean_grid(sv_dtype dt, const MeanArgs &a, int grid, bool write, cudaStream_t s) {
    if (mean_tile_mode()) {
        const uint64_t nt = mean_tiles(a.N, dt);
        SV_CHECK(a.tilepart != nullptr, SV_EINVAL, "internal: mean tile partials not allocated");
        SV_CHECK(nt <= 0x7fffffffull, SV_EINVAL, "internal: too many mean tiles");
        if (dt == SV_C64) {
            if (write) mean_tile_kernel<float2, true><<<(unsigned)nt, kMeanThreads, 0, s>>>(a);
            else mean_tile_kernel<float2, false><<<(unsigned)nt, kMeanThreads, 0, s>>>(a);
        } else {
            if (write) mean_tile_kernel<double2, true><<<(unsigned)nt, kMeanThreads, 0, s>>>(a);
            else mean_tile_kernel<double2, false><<<(unsigned)nt, kMeanThreads, 0, s>>>(a);
        }
        SV_CUDA(cudaGetLastError());
        unsigned int g = (unsigned int)((nt + 2047) / 2048);  // <= 2048 pairs per block
        if (g < 1) g = 1;
        if (g > (unsigned)grid_cap_pairs) g = (unsigned)grid_cap_pairs;
        sum_pairs_kernel<<<g, kMeanThreads, 0, s>>>(a.tilepart, nt, a.partials, a.counter, a.sum_out);
        SV_CUDA(cudaGetLastError());
        return;
    }
    if (dt == SV_C64) {
        if (write) mean_kernel<float2, true><<<grid, kMeanThreads, 0, s>>>(a);
        else mean_kernel<float2, false><<<grid, kMeanThreads, 0, s>>>(a);
    } else {
        if (write) mean_kernel<double2, true><<<grid, kMeanThreads, 0, s>>>(a);
        else mean_kernel<double2, false><<<grid, kMeanThreads, 0, s>>>(a);
    }
    SV_CUDA(cudaGetLastError());
}

}  // namespace sv
