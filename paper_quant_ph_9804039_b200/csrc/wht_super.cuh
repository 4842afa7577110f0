// wht_super.cuh -- L2-staged supertile pass of the WHT (sm_100a), built from
// the tile machinery of wht_kernels.cuh.  Instantiated per stage flavour by
// wht_super.cu (ideal), wht_super_noisy.cu, wht_super_angle.cu.
//
// What it computes: one visit of the F0 group G (the slots [T, nl), i.e. all
// qubits above the contiguous group) fused with F0:
//     stages(G, transform 1) ; F0 ; stages(G, transform 2)
// as "a sequence of V/2 independent 2x2 transformations" per qubit (section
// 2.1) -- exactly the butterflies of the plain schedule, split
// into three dependent sub-passes over each SUPERTILE (the 2^|st| amplitudes
// whose indices differ only in G's slots and two carry slots):
//     sub-pass 0: level-A slots' stages (transform 1)
//     sub-pass 1: level-B slots' stages, F0, level-B slots' stages (transform 2)
//     sub-pass 2: level-A slots' stages (transform 2)
// Each sub-pass is a set of ordinary 2^T-amplitude tiles (registers + one
// shared-memory tile, the relayouts of wht_kernels.cuh).
//
// Why (B200 design): a transform must read and
// write the state at least once, so an iteration costs at least 2 HBM passes;
// the plain schedule needs 4 at n = 28..33 because a 64 KiB tile holds only
// 10 strided slots.  A supertile of <= 16 MiB stays in the 126 MB L2 between
// its sub-passes, so the whole group costs one HBM read + write; the extra
// traffic is L2 traffic (measured: 12.5-13 TB/s read+write L2-resident vs
// 6.0-7.0 TB/s HBM, profiles/r2_xfer_probe.txt).
//
// How: one persistent kernel (2 CTAs per SM).  Work items = (supertile s,
// sub-pass j, tile t) in a host-built segment order that keeps sub-pass j of
// supertile s a few supertiles behind sub-pass j-1 (software pipelining); a
// CTA claims items from a global ticket in increasing order, waits until the
// previous sub-pass of its supertile has completed (per-(s, j) completion
// counters, release/acquire at gpu scope), runs the tile, publishes.  Items are
// claimed in order and only wait on earlier items, so the smallest unfinished
// item can always run: no deadlock, no co-residency assumption.
#pragma once
#include "wht_kernels.cuh"

namespace sv {

template <int NOISY>
struct SuperParamsT {
    KParamsT<NOISY> sp[3];            // per sub-pass: slot map, in-supertile tile-id runs, op, coefficients
    int st_nruns;                     // supertile index -> the slots outside the supertile (runs)
    unsigned char st_start[8], st_len[8];
    const unsigned int *seg;          // segment -> (supertile << 2) | sub-pass
    unsigned int tps_log2;            // tiles per (supertile, sub-pass)
    unsigned long long nitems;
    unsigned int *ticket;             // zeroed before the launch
    unsigned int *done;               // [supertile * 3 + sub-pass], zeroed before the launch
};

#ifdef SV_SUPER_STATS
// measurement builds only: [0] items, [1] items that waited, [2] wait cycles,
// [3] claim-to-start cycles, [4] item cycles (start to publish)
__device__ unsigned long long g_super_stats[8];
#endif

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int NOISY>
__device__ __forceinline__ unsigned long long st_base(unsigned long long s, const SuperParamsT<NOISY> &P) {
    unsigned long long base = 0;
    int off = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        if (r < P.st_nruns) {
            const int len = P.st_len[r];
            base |= ((s >> off) & ((1ull << len) - 1ull)) << P.st_start[r];
            off += len;
        }
    }
    return base;
}

// One tile of sub-pass J (U = its unprocessed tile bits).
template <int J, int U, int NOISY>
__device__ __forceinline__ void super_tile(const KParamsT<NOISY> &p, unsigned long long base, int tid, float2 *sm) {
    constexpr bool PRE = J != 2, POST = J != 0;
    __shared__ unsigned long long s_dummy;
    float2 x[32];
    if constexpr (U >= 3 && U <= SV_2LAYOUT_MAX_U) {
        using L = Layout2<kTileBitsC64, kRegBitsC64>;
        global_load<L, 0>(x, reinterpret_cast<const float2 *>(p.in) + base, p, tid);
        if constexpr (NOISY == 2) apply_scalef(x, p.pass_scalef);
        tile_body2<L, PRE, POST, U, NOISY, false>(x, sm, p, base, reinterpret_cast<float2 *>(p.out) + base, tid,
                                                  static_cast<float2 *const *>(nullptr), false, &s_dummy, &s_dummy);
    } else {
        using L = Layout<float2, kTileBitsC64, kRegBitsC64>;
        global_load<L, 0>(x, reinterpret_cast<const float2 *>(p.in) + base, p, tid);
        if constexpr (NOISY == 2) apply_scalef(x, p.pass_scalef);
        tile_body<L, PRE, POST, U, NOISY, false>(x, sm, p, base, reinterpret_cast<float2 *>(p.out) + base, tid,
                                                 static_cast<float2 *const *>(nullptr), false, &s_dummy, &s_dummy);
    }
}

template <int UA, int UB, int NOISY>
__global__ void __launch_bounds__(256, 2) wht_super_kernel(const __grid_constant__ SuperParamsT<NOISY> P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *sm = reinterpret_cast<float2 *>(smem_raw);
    __shared__ unsigned int s_item;
    const int tid = threadIdx.x;
    const unsigned int tmask = (1u << P.tps_log2) - 1u;
    // thread 0 claims the NEXT item while this one runs (the ticket's round
    // trip is off the critical path)
    unsigned int next = 0;
    if (tid == 0) next = atomicAdd(P.ticket, 1u);
    for (;;) {
        __syncthreads();  // the previous item's shared-memory reads are done
        if (tid == 0) {
            s_item = next;
            if (next < P.nitems) next = atomicAdd(P.ticket, 1u);
        }
        __syncthreads();
        const unsigned int item = s_item;
        if (item >= P.nitems) break;
        const unsigned int seg = __ldg(&P.seg[item >> P.tps_log2]);
        const unsigned int s = seg >> 2, j = seg & 3u;
#ifdef SV_SUPER_STATS
        const long long t0 = clock64();
        bool waited = false;
#endif
        if (j > 0) {
            if (tid == 0) {
                const unsigned int *d = &P.done[s * 3 + j - 1];
                while (ld_acquire_gpu(d) < tmask + 1u) {
#ifdef SV_SUPER_STATS
                    waited = true;
#endif
                    __nanosleep(100);
                }
            }
            __syncthreads();
        }
#ifdef SV_SUPER_STATS
        const long long t1 = clock64();
#endif
        const unsigned long long sb = st_base(s, P);
        const unsigned int t = item & tmask;
        if (j == 0) super_tile<0, UA, NOISY>(P.sp[0], sb | tile_base(t, P.sp[0]), tid, sm);
        else if (j == 1) super_tile<1, UB, NOISY>(P.sp[1], sb | tile_base(t, P.sp[1]), tid, sm);
        else super_tile<2, UA, NOISY>(P.sp[2], sb | tile_base(t, P.sp[2]), tid, sm);
        __syncthreads();  // every thread's stores of this tile are issued
        if (tid == 0) {  // publish: release at gpu scope (cumulative over the CTA's stores via the barrier)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&P.done[s * 3 + j]) : "memory");
#ifdef SV_SUPER_STATS
            const long long t2 = clock64();
            atomicAdd(&g_super_stats[0], 1ull);
            if (waited) atomicAdd(&g_super_stats[1], 1ull);
            atomicAdd(&g_super_stats[2], (unsigned long long)(t1 - t0));
            atomicAdd(&g_super_stats[4], (unsigned long long)(t2 - t1));
#endif
        }
    }
}

// (UA, UB) pairs the planner may produce (plan.cpp): production level A of 11
// slots (UA = 2) with level B of 1..8 slots; the test-only SV_SUPER_A=4 shape
// (UA = 9, UB = 5) gives small states n = 32's level-B tile.
template <int NOISY>
void launch_super_uab(int ua, int ub, const SuperParamsT<NOISY> &P, int grid, cudaStream_t s) {
    void (*fn)(const SuperParamsT<NOISY>) = nullptr;
#define SV_SUPER_CASE(A, B) \
    if (ua == A && ub == B) fn = wht_super_kernel<A, B, NOISY>;
    SV_SUPER_CASE(2, 5) SV_SUPER_CASE(2, 6) SV_SUPER_CASE(2, 7) SV_SUPER_CASE(2, 8) SV_SUPER_CASE(2, 9)
    SV_SUPER_CASE(2, 10) SV_SUPER_CASE(2, 11) SV_SUPER_CASE(2, 12) SV_SUPER_CASE(9, 5)
#undef SV_SUPER_CASE
    SV_CHECK(fn != nullptr, SV_EINVAL, "internal: no supertile kernel for this level split");
    const int smem = (1 << kTileBitsC64) * (int)sizeof(float2);
    SV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    fn<<<grid, 256, smem, s>>>(P);
    SV_CUDA(cudaGetLastError());
}


}  // namespace sv
