// tma_probe.cu -- microbenchmark (not part of libsv): in-place read + write of
// the strided tile shape of the WHT passes (64-B runs at a 64 KiB row stride,
// 1024 rows per 64 KiB tile; and contiguous 64 KiB tiles) with
//   (a) per-thread 8-byte LDG/STG, 2 CTAs/SM, one tile per CTA (the current
//       strided tile kernels' access pattern);
//   (b) one 5-D TMA tensor load per tile into a 2-stage shared-memory ring fed
//       by a producer warp (mbarrier hand-off), STG stores by 8 consumer warps,
//       one persistent CTA per SM;
//   (c) as (b) with a TMA tensor store from shared memory.
// Prints GB/s = 2 x bytes / kernel time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; }      \
    } while (0)

constexpr int N_BITS = 28;      // 2^28 x 8 B = 2 GiB
constexpr int TB = 13;          // tile = 2^13 elements = 64 KiB

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, unsigned ph) {
    asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(su32(b)), "r"(ph) : "memory");
}

// slots of the tile (ascending) and of the tile id
struct Geo {
    int tslot[16];
    int fslot[32];
    int nfree;
};

__device__ __forceinline__ unsigned long long tile_base(unsigned long long t, const Geo &g) {
    unsigned long long b = 0;
    for (int i = 0; i < g.nfree; ++i)
        if ((t >> i) & 1) b |= 1ull << g.fslot[i];
    return b;
}

// (a) LDG/STG, one tile per CTA, element e = tid + 256 j
__global__ void __launch_bounds__(256, 2) k_ldg(uint64_t *buf, Geo g) {
    const unsigned long long base = tile_base(blockIdx.x, g);
    uint64_t r[32];
    unsigned long long off[32], ot = 0;
    for (int b = 0; b < 8; ++b)
        if ((threadIdx.x >> b) & 1) ot += 1ull << g.tslot[b];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        unsigned long long o = ot;
#pragma unroll
        for (int b = 0; b < 5; ++b)
            if ((j >> b) & 1) o += 1ull << g.tslot[8 + b];
        off[j] = base + o;
        r[j] = __ldcg(buf + off[j]);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) buf[off[j]] = r[j] ^ 0x8000000000000000ull;
}

// (b)/(c) persistent TMA pipeline
template <bool TMA_STORE>
__global__ void __launch_bounds__(288, 1) k_tma(const __grid_constant__ CUtensorMap tm, uint64_t *buf, Geo g,
                                                 unsigned long long ntiles, int rank, int cdim_free0, int cdim_free1,
                                                 int free0_bits) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *st[2] = {reinterpret_cast<uint64_t *>(smem), reinterpret_cast<uint64_t *>(smem + 65536)};
    __shared__ __align__(8) uint64_t full[2], empty[2];
    const int tid = threadIdx.x;
    if (tid == 0) {
        mb_init(&full[0], 1); mb_init(&full[1], 1); mb_init(&empty[0], 1); mb_init(&empty[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid >= 256) {
        if (tid != 256) return;
        int it = 0;
        for (unsigned long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int s = it & 1;
            const unsigned ph = (it >> 1) & 1;
            mb_wait(&empty[s], ph ^ 1);
            mb_expect(&full[s], 65536);
            int c[5] = {0, 0, 0, 0, 0};
            // tile id bits: low free0_bits -> dim cdim_free0, the rest -> dim cdim_free1
            c[cdim_free0] = (int)(t & ((1ull << free0_bits) - 1));
            if (cdim_free1 >= 0) c[cdim_free1] = (int)(t >> free0_bits);
            if (rank == 5)
                asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                             ::"r"(su32(st[s])), "l"(&tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su32(&full[s])) : "memory");
            else
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                             ::"r"(su32(st[s])), "l"(&tm), "r"(c[0]), "r"(c[1]), "r"(su32(&full[s])) : "memory");
        }
        return;
    }
    int it = 0;
    for (unsigned long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it & 1;
        const unsigned ph = (it >> 1) & 1;
        mb_wait(&full[s], ph);
        uint64_t *x = st[s];
        if (TMA_STORE) {
            for (int j = tid; j < 8192; j += 256) x[j] ^= 0x8000000000000000ull;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (tid == 0) {
                int c[5] = {0, 0, 0, 0, 0};
                c[cdim_free0] = (int)(t & ((1ull << free0_bits) - 1));
                if (cdim_free1 >= 0) c[cdim_free1] = (int)(t >> free0_bits);
                if (rank == 5)
                    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                                 ::"l"(&tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su32(x)) : "memory");
                else
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                                 ::"l"(&tm), "r"(c[0]), "r"(c[1]), "r"(su32(x)) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                mb_arrive(&empty[s]);
            }
        } else {
            const unsigned long long base = tile_base(t, g);
            unsigned long long ot = 0;
            for (int b = 0; b < 8; ++b)
                if ((tid >> b) & 1) ot += 1ull << g.tslot[b];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                unsigned long long o = ot;
#pragma unroll
                for (int b = 0; b < 5; ++b)
                    if ((j >> b) & 1) o += 1ull << g.tslot[8 + b];
                buf[base + o] = x[tid + 256 * j] ^ 0x8000000000000000ull;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (tid == 0) mb_arrive(&empty[s]);
        }
    }
}

// (d) persistent, 1 CTA/SM, 256 threads: LDGSTS (cp.async 8 B) of tile i+1
// into the second shared-memory stage while tile i goes out with STG
__global__ void __launch_bounds__(256, 1) k_ldgsts(uint64_t *buf, Geo g, unsigned long long ntiles) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *st[2] = {reinterpret_cast<uint64_t *>(smem), reinterpret_cast<uint64_t *>(smem + 65536)};
    const int tid = threadIdx.x;
    unsigned long long ot = 0;
    for (int b = 0; b < 8; ++b)
        if ((tid >> b) & 1) ot += 1ull << g.tslot[b];
    unsigned long long oreg[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        unsigned long long o = ot;
#pragma unroll
        for (int b = 0; b < 5; ++b)
            if ((j >> b) & 1) o += 1ull << g.tslot[8 + b];
        oreg[j] = o;
    }
    auto issue = [&](unsigned long long t, uint64_t *dst) {
        const unsigned long long base = tile_base(t, g);
#pragma unroll
        for (int j = 0; j < 32; ++j)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(dst + tid + 256 * j)),
                         "l"(buf + base + oreg[j]) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    unsigned long long t = blockIdx.x;
    if (t < ntiles) issue(t, st[0]);
    for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
        const unsigned long long tn = t + gridDim.x;
        if (tn < ntiles) issue(tn, st[(it + 1) & 1]);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        uint64_t *x = st[it & 1];
        const unsigned long long base = tile_base(t, g);
#pragma unroll
        for (int j = 0; j < 32; ++j) buf[base + oreg[j]] = x[tid + 256 * j] ^ 0x8000000000000000ull;
        __syncthreads();
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t N = 1ull << N_BITS;
    uint64_t *buf;
    CK(cudaMalloc(&buf, N * 8));
    CK(cudaMemset(buf, 0, N * 8));
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaFuncSetAttribute(k_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    CK(cudaFuncSetAttribute(k_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    CK(cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int pat = 0; pat < 2; ++pat) {
        Geo g{};
        CUtensorMap tm;
        int rank, cf0, cf1, f0bits;
        if (pat == 0) {  // tile slots {0,1,2} u {13..22}; free {3..12} u {23..27}
            int k = 0;
            for (int s = 0; s < 3; ++s) g.tslot[k++] = s;
            for (int s = 13; s < 23; ++s) g.tslot[k++] = s;
            for (int s = 3; s < 13; ++s) g.fslot[g.nfree++] = s;
            for (int s = 23; s < N_BITS; ++s) g.fslot[g.nfree++] = s;
            // dims (elements of 8 B): {8 (slots 0-2), 1024 (3-12), 256 (13-20), 4 (21-22), 32 (23-27)}
            cuuint64_t dim[5] = {8, 1024, 256, 4, 1ull << (N_BITS - 23)};
            cuuint64_t str[4] = {8ull * 8, 8ull << 13, 8ull << 21, 8ull << 23};
            cuuint32_t box[5] = {8, 1, 256, 4, 1}, es[5] = {1, 1, 1, 1, 1};
            if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, buf, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); return 1; }
            rank = 5; cf0 = 1; cf1 = 4; f0bits = 10;
        } else {  // contiguous tiles
            for (int s = 0; s < TB; ++s) g.tslot[s] = s;
            for (int s = TB; s < N_BITS; ++s) g.fslot[g.nfree++] = s;
            cuuint64_t dim[2] = {8192, 1ull << (N_BITS - 13)};
            cuuint64_t str[1] = {8ull << 13};
            cuuint32_t box[2] = {256, 1}, es[2] = {1, 1};
            (void)box;
            // a 64 KiB contiguous tile as a 2-D box {8192? max 256} -> use dims {256, 32, rows}: not expressible in
            // 2-D with box <= 256, so describe it as 3-D folded into the 5-D path
            cuuint64_t dim5[5] = {256, 32, 1ull << (N_BITS - 13), 1, 1};
            cuuint64_t str5[4] = {8ull * 256, 8ull << 13, 8ull << N_BITS, 8ull << N_BITS};
            cuuint32_t box5[5] = {256, 32, 1, 1, 1}, es5[5] = {1, 1, 1, 1, 1};
            (void)dim; (void)str; (void)es;
            if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, buf, dim5, str5, box5, es5, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); return 1; }
            rank = 5; cf0 = 2; cf1 = -1; f0bits = N_BITS - 13;
        }
        const unsigned long long ntiles = N >> TB;
        const double bytes = 2.0 * N * 8;
        for (int mode = 0; mode < 4; ++mode) {
            auto launch = [&]() {
                if (mode == 0) k_ldg<<<(unsigned)ntiles, 256>>>(buf, g);
                else if (mode == 1) k_tma<false><<<sms, 288, 131072>>>(tm, buf, g, ntiles, rank, cf0, cf1, f0bits);
                else if (mode == 2) k_tma<true><<<sms, 288, 131072>>>(tm, buf, g, ntiles, rank, cf0, cf1, f0bits);
                else k_ldgsts<<<sms, 256, 131072>>>(buf, g, ntiles);
            };
            launch();
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) launch();
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%s  %-28s %8.1f GB/s  (%.3f ms/pass)\n", pat == 0 ? "strided 64B x 64KiB" : "contiguous 64KiB   ",
                   mode == 0 ? "LDG/STG 2 CTA/SM" : (mode == 1 ? "TMA load + STG, pipelined" : (mode == 2 ? "TMA load + TMA store" : "LDGSTS 2-stage + STG, 1 CTA/SM")),
                   bytes * 5 / (ms / 1e3) / 1e9, ms / 5);
        }
    }
    // correctness spot check: after 1 + 5 + ... flips the sign bit parity is known; skip
    return 0;
}
