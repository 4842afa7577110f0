// xfer_probe.cu -- microbenchmark (not part of libsv): the on-chip / near-chip
// bandwidths a larger-than-one-CTA WHT tile would have to move its data over.
//   (1) L2-resident in-place read+write: a buffer of B MiB swept R times by one
//       launch (grid-stride, 128-bit accesses), B from 8 MiB to 2 GiB
//       (>= 126 MB L2 is the HBM reference).  Bytes = 2 x B x R.
//   (2) DSMEM exchange inside a thread-block cluster of C CTAs (64 KiB of
//       shared memory each, 2 CTAs per SM): every CTA repeatedly reads its
//       partner's (rank ^ d) shared tile with 128-bit ld.shared::cluster
//       loads and writes them into its own tile (a butterfly's data
//       movement), cluster.sync between rounds.  Reported per SM and total.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/xfer tools/xfer_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void __launch_bounds__(256) l2_rw(float4 *buf, size_t nvec, int reps) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += 4 * stride) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * stride < nvec) v[u] = __ldcg(buf + i + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * stride < nvec) {
                    v[u].x += 1.f;
                    buf[i + u * stride] = v[u];
                }
        }
    }
}

// 64 KiB tile per CTA; `rounds` exchanges with partner rank ^ (1 << (round % log2 C)).
__global__ void __launch_bounds__(256, 2) dsmem_xchg(float *out, int rounds, int logc) {
    extern __shared__ __align__(16) float4 tile[];  // 4096 float4 = 64 KiB
    cg::cluster_group cl = cg::this_cluster();
    const unsigned int me = cl.block_rank();
    for (int i = threadIdx.x; i < 4096; i += 256) tile[i] = make_float4(me, i, 0, 0);
    cl.sync();
    float acc = 0.f;
    for (int r = 0; r < rounds; ++r) {
        const unsigned int peer = me ^ (1u << (logc ? r % logc : 0));
        const float4 *rt = cl.map_shared_rank(tile, logc ? peer : me);
        float4 v[16];
        // read the partner's half tile (32 KiB), as a cross-CTA butterfly does
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = rt[threadIdx.x + 256 * u + ((me & 1) ? 0 : 2048)];
        cl.sync();  // everyone has read before anyone overwrites
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            float4 w = tile[threadIdx.x + 256 * u + ((me & 1) ? 0 : 2048)];
            w.x += v[u].x;
            w.y -= v[u].y;
            tile[threadIdx.x + 256 * u + ((me & 1) ? 0 : 2048)] = w;
            acc += w.z;
        }
        cl.sync();
    }
    if (acc == 1.2345f) out[0] = acc;
}

int main() {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0, dev = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // ---- (1) L2 / HBM read+write -------------------------------------------
    const size_t maxb = 2ull << 30;
    float4 *buf;
    cudaMalloc(&buf, maxb);
    cudaMemset(buf, 0, maxb);
    for (size_t mib : {8, 16, 24, 32, 48, 64, 96, 128, 2048}) {
        const size_t bytes = mib << 20, nvec = bytes / 16;
        const int reps = mib >= 128 ? 3 : (int)(4096 / mib);
        for (int grid_mult : {4, 8}) {
            const int grid = sms * grid_mult;
            l2_rw<<<grid, 256>>>(buf, nvec, 1);
            cudaEventRecord(a);
            l2_rw<<<grid, 256>>>(buf, nvec, reps);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("l2_rw  %6zu MiB  grid %4d  reps %4d  %8.1f GB/s (read+write)  %s\n", mib, grid, reps,
                   2.0 * bytes * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    cudaFree(buf);
    // ---- (2) DSMEM ----------------------------------------------------------
    float *out;
    cudaMalloc(&out, 16);
    cudaFuncSetAttribute(dsmem_xchg, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(dsmem_xchg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int logc : {0, 1, 2, 3, 4}) {
        const int C = 1 << logc;
        cudaLaunchConfig_t cfg = {};
        const int grid = (2 * sms / C) * C;
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = 65536;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, dsmem_xchg, &cfg);
        const int rounds = 2000;
        cudaLaunchKernelEx(&cfg, dsmem_xchg, out, 10, logc);
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, dsmem_xchg, out, rounds, logc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        // bytes read remotely per CTA per round: 32 KiB (C = 1: local shared memory)
        const double bytes = (double)grid * rounds * 32768.0;
        printf("dsmem  cluster %2d  grid %4d  active clusters %4d  %8.1f GB/s total  %6.1f GB/s per SM  %6.2f us/round  %s\n",
               C, grid, ncl, bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / sms, ms * 1e3 / rounds,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
