// strided_rw_probe.cu -- microbenchmark (not part of libsv): in-place
// read+write of a 2 GiB buffer in contiguous runs of R bytes at a large row
// stride, the access shape of the strided WHT tile passes.  Prints achieved
// GB/s (read + write bytes / kernel time) per run length.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe tools/strided_rw_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

// Each CTA owns `rows` runs of R bytes (one per row, rows at stride `stride`
// bytes); consecutive CTAs take consecutive runs of the same rows.
__global__ void probe(float4 *buf, size_t stride_v, int run_v, int rows, size_t ncols) {
    const size_t col = blockIdx.x % ncols;           // which run within a row
    const size_t rgrp = blockIdx.x / ncols;          // which group of rows
    const int per_row = run_v;                       // float4 per run
    float4 r[16];
    const int nthr = blockDim.x;
    const int items = rows * per_row;                // float4 per CTA
    for (int base = threadIdx.x; base < items; base += nthr * 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            int it = base + u * nthr;
            if (it < items) {
                int row = it / per_row, c = it % per_row;
                size_t idx = (rgrp * rows + row) * stride_v + col * per_row + c;
                r[u] = buf[idx];
            }
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            int it = base + u * nthr;
            if (it < items) {
                int row = it / per_row, c = it % per_row;
                size_t idx = (rgrp * rows + row) * stride_v + col * per_row + c;
                r[u].x = -r[u].x;
                buf[idx] = r[u];
            }
        }
    }
}

int main() {
    const size_t bytes = 1ull << 31;
    float4 *buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    const size_t nvec = bytes / 16;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int wide = 0; wide < 2; ++wide)
    for (int run_bytes : {16, 32, 64, 128, 256, 512, 1024, 4096, 65536}) {
        int run_v = run_bytes / 16;
        // tile = 64 KiB = rows * run_bytes; row stride 64 KiB (wide = 0) or
        // the whole buffer / rows (wide = 1)
        int rows = 65536 / (run_v * 16);
        size_t stride_v = wide ? nvec / rows : (size_t)4096;
        if (stride_v < (size_t)run_v) stride_v = run_v;
        size_t ncols = stride_v / run_v;                 // runs per row
        size_t nrowgrp = nvec / stride_v / rows;
        size_t grid = ncols * nrowgrp;
        probe<<<(unsigned)grid, 256>>>(buf, stride_v, run_v, rows, ncols);
        cudaEventRecord(a);
        for (int it = 0; it < 5; ++it) probe<<<(unsigned)grid, 256>>>(buf, stride_v, run_v, rows, ncols);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double moved = 2.0 * (double)grid * rows * run_v * 16 * 5;
        printf("stride %10zu B run %6d B  rows/CTA %5d  grid %8zu  %8.1f GB/s  (%s)\n", stride_v * 16, run_bytes, rows, grid, moved / (ms / 1e3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
