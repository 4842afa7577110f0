// reduce.cuh -- deterministic fp64 grid reduction helpers (device only).
// Fixed-order tree: warp shuffle -> block -> per-block partials -> the last
// block to arrive sums the partials in block order (no floating-point
// atomics, so results are bitwise reproducible for a fixed grid; G14).
#pragma once
#include <cuda_runtime.h>

namespace sv {

// Block sum of (re, im); result valid in thread 0.
__device__ __forceinline__ void block_sum2(double &re, double &im, double *red) {
    for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { red[2 * w] = re; red[2 * w + 1] = im; }
    __syncthreads();
    if (threadIdx.x == 0) {
        re = 0.0; im = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { re += red[2 * i]; im += red[2 * i + 1]; }
    }
}

// Partials -> last block writes the fixed-order total to out[0..1].
__device__ __forceinline__ void finalize(double re, double im, double *partials, unsigned int *counter,
                                         double *out, double *red) {
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = re;
        partials[2 * blockIdx.x + 1] = im;
        __threadfence();
        unsigned int t = atomicAdd(counter, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double r = 0.0, m = 0.0;
    for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        r += __ldcg(&partials[2 * b]);
        m += __ldcg(&partials[2 * b + 1]);
    }
    __syncthreads();  // red reuse
    block_sum2(r, m, red);
    if (threadIdx.x == 0) {
        out[0] = r;
        out[1] = m;
        *counter = 0u;
    }
}


}  // namespace sv
