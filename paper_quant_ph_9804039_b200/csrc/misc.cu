// misc.cu -- initial states, seeded generators, oracle scatter and readouts.
#include <cuda_runtime.h>
#include <math.h>

#include "reduce.cuh"
#include "sv_internal.h"

namespace sv {

constexpr int kThreads = 256;

static unsigned int grid_for(uint64_t work, int per_thread = 4) {
    uint64_t g = (work + (uint64_t)kThreads * per_thread - 1) / ((uint64_t)kThreads * per_thread);
    if (g < 1) g = 1;
    if (g > 148ull * 64) g = 148ull * 64;
    return (unsigned int)g;
}

// ------------------------------------------------------------------------- //
// Seeded generators (G6, G8).  The CPU oracle has its own implementation;   //
// tests/test_parity_*.py check that both produce identical integers.        //
// ------------------------------------------------------------------------- //
#define SV_TAG_MARK 0x4D41524B00000000ull /* "MARK" */
#define SV_TAG_INIT 0x494E495400000000ull /* "INIT" */

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t splitmix64_next(uint64_t &state) {
    state += 0x9E3779B97F4A7C15ull;
    return mix64(state);
}

uint64_t hash64(uint64_t x) { return mix64(x + 0x9E3779B97F4A7C15ull); }

uint64_t gauss_key(uint64_t seed) { return hash64(seed ^ SV_TAG_INIT); }

uint64_t perm_seeded(int n, uint64_t seed, uint64_t x) {
    uint64_t st = seed ^ SV_TAG_MARK;
    const uint64_t k1 = splitmix64_next(st) | 1ull;
    const uint64_t k2 = splitmix64_next(st);
    const uint64_t k3 = splitmix64_next(st) | 1ull;
    const uint64_t mask = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    const int s = (n + 1) / 2;
    x = (x * k1 + k2) & mask;
    x ^= x >> s;
    x = (x * k3) & mask;
    x ^= x >> s;
    return x;
}

// Angle error of qubit q in transform w of iteration t (G20):
// sigma * sqrt(-2 ln u0) cos(2 pi u1) from the counter hashes of
// c = (2t + w) * 64 + q under key hash64(seed ^ "NOIS").
double noise_delta(uint64_t seed, uint64_t t, int w, int q, double sigma) {
    const uint64_t key = hash64(seed ^ 0x4E4F495300000000ull);
    const uint64_t c = (2ull * t + (uint64_t)w) * 64ull + (uint64_t)q;
    const double u0 = ((double)(hash64(key ^ (2ull * c)) >> 11) + 0.5) * 0x1.0p-53;
    const double u1 = ((double)(hash64(key ^ (2ull * c + 1ull)) >> 11) + 0.5) * 0x1.0p-53;
    return sigma * (sqrt(-2.0 * log(u0)) * cos(6.283185307179586 * u1));
}

// Decoherence site after laser operation q of transform w, iteration t (G22):
// hash64(hash64(seed ^ "DECO") ^ c) mod n, c = (2t + w) * 64 + q.
int decay_site(int n, uint64_t seed, uint64_t t, int w, int q) {
    const uint64_t key = hash64(seed ^ 0x4445434F00000000ull);
    const uint64_t c = (2ull * t + (uint64_t)w) * 64ull + (uint64_t)q;
    return (int)(hash64(key ^ c) % (uint64_t)n);
}

// Box-Muller on two counter hashes (G8): u = ((h >> 11) + 0.5) 2^-53.
__device__ __forceinline__ void gauss_draw(uint64_t key, uint64_t i, double &re, double &im) {
    const uint64_t h0 = mix64((key ^ (2ull * i)) + 0x9E3779B97F4A7C15ull);
    const uint64_t h1 = mix64((key ^ (2ull * i + 1ull)) + 0x9E3779B97F4A7C15ull);
    const double u0 = ((double)(h0 >> 11) + 0.5) * 0x1.0p-53;
    const double u1 = ((double)(h1 >> 11) + 0.5) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u0));
    const double phi = 6.283185307179586 * u1;
    double s, c;
    sincos(phi, &s, &c);
    re = r * c;
    im = r * s;
}

// ------------------------------------------------------------------------- //
// Initial states                                                            //
// ------------------------------------------------------------------------- //
template <typename E>
__global__ void fill_kernel(E *a, uint64_t N, double re) {
    using R = decltype(E{}.x);
    const R v = (R)re;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        E e;
        e.x = v;
        e.y = (R)0;
        a[i] = e;
    }
}

void launch_init_uniform(sv_dtype dt, void *a, uint64_t N, int n, cudaStream_t s) {
    // |s> = H^n |0>: 2^{-n/2} (Fig. 1(b) is n = 1)
    const double v = sqrt(ldexp(1.0, -n));
    if (dt == SV_C64) fill_kernel<float2><<<grid_for(N), kThreads, 0, s>>>((float2 *)a, N, v);
    else fill_kernel<double2><<<grid_for(N), kThreads, 0, s>>>((double2 *)a, N, v);
    SV_CUDA(cudaGetLastError());
}

void launch_init_zero(sv_dtype dt, void *a, uint64_t N, int has_origin, cudaStream_t s) {
    if (dt == SV_C64) fill_kernel<float2><<<grid_for(N), kThreads, 0, s>>>((float2 *)a, N, 0.0);
    else fill_kernel<double2><<<grid_for(N), kThreads, 0, s>>>((double2 *)a, N, 0.0);
    SV_CUDA(cudaGetLastError());
    if (has_origin) {  // |0...0>: amplitude 1 at global index 0 (Fig. 1(a))
        if (dt == SV_C64) fill_kernel<float2><<<1, 32, 0, s>>>((float2 *)a, 1, 1.0);
        else fill_kernel<double2><<<1, 32, 0, s>>>((double2 *)a, 1, 1.0);
        SV_CUDA(cudaGetLastError());
    }
}

__global__ void __launch_bounds__(kThreads) gauss_norm_kernel(uint64_t key, uint64_t off, uint64_t N,
                                                               double *partials, unsigned int *counter,
                                                               double *out) {
    __shared__ double red[2 * (kThreads / 32)];
    double s = 0.0, dummy = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        double re, im;
        gauss_draw(key, off + i, re, im);
        s += re * re + im * im;
    }
    block_sum2(s, dummy, red);
    finalize(s, dummy, partials, counter, out, red);
}

template <typename E>
__global__ void gauss_write_kernel(E *a, uint64_t key, uint64_t off, uint64_t N, const double *norm) {
    using R = decltype(E{}.x);
    const double scale = 1.0 / sqrt(norm[0]);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        double re, im;
        gauss_draw(key, off + i, re, im);
        E e;
        e.x = (R)(re * scale);
        e.y = (R)(im * scale);
        a[i] = e;
    }
}

static unsigned int gauss_grid(uint64_t N) {
    unsigned int g = grid_for(N, 8);
    return g > 4096 ? 4096 : g;  // partials capacity (sv_api.cu kMaxGrid)
}

void launch_gauss_norm(uint64_t key, uint64_t off, uint64_t N, double *partials, unsigned int *counter,
                       double *norm_out, cudaStream_t s) {
    gauss_norm_kernel<<<gauss_grid(N), kThreads, 0, s>>>(key, off, N, partials, counter, norm_out);
    SV_CUDA(cudaGetLastError());
}

void launch_gauss_write(sv_dtype dt, void *a, uint64_t key, uint64_t off, uint64_t N, const double *norm,
                        cudaStream_t s) {
    if (dt == SV_C64) gauss_write_kernel<float2><<<grid_for(N), kThreads, 0, s>>>((float2 *)a, key, off, N, norm);
    else gauss_write_kernel<double2><<<grid_for(N), kThreads, 0, s>>>((double2 *)a, key, off, N, norm);
    SV_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------------- //
// Renormalisation (decoherence, G22): the paper's "accumulate and           //
// redistribute a sum" (Eq. 3)                                   //
// ------------------------------------------------------------------------- //
template <typename E>
__global__ void __launch_bounds__(kThreads) norm2_kernel(const E *a, uint64_t N, double *partials,
                                                          unsigned int *counter, double *out) {
    __shared__ double red[2 * (kThreads / 32)];
    double s = 0.0, dummy = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        const E v = a[i];
        s += (double)v.x * (double)v.x + (double)v.y * (double)v.y;
    }
    block_sum2(s, dummy, red);
    finalize(s, dummy, partials, counter, out, red);
}

void launch_norm2(sv_dtype dt, const void *a, uint64_t N, double *partials, unsigned int *counter, double *sum,
                  cudaStream_t s) {
    unsigned int g = grid_for(N, 8);
    if (g > 4096) g = 4096;  // partials capacity
    if (dt == SV_C64) norm2_kernel<float2><<<g, kThreads, 0, s>>>((const float2 *)a, N, partials, counter, sum);
    else norm2_kernel<double2><<<g, kThreads, 0, s>>>((const double2 *)a, N, partials, counter, sum);
    SV_CUDA(cudaGetLastError());
}

// Partials (one per tile of the pass that produced them) -> fixed-order sum:
// block b sums a contiguous segment, thread-strided, then the warp tree and
// the last-block finalize of reduce.cuh (G14: deterministic for a fixed grid).
__global__ void __launch_bounds__(kThreads) sum_partials_kernel(const double *in, uint64_t count, double *partials,
                                                                 unsigned int *counter, double *out) {
    __shared__ double red[2 * (kThreads / 32)];
    const uint64_t per = (count + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = per * blockIdx.x, hi = lo + per < count ? lo + per : count;
    double s = 0.0, dummy = 0.0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += __ldcg(in + i);
    block_sum2(s, dummy, red);
    finalize(s, 0.0, partials, counter, out, red);
}

void launch_sum_partials(const double *in, uint64_t count, double *partials, unsigned int *counter, double *sum,
                         cudaStream_t s) {
    unsigned int g = (unsigned int)((count + 4095) / 4096);
    if (g < 1) g = 1;
    if (g > 1024) g = 1024;
    sum_partials_kernel<<<g, kThreads, 0, s>>>(in, count, partials, counter, sum);
    SV_CUDA(cudaGetLastError());
}

__global__ void norm_finalize_kernel(const double *sum, double *scale_out, double *survival) {
    if (scale_out) *scale_out = 1.0 / sqrt(sum[0]);
    if (survival) *survival = sum[0];
}

void launch_norm_finalize(const double *sum, double *scale_out, double *survival, cudaStream_t s) {
    norm_finalize_kernel<<<1, 1, 0, s>>>(sum, scale_out, survival);
    SV_CUDA(cudaGetLastError());
}

template <typename E>
__global__ void scale_kernel(E *a, uint64_t N, const double *scale) {
    using R = decltype(E{}.x);
    const R sc = (R)scale[0];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        E v = a[i];
        v.x *= sc;
        v.y *= sc;
        a[i] = v;
    }
}

void launch_scale(sv_dtype dt, void *a, uint64_t N, const double *scale, cudaStream_t s) {
    if (dt == SV_C64) scale_kernel<float2><<<grid_for(N), kThreads, 0, s>>>((float2 *)a, N, scale);
    else scale_kernel<double2><<<grid_for(N), kThreads, 0, s>>>((double2 *)a, N, scale);
    SV_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------------- //
// Oracle scatter and readouts                                               //
// ------------------------------------------------------------------------- //
template <typename E>
__global__ void scatter_flip_kernel(E *a, const unsigned long long *mk, uint64_t m) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x) {
        E v = a[mk[j]];
        v.x = -v.x;
        v.y = -v.y;
        a[mk[j]] = v;
    }
}

void launch_oracle_scatter(sv_dtype dt, void *a, const uint64_t *marked, uint64_t m, cudaStream_t s) {
    if (m == 0) return;
    const auto mk = reinterpret_cast<const unsigned long long *>(marked);
    if (dt == SV_C64) scatter_flip_kernel<float2><<<grid_for(m, 1), kThreads, 0, s>>>((float2 *)a, mk, m);
    else scatter_flip_kernel<double2><<<grid_for(m, 1), kThreads, 0, s>>>((double2 *)a, mk, m);
    SV_CUDA(cudaGetLastError());
}

// "The probability of each state is defined as the square of this complex
// amplitude": p = re^2 + im^2 in fp64.
template <typename E>
__global__ void prob_kernel(const E *a, double *p, uint64_t N) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
        const E v = a[i];
        const double re = (double)v.x, im = (double)v.y;
        p[i] = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
    }
}

void launch_probabilities(sv_dtype dt, const void *a, double *p, uint64_t N, cudaStream_t s) {
    if (dt == SV_C64) prob_kernel<float2><<<grid_for(N), kThreads, 0, s>>>((const float2 *)a, p, N);
    else prob_kernel<double2><<<grid_for(N), kThreads, 0, s>>>((const double2 *)a, p, N);
    SV_CUDA(cudaGetLastError());
}

// One block, fixed order: sum over the marked list of |a_m|^2 (fp64).
template <typename E>
__global__ void __launch_bounds__(kThreads) marked_mass_kernel(const E *a, const unsigned long long *mk, uint64_t m,
                                                                double *out) {
    __shared__ double red[2 * (kThreads / 32)];
    double s = 0.0, dummy = 0.0;
    for (uint64_t j = threadIdx.x; j < m; j += blockDim.x) {
        const E v = a[mk[j]];
        const double re = (double)v.x, im = (double)v.y;
        s += re * re + im * im;
    }
    block_sum2(s, dummy, red);
    if (threadIdx.x == 0) out[0] = s;
}

void launch_marked_mass(sv_dtype dt, const void *a, const uint64_t *marked, uint64_t m, double *out,
                        cudaStream_t s) {
    const auto mk = reinterpret_cast<const unsigned long long *>(marked);
    if (dt == SV_C64) marked_mass_kernel<float2><<<1, kThreads, 0, s>>>((const float2 *)a, mk, m, out);
    else marked_mass_kernel<double2><<<1, kThreads, 0, s>>>((const double2 *)a, mk, m, out);
    SV_CUDA(cudaGetLastError());
}

}  // namespace sv
