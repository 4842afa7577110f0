/*
 * sv_oracle.c -- plain, slow, obviously-correct CPU oracle for the Grover
 * state-vector hot path (arxiv quant-ph/9804039, Obenland & Despain,
 * "A Parallel Quantum Computer Simulator").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline leg and --impl reference) may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * under paper_quant_ph_9804039_b200/csrc/; neither side includes the other.
 *
 * Arithmetic: complex double (C99 _Complex), plain loops, no SIMD intrinsics,
 * no blocking, no fusion.  Sums use long double with Kahan compensation.
 *
 * Citation keys: P:NNNN = line of /root/reference/PAPER.md (the paper's
 * PostScript text), S:NNN = line of SPEC.md; "G<k>" = a reading listed in
 * DESIGN.md section "Readings" (the paper is silent on Grover's iteration:
 * it only cites [Grov96] in section 1.5).
 *
 * Index convention ("The bit value of a state corresponds to the
 * index of that state in the vector"; Fig. 3, P:3144-3380 pairs (a0,a1) and
 * (a2,a3) for the low bit): qubit q is bit q of the amplitude index.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* ------------------------------------------------------------------------ */
/* Seeded generators (G6, G8).  Implemented here independently of the CUDA  */
/* library, which has its own implementation; tests check they agree.      */
/* ------------------------------------------------------------------------ */

#define OR_TAG_MARK 0x4D41524B00000000ULL /* "MARK" */
#define OR_TAG_INIT 0x494E495400000000ULL /* "INIT" */

/* SplitMix64 step: state += golden gamma, then the 64-bit finaliser. */
uint64_t or_splitmix64_next(uint64_t *state)
{
    uint64_t z;
    *state = *state + 0x9E3779B97F4A7C15ULL;
    z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Counter hash: one SplitMix64 output from state x (G8). */
uint64_t or_hash64(uint64_t x)
{
    uint64_t s = x;
    return or_splitmix64_next(&s);
}

/* Keyed bijection pi_seed on n-bit integers (G6):
 *   x <- (x*k1 + k2) mod 2^n ; x ^= x >> s ; x <- (x*k3) mod 2^n ; x ^= x >> s
 * with s = ceil(n/2), k1 and k3 odd, (k1,k2,k3) = first three SplitMix64
 * outputs from state seed ^ TAG_MARK. */
static void or_perm_keys(int n, uint64_t seed, uint64_t k[3])
{
    uint64_t st = seed ^ OR_TAG_MARK;
    (void)n;
    k[0] = or_splitmix64_next(&st) | 1ULL;
    k[1] = or_splitmix64_next(&st);
    k[2] = or_splitmix64_next(&st) | 1ULL;
}

uint64_t or_perm(int n, uint64_t seed, uint64_t x)
{
    uint64_t k[3];
    uint64_t mask = (n >= 64) ? ~0ULL : ((1ULL << n) - 1ULL);
    int s = (n + 1) / 2;
    or_perm_keys(n, seed, k);
    x = (x * k[0] + k[1]) & mask;
    x ^= x >> s;
    x = (x * k[2]) & mask;
    x ^= x >> s;
    return x;
}

static int cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* Marked set M = sort{ pi_seed(j) : 0 <= j < m }  (G6 / G7).  Returns 0, or
 * -1 if m > 2^n. */
int or_marked_from_seed(int n, uint64_t m, uint64_t seed, uint64_t *out)
{
    uint64_t N = 1ULL << n, j;
    if (m > N) return -1;
    for (j = 0; j < m; ++j) out[j] = or_perm(n, seed, j);
    qsort(out, (size_t)m, sizeof(uint64_t), cmp_u64);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Initial states                                                           */
/* ------------------------------------------------------------------------ */

/* |s> = H^{(x)n}|0>: every amplitude 2^{-n/2} (Fig. 1(b), P:2284-2286 is the
 * n = 1 case: amplitudes 1/sqrt2, probabilities 1/2). */
void or_init_uniform(int n, cplx *a)
{
    uint64_t N = 1ULL << n, i;
    double v = ldexp(1.0, -n);          /* 2^{-n} */
    v = sqrt(v);                         /* 2^{-n/2}, exact for even n */
    for (i = 0; i < N; ++i) a[i] = v;
}

/* |0...0> (Fig. 1(a)). */
void or_init_zero_state(int n, cplx *a)
{
    uint64_t N = 1ULL << n, i;
    for (i = 0; i < N; ++i) a[i] = 0.0;
    a[0] = 1.0;
}

/* Unnormalised complex Gaussian draw for amplitude i (G8):
 *   u_j = ((hash64(key ^ (2i+j)) >> 11) + 0.5) * 2^-53,  j = 0, 1
 *   r = sqrt(-2 ln u_0), phi = 2 pi u_1, z = r cos(phi) + i r sin(phi). */
void or_gauss_draw(uint64_t key, uint64_t i, double *re, double *im)
{
    uint64_t h0 = or_hash64(key ^ (2ULL * i));
    uint64_t h1 = or_hash64(key ^ (2ULL * i + 1ULL));
    double u0 = ((double)(h0 >> 11) + 0.5) * 0x1.0p-53;
    double u1 = ((double)(h1 >> 11) + 0.5) * 0x1.0p-53;
    double r = sqrt(-2.0 * log(u0));
    double phi = 6.283185307179586 * u1;
    *re = r * cos(phi);
    *im = r * sin(phi);
}

uint64_t or_gauss_key(uint64_t seed) { return or_hash64(seed ^ OR_TAG_INIT); }

/* Seeded complex Gaussian start normalised to ||a||_2 = 1 (G8).  If
 * round_to_c64 != 0 the normalised amplitudes are rounded to float (the
 * c64 dtype) and the oracle continues in double from the rounded values
 * (G12). */
void or_init_gaussian(int n, uint64_t seed, int round_to_c64, cplx *a)
{
    uint64_t N = 1ULL << n, i, key = or_gauss_key(seed);
    long double s = 0.0L, c = 0.0L;
    double scale;
    for (i = 0; i < N; ++i) {
        double re, im;
        long double y, t;
        or_gauss_draw(key, i, &re, &im);
        a[i] = CMPLX(re, im);
        y = (long double)(re * re + im * im) - c;   /* Kahan */
        t = s + y;
        c = (t - s) - y;
        s = t;
    }
    scale = 1.0 / sqrt((double)s);
    for (i = 0; i < N; ++i) {
        double re = creal(a[i]) * scale, im = cimag(a[i]) * scale;
        if (round_to_c64) { re = (double)(float)re; im = (double)(float)im; }
        a[i] = CMPLX(re, im);
    }
}

/* ------------------------------------------------------------------------ */
/* The operations of one Grover iteration                                   */
/* ------------------------------------------------------------------------ */

/* Phase oracle O = I - 2 sum_m |m><m| (G3): negate every listed amplitude. */
void or_oracle_flip(cplx *a, const uint64_t *marked, uint64_t m)
{
    uint64_t j;
    for (j = 0; j < m; ++j) a[marked[j]] = -a[marked[j]];
}

/* One general 2x2 transformation [w x; y z] on qubit q: "a 2x2 transformation
 * on a vector of size V, is a sequence of V/2 independent 2x2
 * transformations ... the simulator splits the state space so that the bit
 * value of the states in the vector differ only in the position of that bit"
 * (section 2.1; Fig. 3). */
void or_apply_2x2(int n, cplx *a, int q, cplx w, cplx x, cplx y, cplx z)
{
    uint64_t N = 1ULL << n, bit = 1ULL << q, i;
    for (i = 0; i < N; ++i) {
        if (i & bit) continue;              /* i has bit q = 0; partner i|bit */
        {
            cplx a0 = a[i], a1 = a[i | bit];
            a[i] = w * a0 + x * a1;
            a[i | bit] = y * a0 + z * a1;
        }
    }
}

/* Unnormalised Walsh-Hadamard transform W = (sqrt2 H)^{(x)n}: for q = 0..n-1
 * apply Fig. 3's 2x2 with w = x = y = 1, z = -1, i.e. (x,y) -> (x+y, x-y). */
void or_wht(int n, cplx *a)
{
    int q;
    for (q = 0; q < n; ++q) or_apply_2x2(n, a, q, 1.0, 1.0, 1.0, -1.0);
}

/* F0 = 2|0><0| - I (G2), with the single exact 2^{-n} normalisation of the
 * two unnormalised transforms folded in (G5). */
void or_f0_scaled(int n, cplx *a)
{
    uint64_t N = 1ULL << n, i;
    double s = ldexp(1.0, -n);
    a[0] = a[0] * s;
    for (i = 1; i < N; ++i) a[i] = -a[i] * s;
}

/* WHT diffusion D = H^n F0 H^n = 2|s><s| - I (north star). */
void or_diffuse_wht(int n, cplx *a)
{
    or_wht(n, a);
    or_f0_scaled(n, a);
    or_wht(n, a);
}

/* Mean diffusion (inversion about the mean): mu = (1/N) sum_i a_i, then
 * a_i <- 2 mu - a_i (north star).  The global sum is the paper's
 * "accumulate and redistribute a sum" (Eq. 3). */
cplx or_sum(int n, const cplx *a)
{
    uint64_t N = 1ULL << n, i;
    long double sr = 0.0L, si = 0.0L, cr = 0.0L, ci = 0.0L;
    for (i = 0; i < N; ++i) {
        long double yr = (long double)creal(a[i]) - cr, yi = (long double)cimag(a[i]) - ci;
        long double tr = sr + yr, ti = si + yi;
        cr = (tr - sr) - yr; ci = (ti - si) - yi;
        sr = tr; si = ti;
    }
    return CMPLX((double)sr, (double)si);
}

void or_diffuse_mean(int n, cplx *a)
{
    uint64_t N = 1ULL << n, i;
    cplx mu = or_sum(n, a) * ldexp(1.0, -n);
    for (i = 0; i < N; ++i) a[i] = 2.0 * mu - a[i];
}

/* k Grover iterations a <- (D O)^k a.  diffusion: 0 = WHT, 1 = mean. */
void or_iterate(int n, cplx *a, const uint64_t *marked, uint64_t m, int k,
                int diffusion)
{
    int it;
    for (it = 0; it < k; ++it) {
        or_oracle_flip(a, marked, m);
        if (diffusion == 0) or_diffuse_wht(n, a);
        else or_diffuse_mean(n, a);
    }
}

/* ------------------------------------------------------------------------ */
/* Operational errors                                  */
/* ------------------------------------------------------------------------ */

/* "Imperfections in the laser apparatus result in deviations in the angle of
 * rotation" (section 2.0; operational errors, section 1.4,
 * P:2609-2614).  Reading G19: every Hadamard of a transform is the
 * reflection-rotation U(phi) = [[cos phi, sin phi], [sin phi, -cos phi]]
 * (Fig. 3's [w x; y z] with w = cos, x = y = sin, z = -cos), phi = pi/4 +
 * delta; ONE delta per (iteration t, transform w in {0,1}, qubit q), i.e. one
 * laser operation per qubit acting on all V/2 pairs.
 * Reading G20: delta = sigma * z, z standard normal by Box-Muller from the
 * counter hash: c = (2t + w) * 64 + q, u_j = ((hash64(key ^ (2c + j)) >> 11)
 * + 0.5) 2^-53, z = sqrt(-2 ln u_0) cos(2 pi u_1), key = hash64(seed ^ "NOIS").
 * With unitary (normalised) transforms F0 = 2|0><0| - I carries no 2^-n. */
#define OR_TAG_NOISE 0x4E4F495300000000ULL /* "NOIS" */

double or_noise_delta(uint64_t seed, uint64_t t, int w, int q, double sigma)
{
    uint64_t key = or_hash64(seed ^ OR_TAG_NOISE);
    uint64_t c = (2ULL * t + (uint64_t)w) * 64ULL + (uint64_t)q;
    uint64_t h0 = or_hash64(key ^ (2ULL * c));
    uint64_t h1 = or_hash64(key ^ (2ULL * c + 1ULL));
    double u0 = ((double)(h0 >> 11) + 0.5) * 0x1.0p-53;
    double u1 = ((double)(h1 >> 11) + 0.5) * 0x1.0p-53;
    return sigma * (sqrt(-2.0 * log(u0)) * cos(6.283185307179586 * u1));
}

/* One noisy transform: for q = 0..n-1 apply U(pi/4 + delta(t, w, q)). */
void or_noisy_transform(int n, cplx *a, uint64_t seed, uint64_t t, int w, double sigma)
{
    int q;
    for (q = 0; q < n; ++q) {
        double phi = 0.78539816339744831 + or_noise_delta(seed, t, w, q, sigma);
        double cs = cos(phi), sn = sin(phi);
        or_apply_2x2(n, a, q, cs, sn, sn, -cs);
    }
}

/* F0 = 2|0><0| - I without scale. */
void or_f0(int n, cplx *a)
{
    uint64_t N = 1ULL << n, i;
    for (i = 1; i < N; ++i) a[i] = -a[i];
}

/* k noisy Grover iterations (global iteration numbers t0 .. t0+k-1):
 * O, noisy transform w = 0, F0, noisy transform w = 1. */
void or_iterate_noisy(int n, cplx *a, const uint64_t *marked, uint64_t m, int k, double sigma,
                      uint64_t seed, uint64_t t0)
{
    int it;
    for (it = 0; it < k; ++it) {
        uint64_t t = t0 + (uint64_t)it;
        or_oracle_flip(a, marked, m);
        or_noisy_transform(n, a, seed, t, 0, sigma);
        or_f0(n, a);
        or_noisy_transform(n, a, seed, t, 1, sigma);
    }
}

/* ------------------------------------------------------------------------ */
/* Decoherence                                         */
/* ------------------------------------------------------------------------ */

/* "The decoherence step adds two additional operations for every laser
 * operation, and requires two messages to accumulate and redistribute the
 * sum" (Eq. 3 text).  Reading G22 (the
 * channel is not given; SPEC S:207-215's choice): after every laser operation
 * (the 2x2 on qubit q), (1) a contraction of a randomly selected site s: the
 * amplitudes with bit s = 1 are scaled by sqrt(1 - rate); (2) a global
 * renormalisation by the accumulated sum sum_i |a_i|^2 (the paper's global
 * sum).  s = hash64(key ^ c) mod n, c = (2t + w) * 64 + q, key = hash64(seed
 * ^ "DECO").  survival[t] = product over iteration t's laser operations of the
 * pre-renormalisation sums.  This follows the paper literally: one global sum
 * per laser operation. */
#define OR_TAG_DECO 0x4445434F00000000ULL /* "DECO" */

double or_norm_sq(int n, const cplx *a);

int or_decay_site(int n, uint64_t seed, uint64_t t, int w, int q)
{
    uint64_t key = or_hash64(seed ^ OR_TAG_DECO);
    uint64_t c = (2ULL * t + (uint64_t)w) * 64ULL + (uint64_t)q;
    return (int)(or_hash64(key ^ c) % (uint64_t)n);
}

static double or_contract_renormalise(int n, cplx *a, int s, double rate)
{
    uint64_t N = 1ULL << n, i, bit = 1ULL << s;
    double c = sqrt(1.0 - rate), sum, inv;
    for (i = 0; i < N; ++i)
        if (i & bit) a[i] = a[i] * c;
    sum = or_norm_sq(n, a);
    inv = 1.0 / sqrt(sum);
    for (i = 0; i < N; ++i) a[i] = a[i] * inv;
    return sum;
}

void or_iterate_decoherent(int n, cplx *a, const uint64_t *marked, uint64_t m, int k, double sigma,
                           double rate, uint64_t seed, uint64_t t0, double *survival)
{
    int it, w, q;
    for (it = 0; it < k; ++it) {
        uint64_t t = t0 + (uint64_t)it;
        double surv = 1.0;
        or_oracle_flip(a, marked, m);
        for (w = 0; w < 2; ++w) {
            if (w == 1) or_f0(n, a);
            for (q = 0; q < n; ++q) {
                double phi = 0.78539816339744831 + or_noise_delta(seed, t, w, q, sigma);
                double cs = cos(phi), sn = sin(phi);
                or_apply_2x2(n, a, q, cs, sn, sn, -cs);                         /* the laser operation */
                surv *= or_contract_renormalise(n, a, or_decay_site(n, seed, t, w, q), rate);
            }
        }
        if (survival) survival[it] = surv;
    }
}

/* ------------------------------------------------------------------------ */
/* Readouts                                                                 */
/* ------------------------------------------------------------------------ */

/* "The probability of each state is defined as the square of this complex
 * amplitude". */
void or_probabilities(int n, const cplx *a, double *p)
{
    uint64_t N = 1ULL << n, i;
    for (i = 0; i < N; ++i) p[i] = creal(a[i]) * creal(a[i]) + cimag(a[i]) * cimag(a[i]);
}

/* Seeded measurement of the whole register.  "This
 * measurement operation forces the state to one of the two values ... we must
 * describe the possible states ... in terms of their probability of
 * occurrence", probability = |a|^2.  Reading G21:
 * shot s draws u_s = ((hash64(key ^ s) >> 11) + 0.5) 2^-53, key =
 * hash64(seed ^ "SAMP"), and returns the smallest index i whose inclusive
 * cumulative probability C_i exceeds u_s * C_{N-1} (inverse CDF, normalised
 * by the total so a norm drift cannot push u past the end). */
#define OR_TAG_SAMPLE 0x53414D5000000000ULL /* "SAMP" */

double or_sample_uniform(uint64_t seed, uint64_t s)
{
    uint64_t key = or_hash64(seed ^ OR_TAG_SAMPLE);
    return ((double)(or_hash64(key ^ s) >> 11) + 0.5) * 0x1.0p-53;
}

/* cdf (N entries, caller-owned) receives the inclusive prefix sums. */
void or_sample(int n, const cplx *a, uint64_t shots, uint64_t seed, uint64_t *out, double *cdf)
{
    uint64_t N = 1ULL << n, i, s;
    long double acc = 0.0L;
    for (i = 0; i < N; ++i) {
        acc += (long double)(creal(a[i]) * creal(a[i]) + cimag(a[i]) * cimag(a[i]));
        cdf[i] = (double)acc;
    }
    for (s = 0; s < shots; ++s) {
        double target = or_sample_uniform(seed, s) * cdf[N - 1];
        uint64_t lo = 0, hi = N - 1;   /* smallest i with cdf[i] > target */
        while (lo < hi) {
            uint64_t md = (lo + hi) >> 1;
            if (cdf[md] > target) hi = md; else lo = md + 1;
        }
        out[s] = lo;
    }
}

double or_marked_mass(const cplx *a, const uint64_t *marked, uint64_t m)
{
    long double s = 0.0L;
    uint64_t j;
    for (j = 0; j < m; ++j) {
        cplx v = a[marked[j]];
        s += (long double)(creal(v) * creal(v) + cimag(v) * cimag(v));
    }
    return (double)s;
}

double or_norm_sq(int n, const cplx *a)
{
    uint64_t N = 1ULL << n, i;
    long double s = 0.0L;
    for (i = 0; i < N; ++i) s += (long double)(creal(a[i]) * creal(a[i]) + cimag(a[i]) * cimag(a[i]));
    return (double)s;
}

/* ------------------------------------------------------------------------ */
/* Brute force: the gate as a 2^n x 2^n matrix (section 1.3)   */
/* ------------------------------------------------------------------------ */

/* K = H (x) H (x) ... (x) H (n factors), H = 2^{-1/2} [[1,1],[1,-1]], built
 * by repeated Kronecker products: K_{m+1}[(r1,r0),(c1,c0)] = H[r1][c1] K_m[r0][c0].
 * Row-major, dim 2^n.  Only for n <= 8. */
int or_dense_hadamard(int n, double *K)
{
    static const double h = 0.70710678118654752440;
    const double H[2][2] = {{h, h}, {h, -h}};
    int m;
    uint64_t dim = 1;
    if (n < 0 || n > 8) return -1;
    K[0] = 1.0;
    for (m = 0; m < n; ++m) {
        uint64_t nd = dim * 2, r, c;
        double *tmp = (double *)malloc(sizeof(double) * nd * nd);
        for (r = 0; r < nd; ++r)
            for (c = 0; c < nd; ++c)
                tmp[r * nd + c] = H[r / dim][c / dim] * K[(r % dim) * dim + (c % dim)];
        memcpy(K, tmp, sizeof(double) * nd * nd);
        free(tmp);
        dim = nd;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Emulated sharding (section 3.1; Fig. 8)         */
/* ------------------------------------------------------------------------ */

/* The owner of a state is the concatenation of the parallel bits, MSB first
 * (P:4102-4103): with P = 2^g shards the parallel bits are the top g
 * bits, so shard r holds global indices [r N_l, (r+1) N_l), N_l = 2^{n-g}.
 *
 * The reorganisation (Fig. 8) that makes the top-g local bits the new
 * parallel bits: block (r, j) = elements of shard r whose top-g local bits
 * equal j; if the owner does not change (j == r) "do nothing", otherwise it
 * is sent to shard j and stored there as block r.  Applied twice it is the
 * identity.  shards[r] points to N_l amplitudes; tmp is scratch of N_l. */
void or_reorganize(int n, int g, cplx **shards, cplx *tmp_all)
{
    uint64_t P = 1ULL << g, Nl = 1ULL << (n - g), B = Nl / P, r, j, i;
    /* tmp_all holds P * N_l amplitudes: new shard j = concat_r old(r, j). */
    for (r = 0; r < P; ++r)
        for (j = 0; j < P; ++j)
            for (i = 0; i < B; ++i)
                tmp_all[j * Nl + r * B + i] = shards[r][j * B + i];
    for (j = 0; j < P; ++j)
        for (i = 0; i < Nl; ++i) shards[j][i] = tmp_all[j * Nl + i];
}

/* Unnormalised WHT over P = 2^g shards: local bits on every shard, one
 * reorganisation, the (new) top-g local bits, reorganise back.  Requires
 * 2g <= n.  Must equal or_wht on the concatenated vector. */
int or_wht_sharded(int n, int g, cplx *a_global)
{
    uint64_t P = 1ULL << g, Nl, r;
    int nl = n - g, q;
    cplx **sh;
    cplx *tmp;
    if (g < 0 || 2 * g > n) return -1;
    Nl = 1ULL << nl;
    sh = (cplx **)malloc(sizeof(cplx *) * P);
    tmp = (cplx *)malloc(sizeof(cplx) * P * Nl);
    for (r = 0; r < P; ++r) sh[r] = a_global + r * Nl;
    for (r = 0; r < P; ++r)
        for (q = 0; q < nl; ++q) or_apply_2x2(nl, sh[r], q, 1.0, 1.0, 1.0, -1.0);
    if (g > 0) {
        or_reorganize(n, g, sh, tmp);
        for (r = 0; r < P; ++r)
            for (q = nl - g; q < nl; ++q) or_apply_2x2(nl, sh[r], q, 1.0, 1.0, 1.0, -1.0);
        or_reorganize(n, g, sh, tmp);
    }
    free(tmp);
    free(sh);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: circuits of general (controlled) 2x2 gates                       */
/* ------------------------------------------------------------------------ */

/* One gate.  Section 2.1: "we describe each operation with a
 * VxV transformation matrix.  Because each gate only operates on a small
 * number of bits, these matrices are simply 2x2 or 4x4 matrices replicated
 * many times."  A gate here is Fig. 3's general 2x2 [w x; y z] on qubit
 * `target`, replicated over the V/2 pairs, and
 * applied only to the pairs whose `controls` qubits are all 1 (a controlled
 * 2x2 is the 4x4 of a two-bit gate, e.g. a controlled-NOT; reading G23).
 * m = {w.re, w.im, x.re, x.im, y.re, y.im, z.re, z.im}.  80 bytes. */
typedef struct {
    int32_t target;
    int32_t reserved;
    uint64_t controls; /* bit q set: qubit q must be 1 */
    double m[8];
} or_gate;

/* The V/2-pair loop of P:3080-3084, restricted to the pairs whose control
 * bits are all set. */
void or_apply_controlled_2x2(int n, cplx *a, int q, uint64_t controls, cplx w, cplx x, cplx y, cplx z)
{
    uint64_t N = 1ULL << n, bit = 1ULL << q, i;
    for (i = 0; i < N; ++i) {
        if (i & bit) continue;
        if ((i & controls) != controls) continue;
        {
            cplx a0 = a[i], a1 = a[i | bit];
            a[i] = w * a0 + x * a1;
            a[i | bit] = y * a0 + z * a1;
        }
    }
}

static int or_gate_valid(int n, const or_gate *g)
{
    uint64_t all = (n >= 64) ? ~0ULL : ((1ULL << n) - 1ULL);
    if (g->target < 0 || g->target >= n) return 0;
    if (g->controls & ~all) return 0;
    if ((g->controls >> g->target) & 1ULL) return 0;
    return 1;
}

/* Apply gates[0..count) in order.  Returns 0, or -1 (nothing applied) if a
 * gate has a target outside [0, n), a control >= n, or controls its own
 * target. */
int or_apply_gates(int n, cplx *a, const or_gate *g, uint64_t count)
{
    uint64_t j;
    for (j = 0; j < count; ++j)
        if (!or_gate_valid(n, &g[j])) return -1;
    for (j = 0; j < count; ++j)
        or_apply_controlled_2x2(n, a, g[j].target, g[j].controls, g[j].m[0] + I * g[j].m[1],
                                g[j].m[2] + I * g[j].m[3], g[j].m[4] + I * g[j].m[5], g[j].m[6] + I * g[j].m[7]);
    return 0;
}

/* The same circuit over P = 2^g shards, the paper's way (section 3.1,
 * P:4097-4113): shard r holds the states whose parallel bits concatenate to
 * r; "all of the processors can run in parallel operating only on local
 * data as long as they do not use any of the QU-bits in the set N.  When the
 * computation needs to operate on one of the bits in N, a new set is picked
 * and the simulator redistributes the data" (Fig. 8, or_reorganize).  The
 * new set is always the top g local positions, so the physical layout is
 * either natural or swapped (positions [nl-g, nl) <-> [nl, n)); a control on
 * a parallel bit is decided by the shard number.  The natural layout is
 * restored at the end.  Must equal or_apply_gates on the concatenated
 * vector.  Returns the number of reorganisations, or -1. */
int or_apply_gates_sharded(int n, int g, const or_gate *gates, uint64_t count, cplx *a_global)
{
    uint64_t P = 1ULL << g, Nl, r, j;
    int nl = n - g, swapped = 0, reorgs = 0, q;
    cplx **sh;
    cplx *tmp;
    if (g < 0 || 2 * g > n) return -1;
    for (j = 0; j < count; ++j)
        if (!or_gate_valid(n, &gates[j])) return -1;
    Nl = 1ULL << nl;
    sh = (cplx **)malloc(sizeof(cplx *) * P);
    tmp = (cplx *)malloc(sizeof(cplx) * P * Nl);
    for (r = 0; r < P; ++r) sh[r] = a_global + r * Nl;
    for (j = 0; j < count; ++j) {
        const or_gate *gt = &gates[j];
        int pt;
        /* physical position of logical qubit q */
#define OR_PHYS(q) ((!swapped) ? (q) : ((q) >= nl ? (q) - g : ((q) >= nl - g ? (q) + g : (q))))
        pt = OR_PHYS(gt->target);
        if (pt >= nl) {
            or_reorganize(n, g, sh, tmp);
            swapped ^= 1;
            ++reorgs;
            pt = OR_PHYS(gt->target);
        }
        for (r = 0; r < P; ++r) {
            uint64_t local_c = 0;
            int ok = 1;
            for (q = 0; q < n; ++q) {
                int pq;
                if (!((gt->controls >> q) & 1ULL)) continue;
                pq = OR_PHYS(q);
                if (pq < nl) local_c |= 1ULL << pq;
                else if (!((r >> (pq - nl)) & 1ULL)) ok = 0; /* parallel bit of shard r is 0 */
            }
            if (!ok) continue;
            or_apply_controlled_2x2(nl, sh[r], pt, local_c, gt->m[0] + I * gt->m[1], gt->m[2] + I * gt->m[3],
                                    gt->m[4] + I * gt->m[5], gt->m[6] + I * gt->m[7]);
        }
#undef OR_PHYS
    }
    if (swapped) {
        or_reorganize(n, g, sh, tmp);
        ++reorgs;
    }
    free(tmp);
    free(sh);
    return reorgs;
}
