// gates.cu -- gate-circuit tile pass: every gate of a
// planned pass (gate_plan.cpp) applied to a 2^T-amplitude tile on-chip, one
// HBM read + write per pass.
//
// What it computes: for each gate, Fig. 3's general 2x2 [w x; y z]
// on the pairs (a_i, a_{i | 2^t}) with bit t of i clear and all
// control bits of i set ("a 2x2 transformation on a vector of size V, is a
// sequence of V/2 independent 2x2 transformations"; G23 for the
// controls).
//
// How (B200 design): the tile machinery of the
// WHT pass (wht_kernels.cuh): 256 threads, 2^R amplitudes per thread in
// registers, three register layouts A/B/C that together cover the T tile
// bits, XOR-swizzled shared-memory relayouts with one barrier each, 128-bit
// coalesced global accesses in layout A.  A gate on tile bit b runs in a
// layout where b is a register bit (complex 2x2 on register pairs, no
// shared-memory traffic); the host orders the pass's ops to minimise
// relayouts (commuting gates only).  A control bit is a register-index
// predicate (register bit), a thread predicate (thread bit), or a tile
// predicate (slot outside the tile); controls on rank bits are decided per
// rank on the host.  The op program lives in device memory and is read with
// uniform (broadcast) loads.
#include <cuda_runtime.h>

#include <string.h>

#include <algorithm>

#include "wht_kernels.cuh"

namespace sv {

template <typename R>
struct alignas(16) GOp {
    R m[8];                  // w, x, y, z as (re, im)
    unsigned int ph;         // register layout (0 = A, 1 = B, 2 = C) | kind << 8
    unsigned int ri;         // register index of the target tile bit (whole kernel: target slot)
    unsigned int jm;         // controls that are register bits of ph (register-index space)
    unsigned int tm;         // controls that are thread bits of ph (tile-element space)
    unsigned long long fm;   // controls outside the tile (local index space; whole kernel: all controls)
};

// Matrix shape, decided on the host from the exact coefficients: the same
// [w x; y z] product with the zero terms (and unit factors) skipped, so the
// result is identical to the general formula up to the rounding of the
// skipped exact zeros / ones.
enum GateKind : unsigned int {
    GK_GENERAL = 0,   // [w x; y z]
    GK_DIAG = 1,      // x = y = 0: (w u, z v)
    GK_PHASE = 2,     // x = y = 0, w = 1: (u, z v)
    GK_ANTI = 3,      // w = z = 0: (x v, y u)
    GK_SWAP = 4,      // w = z = 0, x = y = 1 (NOT): (v, u)
};

// (u, v) <- (w u + x v, y u + z v), complex.
template <typename E, typename R>
__device__ __forceinline__ void cmat(E &u, E &v, const R (&m)[8]) {
    const E a = u, b = v;
    u.x = m[0] * a.x - m[1] * a.y + m[2] * b.x - m[3] * b.y;
    u.y = m[0] * a.y + m[1] * a.x + m[2] * b.y + m[3] * b.x;
    v.x = m[4] * a.x - m[5] * a.y + m[6] * b.x - m[7] * b.y;
    v.y = m[4] * a.y + m[5] * a.x + m[6] * b.y + m[7] * b.x;
}

// c <- (re, im) * c, complex
template <typename E, typename R>
__device__ __forceinline__ void cscale(E &c, R re, R im) {
    const E a = c;
    c.x = re * a.x - im * a.y;
    c.y = re * a.y + im * a.x;
}

template <unsigned int K, typename E, typename R>
__device__ __forceinline__ void cmat_k(E &u, E &v, const R (&m)[8]) {
    if constexpr (K == GK_GENERAL) {
        cmat(u, v, m);
    } else if constexpr (K == GK_DIAG) {
        cscale(u, m[0], m[1]);
        cscale(v, m[6], m[7]);
    } else if constexpr (K == GK_PHASE) {
        cscale(v, m[6], m[7]);
    } else if constexpr (K == GK_ANTI) {
        const E a = u, b = v;
        u.x = m[2] * b.x - m[3] * b.y;
        u.y = m[2] * b.y + m[3] * b.x;
        v.x = m[4] * a.x - m[5] * a.y;
        v.y = m[4] * a.y + m[5] * a.x;
    } else {
        const E a = u;
        u = v;
        v = a;
    }
}

template <int I, unsigned int K, int NR, typename E, typename R>
__device__ __forceinline__ void gate_apply(E (&x)[NR], const R (&m)[8], unsigned int jm) {
#pragma unroll
    for (int j = 0; j < NR; ++j)
        if (!(j & (1 << I)))
            if (((unsigned int)j & jm) == jm) cmat_k<K>(x[j], x[j | (1 << I)], m);
}

#ifndef SV_GATE_KINDS
#define SV_GATE_KINDS 2  // 2: all shapes; 1: general + phase; 0: general only (smaller code)
#endif
template <int I, int NR, typename E, typename R>
__device__ __forceinline__ void gate_apply_kind(E (&x)[NR], const R (&m)[8], unsigned int jm, unsigned int kind) {
#if SV_GATE_KINDS >= 2
    switch (kind) {
        case GK_DIAG: gate_apply<I, GK_DIAG>(x, m, jm); break;
        case GK_PHASE: gate_apply<I, GK_PHASE>(x, m, jm); break;
        case GK_ANTI: gate_apply<I, GK_ANTI>(x, m, jm); break;
        case GK_SWAP: gate_apply<I, GK_SWAP>(x, m, jm); break;
        default: gate_apply<I, GK_GENERAL>(x, m, jm); break;
    }
#elif SV_GATE_KINDS == 1
    if (kind == GK_PHASE) gate_apply<I, GK_PHASE>(x, m, jm);
    else gate_apply<I, GK_GENERAL>(x, m, jm);
#else
    (void)kind;
    gate_apply<I, GK_GENERAL>(x, m, jm);
#endif
}

template <class L, typename E, typename R>
__device__ __forceinline__ void gate_dispatch(E (&x)[L::NR], const R (&m)[8], unsigned int ri, unsigned int jm,
                                              unsigned int kind) {
    switch (ri) {
        case 0: gate_apply_kind<0>(x, m, jm, kind); break;
        case 1: gate_apply_kind<1>(x, m, jm, kind); break;
        case 2: gate_apply_kind<2>(x, m, jm, kind); break;
        case 3: gate_apply_kind<3>(x, m, jm, kind); break;
        default:
            if constexpr (L::kRB > 4) gate_apply_kind<(L::kRB > 4 ? 4 : 0)>(x, m, jm, kind);
            break;
    }
}

template <class L, typename E>
__device__ __forceinline__ void relayout_dyn(E (&x)[L::NR], E *sm, int tid, unsigned int from, unsigned int to) {
    switch (from * 3 + to) {
        case 1: relayout<L, 0, 1>(x, sm, tid); break;
        case 2: relayout<L, 0, 2>(x, sm, tid); break;
        case 3: relayout<L, 1, 0>(x, sm, tid); break;
        case 5: relayout<L, 1, 2>(x, sm, tid); break;
        case 6: relayout<L, 2, 0>(x, sm, tid); break;
        case 7: relayout<L, 2, 1>(x, sm, tid); break;
        default: break;
    }
}

template <typename R>
__device__ __forceinline__ void load_op(const GOp<R> *op, R (&m)[8], unsigned int &ph, unsigned int &ri,
                                        unsigned int &jm, unsigned int &tm, unsigned long long &fm) {
#pragma unroll
    for (int e = 0; e < 8; ++e) m[e] = __ldg(&op->m[e]);
    ph = __ldg(&op->ph);
    ri = __ldg(&op->ri);
    jm = __ldg(&op->jm);
    tm = __ldg(&op->tm);
    fm = __ldg(&op->fm);
}

template <typename E, int TB, int RB, bool XCHG>
__global__ void __launch_bounds__(1 << (TB - RB), (TB - RB <= 7) ? 4 : 2)
    gate_tile_kernel(const KParams p, const GOp<typename RealOf<E>::T> *__restrict__ ops, int nops) {
    using L = Layout<E, TB, RB>;
    using R = typename RealOf<E>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E *sm = reinterpret_cast<E *>(smem_raw);
    __shared__ E *s_dst[XCHG ? 8 : 1];
    if constexpr (XCHG) load_xdst(p, threadIdx.x, s_dst);
    const int tid = threadIdx.x;
    const unsigned long long base = tile_base(blockIdx.x, p.free_mask);
    E x[L::NR];
    global_load<L, 0>(x, reinterpret_cast<const E *>(p.in) + base, p, tid);
    const unsigned int eth[3] = {L::ethr(0, tid), L::ethr(1, tid), L::ethr(2, tid)};
    unsigned int cur = 0;
    for (int k = 0; k < nops; ++k) {
        R m[8];
        unsigned int ph, ri, jm, tm;
        unsigned long long fm;
        load_op(ops + k, m, ph, ri, jm, tm, fm);
        const unsigned int kind = ph >> 8;
        ph &= 0xffu;
        if (ph != cur) {
            relayout_dyn<L>(x, sm, tid, cur, ph);
            cur = ph;
        }
        const unsigned int et = cur == 0 ? eth[0] : (cur == 1 ? eth[1] : eth[2]);
        if ((et & tm) == tm && (base & fm) == fm) gate_dispatch<L>(x, m, ri, jm, kind);
    }
    E *gout = reinterpret_cast<E *>(p.out) + base;
    if (cur == 0) pass_store<L, 0, XCHG>(x, gout, base, p, tid, s_dst);
    else if (cur == 1) pass_store<L, 1, XCHG>(x, gout, base, p, tid, s_dst);
    else pass_store<L, 2, XCHG>(x, gout, base, p, tid, s_dst);
}

// Whole state (n <= T) in one CTA: every gate as a V/2-pair loop over shared
// memory, one barrier per gate.
template <typename E>
__global__ void __launch_bounds__(512) gate_whole_kernel(E *a, int n, const GOp<typename RealOf<E>::T> *ops,
                                                         int nops) {
    using R = typename RealOf<E>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    E *s = reinterpret_cast<E *>(smem_raw);
    const unsigned int N = 1u << n, tid = threadIdx.x, nt = blockDim.x;
    for (unsigned int i = tid; i < N; i += nt) s[i] = a[i];
    __syncthreads();
    for (int k = 0; k < nops; ++k) {
        R m[8];
        unsigned int ph, q, jm, tm;
        unsigned long long cm;
        load_op(ops + k, m, ph, q, jm, tm, cm);
        const unsigned int kind = ph >> 8;
        const unsigned int bit = 1u << q;
        for (unsigned int pr = tid; pr < N / 2; pr += nt) {
            const unsigned int i = ((pr >> q) << (q + 1)) | (pr & (bit - 1));
            if ((i & (unsigned int)cm) == (unsigned int)cm) {
                switch (kind) {
                    case GK_DIAG: cmat_k<GK_DIAG>(s[i], s[i | bit], m); break;
                    case GK_PHASE: cmat_k<GK_PHASE>(s[i], s[i | bit], m); break;
                    case GK_ANTI: cmat_k<GK_ANTI>(s[i], s[i | bit], m); break;
                    case GK_SWAP: cmat_k<GK_SWAP>(s[i], s[i | bit], m); break;
                    default: cmat_k<GK_GENERAL>(s[i], s[i | bit], m); break;
                }
            }
        }
        __syncthreads();
    }
    for (unsigned int i = tid; i < N; i += nt) a[i] = s[i];
}

// ------------------------------------------------------------------------- //
// Host: op programs                                                          //
// ------------------------------------------------------------------------- //
namespace {

unsigned int gate_kind(const sv_gate &g) {
    const double *m = g.m;
    const bool offzero = m[2] == 0.0 && m[3] == 0.0 && m[4] == 0.0 && m[5] == 0.0;
    const bool diagzero = m[0] == 0.0 && m[1] == 0.0 && m[6] == 0.0 && m[7] == 0.0;
    if (offzero) return (m[0] == 1.0 && m[1] == 0.0) ? GK_PHASE : GK_DIAG;
    if (diagzero) return (m[2] == 1.0 && m[3] == 0.0 && m[4] == 1.0 && m[5] == 0.0) ? GK_SWAP : GK_ANTI;
    return GK_GENERAL;
}

template <typename R>
GOp<R> op_coefs(const sv_gate &g) {
    GOp<R> o{};
    for (int e = 0; e < 8; ++e) o.m[e] = (R)g.m[e];
    o.ph = gate_kind(g) << 8;
    return o;
}

// Program of one tile pass for the three-layout family L: tile bits, the
// layout schedule and the per-op predicates.
template <class L, typename R>
void build_tile_ops(const GatePassArgs &a, std::vector<GOp<R>> &out) {
    int slot2bit[64];
    for (int i = 0; i < 64; ++i) slot2bit[i] = -1;
    int b = 0;
    for (int sl = 0; sl < 64; ++sl)
        if ((a.tile_mask >> sl) & 1) slot2bit[sl] = b++;
    struct Pend {
        sv_gate g;           // the gate (matrix possibly fused with later ones)
        int bt;              // target tile bit
        unsigned int tc;     // controls on tile bits (tile-element space)
        unsigned long long fm;
    };
    std::vector<Pend> pend;
    for (uint64_t k = 0; k < a.count; ++k) {
        const sv_gate &g = a.gates[a.order[k]];
        const int pt = gate_phys(g.target, a.nl, a.g, a.swapped);
        SV_CHECK(slot2bit[pt] >= 0, SV_EINVAL, "internal: gate target outside its pass tile");
        Pend pd{g, slot2bit[pt], 0u, 0ull};
        bool live = true;
        for (int q = 0; q < a.n; ++q) {
            if (!((g.controls >> q) & 1ull)) continue;
            const int pq = gate_phys(q, a.nl, a.g, a.swapped);
            if (pq >= a.nl && !a.emulated) {  // rank bit of a real rank
                if (!((a.rank >> (pq - a.nl)) & 1)) live = false;
            } else if (slot2bit[pq] >= 0) {
                pd.tc |= 1u << slot2bit[pq];
            } else {
                pd.fm |= 1ull << pq;
            }
        }
        if (!live) continue;
        // Fusion: a gate with the same target and controls as an earlier op
        // of this pass, with only commuting ops in between, is multiplied
        // into it (host fp64 2x2 product M_later * M_earlier).
        bool fused = false;
        CommuteSet between;
        for (size_t i = pend.size(); i-- > 0;) {
            sv_gate &e = pend[i].g;
            if (e.target == g.target && e.controls == g.controls && between.commutes(g)) {
                double r[8];
                for (int rr = 0; rr < 2; ++rr)
                    for (int cc = 0; cc < 2; ++cc) {
                        double re = 0.0, im = 0.0;
                        for (int kk = 0; kk < 2; ++kk) {
                            const double ar = g.m[2 * (2 * rr + kk)], ai = g.m[2 * (2 * rr + kk) + 1];
                            const double br = e.m[2 * (2 * kk + cc)], bi = e.m[2 * (2 * kk + cc) + 1];
                            re += ar * br - ai * bi;
                            im += ar * bi + ai * br;
                        }
                        r[2 * (2 * rr + cc)] = re;
                        r[2 * (2 * rr + cc) + 1] = im;
                    }
                for (int t = 0; t < 8; ++t) e.m[t] = r[t];
                fused = true;
                break;
            }
            between.add(e);
            if (!between.commutes(g)) break;
        }
        if (!fused) pend.push_back(pd);
    }
    // Layout schedule: in the current layout run every ready op (commutes
    // with all earlier pending ops) whose target is a register bit; when none
    // is left, move to the layout that runs the most ready ops next.
    auto ready_in = [&](int ph, std::vector<size_t> *take) {
        CommuteSet skipped;
        int cnt = 0;
        for (size_t i = 0; i < pend.size(); ++i) {
            if (skipped.commutes(pend[i].g) && L::is_reg(ph, pend[i].bt)) {
                ++cnt;
                if (take) take->push_back(i);
            } else {
                skipped.add(pend[i].g);
            }
        }
        return cnt;
    };
    int cur = 0;
    std::vector<size_t> take;
    while (!pend.empty()) {
        take.clear();
        ready_in(cur, &take);
        if (take.empty()) {
            int best = -1, bc = -1;
            for (int ph = 0; ph < 3; ++ph) {
                if (ph == cur) continue;
                const int c = ready_in(ph, nullptr);
                if (c > bc) { bc = c; best = ph; }
            }
            SV_CHECK(bc > 0, SV_EINVAL, "internal: gate layout schedule stuck");
            cur = best;
            continue;
        }
        std::vector<char> used(pend.size(), 0);
        for (size_t i : take) {
            const Pend &pd = pend[i];
            GOp<R> o = op_coefs<R>(pd.g);
            o.ph |= (unsigned int)cur;
            o.ri = 0;
            for (int r = 0; r < L::kRB; ++r)
                if (L::reg_bit(cur, r) == pd.bt) o.ri = (unsigned int)r;
            o.jm = 0;
            o.tm = 0;
            for (int tbit = 0; tbit < L::kTB; ++tbit) {
                if (!((pd.tc >> tbit) & 1u)) continue;
                bool reg = false;
                for (int r = 0; r < L::kRB; ++r)
                    if (L::reg_bit(cur, r) == tbit) { o.jm |= 1u << r; reg = true; }
                if (!reg) o.tm |= 1u << tbit;
            }
            o.fm = pd.fm;
            out.push_back(o);
            used[i] = 1;
        }
        std::vector<Pend> rest;
        for (size_t i = 0; i < pend.size(); ++i)
            if (!used[i]) rest.push_back(pend[i]);
        pend.swap(rest);
    }
}

template <typename R>
size_t append_ops(const std::vector<GOp<R>> &ops, std::vector<unsigned char> &prog) {
    const size_t off = prog.size();
    prog.resize(off + ops.size() * sizeof(GOp<R>));
    if (!ops.empty()) memcpy(prog.data() + off, ops.data(), ops.size() * sizeof(GOp<R>));
    return ops.size();
}

template <typename E, int TB, int RB>
void launch_tile_gates(const GatePassArgs &a, const void *dev_ops, uint64_t nops, cudaStream_t s) {
    using L = Layout<E, TB, RB>;
    using R = typename RealOf<E>::T;
    KParams kp{};
    kp.in = a.in;
    kp.out = a.out;
    kp.xchg = a.xchg_nl > 0 ? 1 : 0;
    if (kp.xchg) {
        SV_CHECK(a.xchg_g >= 1 && a.xchg_g <= 3 && a.xchg_nl - a.xchg_g >= 1, SV_EINVAL,
                 "internal: fused exchange supports 2..8 ranks");
        kp.xnl = a.xchg_nl;
        kp.xg = a.xchg_g;
        kp.xrank = a.xchg_rank;
        for (int i = 0; i < 8; ++i) kp.xdst[i] = i < (1 << a.xchg_g) ? a.xchg_dst[i] : nullptr;
    }
    int b = 0, f = 0;
    kp.free_mask = 0;
    for (int sl = 0; sl < a.total_bits; ++sl) {
        if ((a.tile_mask >> sl) & 1) {
            SV_CHECK(b < 16, SV_EINVAL, "internal: tile too large");
            kp.slot[b++] = (signed char)sl;
        } else {
            kp.free_mask |= 1ull << sl;
            ++f;
        }
    }
    SV_CHECK(b == TB, SV_EINVAL, "internal: gate tile mask does not have T slots");
    SV_CHECK(nops <= 0x7fffffffull, SV_EINVAL, "too many gates in one pass");
    const unsigned long long ntiles = 1ull << f;
    SV_CHECK(ntiles <= 0x7fffffffull, SV_EINVAL, "too many tiles for one launch");
    auto fn = kp.xchg ? gate_tile_kernel<E, TB, RB, true> : gate_tile_kernel<E, TB, RB, false>;
    const int smem = (1 << TB) * (int)sizeof(E);
    static bool attr = false;
    if (!attr) {
        SV_CUDA(cudaFuncSetAttribute(gate_tile_kernel<E, TB, RB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
        SV_CUDA(cudaFuncSetAttribute(gate_tile_kernel<E, TB, RB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
        attr = true;
    }
    fn<<<(unsigned int)ntiles, L::NT, smem, s>>>(kp, reinterpret_cast<const GOp<R> *>(dev_ops), (int)nops);
    SV_CUDA(cudaGetLastError());
}

template <typename E>
void whole_ops(const GatePassArgs &a, std::vector<GOp<typename RealOf<E>::T>> &ops) {
    using R = typename RealOf<E>::T;
    for (uint64_t k = 0; k < a.count; ++k) {
        const sv_gate &g = a.gates[a.order[k]];
        GOp<R> o = op_coefs<R>(g);
        o.ri = (unsigned int)g.target;
        o.fm = g.controls;
        ops.push_back(o);
    }
}

template <typename E>
void launch_whole_gates(const GatePassArgs &a, const void *dev_ops, uint64_t nops, cudaStream_t s) {
    using R = typename RealOf<E>::T;
    if (nops == 0) return;
    SV_CHECK(nops <= 0x7fffffffull, SV_EINVAL, "too many gates");
    const unsigned int N = 1u << a.n;
    const int threads = N >= 1024 ? 512 : (N / 2 >= 32 ? (int)(N / 2) : 32);
    const int smem = (int)(N * sizeof(E));
    SV_CUDA(cudaFuncSetAttribute(gate_whole_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    gate_whole_kernel<E><<<1, threads, smem, s>>>(reinterpret_cast<E *>(a.in), a.n,
                                                   reinterpret_cast<const GOp<R> *>(dev_ops), (int)nops);
    SV_CUDA(cudaGetLastError());
}

}  // namespace

uint64_t build_gate_ops(sv_dtype dt, const GatePassArgs &a, bool whole, std::vector<unsigned char> &prog) {
    // every op record is 16-byte aligned inside the program
    prog.resize((prog.size() + 15) & ~(size_t)15);
    if (dt == SV_C64) {
        std::vector<GOp<float>> ops;
        if (whole) whole_ops<float2>(a, ops);
        else build_tile_ops<Layout<float2, kGateTileBitsC64, kRegBitsC64>, float>(a, ops);
        return append_ops(ops, prog);
    }
    std::vector<GOp<double>> ops;
    if (whole) whole_ops<double2>(a, ops);
    else build_tile_ops<Layout<double2, kTileBitsC128, kRegBitsC128>, double>(a, ops);
    return append_ops(ops, prog);
}

void launch_gate_pass(sv_dtype dt, const GatePassArgs &a, const void *dev_ops, uint64_t nops, cudaStream_t s) {
    if (dt == SV_C64) launch_tile_gates<float2, kGateTileBitsC64, kRegBitsC64>(a, dev_ops, nops, s);
    else launch_tile_gates<double2, kTileBitsC128, kRegBitsC128>(a, dev_ops, nops, s);
}

void launch_gate_whole(sv_dtype dt, const GatePassArgs &a, const void *dev_ops, uint64_t nops, cudaStream_t s) {
    if (dt == SV_C64) launch_whole_gates<float2>(a, dev_ops, nops, s);
    else launch_whole_gates<double2>(a, dev_ops, nops, s);
}

}  // namespace sv
