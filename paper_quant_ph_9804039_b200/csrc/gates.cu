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
#include <complex>
#include <memory>

#include "gate_kernels.cuh"

namespace sv {

// gate_jit.cu: pass-specialised kernels compiled at run time (complex64, no exchange store)
void *gate_jit_prepare(const void *host_ops, uint64_t nops, bool lin, bool param, bool l2, unsigned long long ntiles,
                       uint64_t call);
void launch_gate_jit(void *kern, const KParams &kp, const void *dev_ops, const void *host_ops, uint64_t nops,
                     bool lin, bool param, unsigned long long ntiles, cudaStream_t s);
size_t gate_jit_compile_only(const void *host_ops, uint64_t nops, bool lin, bool glb, bool l2);
void gate_jit_stats(uint64_t *compiles, double *seconds);

// ------------------------------------------------------------------------- //
// Host: op programs                                                          //
// ------------------------------------------------------------------------- //
namespace {

// SV_GATE_L2=0: every tile pass on the three-layout family (A/B).
bool gate_l2_enabled() {
    static const bool on = [] {
        const char *e = getenv("SV_GATE_L2");
        return !(e && strcmp(e, "0") == 0);
    }();
    return on;
}

bool gate_pass_l2(sv_dtype dt, const GatePassArgs &a);

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
    if constexpr (kNM<R> == 16)
        for (int q = 0; q < 4; ++q) {
            o.m[8 + 2 * q] = -(R)g.m[2 * q + 1];
            o.m[9 + 2 * q] = (R)g.m[2 * q + 1];
        }
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
    struct LinEntry {
        int where;   // 0 tile bit, 1 free slot, 2 none
        int bit;     // tile bit / slot
        double zr, zi;
        sv_gate src;           // the original gate (a short run is emitted gate by gate)
        unsigned int tc;
        unsigned long long fm;
    };
    struct Pend {
        sv_gate g;           // the gate (matrix possibly fused with later ones); for a merged phase
                             // run: diag(1, 1) with the union of the controls (commutation proxy)
        int bt;              // target tile bit
        unsigned int tc;     // controls on tile bits (tile-element space)
        unsigned long long fm;
        std::vector<LinEntry> lin;  // non-empty: a merged run of phase gates (GK_LINPHASE)
    };
    std::vector<Pend> pend;
    for (uint64_t k = 0; k < a.count; ++k) {
        const sv_gate &g = a.gates[a.order[k]];
        const int pt = gate_phys(g.target, a.nl, a.g, a.swapped);
        SV_CHECK(slot2bit[pt] >= 0, SV_EINVAL, "internal: gate target outside its pass tile");
        Pend pd{g, slot2bit[pt], 0u, 0ull, {}};
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
        // Phase gates diag(1, z) with at most one (live) control are merged
        // into a run on their target (GK_LINPHASE) when only commuting ops lie
        // between -- checked before the 2x2 fusion below.
        const bool phase1 = gate_kind(g) == GK_PHASE && __builtin_popcount(pd.tc) + __builtin_popcountll(pd.fm) <= 1;
        if (phase1) {
            LinEntry le{2, 0, g.m[6], g.m[7], g, pd.tc, pd.fm};
            if (pd.tc) { le.where = 0; le.bit = __builtin_ctz(pd.tc); }
            else if (pd.fm) { le.where = 1; le.bit = __builtin_ctzll(pd.fm); }
            bool merged = false;
            CommuteSet between;
            for (size_t i = pend.size(); i-- > 0;) {
                Pend &e = pend[i];
                if (!e.lin.empty() && e.bt == pd.bt && between.commutes(g)) {
                    e.lin.push_back(le);
                    e.g.controls |= g.controls;
                    merged = true;
                    break;
                }
                between.add(e.g);
                if (!between.commutes(g)) break;
            }
            if (merged) continue;
            pd.lin.push_back(le);
            pd.g.m[6] = 1.0;  // proxy: diagonal, support = target + controls
            pd.g.m[7] = 0.0;
            pend.push_back(pd);
            continue;
        }
        // Fusion: a gate with the same target and controls as an earlier op
        // of this pass, with only commuting ops in between, is multiplied
        // into it (host fp64 2x2 product M_later * M_earlier).
        bool fused = false;
        CommuteSet between;
        for (size_t i = pend.size(); i-- > 0;) {
            sv_gate &e = pend[i].g;
            if (pend[i].lin.empty() && e.target == g.target && e.controls == g.controls && between.commutes(g)) {
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
    // A merged phase run pays ~40 complex multiplies per thread for its
    // factor tables: runs of fewer than kMinLinRun gates go back to one op
    // per gate (all diagonal: they commute, so their order is free).
    constexpr size_t kMinLinRun = 4;
    {
        std::vector<Pend> expanded;
        for (Pend &pd : pend) {
            if (pd.lin.empty() || pd.lin.size() >= kMinLinRun) {
                expanded.push_back(std::move(pd));
                continue;
            }
            for (const LinEntry &le : pd.lin) expanded.push_back(Pend{le.src, pd.bt, le.tc, le.fm, {}});
        }
        pend.swap(expanded);
    }
    // Layout schedule: in the current layout run every ready op (commutes
    // with all earlier pending ops) whose target is a register bit; when none
    // is left, move to the layout that runs the most ready ops next.
    auto ready_in = [&](int ph, std::vector<size_t> *take) {
        CommuteSet skipped;
        int cnt = 0;
        for (size_t i = 0; i < pend.size(); ++i) {
            // a merged phase run or a diagonal gate needs no register target: it runs in any layout
            if (skipped.commutes(pend[i].g) &&
                (!pend[i].lin.empty() || gate_diag(pend[i].g) || L::is_reg(ph, pend[i].bt))) {
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
            for (int ph = 0; ph < L::kNPH; ++ph) {
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
            if (!pd.lin.empty()) {
                GOp<R> o{};
                o.ph = (GK_LINPHASE << 8) | (unsigned int)cur;
                o.ri = LP_THR;
                o.jm = (unsigned int)pd.bt;
                for (int r = 0; r < L::kRB; ++r)
                    if (L::reg_bit(cur, r) == pd.bt) { o.ri = LP_REG; o.jm = (unsigned int)r; }
                // host fp64 products: per register bit of this layout, per
                // thread tile bit, per free slot, and the constant factor
                std::complex<double> preg[16], pthr[16], pconst(1.0, 0.0);
                std::vector<std::pair<int, std::complex<double>>> pfree;
                for (int r = 0; r < 16; ++r) { preg[r] = 1.0; pthr[r] = 1.0; }
                for (const LinEntry &le : pd.lin) {
                    const std::complex<double> z(le.zr, le.zi);
                    if (le.where == 2) { pconst *= z; continue; }
                    if (le.where == 1) {
                        bool found = false;
                        for (auto &f : pfree)
                            if (f.first == le.bit) { f.second *= z; found = true; }
                        if (!found) pfree.push_back({le.bit, z});
                        continue;
                    }
                    int reg = -1;
                    for (int r = 0; r < L::kRB; ++r)
                        if (L::reg_bit(cur, r) == le.bit) reg = r;
                    if (reg >= 0) preg[reg] *= z;
                    else pthr[le.bit] *= z;
                }
                std::vector<GOp<R>> ent;
                auto rec = [&](unsigned int w, unsigned int bit, std::complex<double> z) {
                    GOp<R> e{};
                    e.m[0] = (R)z.real();
                    e.m[1] = (R)z.imag();
                    e.ri = w;
                    e.jm = bit;
                    ent.push_back(e);
                };
                for (int r = 0; r < L::kRB; ++r) rec(LP_REG, (unsigned int)r, preg[r]);
                for (int t = 0; t < L::kTB; ++t)
                    if (pthr[t] != std::complex<double>(1.0, 0.0)) rec(LP_THR, (unsigned int)t, pthr[t]);
                o.fm = ent.size() - (size_t)L::kRB;  // thread-bit entries come first
                if (pconst != std::complex<double>(1.0, 0.0)) rec(LP_CONST, 0u, pconst);
                for (auto &f : pfree) rec(LP_FREE, (unsigned int)f.first, f.second);
                o.tm = (unsigned int)ent.size();
                out.push_back(o);
                out.insert(out.end(), ent.begin(), ent.end());
                used[i] = 1;
                continue;
            }
            GOp<R> o = op_coefs<R>(pd.g);
            o.ph |= (unsigned int)cur;
            o.ri = 0;
            bool treg = false;
            for (int r = 0; r < L::kRB; ++r)
                if (L::reg_bit(cur, r) == pd.bt) { o.ri = (unsigned int)r; treg = true; }
            if (!treg) {  // only diagonal gates are scheduled off a register target
                SV_CHECK(gate_diag(pd.g), SV_EINVAL, "internal: non-diagonal gate without a register target");
                o.ph = (GK_DIAGT << 8) | (unsigned int)cur;
                o.ri = (unsigned int)pd.bt;
            }
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
uint64_t relayouts_of(const std::vector<GOp<R>> &ops) {
    uint64_t r = 0;
    unsigned int cur = 0;
    for (size_t k = 0; k < ops.size(); ++k) {  // as the kernel's op loop walks the program
        const unsigned int ph = ops[k].ph & 0xffu, kind = ops[k].ph >> 8;
        if (ph != cur) {
            ++r;
            cur = ph;
        }
        if (kind == GK_LINPHASE) k += ops[k].tm;  // its entry records
    }
    return r;
}

// The two-layout family (Layout2, wht_kernels.cuh) for a complex64 tile pass
// whose non-diagonal gate targets all lie on tile bits >= 3 with the lowest at
// 3 or 4 -- a strided pass with 64-128 B runs, the WHT's rule for Layout2
// (SV_2LAYOUT_MAX_U) -- unless its program needs more relayouts there than on
// the three-layout family (gates alternating between A- and B-layout targets
// without commuting).  Diagonal gates and merged phase runs need no register
// target.  A pure function of the pass, so the program builder, the launcher
// and the relayout count agree.
bool gate_pass_l2(sv_dtype dt, const GatePassArgs &a) {
    if (dt != SV_C64 || !gate_l2_enabled()) return false;
    int slot2bit[64];
    for (int i = 0; i < 64; ++i) slot2bit[i] = -1;
    int b = 0;
    for (int sl = 0; sl < 64; ++sl)
        if ((a.tile_mask >> sl) & 1) slot2bit[sl] = b++;
    if (b != kGateTileBitsC64) return false;
    int lo = 64;
    for (uint64_t k = 0; k < a.count; ++k) {
        const sv_gate &g = a.gates[a.order[k]];
        if (gate_diag(g)) continue;
        const int bt = slot2bit[gate_phys(g.target, a.nl, a.g, a.swapped)];
        if (bt >= 0 && bt < lo) lo = bt;
    }
    static const int max_u = [] {  // SV_GATE_L2_MAXU: A/B of the upper bound
        const char *e = getenv("SV_GATE_L2_MAXU");
        return e ? atoi(e) : SV_2LAYOUT_MAX_U;
    }();
    if (!(lo >= 3 && lo <= max_u && lo < 64)) return false;
    std::vector<GOp<float>> o2, o3;
    build_tile_ops<Layout2<kGateTileBitsC64, kRegBitsC64>, float>(a, o2);
    build_tile_ops<Layout<float2, kGateTileBitsC64, kRegBitsC64>, float>(a, o3);
    return relayouts_of(o2) <= relayouts_of(o3);
}

template <typename R>
size_t append_ops(const std::vector<GOp<R>> &ops, std::vector<unsigned char> &prog) {
    const size_t off = prog.size();
    prog.resize(off + ops.size() * sizeof(GOp<R>));
    if (!ops.empty()) memcpy(prog.data() + off, ops.data(), ops.size() * sizeof(GOp<R>));
    return ops.size();
}

// SV_GATE_PARAM_OPS=0: always read the op program from global memory (A/B).
inline bool gate_param_ops() {
    static const int mode = [] {
        const char *e = getenv("SV_GATE_PARAM_OPS");
        return e ? atoi(e) : 1;
    }();
    return mode != 0;
}

template <typename E, int TB, int RB>
void launch_tile_gates(const GatePassArgs &a, const void *dev_ops, const void *host_ops, uint64_t nops, bool lin,
                       cudaStream_t s) {
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
    kp_set_free_runs(kp);
    SV_CHECK(nops <= 0x7fffffffull, SV_EINVAL, "too many gates in one pass");
    const unsigned long long ntiles = 1ull << f;
    SV_CHECK(ntiles <= 0x7fffffffull, SV_EINVAL, "too many tiles for one launch");
    const int smem = (1 << TB) * (int)sizeof(E);
    const bool l2 = gate_pass_l2(sizeof(E) == 8 ? SV_C64 : SV_C128, a);
    static bool attr = false;
    if (!attr) {
        for (auto f : {gate_tile_kernel<E, TB, RB, true, true>, gate_tile_kernel<E, TB, RB, false, true>,
                       gate_tile_kernel<E, TB, RB, true, false>, gate_tile_kernel<E, TB, RB, false, false>})
            SV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (auto f : {gate_tile_kernel_p<E, TB, RB, true, true>, gate_tile_kernel_p<E, TB, RB, false, true>,
                       gate_tile_kernel_p<E, TB, RB, true, false>, gate_tile_kernel_p<E, TB, RB, false, false>})
            SV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        if constexpr (sizeof(E) == 8) {
            for (auto f : {gate_tile_kernel<E, TB, RB, true, true, true>, gate_tile_kernel<E, TB, RB, false, true, true>,
                           gate_tile_kernel<E, TB, RB, true, false, true>, gate_tile_kernel<E, TB, RB, false, false, true>})
                SV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            for (auto f : {gate_tile_kernel_p<E, TB, RB, true, true, true>, gate_tile_kernel_p<E, TB, RB, false, true, true>,
                           gate_tile_kernel_p<E, TB, RB, true, false, true>,
                           gate_tile_kernel_p<E, TB, RB, false, false, true>})
                SV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        }
        attr = true;
    }
    constexpr uint64_t cap = sizeof(GProg<R>) / sizeof(GOp<R>);
    if constexpr (sizeof(E) == 8 && TB == kGateTileBitsC64) {
        // complex64, no exchange store: the pass-specialised kernel (bitwise the
        // interpreter's result; same program flavour for merged phase runs)
        const bool param = host_ops != nullptr && nops <= cap && gate_param_ops();
        if (a.jit_prepare) {
            if (!kp.xchg && a.jit_kern)
                *a.jit_kern = gate_jit_prepare(host_ops, nops, lin, param, l2, ntiles, a.jit_prepare);
            return;
        }
        if (!kp.xchg && a.jit_kern && *a.jit_kern) {
            launch_gate_jit(*a.jit_kern, kp, dev_ops, host_ops, nops, lin, param, ntiles, s);
            return;
        }
    }
    if (a.jit_prepare) return;
    const bool param = host_ops != nullptr && nops <= cap && gate_param_ops();
    // (xchg, lin, l2) -> instantiation
    auto pick = [&](auto k_ff, auto k_tf, auto k_ft, auto k_tt) { return kp.xchg ? (lin ? k_tt : k_tf) : (lin ? k_ft : k_ff); };
    if (param) {
        auto prog = std::make_unique<GProg<R>>();
        memcpy(prog->op, host_ops, nops * sizeof(GOp<R>));
        auto fn = pick(gate_tile_kernel_p<E, TB, RB, false, false>, gate_tile_kernel_p<E, TB, RB, true, false>,
                       gate_tile_kernel_p<E, TB, RB, false, true>, gate_tile_kernel_p<E, TB, RB, true, true>);
        if constexpr (sizeof(E) == 8)
            if (l2)
                fn = pick(gate_tile_kernel_p<E, TB, RB, false, false, true>, gate_tile_kernel_p<E, TB, RB, true, false, true>,
                          gate_tile_kernel_p<E, TB, RB, false, true, true>, gate_tile_kernel_p<E, TB, RB, true, true, true>);
        fn<<<(unsigned int)ntiles, L::NT, smem, s>>>(kp, *prog, (int)nops);
    } else {
        auto fn = pick(gate_tile_kernel<E, TB, RB, false, false>, gate_tile_kernel<E, TB, RB, true, false>,
                       gate_tile_kernel<E, TB, RB, false, true>, gate_tile_kernel<E, TB, RB, true, true>);
        if constexpr (sizeof(E) == 8)
            if (l2)
                fn = pick(gate_tile_kernel<E, TB, RB, false, false, true>, gate_tile_kernel<E, TB, RB, true, false, true>,
                          gate_tile_kernel<E, TB, RB, false, true, true>, gate_tile_kernel<E, TB, RB, true, true, true>);
        fn<<<(unsigned int)ntiles, L::NT, smem, s>>>(kp, reinterpret_cast<const GOp<R> *>(dev_ops), (int)nops);
    }
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

uint64_t build_gate_ops(sv_dtype dt, const GatePassArgs &a, bool whole, std::vector<unsigned char> &prog,
                        bool *has_lin) {
    // every op record is 16-byte aligned inside the program
    prog.resize((prog.size() + 15) & ~(size_t)15);
    auto lin_in = [](const auto &ops) {
        for (const auto &o : ops)
            if ((o.ph >> 8) == GK_LINPHASE) return true;
        return false;
    };
    if (dt == SV_C64) {
        std::vector<GOp<float>> ops;
        if (whole) whole_ops<float2>(a, ops);
        else if (gate_pass_l2(dt, a)) build_tile_ops<Layout2<kGateTileBitsC64, kRegBitsC64>, float>(a, ops);
        else build_tile_ops<Layout<float2, kGateTileBitsC64, kRegBitsC64>, float>(a, ops);
        if (has_lin) *has_lin = lin_in(ops);
        return append_ops(ops, prog);
    }
    std::vector<GOp<double>> ops;
    if (whole) whole_ops<double2>(a, ops);
    else build_tile_ops<Layout<double2, kTileBitsC128, kRegBitsC128>, double>(a, ops);
    if (has_lin) *has_lin = lin_in(ops);
    return append_ops(ops, prog);
}

uint64_t count_gate_relayouts(sv_dtype dt, const GatePassArgs &a) {
    if (dt == SV_C64) {
        std::vector<GOp<float>> ops;
        if (gate_pass_l2(dt, a)) build_tile_ops<Layout2<kGateTileBitsC64, kRegBitsC64>, float>(a, ops);
        else build_tile_ops<Layout<float2, kGateTileBitsC64, kRegBitsC64>, float>(a, ops);
        return relayouts_of(ops);
    }
    std::vector<GOp<double>> ops;
    build_tile_ops<Layout<double2, kTileBitsC128, kRegBitsC128>, double>(a, ops);
    return relayouts_of(ops);
}

void launch_gate_pass(sv_dtype dt, const GatePassArgs &a, const void *dev_ops, const void *host_ops, uint64_t nops,
                      bool has_lin, cudaStream_t s) {
    if (dt == SV_C64) launch_tile_gates<float2, kGateTileBitsC64, kRegBitsC64>(a, dev_ops, host_ops, nops, has_lin, s);
    else launch_tile_gates<double2, kTileBitsC128, kRegBitsC128>(a, dev_ops, host_ops, nops, has_lin, s);
}

void launch_gate_whole(sv_dtype dt, const GatePassArgs &a, const void *dev_ops, uint64_t nops, cudaStream_t s) {
    if (dt == SV_C64) launch_whole_gates<float2>(a, dev_ops, nops, s);
    else launch_whole_gates<double2>(a, dev_ops, nops, s);
}

}  // namespace sv

extern "C" sv_status sv_debug_gate_jit(int n, sv_dtype dtype, const sv_gate *gates, uint64_t count, int compile,
                                       uint64_t *passes, uint64_t *compiles, double *compile_seconds) {
    using namespace sv;
    try {
        if (compile == 1) {
            SV_CHECK(dtype == SV_C64, SV_EINVAL, "the gate JIT is complex64 only");
            const GatePlan gp = plan_gates(n, 0, dtype, gates, count);
            uint64_t np = 0;
            for (const GateStep &st : gp.steps) {
                if (st.kind != GSTEP_PASS) continue;
                GatePassArgs a;
                a.tile_mask = st.tile;
                a.total_bits = gp.nl;
                a.n = gp.n;
                a.nl = gp.nl;
                a.gates = gates;
                a.order = gp.order.data() + st.first;
                a.count = st.count;
                std::vector<unsigned char> prog;
                bool lin = false;
                const uint64_t nops = build_gate_ops(dtype, a, false, prog, &lin);
                const bool l2 = gate_pass_l2(dtype, a);
                for (bool glb : {false, true})
                    SV_CHECK(gate_jit_compile_only(prog.data(), nops, lin, glb, l2) > 0, SV_ECUDA, "empty cubin");
                ++np;
            }
            if (passes) *passes = np;
        }
        gate_jit_stats(compiles, compile_seconds);
        set_error("");
        return SV_OK;
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    } catch (...) {
        set_error("unexpected exception");
        return SV_ECUDA;
    }
}
