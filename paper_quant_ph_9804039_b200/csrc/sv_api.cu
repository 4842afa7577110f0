// sv_api.cu -- the C ABI of include/sv.h: context, validation, dispatch of
// the device schedule, NCCL plumbing, profiling.
#include <atomic>
#include <cuda_runtime.h>
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <new>
#include <thread>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (CUDA toolkit): ranges for nsys / ncu --nvtx

#include "sv_internal.h"

namespace sv {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

constexpr int kMaxGrid = 4096;  // capacity of the reduction partials

}  // namespace sv

using namespace sv;

struct ProfEvent {
    cudaEvent_t a, b;
    int kind;
};

struct sv_ctx {
    int n = 0, g = 0, rank = 0, world = 1;
    bool emulated = false;
    sv_dtype dt = SV_C64;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    ncclComm_t comm = nullptr;
    void *state = nullptr;
    bool owns_state = true;   // false after sv_attach: the caller owns the buffer
    void *recv = nullptr;
    uint64_t nres = 0;       // resident amplitudes (2^{n-g}; 2^n emulated)
    uint64_t nl_amps = 0;    // amplitudes per rank (2^{n-g})
    uint64_t *d_marked = nullptr;
    uint64_t marked_cap = 0;
    unsigned int *d_tilemap = nullptr;  // one bit per tile of the O-group (holds a marked index)
    uint64_t *d_okeys = nullptr;        // sorted (tile id << 16 | element) of the marked entries
    uint64_t okeys_cap = 0;
    unsigned int *d_chunkmap = nullptr; // one bit per mean-kernel chunk (holds a marked index)
    // fused exchange: peer buffers (own buffers at index rank; CUDA IPC maps
    // of the other ranks' state / recv), or the emulated shards
    bool fused_xchg = false;
    bool xchg_capable = false;
    void *peer_state[8] = {};
    void *peer_recv[8] = {};
    int *d_barrier = nullptr;
    double *d_coefs = nullptr;          // angle-error coefficients of the one-CTA kernel
    size_t coefs_cap = 0;
    double *d_deco = nullptr;           // decoherence: {sum, scale, survival[k]}
    unsigned char *d_gprog = nullptr;   // gate circuits: op programs of every pass of a call
    size_t gprog_cap = 0;
    // CUDA graphs of launch-bound WHT schedules (small states, one GPU):
    // (k, fused exchange, marked epoch) -> executable graph
    struct GraphEntry {
        int k;
        bool fused;
        uint64_t epoch;
        cudaGraphExec_t exec;
    };
    std::vector<GraphEntry> graphs;
    uint64_t marked_epoch = 0;
    bool use_graphs = true;             // SV_GRAPHS=0 disables
    unsigned char *h_gprog = nullptr;   // pinned staging of the program (truly asynchronous upload)
    size_t h_gprog_cap = 0;
    cudaEvent_t gprog_ev = nullptr;     // the last upload from h_gprog has completed
    bool gprog_pending = false;
    size_t deco_cap = 0;
    unsigned int *d_superctr = nullptr;   // supertile pass: ticket + per-(supertile, sub-pass) counters
    unsigned int *d_superseg = nullptr;   // supertile pass: segment order
    uint64_t super_nseg = 0;
    int super_grid = 0;
    double *d_tilepart = nullptr;       // decoherence: per-tile sum |a|^2 of an iteration's last pass
    double *d_meanpart = nullptr;       // mean kernel (tile form): per-tile (re, im) partials
    size_t tilepart_cap = 0;
    double *d_samp = nullptr;           // sampler: chunk prefixes + rank totals + window
    uint64_t *d_shots = nullptr;        // sampler: device output for host-returning calls
    uint64_t shots_cap = 0;
    uint64_t n_marked = 0;   // resident (local) marked entries
    bool has_marked = false;
    double *d_partials = nullptr;  // 2 * kMaxGrid
    double *d_sums = nullptr;      // [0..1], [2..3] ping-pong; [4] norm; [6] scalar out
    unsigned int *d_counter = nullptr;
    unsigned int *d_gbar = nullptr;  // grid barrier of the persistent mean kernel {count, generation}
    void *d_res_slots = nullptr;     // resident mean kernel: per-block published totals (two rounds)
    unsigned long long res_epoch = 0;  // last epoch handed to the resident mean kernel
    void *d_res_acc = nullptr;       // resident mean kernel: fixed-point per-iteration sums (512 B each)
    size_t res_acc_cap = 0;          // iterations d_res_acc holds
    bool mean_resident = true;       // SV_MEAN_RESIDENT=0 disables the one-launch path
    bool mean_resreg = true;         // SV_MEAN_RESIDENT=smem: the shared-memory resident kernel (A/B)
    int mgrid = 1;
    Plan plan;
    bool broken = false;   // the communicator was aborted (sync_ctx): every call fails with SV_ENCCL
    // host-only schedule description (sv_debug_wht_variants): tile passes are
    // described instead of launched, swaps and scatters are skipped
    std::vector<TileVariant> *dry = nullptr;
    // profiling
    bool prof = false;
    std::vector<ProfEvent> pending;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
    uint64_t launches[SV_K_COUNT] = {};
    double ms[SV_K_COUNT] = {};
    std::vector<std::pair<int, double>> timeline;  // (kind, ms) per profiled launch, in order
};

namespace {

// Host-synchronising wait on the context's stream.  With a communicator it
// polls instead of blocking, so a failed or vanished peer cannot hang the
// caller forever: ncclCommGetAsyncError is checked on every poll and, on an
// asynchronous NCCL error or after SV_NCCL_TIMEOUT_S seconds (default 600)
// without progress, the communicator is aborted (ncclCommAbort, which also
// releases kernels blocked in collectives) and the call fails with SV_ENCCL
// (the context must then be freed, as after any SV_ENCCL).
void sync_ctx(sv_ctx *c) {
    if (c->comm == nullptr) {
        SV_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    static const double timeout_s = [] {
        const char *e = getenv("SV_NCCL_TIMEOUT_S");
        const double v = e ? atof(e) : 0.0;
        return v > 0.0 ? v : 600.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(c->stream);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) SV_CUDA(q);
        ncclResult_t ae = ncclSuccess;
        const ncclResult_t r = ncclCommGetAsyncError(c->comm, &ae);
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (r != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress) || el > timeout_s) {
            const std::string why = r != ncclSuccess ? std::string("ncclCommGetAsyncError: ") + ncclGetErrorString(r)
                                    : (ae != ncclSuccess && ae != ncclInProgress)
                                        ? std::string("asynchronous NCCL error: ") + ncclGetErrorString(ae)
                                        : "no progress within SV_NCCL_TIMEOUT_S = " + std::to_string(timeout_s) + " s";
            ncclCommAbort(c->comm);
            c->comm = nullptr;
            c->broken = true;
            throw Error{SV_ENCCL, why + " (communicator aborted; free the context)"};
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

template <class F>
sv_status guarded(F &&f) {
    try {
        f();
        g_err.clear();
        return SV_OK;
    } catch (const Error &e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc &) {
        g_err = "host allocation failed";
        return SV_ENOMEM;
    } catch (...) {
        g_err = "unexpected exception";
        return SV_ECUDA;
    }
}

void dmalloc(void **p, size_t bytes, const char *what) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw Error{SV_ENOMEM, std::string("cudaMalloc(") + what + ", " + std::to_string(bytes) + " B) failed"};
    }
    SV_CUDA(e);
}

// NVTX range names per kernel kind (sv_kernel_kind order): every enqueued
// device operation is bracketed by a host-side range, so an nsys timeline or
// `ncu --nvtx --nvtx-include` can attribute launches to the schedule's phases
// (tile passes, exchanges, allreduces -- the Fig. 12 split).
static const char *const kKindName[SV_K_COUNT] = {"sv.wht_tile", "sv.wht_whole", "sv.mean", "sv.reduce",
                                                  "sv.init", "sv.oracle", "sv.readout", "sv.exchange",
                                                  "sv.allreduce", "sv.gate_tile", "sv.scale"};

struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Bracket one device operation with events when profiling; count launches.
template <class F>
void run(sv_ctx *c, int kind, F &&f) {
    c->launches[kind] += 1;
    NvtxRange range(kKindName[kind]);
    if (!c->prof) {
        f();
        return;
    }
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    if (!c->pool.empty()) {
        ev = c->pool.back();
        c->pool.pop_back();
    } else {
        SV_CUDA(cudaEventCreate(&ev.first));
        SV_CUDA(cudaEventCreate(&ev.second));
    }
    SV_CUDA(cudaEventRecord(ev.first, c->stream));
    f();
    SV_CUDA(cudaEventRecord(ev.second, c->stream));
    c->pending.push_back({ev.first, ev.second, kind});
}

void drain_profile(sv_ctx *c) {
    if (c->pending.empty()) return;
    sync_ctx(c);
    for (auto &p : c->pending) {
        float ms = 0.f;
        SV_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        c->ms[p.kind] += ms;
        c->timeline.emplace_back(p.kind, (double)ms);
        c->pool.push_back({p.a, p.b});
    }
    c->pending.clear();
}

bool origin_here(const sv_ctx *c) { return c->emulated || c->rank == 0; }

void allreduce_sum(sv_ctx *c, double *buf, size_t count) {
    if (c->comm == nullptr) return;
    run(c, SV_K_ALLREDUCE, [&] {
        SV_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, c->stream));
    });
}

void do_init(sv_ctx *c, uint64_t seed, sv_init_kind kind) {
    SV_CUDA(cudaSetDevice(c->device));
    switch (kind) {
        case SV_INIT_UNIFORM:
            run(c, SV_K_INIT, [&] { launch_init_uniform(c->dt, c->state, c->nres, c->n, c->stream); });
            break;
        case SV_INIT_ZERO_STATE:
            run(c, SV_K_INIT, [&] { launch_init_zero(c->dt, c->state, c->nres, origin_here(c) ? 1 : 0, c->stream); });
            break;
        case SV_INIT_GAUSSIAN: {
            const uint64_t key = gauss_key(seed);
            const uint64_t off = c->emulated ? 0 : (uint64_t)c->rank * c->nl_amps;
            double *norm = c->d_sums + 4;
            run(c, SV_K_INIT, [&] {
                launch_gauss_norm(key, off, c->nres, c->d_partials, c->d_counter, norm, c->stream);
            });
            allreduce_sum(c, norm, 1);
            run(c, SV_K_INIT, [&] { launch_gauss_write(c->dt, c->state, key, off, c->nres, norm, c->stream); });
            break;
        }
        default:
            throw Error{SV_EINVAL, "unknown sv_init_kind"};
    }
}

void exchange(sv_ctx *c) {
    const size_t eb = elem_bytes(c->dt);
    const uint64_t P = 1ull << c->g;
    const uint64_t B = c->nl_amps / P;  // amplitudes per (rank, peer) block
    run(c, SV_K_EXCHANGE, [&] {
        if (c->comm != nullptr) {
            // chunk j of the shard (top-g local bits == j) goes to rank j and
            // lands as its chunk `rank` (Fig. 8: blocks whose owner changes
            // are sent; chunk j == rank stays local).
            SV_NCCL(ncclAlltoAll(c->state, c->recv, B * (eb / 8), ncclUint64, c->comm, c->stream));
        } else {
            char *src = (char *)c->state, *dst = (char *)c->recv;
            for (uint64_t r = 0; r < P; ++r)
                for (uint64_t j = 0; j < P; ++j)
                    SV_CUDA(cudaMemcpyAsync(dst + (j * c->nl_amps + r * B) * eb, src + (r * c->nl_amps + j * B) * eb,
                                            B * eb, cudaMemcpyDeviceToDevice, c->stream));
        }
    });
}

// Cross-rank ordering point after a fused exchange pass: every rank's
// peer stores have landed before anyone reads its buffer.  Real ranks: a
// one-integer ncclAllReduce on the stream (completes only after every rank's
// exchange kernel has completed); emulation: stream order is enough.
void xchg_barrier(sv_ctx *c) {
    if (c->comm == nullptr) return;
    run(c, SV_K_EXCHANGE, [&] {
        SV_NCCL(ncclAllReduce(c->d_barrier, c->d_barrier, 1, ncclInt32, ncclSum, c->comm, c->stream));
    });
}

// General per-qubit 2x2 transforms (NEXT-1 angle errors G19/G20, NEXT-2
// decoherence G22); iteration numbers t0 ...
struct Noise {
    double sigma;
    double rate;                      // decoherence rate per laser operation (0 = none)
    uint64_t seed;
    uint64_t t0;
    const double *scale_first = nullptr;  // device scalar folded into the first pass's load
    double *sumsq = nullptr;              // device: per-tile sum |a|^2 written by the last pass
};

// [w x; y z] of logical qubit q in transform tr (= 2 x iteration + w) of the
// call, for all q.  Angle errors: U(pi/4 + delta) = [[c, s], [s, -c]].
// Decoherence: the laser operations of a transform run q = 0..n-1, each
// followed by a contraction diag(1, sqrt(1-rate)) of a drawn site d_q.  Such a
// contraction commutes with every 2x2 except its own site's, so on qubit s it
// sits BEFORE U_s if it follows an earlier operation (q < s) and AFTER U_s
// otherwise: M_s = diag(1, post_s) U_s diag(1, pre_s) with pre_s / post_s the
// products of those factors.  The renormalisations are scalars (applied once
// per iteration by the caller).
static void transform_coefs(const Noise &nz, int tr, int n, std::vector<double> &m) {
    const uint64_t t = nz.t0 + (uint64_t)(tr / 2);
    const int w = tr % 2;
    m.assign((size_t)n * 4, 0.0);
    std::vector<double> pre(n, 1.0), post(n, 1.0);
    if (nz.rate > 0.0) {
        const double cf = sqrt(1.0 - nz.rate);
        for (int q = 0; q < n; ++q) {
            const int d = decay_site(n, nz.seed, t, w, q);
            if (q < d) pre[d] *= cf;
            else post[d] *= cf;
        }
    }
    for (int q = 0; q < n; ++q) {
        const double phi = 0.78539816339744831 + noise_delta(nz.seed, t, w, q, nz.sigma);
        const double cs = cos(phi), sn = sin(phi);
        m[4 * q + 0] = cs;
        m[4 * q + 1] = sn * pre[q];
        m[4 * q + 2] = post[q] * sn;
        m[4 * q + 3] = -post[q] * cs * pre[q];
    }
}

// The supertile group's visit (always fused with F0, plan.cpp): level A
// stages of the first transform, level B stages + F0 + level B stages, level A
// stages of the second transform, as three sub-passes of one persistent launch
// (wht_super.cu).  tcoef: per-transform coefficients of the noisy flavours.
void run_super_step(sv_ctx *c, const Step &s, int total_bits, const std::vector<std::vector<double>> *tcoef) {
    const SuperSpec &sp = c->plan.sup;
    SV_CHECK(s.pre && s.post && s.mid == MID_F0 && !s.pre_swap && s.layout == 0, SV_EINVAL,
             "internal: the supertile group is visited only fused with F0");
    SuperArgs sa;
    sa.st_mask = sp.st;
    sa.ua = c->plan.T - __builtin_popcountll(sp.procA);
    sa.ub = sp.uB;
    sa.ctr = c->d_superctr;
    sa.seg = c->d_superseg;
    sa.nseg = c->super_nseg;
    sa.grid = c->super_grid;
    const uint64_t tiles[3] = {sp.tileA, sp.tileB, sp.tileA};
    const uint64_t procs[3] = {sp.procA, sp.procB, sp.procA};
    for (int j = 0; j < 3; ++j) {
        PassArgs &a = sa.sub[j];
        a.in = c->state;
        a.out = c->state;
        a.f0_scale = tcoef ? 1.0 : ldexp(1.0, -c->n);
        a.has_origin = origin_here(c) ? 1 : 0;
        a.pre = j < 2 ? 1 : 0;
        a.post = j > 0 ? 1 : 0;
        a.mid = j == 1 ? MID_F0 : MID_NONE;
        a.tile_mask = tiles[j];
        a.proc_mask = procs[j];
        a.total_bits = total_bits;
        if (tcoef) {
            a.noisy = 1;
            for (int sl = 0; sl < 64; ++sl) {
                if (!((procs[j] >> sl) & 1)) continue;
                for (int e = 0; e < 4; ++e) {  // natural layout: slot = logical qubit (g == 0)
                    if (a.pre) a.coef[0][sl][e] = (*tcoef)[s.tr_pre][4 * sl + e];
                    if (a.post) a.coef[1][sl][e] = (*tcoef)[s.tr_post][4 * sl + e];
                }
            }
        }
    }
    if (c->dry) {
        TileVariant v[3];
        launch_wht_super_pass(c->dt, sa, nullptr, v);
        for (int j = 0; j < 3; ++j) c->dry->push_back(v[j]);
        return;
    }
    run(c, SV_K_WHT_TILE, [&] { launch_wht_super_pass(c->dt, sa, c->stream); });
}

// Work order of the supertile kernel: step w runs sub-pass 0 of supertile w,
// sub-pass 1 of w - L and sub-pass 2 of w - 2L, so a sub-pass starts 3 L
// segments (3 L x tiles-per-segment items) after the one it depends on --
// more than the CTAs in flight, so CTAs rarely wait -- and about 2 L + 1
// supertiles are live in L2.  SV_SUPER_LAG overrides L.
void setup_super(sv_ctx *c) {
    if (!c->plan.super) return;
    const int stb = __builtin_popcountll(c->plan.sup.st);
    const uint64_t nst = 1ull << (c->plan.nl - stb);
    const uint64_t tps = 1ull << (stb - c->plan.T);
    c->super_grid = super_grid();
    int L = (int)((3 * (uint64_t)c->super_grid + 6 * tps - 1) / (6 * tps));  // ~1.5 x grid / (3 tps)
    if (const char *e = getenv("SV_SUPER_LAG")) L = atoi(e);
    if (L < 1) L = 1;
    std::vector<unsigned int> seg;
    seg.reserve(3 * nst);
    for (uint64_t w = 0; w < nst + 2 * (uint64_t)L; ++w)
        for (int j = 0; j < 3; ++j) {
            const int64_t st = (int64_t)w - (int64_t)j * L;
            if (st >= 0 && st < (int64_t)nst) seg.push_back((unsigned int)(st << 2) | (unsigned int)j);
        }
    SV_CHECK(seg.size() == 3 * nst && nst < (1ull << 30), SV_EINVAL, "internal: supertile segment table");
    dmalloc((void **)&c->d_superseg, seg.size() * sizeof(unsigned int), "supertile segments");
    dmalloc((void **)&c->d_superctr, (3 * nst + 1) * sizeof(unsigned int), "supertile counters");
    SV_CUDA(cudaMemcpyAsync(c->d_superseg, seg.data(), seg.size() * sizeof(unsigned int), cudaMemcpyHostToDevice,
                            c->stream));
    SV_CUDA(cudaStreamSynchronize(c->stream));
    c->super_nseg = seg.size();
}

void run_wht_schedule(sv_ctx *c, int k, bool with_oracle, const Noise *noise = nullptr, double *survival = nullptr) {
    std::vector<std::vector<double>> tcoef;  // per transform of the call
    if (noise) {
        const int ntr = 2 * (with_oracle ? k : 1);
        tcoef.resize(ntr);
        for (int tr = 0; tr < ntr; ++tr) transform_coefs(*noise, tr, c->n, tcoef[tr]);
    }
    if (c->plan.whole) {
        if (with_oracle && k == 0) return;
        if (c->dry) {
            TileVariant v;  // family 0: the one-CTA whole-state kernel
            v.noisy = noise ? 1 : 0;
            c->dry->push_back(v);
            return;
        }
        const int reps = with_oracle ? k : 1;
        const double *coefs = nullptr;
        if (noise) {  // per (iteration, transform, qubit) coefficients for the one-CTA kernel
            std::vector<double> h;
            for (const auto &v : tcoef) h.insert(h.end(), v.begin(), v.end());
            if (h.size() > c->coefs_cap) {
                if (c->d_coefs) SV_CUDA(cudaFree(c->d_coefs));
                c->d_coefs = nullptr;
                c->coefs_cap = 0;
                dmalloc((void **)&c->d_coefs, h.size() * sizeof(double), "angle-error coefficients");
                c->coefs_cap = h.size();
            }
            SV_CUDA(cudaMemcpyAsync(c->d_coefs, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            sync_ctx(c);
            coefs = c->d_coefs;
        }
        run(c, SV_K_WHT_WHOLE, [&] {
            launch_whole_state(c->dt, c->state, c->n, reps, with_oracle ? 1 : 0, SV_DIFFUSE_WHT, c->d_marked,
                               c->n_marked, c->stream, coefs, survival);
        });
        return;
    }
    bool first_pass = true;
    const std::vector<Step> steps = schedule_wht(c->plan, k, with_oracle);
    size_t last_pass = steps.size();
    for (size_t i = 0; i < steps.size(); ++i)
        if (steps[i].kind == STEP_PASS) last_pass = i;
    const int total_bits = c->emulated ? c->n : c->plan.nl;
    // cur = the buffer holding the state.  Unfused: passes write `state`, a
    // swap is an all-to-all state -> recv.  Fused: the pass before a swap
    // stores every element straight into its new owner's other buffer
    // (peer memory over NVLink, or the emulated shard), a swap is only a
    // barrier; passes after it continue in that buffer.
    void *cur = c->state;
    void *next = nullptr;
    for (size_t si = 0; si < steps.size(); ++si) {
        const Step &s = steps[si];
        if (s.kind == STEP_SWAP) {
            if (c->dry) {
                cur = c->fused_xchg ? next : c->recv;
                continue;
            }
            if (c->fused_xchg) {
                xchg_barrier(c);
                cur = next;
            } else {
                exchange(c);
                cur = c->recv;
            }
            continue;
        }
        if (s.kind == STEP_SCATTER) {
            if (s.mid == MID_ORACLE && !c->dry)
                run(c, SV_K_ORACLE, [&] { launch_oracle_scatter(c->dt, c->state, c->d_marked, c->n_marked, c->stream); });
            continue;
        }
        if (c->plan.super && s.group == c->plan.sup.group) {
            run_super_step(c, s, total_bits, noise ? &tcoef : nullptr);
            first_pass = false;
            continue;
        }
        PassArgs a;
        a.in = cur;
        a.out = c->fused_xchg ? cur : c->state;
        if (c->fused_xchg && s.pre_swap) {
            const bool to_recv = (cur == c->state);
            next = to_recv ? c->recv : c->state;
            a.xchg_nl = c->plan.nl;
            a.xchg_g = c->g;
            a.xchg_rank = c->emulated ? -1 : c->rank;
            for (int j = 0; j < (1 << c->g); ++j) {
                if (c->emulated)
                    a.xchg_dst[j] = (char *)next + (size_t)j * c->nl_amps * elem_bytes(c->dt);
                else
                    a.xchg_dst[j] = to_recv ? c->peer_recv[j] : c->peer_state[j];
            }
        }
        if (!c->fused_xchg) cur = c->state;
        a.marked = c->d_okeys;  // O-group lookup keys (only read by oracle passes)
        a.n_marked = c->n_marked;
        a.tilemap = c->d_tilemap;
        a.f0_scale = noise ? 1.0 : ldexp(1.0, -c->n);  // unitary transforms carry no 2^-n
        if (noise) {
            a.noisy = 1;
            const uint64_t proc = c->plan.groups[s.group].proc;
            const int u0 = c->plan.nl - c->g;  // first top-g local slot
            for (int sl = 0; sl < 64; ++sl) {
                if (!((proc >> sl) & 1)) continue;
                // logical qubit of this slot: in the swapped layout the top-g
                // local slots hold the rank qubits nl .. n-1
                const int q = (s.layout == 1 && sl >= u0) ? c->plan.nl + (sl - u0) : sl;
                for (int e = 0; e < 4; ++e) {
                    if (s.pre) a.coef[0][sl][e] = tcoef[s.tr_pre][4 * q + e];
                    if (s.post) a.coef[1][sl][e] = tcoef[s.tr_post][4 * q + e];
                }
            }
            if (first_pass) a.scale_in = noise->scale_first;
            if (si == last_pass) {
                // the decoherence step's global sum (Eq. 3) rides on the last
                // pass's stores; it must leave the state in natural order
                SV_CHECK(!s.pre_swap && s.layout == 0, SV_EINVAL, "internal: sumsq on a swapped pass");
                a.sumsq = noise->sumsq;
            }
        }
        first_pass = false;
        a.mid = s.mid;
        a.has_origin = origin_here(c) ? 1 : 0;
        a.pre = s.pre;
        a.post = s.post;
        a.tile_mask = c->plan.groups[s.group].tile;
        a.proc_mask = c->plan.groups[s.group].proc;
        a.total_bits = total_bits;
        if (c->dry) {
            c->dry->push_back(describe_tile_pass(c->dt, a));
            continue;
        }
        run(c, SV_K_WHT_TILE, [&] { launch_wht_tile_pass(c->dt, a, c->stream); });
    }
}

// Gate circuit (NEXT-4): the planned passes (gate_plan.cpp) and qubit swaps.
// All passes' op programs are built on the host and uploaded once, then the
// passes run back to back on the stream.  Buffers as in run_wht_schedule:
// unfused, a swap is an all-to-all state -> recv and the next pass reads recv
// and writes state; fused, the pass before a swap stores every element into
// its new owner's other buffer and the swap is a barrier.
void run_gates(sv_ctx *c, const sv_gate *gates, uint64_t count) {
    const GatePlan gp = plan_gates(c->n, c->g, c->dt, gates, count);
    if (gp.steps.empty()) return;
    const int total_bits = c->emulated ? c->n : gp.nl;
    auto args = [&](const GateStep &st) {
        GatePassArgs a;
        a.tile_mask = st.tile;
        a.total_bits = total_bits;
        a.g = gp.g;
        a.rank = c->rank;
        a.emulated = c->emulated ? 1 : 0;
        a.swapped = st.swapped;
        a.n = gp.n;
        a.nl = gp.nl;
        a.gates = gates;
        a.order = gp.order.data() + st.first;
        a.count = st.count;
        return a;
    };
    std::vector<unsigned char> prog;
    std::vector<std::pair<size_t, uint64_t>> where(gp.steps.size(), {0, 0});
    std::vector<char> lin(gp.steps.size(), 0);
    for (size_t i = 0; i < gp.steps.size(); ++i) {
        const GateStep &st = gp.steps[i];
        if (st.kind == GSTEP_SWAP) continue;
        const size_t off = (prog.size() + 15) & ~(size_t)15;
        bool hl = false;
        where[i] = {off, build_gate_ops(c->dt, args(st), st.kind == GSTEP_WHOLE, prog, &hl)};
        lin[i] = hl ? 1 : 0;
    }
    if (prog.size() > c->gprog_cap) {
        if (c->d_gprog) SV_CUDA(cudaFree(c->d_gprog));  // (cudaFree waits for the kernels still using it)
        c->d_gprog = nullptr;
        c->gprog_cap = 0;
        dmalloc((void **)&c->d_gprog, prog.size(), "gate program");
        c->gprog_cap = prog.size();
    }
    if (!prog.empty()) {
        // stage in pinned memory so the upload (and the call) stays asynchronous;
        // the staging buffer is reused once the previous upload has completed
        if (c->gprog_ev == nullptr) SV_CUDA(cudaEventCreateWithFlags(&c->gprog_ev, cudaEventDisableTiming));
        if (c->gprog_pending) SV_CUDA(cudaEventSynchronize(c->gprog_ev));
        if (prog.size() > c->h_gprog_cap) {
            if (c->h_gprog) SV_CUDA(cudaFreeHost(c->h_gprog));
            c->h_gprog = nullptr;
            c->h_gprog_cap = 0;
            SV_CUDA(cudaMallocHost((void **)&c->h_gprog, prog.size()));
            c->h_gprog_cap = prog.size();
        }
        memcpy(c->h_gprog, prog.data(), prog.size());
        SV_CUDA(cudaMemcpyAsync(c->d_gprog, c->h_gprog, prog.size(), cudaMemcpyHostToDevice, c->stream));
        SV_CUDA(cudaEventRecord(c->gprog_ev, c->stream));
        c->gprog_pending = true;
    }
    // gate JIT: decide (and compile where due) every pass's specialised kernel
    // before the first launch -- host work outside the passes' events
    static std::atomic<uint64_t> calls{0};
    const uint64_t call = ++calls;
    std::vector<void *> jit(gp.steps.size(), nullptr);
    for (size_t i = 0; i < gp.steps.size(); ++i) {
        const GateStep &st = gp.steps[i];
        if (st.kind != GSTEP_PASS) continue;
        GatePassArgs a = args(st);
        const bool pre_swap = i + 1 < gp.steps.size() && gp.steps[i + 1].kind == GSTEP_SWAP;
        if (c->fused_xchg && pre_swap) continue;  // exchange-store passes keep the interpreter
        a.jit_prepare = call;
        a.jit_kern = &jit[i];
        launch_gate_pass(c->dt, a, nullptr, prog.data() + where[i].first, where[i].second, lin[i] != 0, c->stream);
    }
    void *cur = c->state, *next = nullptr;
    for (size_t i = 0; i < gp.steps.size(); ++i) {
        const GateStep &st = gp.steps[i];
        if (st.kind == GSTEP_SWAP) {
            if (c->fused_xchg && next != nullptr) {
                xchg_barrier(c);
                cur = next;
                next = nullptr;
            } else {  // unfused, or a swap with no pass before it to carry it
                if (cur != c->state)
                    SV_CUDA(cudaMemcpyAsync(c->state, cur, c->nres * elem_bytes(c->dt), cudaMemcpyDeviceToDevice,
                                            c->stream));
                exchange(c);
                cur = c->recv;
            }
            continue;
        }
        GatePassArgs a = args(st);
        const void *ops = c->d_gprog + where[i].first;
        if (st.kind == GSTEP_WHOLE) {
            a.in = c->state;
            run(c, SV_K_GATE_TILE, [&] { launch_gate_whole(c->dt, a, ops, where[i].second, c->stream); });
            continue;
        }
        a.in = cur;
        a.out = c->fused_xchg ? cur : c->state;
        const bool pre_swap = i + 1 < gp.steps.size() && gp.steps[i + 1].kind == GSTEP_SWAP;
        if (c->fused_xchg && pre_swap) {
            const bool to_recv = (cur == c->state);
            next = to_recv ? c->recv : c->state;
            a.xchg_nl = gp.nl;
            a.xchg_g = c->g;
            a.xchg_rank = c->emulated ? -1 : c->rank;
            for (int j = 0; j < (1 << c->g); ++j) {
                if (c->emulated)
                    a.xchg_dst[j] = (char *)next + (size_t)j * c->nl_amps * elem_bytes(c->dt);
                else
                    a.xchg_dst[j] = to_recv ? c->peer_recv[j] : c->peer_state[j];
            }
        }
        a.jit_kern = &jit[i];
        run(c, SV_K_GATE_TILE, [&] {
            launch_gate_pass(c->dt, a, ops, prog.data() + where[i].first, where[i].second, lin[i] != 0, c->stream);
        });
        if (!c->fused_xchg) cur = c->state;
    }
    if (cur != c->state)
        SV_CUDA(cudaMemcpyAsync(c->state, cur, c->nres * elem_bytes(c->dt), cudaMemcpyDeviceToDevice, c->stream));
}

// Launch-bound regime (states of a few MiB: a tile pass is a few us, about
// its launch latency): replay the k-iteration schedule as one CUDA graph,
// captured on first use and cached per (k, exchange mode, marked set).  Not
// while profiling (events per launch), not with NCCL (multi-process), not for
// the one-CTA path (a single launch already).
void run_wht_graphed(sv_ctx *c, int k) {
    constexpr uint64_t kGraphMaxBytes = 64ull << 20;
    const bool small = c->nres * elem_bytes(c->dt) <= kGraphMaxBytes;
    if (!c->use_graphs || c->prof || c->comm != nullptr || c->plan.whole || !small || k < 2) {
        run_wht_schedule(c, k, true);
        return;
    }
    // bounded graphs: k iterations = consecutive calls of at most kGraphIters
    // (each call is the same product; one extra unfused pass per chunk)
    constexpr int kGraphIters = 256;
    if (k > kGraphIters) {
        for (int done = 0; done < k; done += kGraphIters) run_wht_graphed(c, std::min(kGraphIters, k - done));
        return;
    }
    for (const auto &ge : c->graphs)
        if (ge.k == k && ge.fused == c->fused_xchg && ge.epoch == c->marked_epoch) {
            SV_CUDA(cudaGraphLaunch(ge.exec, c->stream));
            return;
        }
    cudaGraph_t graph = nullptr;
    SV_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
        run_wht_schedule(c, k, true);
    } catch (...) {
        cudaStreamEndCapture(c->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    SV_CUDA(cudaStreamEndCapture(c->stream, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    SV_CUDA(e);
    if (c->graphs.size() >= 8) {
        cudaGraphExecDestroy(c->graphs.front().exec);
        c->graphs.erase(c->graphs.begin());
    }
    c->graphs.push_back({k, c->fused_xchg, c->marked_epoch, exec});
    SV_CUDA(cudaGraphLaunch(exec, c->stream));
}

MeanArgs mean_args(sv_ctx *c, bool with_oracle) {
    MeanArgs m;
    m.a = c->state;
    m.N = c->nres;
    m.inv_total = ldexp(1.0, -c->n);
    m.marked = with_oracle ? c->d_marked : nullptr;
    m.n_marked = with_oracle ? c->n_marked : 0;
    m.chunkmap = c->d_chunkmap;
    m.partials = c->d_partials;
    m.counter = c->d_counter;
    if (mean_tile_mode()) {
        if (c->d_meanpart == nullptr)
            dmalloc((void **)&c->d_meanpart, 2 * mean_tiles(c->nres, c->dt) * sizeof(double), "mean tile partials");
        m.tilepart = c->d_meanpart;
    }
    return m;
}

void run_mean(sv_ctx *c, int k, bool with_oracle) {
    if (c->plan.whole) {
        if (with_oracle && k == 0) return;
        run(c, SV_K_WHT_WHOLE, [&] {
            launch_whole_state(c->dt, c->state, c->n, with_oracle ? k : 1, with_oracle ? 1 : 0, SV_DIFFUSE_MEAN,
                               c->d_marked, c->n_marked, c->stream);
        });
        return;
    }
    const int reps = with_oracle ? k : 1;
    if (reps == 0) return;
    // single GPU, state within the aggregate shared memory: all iterations in
    // one persistent launch (mean_resident.cu)
    if (c->comm == nullptr && c->mean_resident && mean_resident_fits(c->dt, c->nres, 2 * kMaxGrid)) {
        if (c->d_res_slots == nullptr) {  // zeroed once: epochs start at 1
            const size_t b = mean_resident_slot_bytes(c->dt, c->nres);
            dmalloc(&c->d_res_slots, b, "resident mean slots");
            SV_CUDA(cudaMemsetAsync(c->d_res_slots, 0, b, c->stream));
        }
        if (c->res_acc_cap < (size_t)reps) {  // grown, never shrunk
            if (c->d_res_acc) SV_CUDA(cudaFree(c->d_res_acc));
            c->d_res_acc = nullptr;
            c->res_acc_cap = 0;
            const size_t cap = std::max<size_t>((size_t)reps, 512);
            dmalloc(&c->d_res_acc, cap * 64 * sizeof(unsigned long long), "resident mean sums");
            c->res_acc_cap = cap;
        }
        const unsigned long long epoch0 = c->res_epoch + 1;
        c->res_epoch += (unsigned long long)reps + 1;  // rounds of this launch: reps (+1 spare)
        run(c, SV_K_MEAN, [&] {
            launch_mean_resident(c->dt, c->state, c->nres, ldexp(1.0, -c->n), with_oracle ? c->d_marked : nullptr,
                                 with_oracle ? c->n_marked : 0, reps, c->d_partials, c->d_gbar, c->d_res_slots,
                                 epoch0, c->mean_resreg, c->d_res_acc, c->stream);
        });
        return;
    }
    MeanArgs m = mean_args(c, with_oracle);
    // first mu: sum of (O a) over the whole register (Eq. 3's accumulate)
    m.sum_out = c->d_sums;
    run(c, SV_K_REDUCE, [&] { launch_mean_grid(c->dt, m, c->mgrid, false, c->stream); });
    allreduce_sum(c, c->d_sums, 2);  // ... and redistribute
    for (int it = 0; it < reps; ++it) {
        m.sum_in = c->d_sums + 2 * (it & 1);
        m.sum_out = c->d_sums + 2 * ((it + 1) & 1);
        run(c, SV_K_MEAN, [&] { launch_mean_grid(c->dt, m, c->mgrid, true, c->stream); });
        if (it + 1 < reps) allreduce_sum(c, m.sum_out, 2);
    }
}

void store_marked(sv_ctx *c, const uint64_t *marked, uint64_t m) {
    c->marked_epoch += 1;  // captured WHT graphs bake the marked-set pointers and counts
    const uint64_t N = 1ull << c->n;
    SV_CHECK(m <= N, SV_EINVAL, "marked set larger than 2^n");
    SV_CHECK(m == 0 || marked != nullptr, SV_EINVAL, "marked is NULL");
    for (uint64_t j = 0; j < m; ++j) {
        SV_CHECK(marked[j] < N, SV_EINVAL, "marked index " + std::to_string(marked[j]) + " >= 2^n");
        SV_CHECK(j == 0 || marked[j] > marked[j - 1], SV_EINVAL,
                 "marked indices must be strictly increasing (duplicates are errors)");
    }
    // resident part, rebased to local indices
    uint64_t lo = 0, hi = m;
    uint64_t base = 0;
    if (!c->emulated && c->world > 1) {
        base = (uint64_t)c->rank * c->nl_amps;
        lo = std::lower_bound(marked, marked + m, base) - marked;
        hi = std::lower_bound(marked, marked + m, base + c->nl_amps) - marked;
    }
    const uint64_t cnt = hi - lo;
    std::vector<uint64_t> loc(cnt);
    for (uint64_t j = 0; j < cnt; ++j) loc[j] = marked[lo + j] - base;
    if (cnt > c->marked_cap) {
        if (c->d_marked) SV_CUDA(cudaFree(c->d_marked));
        c->d_marked = nullptr;
        c->marked_cap = 0;
        dmalloc((void **)&c->d_marked, std::max<uint64_t>(cnt, 1) * 8, "marked");
        c->marked_cap = cnt;
    }
    if (cnt) SV_CUDA(cudaMemcpyAsync(c->d_marked, loc.data(), cnt * 8, cudaMemcpyHostToDevice, c->stream));
    // Per-tile lookup for the O-group's oracle-fused passes: a bitmap over its
    // tiles and the sorted keys (tile id << 16 | tile element) of the marked
    // entries -- tile id / element = the index's free / tile slot bits.
    std::vector<unsigned int> map;
    std::vector<uint64_t> keys(cnt);
    if (!c->plan.whole) {
        const int total_bits = c->emulated ? c->n : c->plan.nl;
        const uint64_t tmask = c->plan.groups[c->plan.fwd[0]].tile;
        const uint64_t fmask = ((total_bits >= 64) ? ~0ull : ((1ull << total_bits) - 1ull)) & ~tmask;
        auto pext = [](uint64_t v, uint64_t m) {
            uint64_t r = 0;
            int k = 0;
            for (int b = 0; b < 64; ++b)
                if ((m >> b) & 1) r |= ((v >> b) & 1ull) << k++;
            return r;
        };
        const uint64_t ntiles = c->nres >> c->plan.T;
        map.assign((ntiles + 31) / 32, 0u);
        for (uint64_t j = 0; j < cnt; ++j) {
            const uint64_t t = pext(loc[j], fmask);
            keys[j] = (t << 16) | pext(loc[j], tmask);
            map[t >> 5] |= 1u << (t & 31);
        }
        std::sort(keys.begin(), keys.end());
        if (!c->d_tilemap) dmalloc((void **)&c->d_tilemap, map.size() * 4, "tile bitmap");
        SV_CUDA(cudaMemcpyAsync(c->d_tilemap, map.data(), map.size() * 4, cudaMemcpyHostToDevice, c->stream));
        if (cnt > c->okeys_cap) {
            if (c->d_okeys) SV_CUDA(cudaFree(c->d_okeys));
            c->d_okeys = nullptr;
            c->okeys_cap = 0;
            dmalloc((void **)&c->d_okeys, cnt * 8, "oracle keys");
            c->okeys_cap = cnt;
        }
        if (cnt) SV_CUDA(cudaMemcpyAsync(c->d_okeys, keys.data(), cnt * 8, cudaMemcpyHostToDevice, c->stream));
    }
    // chunk bitmap of the mean kernel
    const uint64_t ce = mean_chunk_elems(c->dt);
    std::vector<unsigned int> cmap(((c->nres + ce - 1) / ce + 31) / 32, 0u);
    for (uint64_t v : loc) cmap[(v / ce) >> 5] |= 1u << ((v / ce) & 31);
    if (!c->d_chunkmap) dmalloc((void **)&c->d_chunkmap, cmap.size() * 4, "chunk bitmap");
    SV_CUDA(cudaMemcpyAsync(c->d_chunkmap, cmap.data(), cmap.size() * 4, cudaMemcpyHostToDevice, c->stream));
    sync_ctx(c);  // loc / map / keys / cmap are freed on return
    c->n_marked = cnt;
    c->has_marked = true;
}

void check_ctx(const sv_ctx *c) {
    SV_CHECK(c != nullptr, SV_EINVAL, "ctx is NULL");
    SV_CHECK(!c->broken, SV_ENCCL, "the context's communicator was aborted after an NCCL failure; free the context");
}

// Fused exchange plumbing.  Emulation: the shards are in one buffer.  Real
// ranks: exchange CUDA IPC handles of every rank's state and receive buffer
// over the library's own NCCL communicator and map them (NVLink peer access);
// any failure leaves the NCCL all-to-all path in place.  SV_XCHG=nccl forces
// the unfused path.
void setup_peers(sv_ctx *c) {
    if (c->world <= 1) return;
    const char *env = getenv("SV_XCHG");
    const bool want = !(env && strcmp(env, "nccl") == 0);
    if (c->emulated) {
        c->xchg_capable = c->world <= 8;
        c->fused_xchg = want && c->xchg_capable;
        return;
    }
    if (c->comm == nullptr || c->world > 8) return;
    dmalloc((void **)&c->d_barrier, sizeof(int), "barrier");
    SV_CUDA(cudaMemsetAsync(c->d_barrier, 0, sizeof(int), c->stream));
    // Every rank takes part in every collective below whatever its local
    // outcome, and the mode is decided by an allreduce(min): ranks can never
    // disagree on fused vs all-to-all (which would deadlock the schedule).
    struct Entry {
        cudaIpcMemHandle_t h[2];
        int ok;
        int pad;
    };
    Entry mine{};
    mine.ok = (cudaIpcGetMemHandle(&mine.h[0], c->state) == cudaSuccess &&
               cudaIpcGetMemHandle(&mine.h[1], c->recv) == cudaSuccess) ? 1 : 0;
    if (!mine.ok) cudaGetLastError();
    const size_t hb = sizeof(Entry);
    char *d_all = nullptr;
    dmalloc((void **)&d_all, hb * c->world + sizeof(int), "ipc handles");
    std::vector<Entry> all(c->world);
    int *d_ok = reinterpret_cast<int *>(d_all + hb * c->world);
    int ok = 0;
    try {
        SV_CUDA(cudaMemcpyAsync(d_all + hb * c->rank, &mine, hb, cudaMemcpyHostToDevice, c->stream));
        SV_NCCL(ncclAllGather(d_all + hb * c->rank, d_all, hb, ncclChar, c->comm, c->stream));
        SV_CUDA(cudaMemcpyAsync(all.data(), d_all, hb * c->world, cudaMemcpyDeviceToHost, c->stream));
        sync_ctx(c);
        ok = 1;
        for (int j = 0; j < c->world; ++j) ok &= all[j].ok;
        for (int j = 0; j < c->world && ok; ++j) {
            if (j == c->rank) continue;
            if (cudaIpcOpenMemHandle(&c->peer_state[j], all[j].h[0], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
                cudaIpcOpenMemHandle(&c->peer_recv[j], all[j].h[1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                ok = 0;
            }
        }
        SV_CUDA(cudaMemcpyAsync(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream));
        SV_NCCL(ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, c->comm, c->stream));
        SV_CUDA(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        sync_ctx(c);
    } catch (...) {
        cudaFree(d_all);
        throw;
    }
    SV_CUDA(cudaFree(d_all));
    c->peer_state[c->rank] = c->state;
    c->peer_recv[c->rank] = c->recv;
    c->xchg_capable = ok != 0;
    c->fused_xchg = want && ok;
}

void destroy(sv_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto &p : c->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    for (auto &p : c->pool) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    if (!c->emulated)
        for (int j = 0; j < 8; ++j) {
            if (j == c->rank) continue;
            if (c->peer_state[j]) cudaIpcCloseMemHandle(c->peer_state[j]);
            if (c->peer_recv[j]) cudaIpcCloseMemHandle(c->peer_recv[j]);
        }
    cudaFree(c->d_barrier);
    cudaFree(c->d_coefs);
    cudaFree(c->d_samp);
    cudaFree(c->d_deco);
    cudaFree(c->d_tilepart);
    cudaFree(c->d_meanpart);
    cudaFree(c->d_superctr);
    cudaFree(c->d_superseg);
    for (auto &ge : c->graphs) cudaGraphExecDestroy(ge.exec);
    cudaFree(c->d_gprog);
    if (c->h_gprog) cudaFreeHost(c->h_gprog);
    if (c->gprog_ev) cudaEventDestroy(c->gprog_ev);
    cudaFree(c->d_shots);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->owns_state) cudaFree(c->state);
    cudaFree(c->recv);
    cudaFree(c->d_marked);
    cudaFree(c->d_tilemap);
    cudaFree(c->d_okeys);
    cudaFree(c->d_chunkmap);
    cudaFree(c->d_partials);
    cudaFree(c->d_sums);
    cudaFree(c->d_counter);
    cudaFree(c->d_gbar);
    cudaFree(c->d_res_acc);
    cudaFree(c->d_res_slots);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

}  // namespace

extern "C" {

const char *sv_last_error(void) { return g_err.c_str(); }

sv_status sv_init(sv_ctx **out, int n, uint64_t seed, sv_dtype dtype, sv_init_kind init, const sv_dist *dist) {
    sv_ctx *c = nullptr;
    sv_status st = guarded([&] {
        SV_CHECK(out != nullptr, SV_EINVAL, "out is NULL");
        *out = nullptr;
        int world = dist ? dist->world : 1;
        SV_CHECK(world >= 1 && (world & (world - 1)) == 0, SV_EINVAL, "world must be a power of two");
        int g = 0;
        while ((1 << g) < world) ++g;
        SV_CHECK(g <= n, SV_EINVAL, "world larger than 2^n");
        c = new sv_ctx();
        c->n = n;
        c->g = g;
        c->world = world;
        c->dt = dtype;
        c->plan = make_plan(n, g, dtype);  // validates n, dtype, shard size
        c->emulated = dist && world > 1 && dist->nccl_id == nullptr;
        c->rank = (dist && !c->emulated) ? dist->rank : 0;
        SV_CHECK(c->rank >= 0 && c->rank < world, SV_EINVAL, "rank out of range");
        c->device = dist ? dist->device : 0;
        if (!dist) SV_CUDA(cudaGetDevice(&c->device));
        SV_CUDA(cudaSetDevice(c->device));
        if (dist && dist->stream) {
            c->stream = (cudaStream_t)dist->stream;
        } else {
            SV_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->own_stream = true;
        }
        c->nl_amps = 1ull << (n - g);
        c->nres = c->emulated ? (1ull << n) : c->nl_amps;
        const size_t bytes = c->nres * elem_bytes(dtype);
        dmalloc(&c->state, bytes, "state");
        if (g > 0) dmalloc(&c->recv, bytes, "swap receive buffer");
        dmalloc((void **)&c->d_partials, 2 * kMaxGrid * sizeof(double), "partials");
        dmalloc((void **)&c->d_sums, 8 * sizeof(double), "sums");
        dmalloc((void **)&c->d_counter, sizeof(unsigned int), "counter");
        dmalloc((void **)&c->d_gbar, 4 * sizeof(unsigned int), "grid barrier");
        SV_CUDA(cudaMemsetAsync(c->d_gbar, 0, 4 * sizeof(unsigned int), c->stream));
        if (const char *e = getenv("SV_MEAN_RESIDENT")) {
            c->mean_resident = strcmp(e, "0") != 0;
            c->mean_resreg = strcmp(e, "smem") != 0;
        }
        if (const char *e = getenv("SV_GRAPHS")) c->use_graphs = strcmp(e, "0") != 0;
        SV_CUDA(cudaMemsetAsync(c->d_counter, 0, sizeof(unsigned int), c->stream));
        SV_CUDA(cudaMemsetAsync(c->d_sums, 0, 8 * sizeof(double), c->stream));
        c->mgrid = std::min(mean_grid(c->nres, dtype), kMaxGrid);
        // world = 1 with an id: a one-rank communicator -- every collective of
        // the schedule (scalar allreduces, the polling waits) runs through NCCL
        // on one GPU (tests/test_nccl_one_rank_gpu.py)
        if (dist && !c->emulated && dist->nccl_id != nullptr) {
            ncclUniqueId id;
            memcpy(&id, dist->nccl_id, sizeof(id));
            SV_NCCL(ncclCommInitRank(&c->comm, world, id, c->rank));
        }
        setup_peers(c);
        setup_super(c);
        do_init(c, seed, init);
        *out = c;
    });
    if (st != SV_OK) {
        std::string msg = g_err;
        destroy(c);
        g_err = msg;
    }
    return st;
}

sv_status sv_reset(sv_ctx *c, uint64_t seed, sv_init_kind init) {
    return guarded([&] {
        check_ctx(c);
        do_init(c, seed, init);
    });
}

sv_status sv_set_marked(sv_ctx *c, const uint64_t *marked, uint64_t m) {
    return guarded([&] {
        check_ctx(c);
        SV_CUDA(cudaSetDevice(c->device));
        store_marked(c, marked, m);
    });
}

sv_status sv_apply_oracle(sv_ctx *c, const uint64_t *marked, uint64_t m) {
    return guarded([&] {
        check_ctx(c);
        SV_CUDA(cudaSetDevice(c->device));
        store_marked(c, marked, m);
        run(c, SV_K_ORACLE, [&] { launch_oracle_scatter(c->dt, c->state, c->d_marked, c->n_marked, c->stream); });
    });
}

sv_status sv_diffuse(sv_ctx *c, sv_diffusion d) {
    return guarded([&] {
        check_ctx(c);
        SV_CUDA(cudaSetDevice(c->device));
        if (d == SV_DIFFUSE_WHT) run_wht_schedule(c, 1, false);
        else if (d == SV_DIFFUSE_MEAN) run_mean(c, 1, false);
        else throw Error{SV_EINVAL, "unknown diffusion"};
    });
}

sv_status sv_iterate_noisy(sv_ctx *c, int k, double sigma, uint64_t seed, uint64_t t0) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(k >= 0, SV_EINVAL, "k must be >= 0");
        SV_CHECK(sigma >= 0.0 && sigma < 10.0, SV_EINVAL, "sigma must be in [0, 10)");
        SV_CHECK(c->n <= 64, SV_EINVAL, "internal: qubit index range");
        SV_CHECK(c->has_marked, SV_ESTATE, "sv_iterate_noisy before any marked set");
        SV_CUDA(cudaSetDevice(c->device));
        const Noise nz{sigma, 0.0, seed, t0};
        run_wht_schedule(c, k, true, &nz);
    });
}

sv_status sv_iterate_decoherent(sv_ctx *c, int k, double sigma, double rate, uint64_t seed, uint64_t t0,
                                double *survival) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(k >= 0, SV_EINVAL, "k must be >= 0");
        SV_CHECK(sigma >= 0.0 && sigma < 10.0, SV_EINVAL, "sigma must be in [0, 10)");
        SV_CHECK(rate >= 0.0 && rate < 1.0, SV_EINVAL, "rate must be in [0, 1)");
        SV_CHECK(c->n <= 64, SV_EINVAL, "internal: qubit index range");
        SV_CHECK(c->has_marked, SV_ESTATE, "sv_iterate_decoherent before any marked set");
        SV_CUDA(cudaSetDevice(c->device));
        if (k == 0) return;
        if ((size_t)k + 2 > c->deco_cap) {
            if (c->d_deco) SV_CUDA(cudaFree(c->d_deco));
            c->d_deco = nullptr;
            c->deco_cap = 0;
            dmalloc((void **)&c->d_deco, ((size_t)k + 2) * sizeof(double), "survival");
            c->deco_cap = (size_t)k + 2;
        }
        double *sum = c->d_deco, *scale = c->d_deco + 1, *surv = c->d_deco + 2;
        if (c->plan.whole) {  // one CTA: renormalises inside, once per iteration
            const Noise nz{sigma, rate, seed, t0};
            run_wht_schedule(c, k, true, &nz, surv);
        } else {
            // The renormalisations are global scalars, so the per-operation
            // factors of an iteration collapse into one: each iteration's last
            // tile pass writes its tiles' sum |a|^2 (Eq. 3's global sum) as it
            // stores them, a small kernel sums those partials in fixed order
            // (allreduced across ranks), and 1/sqrt(sum) is folded into the
            // next iteration's first load -- no extra read pass of the state.
            const size_t ntiles = (size_t)(c->nres >> c->plan.T);
            if (ntiles > c->tilepart_cap) {
                if (c->d_tilepart) SV_CUDA(cudaFree(c->d_tilepart));
                c->d_tilepart = nullptr;
                c->tilepart_cap = 0;
                dmalloc((void **)&c->d_tilepart, ntiles * sizeof(double), "per-tile sums");
                c->tilepart_cap = ntiles;
            }
            for (int it = 0; it < k; ++it) {
                Noise nz{sigma, rate, seed, t0 + (uint64_t)it, it == 0 ? nullptr : scale};
                nz.sumsq = c->d_tilepart;
                run_wht_schedule(c, 1, true, &nz);
                run(c, SV_K_REDUCE, [&] {
                    launch_sum_partials(c->d_tilepart, ntiles, c->d_partials, c->d_counter, sum, c->stream);
                });
                allreduce_sum(c, sum, 1);
                run(c, SV_K_REDUCE, [&] { launch_norm_finalize(sum, scale, surv + it, c->stream); });
            }
            run(c, SV_K_SCALE, [&] { launch_scale(c->dt, c->state, c->nres, scale, c->stream); });
        }
        if (survival) {
            SV_CUDA(cudaMemcpyAsync(survival, surv, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            sync_ctx(c);
        }
    });
}

sv_status sv_iterate(sv_ctx *c, int k, sv_diffusion d) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(k >= 0, SV_EINVAL, "k must be >= 0");
        SV_CHECK(c->has_marked, SV_ESTATE, "sv_iterate before any marked set (sv_set_marked / sv_apply_oracle)");
        SV_CUDA(cudaSetDevice(c->device));
        if (d == SV_DIFFUSE_WHT) run_wht_graphed(c, k);
        else if (d == SV_DIFFUSE_MEAN) run_mean(c, k, true);
        else throw Error{SV_EINVAL, "unknown diffusion"};
    });
}

sv_status sv_probabilities(sv_ctx *c, double *out, uint64_t len, int on_device) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(out != nullptr, SV_EINVAL, "out is NULL");
        SV_CHECK(len == c->nres, SV_EINVAL, "len must equal the resident length");
        SV_CUDA(cudaSetDevice(c->device));
        if (on_device) {
            run(c, SV_K_READOUT, [&] { launch_probabilities(c->dt, c->state, out, c->nres, c->stream); });
            return;
        }
        SV_CHECK(c->nres <= (1ull << 26), SV_ETOOBIG, "host gather above 2^26 entries");
        double *tmp = nullptr;
        dmalloc((void **)&tmp, c->nres * sizeof(double), "probabilities");
        try {
            run(c, SV_K_READOUT, [&] { launch_probabilities(c->dt, c->state, tmp, c->nres, c->stream); });
            SV_CUDA(cudaMemcpyAsync(out, tmp, c->nres * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            sync_ctx(c);
        } catch (...) {
            cudaFree(tmp);
            throw;
        }
        SV_CUDA(cudaFree(tmp));
    });
}

sv_status sv_sample(sv_ctx *c, uint64_t shots, uint64_t seed, uint64_t *out, int out_on_device) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(out != nullptr || shots == 0, SV_EINVAL, "out is NULL");
        SV_CHECK(out_on_device || shots <= (1ull << 26), SV_ETOOBIG, "host sample list above 2^26 shots");
        SV_CUDA(cudaSetDevice(c->device));
        const uint64_t nch = sample_chunks(c->nres);
        const int world = c->comm ? c->world : 1;
        const int rank = c->comm ? c->rank : 0;
        // chunk prefixes [nch], every rank's total [world], window [3], scan
        // segments [nb], chunk-local row prefixes [32 nch] (1/128 of the amplitudes)
        const uint64_t nb = sample_scan_blocks(c->nres);
        if (!c->d_samp)
            dmalloc((void **)&c->d_samp, (nch + (size_t)world + 3 + nb + 32 * nch) * sizeof(double), "sampler scratch");
        double *totals = c->d_samp + nch;  // [world]
        double *g = totals + world;         // window {global total, own offset, next rank's offset}
        double *bscr = g + 3;               // [nb]
        double *rowp = bscr + nb;           // [32 nch]
        uint64_t *dout = out;
        if (!out_on_device) {
            if (shots > c->shots_cap) {
                if (c->d_shots) SV_CUDA(cudaFree(c->d_shots));
                c->d_shots = nullptr;
                c->shots_cap = 0;
                dmalloc((void **)&c->d_shots, std::max<uint64_t>(shots, 1) * 8, "sample list");
                c->shots_cap = shots;
            }
            dout = c->d_shots;
        }
        const uint64_t key = hash64(seed ^ 0x53414D5000000000ull);  // "SAMP" (G21)
        run(c, SV_K_READOUT, [&] {
            launch_sample_prefix(c->dt, c->state, c->nres, c->d_samp, totals + rank, bscr, rowp, c->stream);
        });
        if (c->comm) {  // every rank's total, in rank order
            run(c, SV_K_ALLREDUCE, [&] {
                SV_NCCL(ncclAllGather(totals + rank, totals, 1, ncclFloat64, c->comm, c->stream));
            });
        }
        const uint64_t base = c->comm ? (uint64_t)c->rank * c->nl_amps : 0;
        run(c, SV_K_READOUT, [&] {
            launch_sample_draw(c->dt, c->state, c->nres, c->d_samp, rowp, totals, world, rank, g, key, shots, base, dout,
                               c->stream);
        });
        if (c->comm && shots) {  // each shot is owned by one rank; the others wrote 0
            run(c, SV_K_ALLREDUCE, [&] {
                SV_NCCL(ncclAllReduce(dout, dout, shots, ncclUint64, ncclSum, c->comm, c->stream));
            });
        }
        if (!out_on_device && shots) {
            SV_CUDA(cudaMemcpyAsync(out, dout, shots * 8, cudaMemcpyDeviceToHost, c->stream));
            sync_ctx(c);
        }
    });
}

sv_status sv_measure_marked_mass(sv_ctx *c, double *out) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(out != nullptr, SV_EINVAL, "out is NULL");
        SV_CHECK(c->has_marked, SV_ESTATE, "no marked set");
        SV_CUDA(cudaSetDevice(c->device));
        double *d = c->d_sums + 6;
        run(c, SV_K_READOUT, [&] { launch_marked_mass(c->dt, c->state, c->d_marked, c->n_marked, d, c->stream); });
        allreduce_sum(c, d, 1);
        SV_CUDA(cudaMemcpyAsync(out, d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        sync_ctx(c);
    });
}

sv_status sv_norm2(sv_ctx *c, double *out) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(out != nullptr, SV_EINVAL, "out is NULL");
        SV_CUDA(cudaSetDevice(c->device));
        double *d = c->d_sums + 7;
        run(c, SV_K_READOUT, [&] { launch_norm2(c->dt, c->state, c->nres, c->d_partials, c->d_counter, d, c->stream); });
        allreduce_sum(c, d, 1);
        SV_CUDA(cudaMemcpyAsync(out, d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        sync_ctx(c);
    });
}

sv_status sv_get_amplitudes(sv_ctx *c, void *host_out, uint64_t offset, uint64_t count) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(host_out != nullptr || count == 0, SV_EINVAL, "host_out is NULL");
        SV_CHECK(offset <= c->nres && count <= c->nres - offset, SV_EINVAL, "range outside the resident state");
        SV_CUDA(cudaSetDevice(c->device));
        const size_t eb = elem_bytes(c->dt);
        SV_CUDA(cudaMemcpyAsync(host_out, (char *)c->state + offset * eb, count * eb, cudaMemcpyDeviceToHost, c->stream));
        sync_ctx(c);
    });
}

sv_status sv_set_amplitudes(sv_ctx *c, const void *host_in, uint64_t offset, uint64_t count) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(host_in != nullptr || count == 0, SV_EINVAL, "host_in is NULL");
        SV_CHECK(offset <= c->nres && count <= c->nres - offset, SV_EINVAL, "range outside the resident state");
        SV_CUDA(cudaSetDevice(c->device));
        const size_t eb = elem_bytes(c->dt);
        SV_CUDA(cudaMemcpyAsync((char *)c->state + offset * eb, host_in, count * eb, cudaMemcpyHostToDevice, c->stream));
        sync_ctx(c);
    });
}

sv_status sv_marked_from_seed(int n, uint64_t m, uint64_t seed, uint64_t *out) {
    return guarded([&] {
        SV_CHECK(n >= 1 && n <= 40, SV_EINVAL, "n must be in [1, 40]");
        SV_CHECK(m <= (1ull << n), SV_EINVAL, "m > 2^n");
        SV_CHECK(out != nullptr || m == 0, SV_EINVAL, "out is NULL");
        for (uint64_t j = 0; j < m; ++j) out[j] = perm_seeded(n, seed, j);
        std::sort(out, out + m);
    });
}

sv_status sv_info(const sv_ctx *c, int *n, int *world, int *rank, uint64_t *local_len, sv_dtype *dtype) {
    return guarded([&] {
        check_ctx(c);
        if (n) *n = c->n;
        if (world) *world = c->world;
        if (rank) *rank = c->rank;
        if (local_len) *local_len = c->nres;
        if (dtype) *dtype = c->dt;
    });
}

sv_status sv_comm_info(const sv_ctx *c, int *nranks, int *comm_rank) {
    return guarded([&] {
        check_ctx(c);
        int nr = 0, ur = -1;
        if (c->comm != nullptr) {
            SV_NCCL(ncclCommCount(c->comm, &nr));
            SV_NCCL(ncclCommUserRank(c->comm, &ur));
        }
        if (nranks) *nranks = nr;
        if (comm_rank) *comm_rank = ur;
    });
}

sv_status sv_attach(sv_ctx *c, void *dev_ptr, uint64_t bytes) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(dev_ptr != nullptr, SV_EINVAL, "dev_ptr is NULL");
        SV_CHECK(bytes == c->nres * elem_bytes(c->dt), SV_EINVAL,
                 "bytes must equal the resident state size (" + std::to_string(c->nres * elem_bytes(c->dt)) + ")");
        SV_CHECK(((uintptr_t)dev_ptr & 15u) == 0, SV_EINVAL, "dev_ptr must be 16-byte aligned");
        SV_CHECK(c->comm == nullptr, SV_ESTATE,
                 "sv_attach is single-process only (peer mappings of the fused exchange are made at sv_init)");
        SV_CUDA(cudaSetDevice(c->device));
        cudaPointerAttributes at{};
        SV_CUDA(cudaPointerGetAttributes(&at, dev_ptr));
        SV_CHECK(at.type == cudaMemoryTypeDevice && at.device == c->device, SV_EINVAL,
                 "dev_ptr is not device memory of the context's GPU");
        sync_ctx(c);  // no pending work on the old buffer
        if (c->owns_state) SV_CUDA(cudaFree(c->state));
        c->state = dev_ptr;
        c->owns_state = false;
        for (auto &ge : c->graphs) cudaGraphExecDestroy(ge.exec);  // graphs bake the state pointer
        c->graphs.clear();
    });
}

sv_status sv_snapshot(sv_ctx *c, const char *path, uint64_t *written) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(path != nullptr, SV_EINVAL, "path is NULL");
        SV_CHECK(c->nres <= (1ull << 26), SV_ETOOBIG, "snapshot above 2^26 resident amplitudes");
        SV_CUDA(cudaSetDevice(c->device));
        FILE *f = fopen(path, "w");
        SV_CHECK(f != nullptr, SV_EINVAL, std::string("cannot open ") + path);
        uint64_t count = 0;
        try {
            const uint64_t base = (!c->emulated && c->world > 1) ? (uint64_t)c->rank * c->nl_amps : 0;
            fprintf(f, "s=2 M=%d\n", c->n);
            const size_t eb = elem_bytes(c->dt);
            constexpr uint64_t kChunk = 1ull << 20;
            std::vector<unsigned char> buf(kChunk * eb);
            for (uint64_t off = 0; off < c->nres; off += kChunk) {
                const uint64_t cnt = std::min<uint64_t>(kChunk, c->nres - off);
                SV_CUDA(cudaMemcpyAsync(buf.data(), (char *)c->state + off * eb, cnt * eb, cudaMemcpyDeviceToHost,
                                        c->stream));
                sync_ctx(c);
                for (uint64_t i = 0; i < cnt; ++i) {
                    double re, im;
                    if (c->dt == SV_C64) {
                        const float *v = reinterpret_cast<const float *>(buf.data()) + 2 * i;
                        re = v[0];
                        im = v[1];
                    } else {
                        const double *v = reinterpret_cast<const double *>(buf.data()) + 2 * i;
                        re = v[0];
                        im = v[1];
                    }
                    if (re == 0.0 && im == 0.0) continue;
                    fprintf(f, "%llu %.17g %.17g\n", (unsigned long long)(base + off + i), re, im);
                    ++count;
                }
            }
        } catch (...) {
            fclose(f);
            throw;
        }
        SV_CHECK(fclose(f) == 0, SV_EINVAL, std::string("write failed: ") + path);
        if (written) *written = count;
    });
}

sv_status sv_set_exchange(sv_ctx *c, int fused) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(!fused || c->xchg_capable, SV_ESTATE, "fused exchange unavailable (1 rank, > 8 ranks or no peer access)");
        c->fused_xchg = fused != 0;
    });
}

sv_status sv_get_exchange(const sv_ctx *c, int *fused) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(fused != nullptr, SV_EINVAL, "fused is NULL");
        *fused = c->fused_xchg ? 1 : 0;
    });
}

sv_status sv_synchronize(sv_ctx *c) {
    return guarded([&] {
        check_ctx(c);
        SV_CUDA(cudaSetDevice(c->device));
        sync_ctx(c);
    });
}

sv_status sv_nccl_unique_id(void *out, size_t len) {
    return guarded([&] {
        SV_CHECK(out != nullptr && len >= sizeof(ncclUniqueId), SV_EINVAL, "need a 128-byte buffer");
        ncclUniqueId id;
        SV_NCCL(ncclGetUniqueId(&id));
        memcpy(out, &id, sizeof(id));
    });
}

sv_status sv_plan_wht(int n, int world, sv_dtype dtype, int k, int with_oracle, sv_plan_step *out, int cap,
                      int *nsteps) {
    return guarded([&] {
        SV_CHECK(world >= 1 && (world & (world - 1)) == 0, SV_EINVAL, "world must be a power of two");
        SV_CHECK(k >= 0, SV_EINVAL, "k must be >= 0");
        int g = 0;
        while ((1 << g) < world) ++g;
        SV_CHECK(g <= n, SV_EINVAL, "world larger than 2^n");
        Plan p = make_plan(n, g, dtype);
        std::vector<Step> steps = schedule_wht(p, k, with_oracle != 0);
        if (nsteps) *nsteps = (int)steps.size();
        for (int i = 0; i < (int)steps.size() && i < cap && out; ++i) {
            const Step &s = steps[i];
            sv_plan_step &o = out[i];
            o.kind = s.kind;
            o.pre = s.pre;
            o.mid = s.mid;
            o.post = s.post;
            o.in_recv = s.in_recv;
            o.tile_bits = p.whole ? p.nl
                          : (p.super && s.group == p.sup.group) ? __builtin_popcountll(p.sup.st) : p.T;
            o.tile_mask = (s.group >= 0) ? p.groups[s.group].tile : 0;
            o.proc_mask = (s.group >= 0) ? p.groups[s.group].proc : 0;
        }
    });
}

sv_status sv_debug_wht_variants(int n, int world, sv_dtype dtype, int flavour, int k, double sigma, double rate,
                                uint64_t seed, int fused, sv_tile_variant *out, int cap, int *count) {
    return guarded([&] {
        SV_CHECK(world >= 1 && (world & (world - 1)) == 0, SV_EINVAL, "world must be a power of two");
        SV_CHECK(k >= 0, SV_EINVAL, "k must be >= 0");
        SV_CHECK(flavour >= 0 && flavour <= 3, SV_EINVAL, "flavour must be 0..3");
        int g = 0;
        while ((1 << g) < world) ++g;
        SV_CHECK(g <= n, SV_EINVAL, "world larger than 2^n");
        // the schedule code of the entry points, on a context without device
        // memory (emulated sharding for world > 1: the same passes per rank)
        sv_ctx c;
        c.n = n;
        c.g = g;
        c.world = world;
        c.dt = dtype;
        c.plan = make_plan(n, g, dtype);
        c.emulated = world > 1;
        c.fused_xchg = fused != 0 && world > 1 && world <= 8;
        c.nl_amps = 1ull << (n - g);
        c.nres = c.emulated ? (1ull << n) : c.nl_amps;
        std::vector<TileVariant> v;
        c.dry = &v;
        static double dummy_scale = 1.0;  // stands for the device renormalisation scalar
        if (flavour == 0) {
            run_wht_schedule(&c, k, true);
        } else if (flavour == 1) {
            const Noise nz{sigma, 0.0, seed, 0};
            run_wht_schedule(&c, k, true, &nz);
        } else if (flavour == 2) {  // as sv_iterate_decoherent
            if (c.plan.whole) {
                const Noise nz{sigma, rate, seed, 0};
                if (k > 0) run_wht_schedule(&c, k, true, &nz, &dummy_scale);
            } else {
                for (int it = 0; it < k; ++it) {
                    Noise nz{sigma, rate, seed, (uint64_t)it, it == 0 ? nullptr : &dummy_scale};
                    nz.sumsq = &dummy_scale;
                    run_wht_schedule(&c, 1, true, &nz);
                }
            }
        } else {
            run_wht_schedule(&c, 1, false);
        }
        if (count) *count = (int)v.size();
        for (int i = 0; i < (int)v.size() && i < cap && out; ++i) {
            out[i].family = v[i].family;
            out[i].u = v[i].u;
            out[i].pre = v[i].pre;
            out[i].mid = v[i].mid;
            out[i].post = v[i].post;
            out[i].noisy = v[i].noisy;
            out[i].xchg = v[i].xchg;
        }
    });
}

sv_status sv_apply_gates(sv_ctx *c, const sv_gate *gates, uint64_t count) {
    return guarded([&] {
        check_ctx(c);
        SV_CUDA(cudaSetDevice(c->device));
        run_gates(c, gates, count);
    });
}

sv_status sv_plan_gates(int n, int world, sv_dtype dtype, const sv_gate *gates, uint64_t count,
                        sv_gate_plan_step *out, int cap, int *nsteps, uint64_t *order) {
    return guarded([&] {
        SV_CHECK(world >= 1 && (world & (world - 1)) == 0, SV_EINVAL, "world must be a power of two");
        int g = 0;
        while ((1 << g) < world) ++g;
        SV_CHECK(g <= n, SV_EINVAL, "world larger than 2^n");
        const GatePlan gp = plan_gates(n, g, dtype, gates, count);
        if (nsteps) *nsteps = (int)gp.steps.size();
        for (int i = 0; i < (int)gp.steps.size() && i < cap && out; ++i) {
            const GateStep &s = gp.steps[i];
            sv_gate_plan_step &o = out[i];
            o.kind = s.kind;
            o.tile_bits = s.kind == GSTEP_WHOLE ? n : gp.T;
            o.tile_mask = s.tile;
            o.proc_mask = s.proc;
            o.first = s.first;
            o.count = s.count;
            o.ops = s.ops;
            o.lin_ops = s.lin_ops;
        }
        if (order)
            for (size_t j = 0; j < gp.order.size(); ++j) order[j] = gp.order[j];
    });
}

sv_status sv_debug_gate_relayouts(int n, int world, sv_dtype dtype, const sv_gate *gates, uint64_t count,
                                  uint64_t *out, int cap, int *nsteps) {
    return guarded([&] {
        SV_CHECK(world >= 1 && (world & (world - 1)) == 0, SV_EINVAL, "world must be a power of two");
        int g = 0;
        while ((1 << g) < world) ++g;
        SV_CHECK(g <= n, SV_EINVAL, "world larger than 2^n");
        const GatePlan gp = plan_gates(n, g, dtype, gates, count);
        if (nsteps) *nsteps = (int)gp.steps.size();
        for (int i = 0; i < (int)gp.steps.size() && i < cap && out; ++i) {
            const GateStep &st = gp.steps[i];
            out[i] = 0;
            if (st.kind != GSTEP_PASS) continue;
            GatePassArgs a;  // rank 0's program (controls on rank bits decided as on rank 0)
            a.tile_mask = st.tile;
            a.total_bits = gp.nl;
            a.g = gp.g;
            a.swapped = st.swapped;
            a.n = gp.n;
            a.nl = gp.nl;
            a.gates = gates;
            a.order = gp.order.data() + st.first;
            a.count = st.count;
            out[i] = count_gate_relayouts(dtype, a);
        }
    });
}

sv_status sv_profile(sv_ctx *c, int enable) {
    return guarded([&] {
        check_ctx(c);
        drain_profile(c);
        c->prof = enable != 0;
        for (int i = 0; i < SV_K_COUNT; ++i) {
            c->launches[i] = 0;
            c->ms[i] = 0.0;
        }
        c->timeline.clear();
    });
}

sv_status sv_profile_timeline(sv_ctx *c, int *kinds, double *ms, uint64_t cap, uint64_t *count) {
    return guarded([&] {
        check_ctx(c);
        drain_profile(c);
        if (count) *count = c->timeline.size();
        for (uint64_t i = 0; i < cap && i < c->timeline.size(); ++i) {
            if (kinds) kinds[i] = c->timeline[i].first;
            if (ms) ms[i] = c->timeline[i].second;
        }
    });
}

sv_status sv_profile_read(sv_ctx *c, int kind, uint64_t *launches, double *total_ms) {
    return guarded([&] {
        check_ctx(c);
        SV_CHECK(kind >= 0 && kind < SV_K_COUNT, SV_EINVAL, "kind out of range");
        drain_profile(c);
        if (launches) *launches = c->launches[kind];
        if (total_ms) *total_ms = c->ms[kind];
    });
}

void sv_free(sv_ctx *c) { destroy(c); }

}  // extern "C"
