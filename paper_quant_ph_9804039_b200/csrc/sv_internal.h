// sv_internal.h -- internal declarations of libsv.so (not part of the ABI).
// Citations: P:NNNN = line of the paper text, S:NNN = SPEC line, G<k> = a
// reading in DESIGN.md.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sv.h"
#include "sv_consts.h"

namespace sv {

// ------------------------------------------------------------------------- //
// Error plumbing                                                             //
// ------------------------------------------------------------------------- //
void set_error(const std::string &msg);

struct Error {
    sv_status code;
    std::string msg;
};

#define SV_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            throw ::sv::Error{SV_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

#define SV_NCCL(call)                                                                     \
    do {                                                                                  \
        ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess)                                                            \
            throw ::sv::Error{SV_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)}; \
    } while (0)

#define SV_CHECK(cond, code, msg)                                   \
    do {                                                            \
        if (!(cond)) throw ::sv::Error{(code), std::string(msg)};   \
    } while (0)

// ------------------------------------------------------------------------- //
// Tile geometry per dtype                       //
// ------------------------------------------------------------------------- //
inline int tile_bits(sv_dtype d) { return d == SV_C64 ? kTileBitsC64 : kTileBitsC128; }
inline int gate_tile_bits(sv_dtype d) { return d == SV_C64 ? kGateTileBitsC64 : kTileBitsC128; }
inline int carry_bits(sv_dtype d) { return d == SV_C64 ? kCarryC64 : kCarryC128; }
inline size_t elem_bytes(sv_dtype d) { return d == SV_C64 ? 8 : 16; }

// ------------------------------------------------------------------------- //
// Schedule (plan.cpp)                                                        //
// ------------------------------------------------------------------------- //
enum StepKind { STEP_PASS = 0, STEP_SWAP = 1, STEP_WHOLE = 2, STEP_SCATTER = 3 };

struct Group {
    uint64_t proc = 0;   // slots whose butterfly stages run in this pass
    uint64_t tile = 0;   // slots spanned by one tile (popcount == T), proc subset
};

struct Step {
    int kind = STEP_PASS;
    int group = -1;
    int pre = 0, mid = MID_NONE, post = 0;
    int in_recv = 0;
    int pre_swap = 0;   // the next step is a qubit swap (its store can BE the exchange)
    int tr_pre = -1;    // transform (2 x iteration + w, within the call) of the pre stages
    int tr_post = -1;   // ... of the post stages
    int layout = 0;     // 0 = natural; 1 = top-g local slots hold the rank qubits
};

// L2-staged supertile pass: the F0 group's
// processed slots plus two carry slots form a supertile of 2^|st| amplitudes
// that stays in L2 while three dependent sub-passes of ordinary 2^T tiles run
// over it -- level A's stages (transform 1), level B's stages + F0 + level B's
// stages, level A's stages (transform 2) -- so the group costs ONE HBM read
// and write of the state however many slots it has.
struct SuperSpec {
    int group = -1;          // index of the supertile group in Plan::groups
    uint64_t st = 0;         // slots of one supertile (carry slots + the group's processed slots)
    uint64_t tileA = 0, procA = 0;  // level A sub-passes: tile slots, processed slots
    uint64_t tileB = 0, procB = 0;  // level B (F0) sub-pass
    int uB = 0;              // unprocessed tile bits of the level B tiles
};

struct Plan {
    int nl = 0;       // local index bits (n - g)
    int g = 0;        // rank bits
    int T = 0;        // tile bits
    bool whole = false;
    bool super = false;      // the F0 group is a supertile group (sup)
    SuperSpec sup;
    std::vector<Group> groups;   // groups[0] = contiguous slots [0, T)
    // fwd[0] hosts the oracle O (natural layout), fwd.back() hosts F0
    std::vector<int> fwd;        // first transform: group indices, -1 = swap
};

// (level A, level B) unprocessed tile bits with a supertile kernel instantiation (wht_super.cuh).
inline bool super_pair_supported(int ua, int ub) {
    return (ua == 2 && ub >= 5 && ub <= 12) || (ua == 9 && ub == 5);
}
// Validates (n, g, dtype) and builds the group structure.  Throws Error.
Plan make_plan(int n, int g, sv_dtype dtype);
// Expand an op sequence to fused device steps.
//   with_oracle: iterations (O, WHT, F0, WHT) x k; else one (WHT, F0, WHT).
std::vector<Step> schedule_wht(const Plan &plan, int k, bool with_oracle);

// ------------------------------------------------------------------------- //
// Gate circuits (gate_plan.cpp)                          //
// ------------------------------------------------------------------------- //
enum GateStepKind { GSTEP_PASS = 0, GSTEP_SWAP = 1, GSTEP_WHOLE = 2 };

struct GateStep {
    int kind = GSTEP_PASS;
    uint64_t proc = 0;   // physical slots targeted by the pass's gates
    uint64_t tile = 0;   // physical slots of one tile (popcount == T)
    int swapped = 0;     // layout during the pass: 0 natural, 1 top-g local <-> rank bits
    uint64_t first = 0;  // gates order[first .. first + count)
    uint64_t count = 0;
    uint64_t ops = 0;    // ops after the host fusion of same-target gates (gates.cu)
    uint64_t lin_ops = 0;  // of which merged phase runs (phase-polynomial ops)
};

struct GatePlan {
    int n = 0, nl = 0, g = 0, T = 0;
    std::vector<GateStep> steps;
    std::vector<uint64_t> order;   // gate indices in execution order
};

// Validates every gate (throws Error{SV_EINVAL}) and builds the schedule.
GatePlan plan_gates(int n, int g, sv_dtype dtype, const sv_gate *gates, uint64_t count);
// Physical slot of logical qubit q in layout `swapped` (section 3.1 swap of
// the top-g local slots [nl-g, nl) with the rank bits [nl, n)).
inline int gate_phys(int q, int nl, int g, int swapped) {
    if (!swapped) return q;
    if (q >= nl) return q - g;
    if (q >= nl - g) return q + g;
    return q;
}

// x = y = 0 exactly: the gate is diagonal (a phase on each basis state).
inline bool gate_diag(const sv_gate &g) { return g.m[2] == 0.0 && g.m[3] == 0.0 && g.m[4] == 0.0 && g.m[5] == 0.0; }

// Gates a later gate must commute with to be moved ahead of them (sufficient
// conditions).  A controlled 2x2 is P0 (x) I + P1 (x) U on its controls:
//  * two non-diagonal gates commute if the targets differ and neither target
//    is a control of the other;
//  * a diagonal gate D commutes with any gate whose target is outside D's
//    support (target + controls): D commutes with the control projectors;
//  * two diagonal gates always commute.
struct CommuteSet {
    uint64_t tnd = 0;   // targets of non-diagonal gates
    uint64_t cnd = 0;   // controls of non-diagonal gates
    uint64_t sd = 0;    // supports of diagonal gates
    void add(const sv_gate &g) {
        const uint64_t t = 1ull << g.target;
        if (gate_diag(g)) sd |= t | g.controls;
        else { tnd |= t; cnd |= g.controls; }
    }
    bool commutes(const sv_gate &g) const {
        const uint64_t t = 1ull << g.target;
        if (gate_diag(g)) return !((t | g.controls) & tnd);
        return !(t & (tnd | cnd | sd)) && !(g.controls & tnd);
    }
};

// One gate-circuit tile pass / the whole-state gate kernel (gates.cu).
struct GatePassArgs {
    void *in = nullptr;
    void *out = nullptr;
    uint64_t tile_mask = 0;       // physical slots of a tile
    int total_bits = 0;           // index bits of the launched buffer
    int g = 0;                    // rank bits
    int rank = 0;                 // own rank (real) -- controls on rank bits are decided on the host
    int emulated = 0;
    int swapped = 0;
    int n = 0, nl = 0;
    const sv_gate *gates = nullptr;  // host
    const uint64_t *order = nullptr; // host: this pass's gate indices (execution order)
    uint64_t count = 0;
    // fused qubit-swap exchange as in PassArgs
    int xchg_nl = 0, xchg_g = 0, xchg_rank = -1;
    void *xchg_dst[8] = {};
    // gate JIT (complex64, gate_jit.cu): jit_prepare = the run_gates call
    // number -> decide / compile only, store the kernel (or nullptr) in
    // *jit_kern, launch nothing; 0 -> launch *jit_kern if set, else the interpreter
    uint64_t jit_prepare = 0;
    void **jit_kern = nullptr;
};
// Append the op program of one pass (whole: the one-CTA kernel) to `prog`
// (16-byte aligned records); returns the op count.  Ops whose rank-bit
// controls fail on this rank are dropped.  *has_lin: the pass holds merged
// phase runs (launched with the kernel instantiation that handles them).
uint64_t build_gate_ops(sv_dtype dt, const GatePassArgs &a, bool whole, std::vector<unsigned char> &prog,
                        bool *has_lin);
// Shared-memory relayouts the tile kernel performs on one pass's program
// (host only; layout changes between consecutive ops).
uint64_t count_gate_relayouts(sv_dtype dt, const GatePassArgs &a);
// dev_ops: the pass's records in device memory; host_ops: the same records on
// the host (NULL = none) -- a program that fits the kernel-parameter space is
// passed by value (constant bank) instead.
void launch_gate_pass(sv_dtype dt, const GatePassArgs &a, const void *dev_ops, const void *host_ops, uint64_t nops,
                      bool has_lin, cudaStream_t s);
void launch_gate_whole(sv_dtype dt, const GatePassArgs &a, const void *dev_ops, uint64_t nops, cudaStream_t s);

// ------------------------------------------------------------------------- //
// Kernel launchers (wht.cu, mean.cu, misc.cu)                                //
// ------------------------------------------------------------------------- //
struct PassArgs {
    void *in = nullptr;
    void *out = nullptr;
    const uint64_t *marked = nullptr;   // sorted local indices (device)
    uint64_t n_marked = 0;
    const unsigned int *tilemap = nullptr;  // bit per contiguous 2^T tile: holds a marked index
    double f0_scale = 0.0;              // 2^-n
    int mid = MID_NONE;
    int has_origin = 0;                 // global index 0 resident at local 0
    int pre = 0, post = 0;
    uint64_t tile_mask = 0;             // slots of one tile
    uint64_t proc_mask = 0;             // processed slots (subset of tile_mask)
    int total_bits = 0;                 // index bits of the launched buffer
    // fused qubit-swap exchange: the pass's store sends every element to its
    // new owner (xchg_nl > 0 enables; see global_store_xchg in wht.cu)
    int xchg_nl = 0;                    // local index bits per rank
    int xchg_g = 0;                     // rank bits
    int xchg_rank = -1;                 // own rank; -1 = emulation (rank = index >> nl)
    void *xchg_dst[8] = {};             // destination buffer base of each rank
    // general 2x2 stages (NEXT-1 angle errors, NEXT-2 decoherence):
    // coef[half][slot] = [w x; y z] for the stages before (half 0) / after
    // (half 1) the elementwise op
    int noisy = 0;
    double coef[2][64][4] = {};
    const double *scale_in = nullptr;   // device scalar multiplied into the loaded tile
    double *sumsq = nullptr;            // device: per-tile fp64 sum |a|^2 of the stored tile (noisy flavours)
};

// Template instantiation a tile pass runs (host-side description).
struct TileVariant {
    int family = 0;   // 0 whole-state kernel, 1 three-layout tile kernel, 2 two-layout (strided c64),
                      // 3 sub-pass of the supertile kernel (three per supertile pass)
    int u = 0;        // unprocessed (carry) tile bits; processed = [u, T)
    int pre = 0, mid = 0, post = 0;
    int noisy = 0;    // 0 ideal butterflies, 1 general real 2x2, 2 angle-error tan form
    int xchg = 0;     // store is the fused qubit-swap exchange
};
// One supertile pass (wht_super.cu): the F0 group's three sub-passes over
// L2-resident supertiles in one persistent launch.
struct SuperArgs {
    PassArgs sub[3];               // sub-pass 0: level A pre; 1: level B pre + F0 + post; 2: level A post
    uint64_t st_mask = 0;          // slots of one supertile
    int ua = 0, ub = 0;            // unprocessed tile bits of the level A / level B tiles
    unsigned int *ctr = nullptr;   // device: ticket + per-(supertile, sub-pass) counters (zeroed by the launch)
    const unsigned int *seg = nullptr;  // device: segment order, (supertile << 2) | sub-pass
    uint64_t nseg = 0;
    int grid = 0;                  // persistent CTAs
};
// describe != nullptr: fill it and launch nothing (no device needed).
void launch_wht_super_pass(sv_dtype dt, const SuperArgs &a, cudaStream_t s, TileVariant *describe = nullptr);
// Persistent CTAs of the supertile kernel (occupancy x SMs; host query).
int super_grid();
// describe != nullptr: fill it and launch nothing (no device needed).
void launch_wht_tile_pass(sv_dtype dt, const PassArgs &a, cudaStream_t s, TileVariant *describe = nullptr);
TileVariant describe_tile_pass(sv_dtype dt, const PassArgs &a);
void launch_whole_state(sv_dtype dt, void *state, int n, int k, int with_oracle, int diffusion,
                        const uint64_t *marked, uint64_t m, cudaStream_t s, const double *coefs = nullptr,
                        double *survival = nullptr);

struct MeanArgs {
    void *a = nullptr;
    uint64_t N = 0;                    // resident amplitudes
    double inv_total = 0.0;            // 1 / 2^n (global N)
    const uint64_t *marked = nullptr;  // sorted local indices
    uint64_t n_marked = 0;
    const unsigned int *chunkmap = nullptr;  // bit per mean_chunk_elems() chunk: holds a marked index
    const double *sum_in = nullptr;    // complex sum of (O a) over all ranks
    double *sum_out = nullptr;         // local complex sum of (O a_new)
    double *partials = nullptr;        // 2 * grid doubles
    unsigned int *counter = nullptr;   // zero-initialised ticket
    double *tilepart = nullptr;        // tile form: 2 * mean_tiles() doubles (per-tile partials)
};
// One wave of blocks (SM count x resident blocks), capped by the work.
int mean_grid(uint64_t N, sv_dtype dt);
uint64_t mean_chunk_elems(sv_dtype dt);  // amplitudes per chunk (tile) of the mean kernel
bool mean_tile_mode();                   // SV_MEAN_TILE (default on): one CTA per 64 KiB tile
uint64_t mean_tiles(uint64_t N, sv_dtype dt);
// write = true: fused flip + invert-about-mean + next-sum; false: read-only
// sum of (O a) (the first mu of an sv_iterate call).
void launch_mean_grid(sv_dtype dt, const MeanArgs &a, int grid, bool write, cudaStream_t s);

// All k mean-diffusion iterations in one cooperative launch when the state
// fits the aggregate shared memory of one wave (mean_resident.cu).
bool mean_resident_fits(sv_dtype dt, uint64_t N, size_t partials_cap);
// slots: mean_resident_slot_bytes() of device memory reserved for the
// kernel's all-gather; epoch0: launch-unique, advanced by >= k + 1 per launch.
// bar: 4 unsigned ints (the shared-memory kernel's {count, generation}, then
// the register kernel's 64-bit arrival counter).  regs: the register-resident
// kernel where its slice fits (else the shared-memory one).  acc: 64 k uint64
// of device memory for the register kernel's fixed-point per-iteration sums
// (zeroed here before the launch), or nullptr (fp64 gather every round).
size_t mean_resident_slot_bytes(sv_dtype dt, uint64_t N);
void launch_mean_resident(sv_dtype dt, void *a, uint64_t N, double inv_N, const uint64_t *marked, uint64_t m, int k,
                          double *partials, unsigned int *bar, void *slots, unsigned long long epoch0, bool regs,
                          void *acc, cudaStream_t s);

void launch_init_uniform(sv_dtype dt, void *a, uint64_t N, int n, cudaStream_t s);
void launch_init_zero(sv_dtype dt, void *a, uint64_t N, int has_origin, cudaStream_t s);
// Gaussian (G8): pass 1 writes the local sum |z|^2 into *norm_out (fp64),
// pass 2 regenerates and scales by 1/sqrt(*norm_in).
void launch_gauss_norm(uint64_t key, uint64_t global_offset, uint64_t N, double *partials,
                       unsigned int *counter, double *norm_out, cudaStream_t s);
void launch_gauss_write(sv_dtype dt, void *a, uint64_t key, uint64_t global_offset, uint64_t N,
                        const double *norm_in, cudaStream_t s);
void launch_oracle_scatter(sv_dtype dt, void *a, const uint64_t *marked, uint64_t m, cudaStream_t s);
void launch_probabilities(sv_dtype dt, const void *a, double *p, uint64_t N, cudaStream_t s);
void launch_marked_mass(sv_dtype dt, const void *a, const uint64_t *marked, uint64_t m, double *out,
                        cudaStream_t s);

// Seeded whole-register measurement (sample.cu; NEXT-3, G21).
uint64_t sample_chunks(uint64_t N);
uint64_t sample_scan_blocks(uint64_t N);  // segments of the chunk-prefix scan (scratch doubles)
void launch_sample_prefix(sv_dtype dt, const void *a, uint64_t N, double *scratch, double *rank_total,
                          double *bscratch, double *rowp, cudaStream_t s);
void launch_sample_draw(sv_dtype dt, const void *a, uint64_t N, const double *scratch, const double *rowp,
                        const double *totals,
                        int world, int rank, double *g, uint64_t key, uint64_t shots, uint64_t index_base,
                        uint64_t *out, cudaStream_t s);

// Seeded generators (host side of the library; G6, G8).
uint64_t splitmix64_next(uint64_t &state);
uint64_t hash64(uint64_t x);
uint64_t gauss_key(uint64_t seed);
uint64_t perm_seeded(int n, uint64_t seed, uint64_t x);
// Angle error of qubit q in transform w of iteration t (G20).
double noise_delta(uint64_t seed, uint64_t t, int w, int q, double sigma);
// Decoherence site after laser operation q of transform w, iteration t (G22).
int decay_site(int n, uint64_t seed, uint64_t t, int w, int q);
// Renormalisation (G22): sum |a|^2 -> *sum (deterministic), then
// scale_out = 1/sqrt(sum), survival = sum (either pointer may be null).
void launch_norm2(sv_dtype dt, const void *a, uint64_t N, double *partials, unsigned int *counter, double *sum,
                  cudaStream_t s);
void launch_norm_finalize(const double *sum, double *scale_out, double *survival, cudaStream_t s);
// Fixed-order fp64 sum of count partials (per-tile sums) -> *sum.
void launch_sum_partials(const double *in, uint64_t count, double *partials, unsigned int *counter, double *sum,
                         cudaStream_t s);
void launch_scale(sv_dtype dt, void *a, uint64_t N, const double *scale, cudaStream_t s);

}  // namespace sv
