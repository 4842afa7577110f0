/*
 * sv.h -- C ABI of the B200-native Grover state-vector hot path
 * (arxiv quant-ph/9804039, Obenland & Despain, "A Parallel Quantum Computer
 * Simulator", HPC'98).
 *
 * Implemented by paper_quant_ph_9804039_b200/libsv.so (hand-written CUDA for
 * sm_100a + NCCL).  C99, extern "C", plain pointers and sizes; no torch types.
 *
 * Citations: P:NNNN is a line of the paper text (reference PAPER.md);
 * S:NNN a line of the reference SPEC.md; G<k> a reading in DESIGN.md
 * ("Readings").  The paper cites quantum search only in section 1.5
 * (P:2946-2965); the iteration a <- D O a is fixed by the north star (G1).
 *
 * Conventions used by every call
 *  - Amplitude store (section 1.2): a dense vector of N = 2^n
 *    complex amplitudes; "the bit value of a state corresponds to the index of
 *    that state in the vector": qubit q is bit q of the index (G4).
 *    Layout is interleaved complex: SV_C64 = {float re, im} (8 B),
 *    SV_C128 = {double re, im} (16 B) -- torch.complex64/complex128 compatible.
 *  - Sharding (section 3.1): with P = 2^g ranks the "parallel
 *    bits" are the top g qubits, concatenated MSB first into the rank
 *    (P:4102-4103): rank r owns global indices [r*N/P, (r+1)*N/P).
 *    local index = global index - r*N/P.  Between calls the layout is always
 *    this natural one (internal qubit swaps are undone before a call returns).
 *  - Status: every sv_status call returns SV_OK (0) or a negative code and
 *    sets a thread-local message readable with sv_last_error().  After
 *    SV_ECUDA / SV_ENCCL the context must be freed.
 *  - Streams: all device work of a context is enqueued on one stream (the
 *    caller's, if given in sv_dist.stream, else a stream the context creates).
 *    Calls returning host data synchronise that stream; others are
 *    asynchronous.  A context is single-writer: no concurrent
 *    calls on the same sv_ctx.
 *  - Ownership: the library owns every device buffer it allocates; input
 *    arrays are copied before the call returns; output buffers belong to the
 *    caller.
 */
#ifndef SV_H
#define SV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SV_OK = 0,
    SV_EINVAL = -1,  /* invalid argument (range, ordering, power-of-two, size) */
    SV_ENOMEM = -2,  /* device or host allocation failed                       */
    SV_ECUDA = -3,   /* CUDA runtime error (message has cudaGetErrorString)    */
    SV_ENCCL = -4,   /* NCCL error (message has ncclGetErrorString)            */
    SV_ESTATE = -5,  /* call not valid in the context's state                  */
    SV_ETOOBIG = -6  /* host gather above the 2^26-entry guard     */
} sv_status;

typedef enum { SV_C64 = 0, SV_C128 = 1 } sv_dtype;

typedef enum {
    SV_INIT_UNIFORM = 0,    /* |s> = H^n|0>: every amplitude 2^{-n/2} (Fig. 1(b)) */
    SV_INIT_GAUSSIAN = 1,   /* seeded complex Gaussian, normalised to ||a||_2 = 1 (G8)          */
    SV_INIT_ZERO_STATE = 2  /* |0...0> (Fig. 1(a))                                      */
} sv_init_kind;

typedef enum {
    SV_DIFFUSE_WHT = 0,   /* D = H^n F0 H^n, F0 = 2|0><0| - I (G2): 2 x n butterfly stages   */
    SV_DIFFUSE_MEAN = 1   /* D a = 2 mean(a) - a: global sum (Eq. 3) + update   */
} sv_diffusion;

typedef struct sv_ctx sv_ctx; /* opaque; one per process (= per GPU rank) */

/* Multi-GPU description (section 3.1).  world = P = 2^g >= 1.
 *  - nccl_id != NULL: real rank `rank` of a P-rank job; nccl_id points to the
 *    128-byte ncclUniqueId produced by sv_nccl_unique_id() on rank 0 and
 *    broadcast by the caller (e.g. torch.distributed).  One GPU per rank.
 *    world = 1 with an id makes a one-rank communicator (the collectives of
 *    the schedule then run through NCCL on one GPU).
 *  - nccl_id == NULL and world > 1: single-process emulation of all P ranks on
 *    one device (the state is held as P shards in rank order; qubit swaps are
 *    device-local copies).  For tests of the sharded schedule on one GPU.
 *  - device: CUDA device ordinal; stream: a cudaStream_t or NULL. */
typedef struct {
    int rank;
    int world;
    const void *nccl_id;
    int device;
    void *stream;
} sv_dist;

/* Create a context holding an n-qubit state and initialise it.
 *   n: 1..40; seed: drives SV_INIT_GAUSSIAN (G8) -- other kinds ignore it;
 *   dist: NULL = one GPU (device 0 / current device), own stream.
 * Device memory: the local shard (2^{n-g} amplitudes) plus, when P > 1, one
 * receive buffer of the same size for the out-of-place qubit swap.
 * Errors: SV_EINVAL (n out of range, world not a power of two, shard too small
 * for the WHT tiles: n - 2g < 13 for c64 / 12 for c128 when P > 1),
 * SV_ENOMEM, SV_ECUDA, SV_ENCCL.  *out is NULL on error. */
sv_status sv_init(sv_ctx **out, int n, uint64_t seed, sv_dtype dtype, sv_init_kind init,
                  const sv_dist *dist);

/* Re-initialise the existing state (no reallocation); the marked set is kept. */
sv_status sv_reset(sv_ctx *ctx, uint64_t seed, sv_init_kind init);

/* Set the marked set used by sv_iterate without applying O.
 *   marked: m GLOBAL indices, strictly increasing, each < 2^n (host memory,
 *   copied).  0 <= m <= 2^n; m = 0 means O = I (G17).
 * Errors: SV_EINVAL (index out of range, not strictly increasing -- duplicates
 * are errors, not double flips). */
sv_status sv_set_marked(sv_ctx *ctx, const uint64_t *marked, uint64_t m);

/* Set the marked set (as sv_set_marked) and apply the phase oracle
 * O = I - 2 sum_m |m><m| once (G3: phase pi on the marked states). */
sv_status sv_apply_oracle(sv_ctx *ctx, const uint64_t *marked, uint64_t m);

/* Apply the diffusion D once (no oracle). */
sv_status sv_diffuse(sv_ctx *ctx, sv_diffusion diffusion);

/* Apply k Grover iterations a <- (D O)^k a with the context's marked set.
 * WHT: each iteration runs both n-stage transforms (the paper's "sequence of
 * V/2 independent 2x2 transformations" per qubit, with w = x = y
 * = 1, z = -1; Fig. 3) around F0 and the exact 2^{-n} scale (G5), fused into
 * multi-stage HBM passes; P > 1 adds one qubit-swap exchange per transform
 * (the paper's reorganisation, Fig. 8).  MEAN: one fused
 * flip + invert-about-mean pass per iteration plus (P > 1) one 2-double
 * allreduce (Eq. 3's accumulate-and-redistribute).  On one GPU
 * a state of <= 16 (complex128) / 32 (complex64) amplitudes per thread of one
 * 512-thread block per SM (c2: n = 20) runs all k MEAN iterations in ONE
 * cooperative launch with the state in registers and one grid-wide sum per
 * iteration (exact fixed-point integer atomics, deterministic; SV_RESREG_FX=0:
 * fp64 partials; SV_MEAN_RESIDENT=0 / smem: per-iteration launches / the
 * shared-memory resident kernel); the results agree within the dtype tolerance.
 * Errors: SV_EINVAL (k < 0), SV_ESTATE (no marked set was ever given). */
sv_status sv_iterate(sv_ctx *ctx, int k, sv_diffusion diffusion);

/* k Grover iterations with operational angle errors:
 * "imperfections in the laser apparatus result in deviations in the angle of
 * rotation" (section 2.0; section 1.4).  Reading G19:
 * every Hadamard of the WHT diffusion becomes U(phi) = [[cos phi, sin phi],
 * [sin phi, -cos phi]] (Fig. 3's [w x; y z]), phi = pi/4 + delta, one delta
 * per (iteration t, transform w, qubit q) shared by all V/2 pairs of that
 * qubit; F0 = 2|0><0| - I (no 2^-n: the transforms are unitary); O exact.
 * Reading G20: delta = sigma * z, z ~ N(0,1) from a counter hash of
 * (seed, t, w, q); iterations are numbered t0, t0+1, ... so a run can be
 * split over calls.  sigma = 0 is the ideal iteration (up to rounding).
 * Errors: SV_EINVAL (k < 0, sigma not in [0, 10)), SV_ESTATE (no marked set). */
sv_status sv_iterate_noisy(sv_ctx *ctx, int k, double sigma, uint64_t seed, uint64_t t0);

/* k noisy Grover iterations with the decoherence step:
 * "the decoherence step adds two additional operations for every laser
 * operation, and requires two messages to accumulate and redistribute the
 * sum" (Eq. 3 text).  Reading G22: after every laser
 * operation (the 2x2 on qubit q of a transform) the amplitudes with bit d = 1
 * of a drawn site d are contracted by sqrt(1 - rate), then the register is
 * renormalised by the global sum |a|^2.  Angle errors as sv_iterate_noisy
 * (sigma = 0: none).  The renormalisations are global scalars, so they are
 * applied once per iteration from one deterministic fp64 reduction
 * (allreduced over ranks); survival[t] (host, k entries, may be NULL) = the
 * product of iteration t's pre-renormalisation sums.  The state is left
 * normalised.  Errors: SV_EINVAL (k < 0, sigma, rate not in [0, 1)),
 * SV_ESTATE (no marked set). */
sv_status sv_iterate_decoherent(sv_ctx *ctx, int k, double sigma, double rate, uint64_t seed, uint64_t t0,
                                double *survival);

/* p_i = re^2 + im^2 in fp64 ("the probability of each state is defined as the
 * square of this complex amplitude") for the context's resident
 * indices (local shard; whole state in emulation), in local index order.
 *   out: len doubles (len must equal the resident length); out_on_device: 1 =
 *   device pointer, 0 = host pointer (host path guarded at 2^26 entries,
 *   SV_ETOOBIG above). */
sv_status sv_probabilities(sv_ctx *ctx, double *out, uint64_t len, int out_on_device);

/* Seeded measurement of the whole register, `shots` times, without collapsing
 * the state: "this measurement operation forces the state
 * to one of the two values ... in terms of their probability of occurrence"
 * (P:2273-2276), probability |a_i|^2.  Reading G21: shot s uses
 * u_s = ((SplitMix64(key ^ s) >> 11) + 0.5) 2^-53, key = SplitMix64(seed ^
 * "SAMP"), and returns the smallest GLOBAL index whose inclusive cumulative
 * probability exceeds u_s times the total (fp64, fixed summation order:
 * deterministic).  out: shots indices (host, guarded at 2^26, or device);
 * identical on every rank.  Errors: SV_EINVAL (out NULL), SV_ETOOBIG. */
sv_status sv_sample(sv_ctx *ctx, uint64_t shots, uint64_t seed, uint64_t *out, int out_on_device);

/* out (host) = sum over the marked set of |a_m|^2, fp64, allreduced over
 * ranks (identical on every rank).  SV_ESTATE if no marked set. */
sv_status sv_measure_marked_mass(sv_ctx *ctx, double *out);

/* Squared norm sum_i |a_i|^2 of the whole register (all ranks; fp64,
 * deterministic fixed-order reduction, allreduced): the norm-drift readout of
 * S:134 / S:125 -- 1 up to rounding after any unitary iteration (ideal or
 * with angle errors) and after every renormalised decoherent iteration.
 * Synchronises.  Errors: SV_EINVAL (NULL out). */
sv_status sv_norm2(sv_ctx *ctx, double *out);

/* Copy `count` resident amplitudes starting at resident offset `offset` to
 * host memory, dtype-native (8 or 16 bytes each).  SV_EINVAL if out of range. */
sv_status sv_get_amplitudes(sv_ctx *ctx, void *host_out, uint64_t offset, uint64_t count);

/* Overwrite `count` resident amplitudes from host memory (dtype-native).
 * Used to start from an arbitrary (test-generated) state. */
sv_status sv_set_amplitudes(sv_ctx *ctx, const void *host_in, uint64_t offset, uint64_t count);

/* The seeded marked set of G6/G7: sort{pi_seed(j) : 0 <= j < m}, pi_seed the
 * keyed bijection on n-bit integers.  Host-only; out has m entries.
 * SV_EINVAL if m > 2^n or n not in 1..40. */
sv_status sv_marked_from_seed(int n, uint64_t m, uint64_t seed, uint64_t *out);

/* Context description; any pointer may be NULL.  local_len = resident
 * amplitudes (2^{n-g}; 2^n in emulation). */
sv_status sv_info(const sv_ctx *ctx, int *n, int *world, int *rank, uint64_t *local_len,
                  sv_dtype *dtype);

/* The context's NCCL communicator as NCCL reports it (ncclCommCount,
 * ncclCommUserRank): *nranks = 0 and *comm_rank = -1 when the context has
 * none (one GPU, or single-process emulation).  Lets a launcher verify that
 * every process joined one communicator of the expected size. */
sv_status sv_comm_info(const sv_ctx *ctx, int *nranks, int *comm_rank);

/* Adopt a caller-owned device buffer as the state (SURVEY 8(b) phase-2
 * option): dev_ptr = bytes of interleaved complex amplitudes in the natural
 * layout (e.g. a torch.complex64 / complex128 CUDA tensor's data_ptr()), on
 * the context's device, 16-byte aligned, bytes = resident length x element
 * size.  The library frees its own state buffer, computes in place in
 * dev_ptr from now on and never frees it -- the caller keeps ownership and
 * must keep it alive until sv_free.  The buffer's current contents are the
 * state (no initialisation).  Single-process contexts only (one GPU or
 * emulation): SV_ESTATE with a communicator (the fused exchange's peer
 * mappings are made at sv_init).  Errors: SV_EINVAL (NULL, size, alignment,
 * not device memory of the context's GPU), SV_ESTATE. */
sv_status sv_attach(sv_ctx *ctx, void *dev_ptr, uint64_t bytes);

/* Debug / oracle snapshot in SPEC's text format: header line
 * "s=2 M=<n>", then one line per nonzero resident amplitude,
 * "<global index base-10> <re> <im>" with 17 significant digits, ascending
 * index.  *written (may be NULL) = amplitude lines.  Synchronises.  Errors:
 * SV_ETOOBIG above 2^26 resident amplitudes (the host-gather guard),
 * SV_EINVAL (NULL path, file not writable). */
sv_status sv_snapshot(sv_ctx *ctx, const char *path, uint64_t *written);

/* Qubit-swap exchange mode (P > 1).  fused = 1: the pass before each swap
 * stores every amplitude straight into its new owner's buffer -- peer memory
 * over NVLink mapped with CUDA IPC, or the emulated shard -- and the swap is
 * a cross-rank barrier (one-integer ncclAllReduce); the reorganisation of
 * Fig. 8 then costs no extra HBM pass.  fused = 0: ncclAlltoAll
 * of contiguous chunks into a receive buffer (emulation: device copies).
 * Default: fused when available (SV_XCHG=nccl in the environment forces 0).
 * SV_ESTATE if fused is requested but unavailable (1 rank, > 8 ranks, or the
 * peers' buffers could not be mapped). */
sv_status sv_set_exchange(sv_ctx *ctx, int fused);
sv_status sv_get_exchange(const sv_ctx *ctx, int *fused);

/* ---- NEXT-4: circuits of general (controlled) 2x2 gates ------------------- */

/* One gate (80 bytes).  Section 2.1: "we describe each
 * operation with a VxV transformation matrix.  Because each gate only
 * operates on a small number of bits, these matrices are simply 2x2 or 4x4
 * matrices replicated many times."  The gate is Fig. 3's general 2x2
 * [w x; y z] on qubit `target`, applied as V/2 independent pair
 * transformations: for every index i with bit `target` = 0 and
 * (i & controls) == controls, (a_i, a_j) <- (w a_i + x a_j, y a_i + z a_j),
 * j = i | 2^target.  A controlled 2x2 is the 4x4 of a two-bit gate (G23).
 *   m = {w.re, w.im, x.re, x.im, y.re, y.im, z.re, z.im} (fp64; rounded to
 *   fp32 for SV_C64 states); reserved must be 0. */
typedef struct {
    int32_t target;
    int32_t reserved;
    uint64_t controls;
    double m[8];
} sv_gate;

/* Apply gates[0..count) to the state, in order (gates may be regrouped only
 * where they commute: different targets and neither controlled by the other's
 * target; a diagonal gate commutes with any gate whose target is outside its
 * support; diagonal gates commute).  Results equal the gate-by-gate product up
 * to rounding: the host multiplies same-target same-control gates separated
 * only by commuting gates into one fp64 2x2, and merges runs of >= 4
 * single-control phase gates on one target into one phase-polynomial op.
 * The host planner packs consecutive runs of gates on up to T
 * local qubits into one tile pass each (one HBM read + write per pass, all of
 * the pass's gates on-chip); a gate on a parallel (rank) qubit first triggers
 * the qubit swap of section 3.1 / Fig. 8 ("when the computation needs to
 * operate on one of the bits in N, a new set is picked and the simulator
 * redistributes the data"); the natural layout is restored
 * before the call returns.  n <= T (13 for c64, 12 for c128) runs all gates
 * in one CTA's shared memory.  gates: host array, copied.
 * Errors: SV_EINVAL (target not in [0, n), control >= n, control == target,
 * reserved != 0, gates NULL with count > 0). */
sv_status sv_apply_gates(sv_ctx *ctx, const sv_gate *gates, uint64_t count);

/* One step of a gate-circuit schedule: kind 0 = tile pass (tile_mask / proc_mask
 * as in sv_plan_step, in PHYSICAL slots of the shard; its gates are
 * order[first .. first + count)), kind 1 = qubit-swap exchange (physical
 * slots [nl - g, nl) <-> the g rank bits), kind 2 = whole state in one CTA.
 * ops: operations the pass runs after the host merging (a gate is multiplied
 * into an earlier one with the same target and controls when only commuting
 * gates lie between them; runs of >= 4 single-control phase gates on one
 * target become one phase-polynomial op); lin_ops: how many of them are such
 * merged phase runs. */
typedef struct {
    int kind;
    int tile_bits;
    uint64_t tile_mask;
    uint64_t proc_mask;
    uint64_t first;
    uint64_t count;
    uint64_t ops;
    uint64_t lin_ops;
} sv_gate_plan_step;

/* The schedule sv_apply_gates enqueues on every rank for an n-qubit state over
 * world = 2^g ranks (host only, no device).  Writes at most cap steps
 * (*nsteps = total) and, if order != NULL, the execution order of the gate
 * indices (count entries).  The layout is natural again after the last step.
 * Errors: as sv_apply_gates, plus invalid (n, world, dtype). */
sv_status sv_plan_gates(int n, int world, sv_dtype dtype, const sv_gate *gates, uint64_t count,
                        sv_gate_plan_step *out, int cap, int *nsteps, uint64_t *order);

/* Block until all work enqueued on the context's stream is done. */
sv_status sv_synchronize(sv_ctx *ctx);

/* Write a fresh ncclUniqueId (len >= 128) for rank 0 to broadcast. */
sv_status sv_nccl_unique_id(void *out, size_t len);

/* ---- schedule introspection (host only; no device needed) ---------------- */

/* One step of a device schedule.  kind: 0 = tile pass, 1 = qubit-swap
 * exchange, 2 = whole-state kernel, 3 = oracle scatter.  For a tile pass the
 * tile is the 2^T amplitudes whose local indices differ only in the slots of
 * tile_mask; the butterfly stages run on the slots of proc_mask before (pre)
 * and/or after (post) the elementwise op `mid` (0 none, 1 oracle O, 2 F0 with
 * the 2^{-n} scale).  in_recv: the pass reads the swap receive buffer. */
typedef struct {
    int kind;
    int pre;
    int mid;
    int post;
    int in_recv;
    int tile_bits;
    uint64_t tile_mask;
    uint64_t proc_mask;
} sv_plan_step;

/* The schedule sv_iterate(k, SV_DIFFUSE_WHT) (with_oracle = 1) or
 * sv_diffuse(SV_DIFFUSE_WHT) (with_oracle = 0, k ignored) enqueues on every
 * rank for an n-qubit state over world = 2^g ranks.  Writes at most cap steps,
 * *nsteps = total.  SV_EINVAL for invalid (n, world, dtype). */
sv_status sv_plan_wht(int n, int world, sv_dtype dtype, int k, int with_oracle,
                      sv_plan_step *out, int cap, int *nsteps);

/* Kernel variant (template instantiation) of one WHT tile pass.  family: 0 =
 * the one-CTA whole-state kernel, 1 = the three-register-layout tile kernel,
 * 2 = the two-layout kernel of strided complex64 tiles; u = unprocessed
 * (carry) tile bits, the butterflies run on tile bits [u, T); pre / mid / post
 * as in sv_plan_step; noisy: 0 ideal butterflies, 1 general real 2x2 (Fig. 3's
 * [w x; y z], angle errors with decoherence contractions), 2 angle-error tan
 * form; xchg: the pass's store is the fused qubit-swap exchange. */
typedef struct {
    int family;
    int u;
    int pre;
    int mid;
    int post;
    int noisy;
    int xchg;
} sv_tile_variant;

/* The kernel variants one call launches, in launch order, without a device:
 * flavour 0 = sv_iterate(k, SV_DIFFUSE_WHT), 1 = sv_iterate_noisy(k, sigma,
 * seed, 0), 2 = sv_iterate_decoherent(k, sigma, rate, seed, 0), 3 =
 * sv_diffuse(SV_DIFFUSE_WHT); world > 1 describes the sharded schedule (each
 * rank launches the same variants), fused selects the fused exchange.  The
 * SV_PLAN_CHUNKS override applies as in sv_init.  Writes at most cap entries,
 * *count = total.  SV_EINVAL as sv_plan_wht, or flavour outside 0..3.  Used by
 * tests/test_variants.py to map every variant a bench launches to a parity
 * test that runs it. */
sv_status sv_debug_wht_variants(int n, int world, sv_dtype dtype, int flavour, int k, double sigma, double rate,
                                uint64_t seed, int fused, sv_tile_variant *out, int cap, int *count);

/* ---- per-kernel device timing (CUDA events on the context's stream) ------ */

typedef enum {
    SV_K_WHT_TILE = 0,   /* multi-stage WHT tile pass                */
    SV_K_WHT_WHOLE = 1,  /* whole state in one CTA (small n)         */
    SV_K_MEAN = 2,       /* fused flip + invert-about-mean           */
    SV_K_REDUCE = 3,     /* read-only flipped-sum reduction          */
    SV_K_INIT = 4,       /* state initialisation                     */
    SV_K_ORACLE = 5,     /* standalone oracle scatter                */
    SV_K_READOUT = 6,    /* probabilities / marked mass              */
    SV_K_EXCHANGE = 7,   /* qubit-swap all-to-all (NCCL or emulated) */
    SV_K_ALLREDUCE = 8,  /* scalar NCCL allreduce                    */
    SV_K_GATE_TILE = 9,  /* gate-circuit tile pass (NEXT-4)          */
    SV_K_SCALE = 10,     /* state x scalar (end of a decoherent call) */
    SV_K_COUNT = 11
} sv_kernel_kind;

/* enable != 0: bracket every launch with CUDA events and count launches per
 * kind (resets the counters); 0: stop recording. */
sv_status sv_profile(sv_ctx *ctx, int enable);

/* Synchronises, then returns launches and summed device milliseconds of one
 * kind since sv_profile(ctx, 1). */
sv_status sv_profile_read(sv_ctx *ctx, int kind, uint64_t *launches, double *total_ms);

/* Synchronises, then writes the kind and device milliseconds of each profiled
 * launch since sv_profile(ctx, 1), in launch order (at most cap entries;
 * *count = total).  Pairs with sv_plan_wht to attribute time to passes. */
sv_status sv_profile_timeline(sv_ctx *ctx, int *kinds, double *ms, uint64_t cap, uint64_t *count);

/* ---- layout introspection (host only; used by tests/test_layouts.py) ----- */

/* Tile element index and swizzled shared-memory slot held by thread `tid`,
 * register `reg` in register layout `phase` (0 = A, 1 = B, 2 = C) of the WHT
 * tile kernel for `dtype` (SV_C64 / SV_C128: the three-layout family; 2: the
 * two-layout family of strided complex64 tiles, phases 0-1).  Returns 0, or
 * -1 for out-of-range arguments. */
int sv_debug_tile_layout(int dtype, int phase, int tid, int reg, int *tile_elem, int *smem_index);
/* 1 if layout `phase` runs the butterfly stage of tile bit `bit`, else 0. */
int sv_debug_tile_owner(int dtype, int phase, int bit);

/* Shared-memory relayouts (register-layout changes between consecutive ops)
 * the gate tile kernel performs in each step of sv_plan_gates' schedule, as
 * rank 0 runs it (host only; 0 for swap / whole-state steps).  Writes at most
 * cap entries, *nsteps = total.  Used by the analytical model (costmodel.py).
 * Errors: as sv_plan_gates. */
sv_status sv_debug_gate_relayouts(int n, int world, sv_dtype dtype, const sv_gate *gates, uint64_t count,
                                  uint64_t *out, int cap, int *nsteps);

/* Gate engine, pass-specialised kernels (gate_jit.cu): with compile == 1,
 * generate and NVRTC-compile (no device needed) the kernel of every tile pass
 * sv_plan_gates gives the circuit on one complex64 GPU, in both program
 * flavours; *passes = passes compiled.  (compile == 2 is accepted and, the
 * automatic mode compiling synchronously, has nothing to wait for.)  Always: *compiles /
 * *compile_seconds = specialised kernels this process has loaded for
 * launches so far / NVRTC seconds spent (any pointer may be NULL).  Errors: SV_EINVAL (gates, dtype), SV_ECUDA (NVRTC
 * failure, with its log in sv_last_error()). */
sv_status sv_debug_gate_jit(int n, sv_dtype dtype, const sv_gate *gates, uint64_t count, int compile,
                            uint64_t *passes, uint64_t *compiles, double *compile_seconds);

/* Release every resource of the context (NULL-safe). */
void sv_free(sv_ctx *ctx);

/* Thread-local message of the last failing call ("" if none). */
const char *sv_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SV_H */
