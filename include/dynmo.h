/*
 * dynmo.h -- C-ABI of the B200-native DynMo per-step rebalancing hot path.
 *
 * DynMo (arXiv 2505.14864) rebalances a pipeline-parallel model whose
 * per-layer work changes during training.  Each step:
 *   1 dynmo_profile_layers   per-layer counters -> int64 cost c_i, all-gather
 *   2 dynmo_partition_stages contiguous layers->stages min-max partition
 *   3 dynmo_diffuse_balance  the paper's decentralised diffusion variant
 *   4 dynmo_repack_workers   fewest workers within a throughput bound
 *   5 dynmo_migrate_layers   move the layers whose GPU changed (NCCL P2P),
 *     or _p2p / _dev: receiver pull over NVLink peer memory (host- or
 *     device-driven; the latter keeps the whole step one graph launch)
 * Beyond the per-step path:
 *     DYNMO_SRC_TIME_NS + dynmo_timestamp   "by Time" profiling (NEXT-1)
 *     dynmo_global_prune                    Alg. 1 global pruning (NEXT-2)
 *     dynmo_ctx_split, dynmo_map_stages     release GPUs / placement (NEXT-3)
 * Citations: P:Lnnn = PAPER.md line (SPEC:Lnnn = SPEC.md line); readings of
 * ambiguous passages (Q1..Q23) are listed in DESIGN.md.
 *
 * Conventions
 *  - Pointers prefixed d_ are DEVICE pointers, h_ are HOST pointers.  The
 *    library never takes ownership of caller memory and never frees it.
 *  - Calls 1-4 are asynchronous on the given cudaStream_t and never
 *    synchronise the host; data-dependent errors are written to device
 *    status words (int32).  Call 5 (NCCL, or dynmo_migrate_layers_p2p) takes
 *    host boundaries (the caller copies the <= 40 B boundary vector D2H
 *    first); dynmo_migrate_layers_dev reads them from device memory, so the
 *    whole step can be one CUDA graph launch.  All calls are stream-ordered.
 *  - Return value: host-checkable status (argument validation, CUDA/NCCL
 *    launch errors).  0 OK, < 0 error, > 0 warning.
 *  - int32 layer/stage indices, int64 costs and bytes.  All results are
 *    deterministic; integer results are bit-exact with the CPU oracle.
 *  - Thread safety: a ctx may be used from one host thread at a time.
 */
#ifndef DYNMO_H
#define DYNMO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t dynmo_status;
#define DYNMO_OK 0
#define DYNMO_E_INVALID (-1)     /* bad argument / malformed instance       */
#define DYNMO_E_INFEASIBLE (-2)  /* no split satisfies the memory cap       */
#define DYNMO_E_OVERFLOW (-3)    /* an int64 cost, sum or phi overflowed     */
#define DYNMO_E_CUDA (-4)        /* CUDA runtime error (see strerror/last)   */
#define DYNMO_E_NCCL (-5)        /* NCCL error (see dynmo_last_error)        */
#define DYNMO_E_NOMEM (-6)       /* device allocation failed (plan create)   */
#define DYNMO_W_NOT_CONVERGED 1  /* diffusion stopped at max_rounds          */
#define DYNMO_W_BOUND_UNMET 2    /* repack could not meet bound / target     */

typedef void *dynmo_stream; /* a cudaStream_t; NULL = legacy default stream */
typedef struct dynmo_ctx_s *dynmo_ctx;
typedef struct dynmo_plan_s *dynmo_plan;

const char *dynmo_strerror(dynmo_status s);
/* Last host-side error message of this thread (CUDA/NCCL string), or "". */
const char *dynmo_last_error(void);
/* Library version string. */
const char *dynmo_version(void);

/* ------------------------------------------------------------------ ctx --
 * One process per GPU ("one MPI rank per GPU"; here torch.distributed
 * ranks).  nranks == 1: no NCCL communicator is created up front (a
 * one-rank communicator is created by the first plan that asks for the NCCL
 * exchange), and the peer window is local.  nranks > 1: every
 * rank passes the same 128-byte id obtained on rank 0 from
 * dynmo_get_unique_id() and broadcast by the caller (e.g. through the torch
 * process group); the ctx owns the resulting ncclComm_t.  device is the CUDA
 * ordinal this rank drives.  ctx_create is collective over the nranks ranks. */
dynmo_status dynmo_get_unique_id(uint8_t h_id_out[128]);
dynmo_status dynmo_ctx_create(int32_t device, int32_t nranks, int32_t rank,
                              const uint8_t *h_nccl_id /* 128 B, or NULL if nranks==1 */,
                              dynmo_ctx *out);
/* Frees the ctx and aborts its communicator without waiting for outstanding
 * collective work: synchronise the streams that use it first (CUDA graphs
 * that captured collectives of this ctx must not be replayed afterwards). */
void dynmo_ctx_destroy(dynmo_ctx ctx);
/* Releasing GPUs after re-packing ("splitting the communicator
 * via ncclCommSplit()"): collective over ctx's ranks.  Ranks passing the
 * same color >= 0 get a new ctx over their group (ranks ordered by key, then
 * by old rank), with its own communicator and peer windows; color < 0 (a
 * released GPU) returns *out = NULL.  The old ctx stays valid (destroy it
 * separately).  E_NCCL on a communicator error. */
dynmo_status dynmo_ctx_split(dynmo_ctx ctx, int32_t color, int32_t key, dynmo_ctx *out);
int32_t dynmo_ctx_nranks(dynmo_ctx ctx);
int32_t dynmo_ctx_rank(dynmo_ctx ctx);

/* Diagnostics: per-phase device timing.  When enabled, the library records a
 * pair of CUDA events on the launching stream around every launch of the
 * phase (the breakdown of the paper's overhead figure: profiling /
 * balancing algorithm / migration).  If the stream is being captured into a
 * CUDA graph, the pair becomes two external event-record nodes that every
 * replay re-records: call timing_poll after each replay has completed.
 * timing_poll adds every recorded pair to the per-phase accumulators;
 * timing_read returns (and resets) the accumulated milliseconds and launch
 * count of a phase.  Off by default (no events recorded). */
enum {
    DYNMO_PHASE_PROFILE = 0,   /* k_profile (the streaming kernel)          */
    DYNMO_PHASE_EPILOGUE = 1,  /* k_epilogue (counters -> cost)            */
    DYNMO_PHASE_EXCHANGE = 2,  /* ncclAllGather + k_unpack                 */
    DYNMO_PHASE_PARTITION = 3, /* k_partition                              */
    DYNMO_PHASE_DIFFUSE = 4,   /* k_diffuse                                */
    DYNMO_PHASE_REPACK = 5,    /* k_repack                                 */
    DYNMO_PHASE_MIGRATE = 6,   /* NCCL send/recv group of migrate_layers   */
    DYNMO_NUM_PHASES = 7
};
/* enable: 0 off, 1 every phase, otherwise a bitmask (bit p = phase p, e.g.
 * 1 << DYNMO_PHASE_PROFILE only; -1 = all). */
dynmo_status dynmo_ctx_set_timing(dynmo_ctx ctx, int32_t enable);
dynmo_status dynmo_ctx_timing_poll(dynmo_ctx ctx);
/* Device-side barrier over the ctx ranks on `stream` (a one-element NCCL
 * all-reduce; no-op for one rank): work enqueued after it starts only when
 * every rank's stream has reached it.  Capturable (the rebalancing step runs
 * at the training-iteration barrier); the graph holding it must be
 * destroyed before the ctx. */
dynmo_status dynmo_ctx_barrier(dynmo_ctx ctx, dynmo_stream stream);
/* Stop polling the event pairs baked into the graphs captured so far (their
 * events stay alive until ctx destruction, so those graphs remain valid):
 * call before capturing a graph whose timings are read separately. */
dynmo_status dynmo_ctx_timing_detach(dynmo_ctx ctx);
dynmo_status dynmo_ctx_timing_read(dynmo_ctx ctx, int32_t phase, double *h_total_ms,
                                   int64_t *h_count);
/* With the profile phase timed, k_profile also records its own span on the
 * device clock (%globaltimer: first CTA start to last CTA end; the event
 * pair around it adds the launch and completion latency, ~5 us on B200,
 * tools/lat/ramp.cu); the epilogue folds each launch's span into an
 * accumulator.  Returns (and resets) the accumulated milliseconds and
 * launch count; synchronous. */
dynmo_status dynmo_ctx_profile_span(dynmo_ctx ctx, double *h_total_ms, int64_t *h_count);

/* Device step timeline, diagnostic builds only (compiled with
 * -DDYNMO_STEP_STAMPS, tools/build_stamps.sh): copies to h_out (host,
 * 4 * 7 uint64) each step kernel's {first-warp start, last-warp end} in
 * %globaltimer ns -- k_profile, k_epilogue, k_publish, then k_partition,
 * k_diffuse (discrete block), k_diffuse (fluid block), k_repack, in two
 * tables of 7 pairs (unused rows {~0, 0}) -- and, if reset != 0, re-arms
 * them.  Synchronous (device-wide copies); not for use inside a capture.
 * Returns 7, or 0 in a normal build (no stamps recorded, h_out untouched). */
int dynmo_diag_step_stamps(unsigned long long *h_out, int reset);
/* Hang analysis: a snapshot of this rank's peer window, copied on a private
 * non-blocking stream (so it completes while the ctx's other streams wait):
 * h_out[0] sticky error, [1] device-migration epoch, [2] exchange epoch,
 * [3..19) backward done words, [19..21) chunks finished (epoch parities),
 * [21..21+n) layer release words, [21+n..21+2n) chunk claim words
 * (n = min(n_layers, 1024)).  INVALID if n_words < 21 + 2n. */
dynmo_status dynmo_ctx_window_snapshot(dynmo_ctx ctx, int32_t n_layers, uint64_t *h_out, int64_t n_words);

/* ----------------------------------------------------------- profiling --
 * Sources of per-layer workload (P:L234-239 pruning p_i, P:L266-283 freezing
 * f_i, P:L340-353 early exit t_i, P:L376-389 MoD r_i t_i, P:L209-214 MoE
 * tokens per expert; P:L632 + P:L720 + P:L743 execution time, the "by Time"
 * balancers).  A segment is a caller-owned device array that
 * contributes to ONE layer (or, for EXIT_U8, to every local layer).  All
 * contributions to a layer are summed, so one layer may have several
 * segments (e.g. its four weight tensors). */
enum {
    DYNMO_SRC_MASK_BITS = 0,   /* uint32 words, 1 bit/param, little-endian bit
                                  order (bit b = word b/32, bit b%32); counts
                                  set bits among the first n_elem  -> nnz_i */
    DYNMO_SRC_MASK_U8 = 1,     /* bool/uint8 mask, n_elem bytes; != 0 -> nnz_i */
    DYNMO_SRC_NZ_BF16 = 2,     /* bf16 weights; (bits & 0x7FFF) != 0 -> nnz_i
                                  (+0 and -0 are pruned, NaN counts)         */
    DYNMO_SRC_NZ_F32 = 3,      /* f32 weights; (bits & 0x7FFFFFFF) != 0      */
    DYNMO_SRC_TOKMASK_BITS = 4,/* per-layer token bitmask (MoD routing or an
                                  early-exit alive mask), n_elem bits -> tok_i */
    DYNMO_SRC_EXIT_U8 = 5,     /* per-token exit depth e[t] (token processed by
                                  layers 0..e[t]-1), n_elem tokens; adds
                                  #{t : e[t] > i} to tok_i of EVERY local layer
                                  i (layer field ignored)                     */
    DYNMO_SRC_EXPERT_I64 = 6,  /* int64 top-k expert ids [T*k] of a MoE layer;
                                  histogram over [0, n_experts)               */
    DYNMO_SRC_EXPERT_I32 = 7,  /* int32 variant                              */
    DYNMO_SRC_TIME_NS = 8      /* int64 (begin, end) timestamp pairs in ns,
                                  n_elem int64 values (even; 8-byte aligned);
                                  adds sum(end - begin) to time_i.  end < begin
                                  is INVALID.  Stamps from dynmo_timestamp (or
                                  any monotonic ns clock); a layer's boundary
                                  stamps s[i], s[i+1] can be the overlapping
                                  segment {&s[i], 2}.                         */
};

typedef struct dynmo_segment {
    const void *d_ptr;   /* device pointer; alignment of its element type   */
    int64_t n_elem;      /* bits (MASK_BITS, TOKMASK_BITS), else elements   */
    int32_t layer;       /* global layer index in [layer_begin, +n_local)   */
    int32_t src_kind;    /* DYNMO_SRC_*                                     */
    int32_t n_experts;   /* EXPERT_*: E in [1, 1024]; all segments of one
                            layer must agree.  Ignored otherwise.            */
    int32_t top_k;       /* EXPERT_*: informational (n_elem = T*k)          */
} dynmo_segment;

/* Per-local-layer cost coefficients (readings Q1-Q6, Q21):
 *   c_i = frozen_i ? F : tok_i * (A + B * nnz_i) + C * moe_i + D * time_i
 * ("by Param" balancing: B = 1; "by Time": D = 1, A = B = C = 0)
 *   moe_i = EP * max_{r<EP} sum_{e in group r} cnt_{i,e}
 * groups = EP contiguous blocks of E/EP experts (EP <= 0 means EP = E;
 * E % EP != 0 is INVALID).  Absent sources default to tok_i = 1, nnz_i = 0,
 * moe_i = 0, time_i = 0.  Checked int64 arithmetic (128-bit intermediates):
 * a result above INT64_MAX is OVERFLOW; a negative coefficient is INVALID. */
typedef struct dynmo_cost_coef {
    int64_t A, B, C, F, D;
    int32_t ep_ranks;
    int32_t pad;
} dynmo_cost_coef;

/* Build the launch plan for this rank's segments (off the hot path; plain
 * host work + two small device allocations owned by the plan).  The plan
 * stores the segment pointers: they must stay valid while the plan is used;
 * rebuild after migration or re-allocation.
 *   layer_begin, n_local: the contiguous global layers this rank profiles.
 *   n_total: length of the global cost vector.
 *   exchange: every rank ends with the global vector (slices must tile
 *     [0, n_total) exactly, else the device status is INVALID; on a
 *     single-rank ctx the exchange runs against the rank itself, so the same
 *     code path -- LL slot encode/decode, slot validation, unpack -- runs on
 *     one GPU):
 *       1 -> over NVLink peer memory: the epilogue stores this rank's slot
 *            straight into every rank's receive area (double-buffered by a
 *            device-side epoch, graph-safe) and releases a flag; the unpack
 *            kernel waits (bounded, 10 s) for every rank's flag.  Plan
 *            creation is then COLLECTIVE (CUDA IPC of the receive areas; a
 *            failure on any rank -- validation, allocation, mapping -- fails
 *            the call on every rank, none is left waiting), and every rank
 *            must make the same sequence of profile calls.
 *       2 -> ncclAllGather of the fixed-size slots on the ctx communicator.
 *     0 -> local only: n_total == n_local and outputs are indexed by local
 *     layer.
 * Errors (returned): INVALID for a null/negative argument, a layer outside
 * the local range, an unknown src_kind, n_experts outside [1, 1024] or
 * inconsistent within a layer, a misaligned pointer; NOMEM; CUDA. */
dynmo_status dynmo_profile_plan_create(dynmo_ctx ctx, const dynmo_segment *h_segs, int32_t n_segs,
                                       int32_t layer_begin, int32_t n_local, int32_t n_total,
                                       int32_t exchange, dynmo_plan *out);
void dynmo_profile_plan_destroy(dynmo_plan plan);
/* Number of work tiles the fused profiling kernel walks (diagnostics). */
int64_t dynmo_plan_num_tiles(dynmo_plan plan);
/* Algorithmic bytes read by one profile launch (sum of segment bytes). */
int64_t dynmo_plan_bytes(dynmo_plan plan);
/* Max experts over segments (0 if no MoE source). */
int32_t dynmo_plan_max_experts(dynmo_plan plan);

/* Call 1 -- profile_layers.  One fused streaming kernel over every segment
 * (128-bit loads, warp-shuffle reductions), the cost epilogue, and (if the
 * plan exchanges) an ncclAllGather of fixed-size per-rank slots over NVLink
 * followed by an unpack kernel.
 *   d_frozen   [n_local] uint8, nullable (no layer frozen)
 *   d_coef     [n_local] dynmo_cost_coef, required
 *   d_mem_local[n_local] int64 caller memory per layer, nullable
 *   d_counters [n_local][5] int64 out, nullable: {nnz_i, tok_i, moe_i, c_i,
 *              time_i} with the defaults applied (tok_i = 1 without a token
 *              source)
 *   d_hist     [n_local][max_experts] int64 out, nullable: cnt_{i,e}
 *   d_cost     [n_total] int64 out: global (exchange) or local cost vector
 *   d_mem      [n_total] int64 out, nullable: gathered d_mem_local (zeros if
 *              d_mem_local is NULL)
 *   d_status   [1] int32 out: OK, INVALID (expert id outside [0,E), a time
 *              pair with end < begin, bad coefficient, slices do not tile),
 *              OVERFLOW; the most negative
 *              code wins.  Layers with an error get c_i = -1.
 * Collective when the plan exchanges: every rank must call it. */
dynmo_status dynmo_profile_layers(dynmo_ctx ctx, dynmo_plan plan, const uint8_t *d_frozen,
                                  const dynmo_cost_coef *d_coef, const int64_t *d_mem_local,
                                  int64_t *d_counters, int64_t *d_hist, int64_t *d_cost,
                                  int64_t *d_mem, int32_t *d_status, dynmo_stream stream);

/* Device timestamp for the "by Time" source (the profiling
 * iteration's layer execution times): enqueues on `stream` a one-thread
 * kernel that stores %globaltimer (ns, monotonic, GPU-wide) into *d_slot when
 * the work enqueued before it on the stream has completed -- call it at layer
 * boundaries of the profiling iteration, no host synchronisation.  Capturable
 * in a CUDA graph.  d_slot: int64 device pointer, caller-owned. */
dynmo_status dynmo_timestamp(dynmo_ctx ctx, int64_t *d_slot, dynmo_stream stream);

/* Publish a step result to the host without a copy-engine transfer: enqueues
 * on `stream` a kernel that stores `bytes` bytes of device memory d_src into
 * h_dst, page-locked host memory mapped into the device address space
 * (cudaHostAlloc / cudaMallocHost / torch pin_memory, unified addressing).
 * The bytes are visible to the host once work recorded after it on the
 * stream (an event) has completed.  The kernel
 * starts programmatically (PDL) and waits for the preceding kernel.  In the
 * bench's step it replaces the D2H copy node of the new boundaries + status
 * (the "result read" of the per-step path, "the new partition is
 * broadcast"): ~6 us of copy-engine latency per step for tens of bytes.
 * Results above 4 KiB go through cudaMemcpyAsync instead (GPU stores to host
 * memory run at a few GB/s: the copy engine is faster there).
 * Capturable.  Errors: INVALID for null pointers, bytes < 0, d_src not device
 * memory, or h_dst (first or last byte) not mapped page-locked host memory --
 * nothing is enqueued then.  bytes = 0 is a no-op. */
dynmo_status dynmo_publish(dynmo_ctx ctx, const void *d_src, void *h_dst, int64_t bytes, dynmo_stream stream);

/* -------------------------------------------------------------- solvers --
 * Batched instance layout shared by calls 2-4 (one CTA per instance):
 *   instance q owns layers [d_layer_off[q], d_layer_off[q+1]) of d_cost /
 *   d_mem; L_q = d_layer_off[q+1] - d_layer_off[q] in [1, max_layers].
 *   Its boundary vector b[0..n_q] (b_0 = 0, b_n = L_q, strictly increasing,
 *   stage s = layers [b_s, b_{s+1})) is stored at d_bnd + d_bnd_off[q];
 *   the caller sizes d_bnd_off[q+1] - d_bnd_off[q] >= n_q + 1.
 *   d_mem nullable (no memory constraint; d_cap ignored); else d_cap[q] is
 *   the inclusive per-stage memory cap (Alg. 2's strict "< MAX_MEM" is
 *   cap = MAX_MEM - 1, reading Q9).
 *   max_layers: host upper bound on every L_q, <= DYNMO_MAX_LAYERS (it picks
 *   the kernel variant; an instance with L_q > max_layers gets INVALID).
 * Per-instance device status d_status[q]; on an error the instance's outputs
 * are b = -1, bottleneck = -1 (imbalance = -1.0). */
#define DYNMO_MAX_LAYERS 1023

/* Call 2 -- partition_stages ("minimize the maximum load among
 * all workers"; P:L496, P:L720 centralised Partition, "binary search and
 * linear probing").  B* = min over contiguous n-splits with every stage
 * mem <= cap of the max stage cost; exact integer multi-section search over
 * B with a warp-parallel greedy feasibility test.  Output boundaries are the
 * lexicographically largest optimal split (reading Q7); d_imbalance (nullable)
 * is Delta L = (L_max - L_min) / ((1/n) sum L) in fp64 (eq:imbalance,
 * P:L193; 0 when sum is 0).  Status INVALID (n < 1, n > L, negative cost or
 * mem), INFEASIBLE (no split meets cap), OVERFLOW (sum of costs > INT64_MAX). */
dynmo_status dynmo_partition_stages(dynmo_ctx ctx, int32_t n_inst, int32_t max_layers,
                                    const int64_t *d_cost, const int64_t *d_mem,
                                    const int32_t *d_layer_off, const int32_t *d_n_stages,
                                    const int64_t *d_cap, const int32_t *d_bnd_off,
                                    int32_t *d_bnd, int64_t *d_bottleneck, double *d_imbalance,
                                    int32_t *d_status, dynmo_stream stream);

/* Call 3 -- diffuse_balance (P:L497 decentralised diffusion; P:L518-549
 * Lemma 2: potential phi = sum_{u<v} |x_u - x_v|, max-neighbor pairing,
 * "largest reductions in imbalance while satisfying memory constraints").
 * Discrete rounds (reading Q10): every adjacent stage pair computes its best
 * re-split j (min of (pair max, |j - b|, j) over mem-feasible j); a pair is
 * improvable iff that lowers the pair max; each stage picks its improvable
 * incident pair with the largest load gap (ties: lower index); mutually
 * picked pairs apply their re-split.  Stops with OK when phi <= gamma[q] or
 * no pair is improvable, with NOT_CONVERGED at max_rounds.  The fluid process
 * of the proof (pairs average real loads) runs alongside from the same
 * start: x in fp64, stop at phi_f <= gamma_f[q] (NOT_CONVERGED at max_rounds).
 *   d_bnd_in / d_bnd_out use the d_bnd_off layout with n_q = d_n_stages[q].
 *   d_gamma nullable (0), d_gamma_fluid nullable (0.0).
 *   Outputs: d_rounds[q], d_phi[q] (final), d_phi0[q] (initial) nullable,
 *   d_fluid_x (nullable) at offset d_bnd_off[q] - q (n_q doubles),
 *   d_fluid_rounds[q], d_fluid_phi[q], d_fluid_status[q] nullable.  The fluid
 *   process runs only if d_fluid_x is given (in its own CTA, concurrently).
 *   d_status[q]: the discrete process (OK, NOT_CONVERGED, INVALID, OVERFLOW);
 *   d_fluid_status[q]: the fluid process (OK, NOT_CONVERGED, INVALID -- also
 *   for gamma_fluid < 0 or NaN --, OVERFLOW).  b_in must be a valid split
 *   (else INVALID); a b_in that violates the cap is accepted and moves never
 *   exceed it. */
dynmo_status dynmo_diffuse_balance(dynmo_ctx ctx, int32_t n_inst, int32_t max_layers,
                                   const int64_t *d_cost, const int64_t *d_mem,
                                   const int32_t *d_layer_off, const int32_t *d_n_stages,
                                   const int64_t *d_cap, const int32_t *d_bnd_off,
                                   const int32_t *d_bnd_in, const int64_t *d_gamma,
                                   const double *d_gamma_fluid, int32_t max_rounds,
                                   int32_t *d_bnd_out, int32_t *d_rounds, int64_t *d_phi,
                                   int64_t *d_phi0, double *d_fluid_x, int32_t *d_fluid_rounds,
                                   double *d_fluid_phi, int32_t *d_fluid_status, int32_t *d_status,
                                   dynmo_stream stream);

/* Call 4 -- repack_workers (P:L556-609 re-packing; "without
 * sacrificing training throughput"; readings Q14-Q16).
 *   mode BOUND: n' = the fewest workers k in [floor, n_cur] such that some
 *     contiguous k-split has every stage cost <= bound[q] and mem <= cap;
 *     boundaries = partition_stages at n' (workers 0..n'-1 stay active, in
 *     pipeline order).  If even n_cur cannot meet the bound: BOUND_UNMET,
 *     n' = n_cur with its optimal split.
 *   mode ALG2: Alg. 2 first-fit merges of adjacent active
 *     workers of the current split d_bnd_in, src ascending, if
 *     mem[src] + mem[dst] <= cap and #active > floor (the target); fixes of
 *     SPEC:L389 (skip and zero a deactivated src).  BOUND_UNMET if the
 *     target is not reached.  d_bound ignored.
 *   d_n_cur[q] plays the role of n_q for the layouts (d_bnd_off capacity
 *   n_cur + 1; d_bnd_in only read in ALG2 mode, nullable otherwise).
 *   Outputs d_n_new[q], d_bnd (n'+1 entries, the rest of the capacity -1),
 *   d_bottleneck[q] = max stage cost of the output split.
 *   INVALID if floor < 1, floor > n_cur, n_cur > L or bound < 0. */
#define DYNMO_REPACK_BOUND 0
#define DYNMO_REPACK_ALG2 1
dynmo_status dynmo_repack_workers(dynmo_ctx ctx, int32_t n_inst, int32_t max_layers,
                                  const int64_t *d_cost, const int64_t *d_mem,
                                  const int32_t *d_layer_off, const int32_t *d_n_cur,
                                  const int64_t *d_cap, const int32_t *d_bnd_off,
                                  const int32_t *d_bnd_in, const int64_t *d_bound,
                                  const int32_t *d_floor, int32_t mode, int32_t *d_n_new,
                                  int32_t *d_bnd, int64_t *d_bottleneck, int32_t *d_status,
                                  dynmo_stream stream);

/* ------------------------------------------------------------ migration --
 * Call 5 -- migrate_layers ("When a layer is migrated from GPU A to
 * GPU B, the memory allocated for the layer ... is released on GPU A and
 * allocated on GPU B"; payload at a step boundary = parameters + optimizer
 * state, reading Q19).  COLLECTIVE: every rank calls it with identical
 * boundary and rank arrays.  Layer i lives on rank h_rank_old[stage_old(i)]
 * before and h_rank_new[stage_new(i)] after; every layer whose rank changes
 * is moved with ncclSend/ncclRecv of each of its n_bufs buffers inside one
 * NCCL group on `stream` (NVLink / NVSwitch peer transfers).
 *   h_send[i*n_bufs + k]: on the OLD owner, the k-th buffer of layer i
 *   (pointer + bytes); h_recv[i*n_bufs + k]: on the NEW owner, a caller-
 *   allocated buffer of the same byte size.  Entries for layers this rank
 *   neither sends nor receives are ignored (may be {NULL, 0}).  A needed
 *   entry that is NULL with bytes > 0 -> INVALID before any transfer.
 *   Sizes must agree between sender and receiver (caller metadata).
 *   The caller frees send buffers after the stream has completed.
 *   h_bytes_sent / h_bytes_recv (nullable): bytes this rank sends/receives.
 * With nranks == 1 every rank entry must be 0 and nothing is transferred. */
typedef struct dynmo_buf {
    void *d_ptr;
    int64_t bytes;
} dynmo_buf;

dynmo_status dynmo_migrate_layers(dynmo_ctx ctx, int32_t n_layers, int32_t n_old,
                                  const int32_t *h_bnd_old, const int32_t *h_rank_old,
                                  int32_t n_new, const int32_t *h_bnd_new,
                                  const int32_t *h_rank_new, const dynmo_buf *h_send,
                                  const dynmo_buf *h_recv, int32_t n_bufs, int64_t *h_bytes_sent,
                                  int64_t *h_bytes_recv, dynmo_stream stream);

/* Call 5, peer-memory variant (nranks > 1): the receivers PULL the moved
 * layers' buffers straight from the senders' memory over NVLink with one copy
 * kernel (128-bit loads; no NCCL in the data path).
 * dynmo_migrate_plan_create is COLLECTIVE and off the hot path: every rank
 * registers the buffers it may send (h_send, layers it owns now; CUDA IPC
 * handles of their cudaMalloc allocations are exchanged over the ctx
 * communicator and mapped by every peer) and the buffers it may receive into
 * (h_recv), same table layout as dynmo_migrate_layers.  The buffers must stay
 * allocated while the plan lives.  A failure on any rank during plan creation
 * fails it on every rank (no rank is left in a setup collective).
 * dynmo_migrate_layers_p2p is collective
 * like call 5: on `stream` the sender marks its buffers ready (release flag in
 * each receiver's peer window, after its prior work), each receiver waits for
 * its senders, copies, and marks done; the sender's stream then waits for its
 * receivers (so it may overwrite or free the send buffers afterwards).  Sizes
 * must match between sender and receiver (INVALID).  The ready/done flags
 * carry one epoch per directed rank pair, advanced only in calls where that
 * pair moves data, so ranks that sit a call out stay in step.  Waits are
 * bounded (10 s): a timeout sets a sticky error readable with
 * dynmo_ctx_p2p_error. */
typedef struct dynmo_mplan_s *dynmo_mplan;
dynmo_status dynmo_migrate_plan_create(dynmo_ctx ctx, int32_t n_layers, int32_t n_bufs,
                                       const dynmo_buf *h_send, const dynmo_buf *h_recv,
                                       dynmo_mplan *out);
void dynmo_migrate_plan_destroy(dynmo_mplan plan);
dynmo_status dynmo_migrate_layers_p2p(dynmo_ctx ctx, dynmo_mplan plan, int32_t n_old,
                                      const int32_t *h_bnd_old, const int32_t *h_rank_old,
                                      int32_t n_new, const int32_t *h_bnd_new,
                                      const int32_t *h_rank_new, int64_t *h_bytes_sent,
                                      int64_t *h_bytes_recv, dynmo_stream stream);
/* Device-driven variant: the boundaries and stage->rank maps are DEVICE
 * arrays (e.g. straight from partition_stages / repack_workers), every kernel
 * derives the moves itself, and the ready/done epochs are device-side, so
 * there is no host round trip and the call can be captured in a CUDA graph
 * together with profile + partition (the whole rebalancing step is then one
 * graph launch).  Collective like call 5 (same call sequence on every rank).
 * n_old / n_new: stage counts of the two maps; n_layers <= 1023.  An invalid
 * boundary vector, a stage -> rank entry outside [0, nranks) (e.g. the -1 of
 * a failed dynmo_map_stages) or a send/receive size mismatch sets the sticky
 * peer error to INVALID and moves nothing (for a size mismatch: that buffer);
 * a wait timeout sets it to NCCL.
 * d_bytes_sent / d_bytes_recv (nullable): this rank's bytes (device). */
dynmo_status dynmo_migrate_layers_dev(dynmo_ctx ctx, dynmo_mplan plan, int32_t n_old,
                                      const int32_t *d_bnd_old, const int32_t *d_rank_old,
                                      int32_t n_new, const int32_t *d_bnd_new,
                                      const int32_t *d_rank_new, int64_t *d_bytes_sent,
                                      int64_t *d_bytes_recv, dynmo_stream stream);
/* SM budget of dynmo_migrate_layers_dev's pull kernel: at most max_ctas
 * CTAs of 512 threads (0 = one per SM, the default; clamped to the SM
 * count).  For a migration overlapped with backward compute on another
 * stream ("moving layers while the gradients calculation take
 * place"): each CTA keeps 64 KB of NVLink loads in flight, so
 * a small budget still fills the link while the other SMs compute.  Host
 * setting, takes effect at the next call (and at graph capture).  INVALID if
 * max_ctas < 0. */
dynmo_status dynmo_migrate_plan_set_ctas(dynmo_mplan plan, int32_t max_ctas);
/* Migration overlapped with the backward pass (NEXT-3; "by moving
 * layers while the gradients calculation take place, from the last to the
 * first layer"; P:L640, P:L672 per-iteration MoE / MoD rebalancing).  The
 * payload tables are the plan's (params + gradients + optimizer state of a
 * layer, any number of buffers per layer); the new split is a DEVICE array
 * computed before the backward pass (profile -> partition after forward).
 * No kernel spins: waits are stream memory operations (cuStreamWaitValue64,
 * polled by the GPU front end), so no SM is held while a layer's gradients
 * are still being computed.  Per iteration, on every rank, in host order:
 *   dynmo_migrate_bwd_begin: collective, once per iteration, before the
 *     other three calls: advances the iteration epoch (host side; nothing is
 *     launched).  DYNMO_E_CUDA if the device lacks 64-bit stream memory
 *     operations.
 *   dynmo_migrate_layer_ready: on the stream that wrote layer `layer`'s
 *     buffers (its gradients), after them: a one-thread kernel fences at
 *     system scope and releases the layer's word in EVERY rank's peer window.
 *     Every layer must be released by its owner (old stage's rank) once per
 *     iteration, last layer first as the backward pass runs.  INVALID if
 *     layer is outside [0, n_layers) or before bwd_begin.
 *   dynmo_migrate_layers_bwd: on a side stream: for each layer in
 *     DESCENDING order, a stream wait for its ready word, then a pull kernel
 *     of max_ctas CTAs that copies the layer over NVLink iff it moves to this
 *     rank (device boundaries / rank maps, as dynmo_migrate_layers_dev);
 *     then releases this rank's done word in every window.  *d_bytes_recv
 *     (nullable) = bytes pulled.  Requires an SM budget
 *     (dynmo_migrate_plan_set_ctas with 0 < max_ctas < SM count, else
 *     INVALID): the pulls share the GPU with this rank's backward pass.
 *   dynmo_migrate_bwd_end: on the stream that reuses / frees the sent
 *     buffers (e.g. the backward stream after its last layer): stream waits
 *     for every rank's done word; *d_bytes_sent (nullable) = bytes of this
 *     rank's layers the others pulled.
 * Errors: a malformed split or rank map, or mismatched buffer sizes, set the
 * ctx's sticky error word (DYNMO_E_INVALID, dynmo_ctx_p2p_error) and move
 * nothing; the handshake still completes.  The waits are unbounded (like a
 * NCCL collective): a rank that skips a call blocks its peers' streams, and
 * between bwd_begin and its last layer_ready a rank's host must not wait on
 * the device (cudaDeviceSynchronize, synchronous copies, a first launch
 * that lazily loads a module): its side stream already waits for releases
 * its own stream has not executed yet, and its peers' streams for its
 * releases.  With the default CUDA_MODULE_LOADING=LAZY, every kernel the
 * backward launches in that window must have run once before (a warm-up
 * iteration; note that e.g. a fill of an unaligned view is a different
 * kernel from the aligned one), or the process sets
 * CUDA_MODULE_LOADING=EAGER.  The library loads its own kernels when the
 * ctx is created.  dynmo_ctx_window_snapshot shows which release or done
 * word a hung rank is waiting for.
 * Host epochs are baked into the stream operations, so these calls are
 * issued eagerly each iteration (not replayed from a captured graph). */
dynmo_status dynmo_migrate_bwd_begin(dynmo_ctx ctx, dynmo_mplan plan, dynmo_stream stream);
dynmo_status dynmo_migrate_layer_ready(dynmo_ctx ctx, dynmo_mplan plan, int32_t layer, dynmo_stream stream);
dynmo_status dynmo_migrate_layers_bwd(dynmo_ctx ctx, dynmo_mplan plan, int32_t n_old,
                                      const int32_t *d_bnd_old, const int32_t *d_rank_old,
                                      int32_t n_new, const int32_t *d_bnd_new,
                                      const int32_t *d_rank_new, int64_t *d_bytes_recv,
                                      dynmo_stream stream);
/* Escape hatch (the waits above are unbounded): releases every layer and
 * done word of the current epoch in this rank's own window and sets the
 * sticky error to DYNMO_E_NCCL, so this rank's streams stop waiting.  For a
 * host watchdog that sees an iteration overrun (a peer that skipped a call
 * or died); copies on a private stream.  The iteration's received payload is
 * undefined; the next iteration (dynmo_migrate_bwd_begin) starts clean. */
dynmo_status dynmo_migrate_bwd_abort(dynmo_ctx ctx, dynmo_mplan plan);
dynmo_status dynmo_migrate_bwd_end(dynmo_ctx ctx, dynmo_mplan plan, int32_t n_old,
                                   const int32_t *d_bnd_old, const int32_t *d_rank_old,
                                   int32_t n_new, const int32_t *d_bnd_new,
                                   const int32_t *d_rank_new, int64_t *d_bytes_sent,
                                   dynmo_stream stream);
/* Sticky device error of the peer-memory paths (0 = none); synchronous. */
dynmo_status dynmo_ctx_p2p_error(dynmo_ctx ctx, int32_t *h_err);
/* Resets the sticky error word to 0 after the device is idle (e.g. after a
 * handled dynmo_migrate_bwd_abort); synchronous. */
dynmo_status dynmo_ctx_p2p_error_clear(dynmo_ctx ctx);

/* Host-only helper (no GPU, no ctx): the migration plan call 5 executes.
 * Writes moves (layer, src_rank, dst_rank), layer ascending, for every layer
 * whose owning rank changes, into h_moves[n_layers][3]; returns the number of
 * moves, or DYNMO_E_INVALID (< 0) if a boundary vector is malformed. */
int32_t dynmo_migration_plan(int32_t n_layers, int32_t n_old, const int32_t *h_bnd_old,
                             const int32_t *h_rank_old, int32_t n_new, const int32_t *h_bnd_new,
                             const int32_t *h_rank_new, int32_t *h_moves);

/* Migration-minimising stage -> rank map (NEXT-3; reading Q23): layer i
 * lives on rank_old[stage_old(i)]; place the n_new stages of the new split on
 * DISTINCT ranks of `allowed` (bit r = rank r may host a stage, ranks < G <=
 * 16) so that the bytes of layers that stay on their rank are maximal (each
 * byte kept is a byte not migrated); among optimal maps the
 * lexicographically smallest rank vector.  Exact (DP over subsets of ranks,
 * one CTA, ctx workspace), asynchronous, capturable; feeds d_rank_new of
 * dynmo_migrate_layers_dev directly.  Several stages per GPU: make the G
 * "ranks" slots (capacity = slots per GPU), give d_rank_old in slot units,
 * and d_slot_rank[G] (nullable) maps each slot to its GPU for the output.
 *   d_bnd_old[n_old+1], d_rank_old[n_old], d_bnd_new[n_new+1] int32 device
 *   d_bytes[n_layers] int64 device (e.g. the mem vector of profile_layers)
 *   out: d_rank_new[n_new] int32 (-1 on error), d_kept[1] int64 (bytes kept,
 *        -1 on error), d_status[1] int32: OK, INVALID (malformed split, rank
 *        outside [0, G), negative bytes), INFEASIBLE (n_new > |allowed|).
 * Host INVALID: n_layers outside [1, 1023], G outside [1, 16], null pointers. */
dynmo_status dynmo_map_stages(dynmo_ctx ctx, int32_t n_layers, int32_t n_old, const int32_t *d_bnd_old,
                              const int32_t *d_rank_old, int32_t n_new, const int32_t *d_bnd_new,
                              const int64_t *d_bytes, int32_t G, uint32_t allowed, const int32_t *d_slot_rank,
                              int32_t *d_rank_new, int64_t *d_kept, int32_t *d_status, dynmo_stream stream);

/* ---------------------------------------- global magnitude pruning (NEXT-2)
 * Algorithm 1: every rank holds a portion of the model; keep
 * exactly k parameters of largest magnitude |w| over ALL ranks (line 2:
 * k = num_params (1 - sparsity), computed by the caller; lines 3-8: local
 * top-k, gather, global top-k, scatter); equal magnitudes are kept in the
 * global order (rank, then segment order, then element index; SPEC
 * S:L175-184).  Same kept set as the paper's gather/scatter, found by an
 * exact distributed radix select on magnitude keys: 1 (all bf16: the 15-bit
 * first digit is the whole magnitude) or 3 HBM-streaming histogram passes
 * over this rank's weights with an NCCL all-reduce of the counters per pass
 * (32769 after the first), then one mask-writing pass. */
enum { DYNMO_W_F32 = 0, DYNMO_W_BF16 = 1 };

typedef struct dynmo_prune_segment {
    const void *d_w;   /* weights, 16-byte aligned, caller-owned           */
    uint8_t *d_mask;   /* out: 1 keep / 0 prune per weight (n bytes)       */
    int64_t n;         /* weights in the segment (>= 0)                    */
    int32_t dtype;     /* DYNMO_W_F32 | DYNMO_W_BF16                       */
    int32_t pad;
} dynmo_prune_segment;

typedef struct dynmo_pplan_s *dynmo_pplan;

/* Plan of this rank's weight segments (in order; off the hot path: tile
 * table + workspace on the device).  Pointers must stay valid while the plan
 * is used.  COLLECTIVE when the ctx has more than one rank (every rank calls
 * it, synchronous): the ranks agree on the passes (an f32 segment on any rank
 * adds the f32 passes on all).  INVALID: unknown dtype, negative n, a
 * misaligned pointer -- on any rank, returned by every rank. */
dynmo_status dynmo_prune_plan_create(dynmo_ctx ctx, const dynmo_prune_segment *h_segs, int32_t n_segs,
                                     dynmo_pplan *out);
void dynmo_prune_plan_destroy(dynmo_pplan plan);

/* Collective (every rank, same k): writes every segment's mask.
 *   k       global number of weights to keep; k < 0 is INVALID (host).
 *   d_info  [6] int64 out, nullable: {tau key (bits of the k-th largest |w|
 *           as f32; -1 if nothing is kept), global non-NaN count, global
 *           count above tau, ties kept on this rank, ties on this rank,
 *           flags: bit 0 = the first digit's bin window (estimated from a
 *           1/32 tile sample) missed and the full first-digit histogram
 *           ran; bit 1 = the tie counts came from the windowed pass (no
 *           tie-count pass over the weights)}.
 *   d_status [1] int32 out: OK; INVALID if k > global non-NaN count (all
 *           masks 0) or a NaN weight exists (NaN is never kept).
 * Asynchronous on `stream`, no host synchronisation; capturable in a CUDA
 * graph (NCCL calls included). */
dynmo_status dynmo_global_prune(dynmo_ctx ctx, dynmo_pplan plan, int64_t k, int64_t *d_info,
                                int32_t *d_status, dynmo_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* DYNMO_H */
