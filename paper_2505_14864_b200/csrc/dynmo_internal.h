// Internal declarations shared by the host library (dynmo_host.cpp) and the
// sm_100a kernels (k_profile.cu, k_solve.cu).  Not part of the C-ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dynmo.h"

// Bounds-checked build (make debug -> libdynmo_dbg.so, DYNMO_DEBUG=1 loads
// it): every scratch / shared-memory / table index is asserted; a violation
// prints its site and traps.  Compiled out of the product library.
#ifdef DYNMO_BOUNDS
#include <cstdio>
#define DYNMO_DCHECK(c)                                                                  \
    do {                                                                                 \
        if (!(c)) {                                                                      \
            printf("DYNMO_BOUNDS %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,     \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                               \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define DYNMO_DCHECK(c) ((void)0)
#endif

namespace dynmo {

// ---------------------------------------------------------------- profiling
// A tile is a contiguous byte range of one segment processed by one warp.
// Vector tiles are 16-byte aligned with a multiple-of-16 length; scalar tiles
// (unaligned heads/tails, < 16 bytes, and the last partial byte of a bit
// mask) are walked element by element.
enum ProfOp : uint16_t {
    OP_POPC = 0,   // count set bits                (MASK_BITS, TOKMASK_BITS)
    OP_NZ8 = 1,    // count bytes != 0              (MASK_U8)
    OP_NZ16 = 2,   // count (h & 0x7FFF) != 0       (NZ_BF16)
    OP_NZ32 = 3,   // count (w & 0x7FFFFFFF) != 0   (NZ_F32)
    OP_EXIT = 4,   // histogram of uint8 exit depths
    OP_EXP64 = 5,  // per-layer histogram of int64 expert ids
    OP_EXP32 = 6,  // per-layer histogram of int32 expert ids
    OP_TIME = 7,   // sum of (end - begin) over int64 timestamp pairs (TIME_NS)
    OP_KINDS = 8,
    OP_SCALAR = 0x10,  // flag: scalar tile
    OP_STRIDED = 0x20, // flag: strided count tile -- whole layers of `bits` 16-byte vectors each,
                       // back to back (layer = tile.layer + vector / bits), see kStrided*
};
// Strided tiles: runs of bit-mask segments of one kind that are contiguous
// in memory, one per consecutive layer, all of the same 16-byte-multiple
// size (e.g. config 5's 4096-bit MoD token masks, 512 B per layer) become
// one descriptor per tile instead of one per layer.
constexpr uint32_t kStridedMinVec = 32, kStridedMaxVec = 256;  // layer sizes 512 B .. 4 KiB
constexpr int kStridedMinRun = 8;                              // layers per run worth merging

// Accumulator slots per local layer in the device workspace.
enum { ACC_NNZ = 0, ACC_TOK = 1, ACC_TIME = 2, ACC_N = 3 };

struct ProfTile {
    const void *ptr;   // first byte
    uint32_t nbytes;   // bytes in the tile
    int32_t layer;     // local layer index (ignored by OP_EXIT)
    uint16_t op;       // ProfOp | OP_SCALAR | OP_STRIDED
    uint16_t aux;      // count ops: accumulator slot; OP_EXP*: E;
    uint32_t bits;     // scalar OP_POPC: valid bits in the (single) last byte, 0 = all 8;
                       // OP_STRIDED: 16-byte vectors per layer
};
static_assert(sizeof(ProfTile) == 24, "tile layout");

// Static per-local-layer source flags, known at plan creation.
enum { SRC_HAS_NNZ = 1, SRC_HAS_TOK = 2, SRC_HAS_MOE = 4, SRC_HAS_EXIT = 8, SRC_HAS_TIME = 16 };
struct LayerInfo {
    int32_t flags;
    int32_t E;   // experts of this layer (0 if no MoE source)
};

// ------------------------------------------------ programmatic dependent launch
// Kernels that follow another kernel of the path on a stream are launched
// with programmatic stream serialization: they may be scheduled while the
// predecessor still runs (hiding launch latency) and execute pdl_wait()
// before touching ANY memory, so the ordering seen by the data is that of a
// normal launch (griddepcontrol.wait returns once the predecessor grid has
// completed and its writes are visible; it is a no-op without the attribute).
// pdl_trigger() lets the successor be scheduled early.  DYNMO_PDL=0 disables.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

// Diagnostic build only (-DDYNMO_STEP_STAMPS, tools/step_stamps.py): every
// step kernel records the first warp start (after its griddepcontrol.wait)
// and the last warp end in %globaltimer ns, per kernel id, in a per-file
// device table read by dynmo_diag_step_stamps.
enum { STAMP_PROFILE = 0, STAMP_EPILOGUE, STAMP_PUBLISH, STAMP_PARTITION, STAMP_DIFFUSE_D, STAMP_DIFFUSE_F,
       STAMP_REPACK, STAMP_N };
#ifdef DYNMO_STEP_STAMPS
__device__ __forceinline__ unsigned long long stamp_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
struct StampScope {
    unsigned long long *row;
    __device__ explicit StampScope(unsigned long long *r) : row(r) {
        if ((threadIdx.x & 31) == 0) atomicMin(&row[0], stamp_now());
    }
    __device__ ~StampScope() {
        if ((threadIdx.x & 31) == 0) atomicMax(&row[1], stamp_now());
    }
};
#define STEP_STAMP(id) StampScope step_stamp_scope_(g_step_stamp[id])
#else
#define STEP_STAMP(id)
#endif
void diag_stamps_profile(unsigned long long *h, bool reset);  // k_profile.cu's kernels
void diag_stamps_solve(unsigned long long *h, bool reset);    // k_solve.cu's kernels

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    if (!pdl_enabled()) {
        k<<<grid, block, smem, s>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

constexpr int kProfThreads = 256;
constexpr uint32_t kTileBytes = 32u << 10;   // max vector tile size (plan picks 4..32 KiB)
constexpr int kExitBins = 256;
constexpr int kColExperts = 64;              // E <= 64: per-lane columns in smem
constexpr int kMaxExperts = 1024;

struct ProfArgs {
    const ProfTile *tiles;
    int64_t n_tiles;
    unsigned long long *acc;    // [n_local][ACC_N]
    unsigned long long *hist;   // [n_local][max_E]
    unsigned long long *exit_hist;  // [kExitBins]
    int32_t max_E;
    int32_t *ws_status;
    int32_t warp_words;  // per-warp histogram scratch (u32 words)
    int32_t n_local;     // layers of the plan (bounds of acc / hist rows)
    int32_t l2_prefetch; // 1: each warp bulk-prefetches its whole tile range into L2 at entry
    // nullable: {~min CTA start, max CTA end} in %globaltimer ns (profile-phase
    // timing: the kernel's own span, without the event-bracket launch and
    // completion latencies); folded and reset by the epilogue's last block
    unsigned long long *span;
};
// Plans whose bytes fit comfortably in the 126 MB L2 issue one L2 bulk
// prefetch per tile at kernel entry (all of a warp's range at once), so the
// HBM queues fill at once instead of one register batch per warp at a time
// (small per-GPU shares are latency / ramp bound).
constexpr int64_t kL2PrefetchMaxBytes = 0;  // off: measured slower (profiles/r02_ab_env.jsonl), knob kept for A/B

struct PeerWindow;
constexpr int kMaxRanksEpi = 16;

struct EpiArgs {
    int32_t layer_begin, n_local, n_total, exchange, max_E;
    // exchange over peer memory (exchange == 1): every rank's slot area is
    // LL words uint64 [2 parity][nranks][2 (3 + 2 n_total)]: every int64 of
    // the slot {layer_begin, n_local, status, cost[n_total], mem[n_total]} as
    // two 8-byte words {32 data bits, 32-bit epoch} (flag in the data: no
    // fence or flag release needed), mapped by every peer
    int32_t p2p, rank, nranks;
    int64_t *peer_slots[kMaxRanksEpi];
    PeerWindow *win;                      // local window (exch_epoch counter)
    PeerWindow *peer_win[kMaxRanksEpi];   // every rank's window (flags)
    const LayerInfo *info;
    unsigned long long *acc;
    unsigned long long *hist;
    unsigned long long *exit_hist;
    const uint8_t *frozen;
    const dynmo_cost_coef *coef;
    const int64_t *mem_local;
    int64_t *counters_out;   // [n_local][4] nullable
    int64_t *hist_out;       // [n_local][max_E] nullable
    int64_t *cost_out;       // local mode: [n_local]
    int64_t *mem_out;        // local mode: [n_local] nullable
    int64_t *slot_send;      // exchange mode: [3 + 2*n_total]
    int32_t *ws_status;
    unsigned int *ws_done;
    int32_t *status_out;     // local mode final status
    unsigned long long *span;  // nullable: [0] ~start, [1] end of k_profile, [2] sum of spans (ns), [3] launches
    // nullable: plan scratch (3 + 2 max_E + 256 + 8 + max_E u64, zero) for the
    // epilogue's code warm-up pass before griddepcontrol.wait
    unsigned long long *warm;
    // peer-memory exchange fused into the last block (p2p && fuse_unpack):
    // this rank's receive area, the decode buffer, the global outputs
    int32_t fuse_unpack;
    const int64_t *p2p_slots;
    int64_t *decoded, *x_cost, *x_mem;
    int32_t *x_status;
};

// ops: bit 0 count ops, bit 1 exit histogram, bit 2 expert histograms
cudaError_t launch_profile(const ProfArgs &a, int ops, int grid, cudaStream_t s);
int profile_blocks_per_sm(int ops, int warp_words);
// per-warp histogram scratch words of one expert layer: E <= 16 counts in
// registers, E <= 64 in lane-private smem columns (32 E words), else E words
inline int expert_words(int E) { return E <= 16 ? 0 : E <= kColExperts ? 32 * E : E; }
// per-warp scratch of a plan: max over its exit source (256 bins) and layers
inline int profile_warp_words(bool any_exit, int max_expert_words) {
    const int w = any_exit ? kExitBins : 0;
    const int m = w > max_expert_words ? w : max_expert_words;
    return m > 0 ? m : 1;
}
// ------------------------------------------------- global pruning (Alg. 1)
struct PruneTile {
    const void *w;    // 16-byte aligned first element
    uint8_t *mask;    // its mask bytes
    uint32_t n;       // elements (<= kPruneTileElems)
    int32_t dtype;    // DYNMO_W_F32 | DYNMO_W_BF16
};
static_assert(sizeof(PruneTile) == 24, "prune tile layout");
constexpr uint32_t kPruneTileElems = 32768;
constexpr int64_t kPruneSampleStride = 32;  // pass-0 sample: every 32nd tile
constexpr int kWinCnt = 16;
constexpr int kPruneCw = 4097;  // counters of the windowed pass's compact histogram (4096 bins + NaN)  // windows up to 16 bins also record per-(tile, warp range) bin counts

struct PruneSel {  // device-side selection state of one call
    long long k, k_rem, above, tie_local, keep_ties, n_global;
    uint32_t prefix, tau;
    int32_t partial, status, done, pad;
    uint32_t win_lo, win_hi;  // pass-0 bin window estimated from the sample histogram
    int32_t miss;             // the k-th key fell outside the window: full pass-0 histogram
    int32_t missed;           // a miss happened in this call (d_info[5])
    int32_t wincnt;           // tile_win holds the per-(tile, warp range) counts of tau's bin
    uint32_t tau_d;           // tau's bin - win_lo
};

struct PruneArgs {
    const PruneTile *tiles;
    int64_t n_tiles;
    unsigned long long *hist_local;   // [32770] (bin 32768: NaN count; 32769: elements, sample pass)
    unsigned long long *hist_global;  // [32770] all-reduced (nranks > 1)
    PruneSel *sel;
    const long long *tie_all;         // [nranks] all-gathered tie counts
    uint32_t *tile_ties;              // [n_tiles]
    unsigned long long *tile_off;     // [n_tiles]
    uint16_t *tile_win;               // [n_tiles][8][kWinCnt] window-bin counts (bf16-only plans), else null
    uint32_t *tile_tot;               // [n_tiles] tau's ties per tile (from tile_win)
    unsigned long long *cw_local;     // [4097] the windowed pass's compact histogram (k_prune.cu kCw)
    unsigned long long *cw_global;    // [4097] all-reduced (nranks > 1)
    long long n_elems;                // this rank's weights
    int32_t rank, nranks, last_pass;
};
cudaError_t launch_prune(const PruneArgs &a, int pass_kind, int grid, cudaStream_t s);
int prune_blocks_per_sm(int kind);
cudaError_t launch_prune_begin(PruneSel *sel, long long k, cudaStream_t s);
cudaError_t launch_prune_info(const PruneArgs &a, long long *d_info, int32_t *d_status, cudaStream_t s);

// --------------------------------------- stage -> rank map (NEXT-3, Q23)
constexpr int kMaxMapRanks = 16;
struct MapArgs {
    int32_t L, n_old, n_new, G;
    uint32_t allowed;
    const int32_t *bnd_old, *rank_old, *bnd_new;
    const int64_t *bytes;
    int32_t *rank_new;
    int64_t *kept;
    int32_t *status;
    long long *work;  // [1 << G]
    const int32_t *slot_rank;  // nullable: output rank_new[s] = slot_rank[slot]
};
cudaError_t launch_map_stages(const MapArgs &a, cudaStream_t s);

cudaError_t launch_epilogue(const EpiArgs &a, cudaStream_t s);
cudaError_t launch_stamp(int64_t *d_slot, cudaStream_t s);
cudaError_t launch_publish(const void *d_src, void *d_dst, int64_t bytes, cudaStream_t s);
cudaError_t launch_unpack(const int64_t *slot_recv, int32_t nranks, int32_t n_total,
                          int64_t *cost_out, int64_t *mem_out, int32_t *status_out,
                          cudaStream_t s);
// peer-memory exchange: waits for every rank's flag of this epoch, then
// unpacks the local slot area (parity of the epoch)
cudaError_t launch_unpack_p2p(const int64_t *slots, PeerWindow *win, int32_t nranks, int32_t n_total,
                              int64_t *decoded, int64_t *cost_out, int64_t *mem_out, int32_t *status_out,
                              cudaStream_t s);

// ------------------------------------------------------------------ solvers
struct SolveArgs {
    int32_t n_inst, max_layers;
    int32_t fluid_spec;  // fluid process: speculative rounds (1) or the exact per-round chain (0)
    const int64_t *cost, *mem;
    const int32_t *layer_off, *n_stages;   // n_stages: n (partition/diffuse) or n_cur (repack)
    const int64_t *cap;
    const int32_t *bnd_off;
    const int32_t *bnd_in;
    int32_t *bnd_out;
    int64_t *bottleneck;
    double *imbalance;
    int32_t *status;
    // diffusion
    const int64_t *gamma;
    const double *gamma_fluid;
    int32_t max_rounds;
    int32_t *rounds;
    int64_t *phi, *phi0;
    double *fluid_x;
    int32_t *fluid_rounds;
    double *fluid_phi;
    int32_t *fluid_status;
    // repack
    const int64_t *bound;
    const int32_t *floor_;
    int32_t mode;
    int32_t *n_new;
};

// ---------------------------------------------------------------- peer P2P
constexpr int kP2PThreads = 512;
constexpr int kP2PMaxItems = 64;
constexpr int kMaxRanks = kMaxRanksEpi;

// Per-rank flag window, mapped by every peer (CUDA IPC).  Peers write their
// own slot [src]; the owner reads.  Epochs only grow.
struct PeerWindow {
    uint64_t ready[kMaxRanks];  // sender src's buffers are ready (migration epoch)
    uint64_t done[kMaxRanks];   // receiver dst finished pulling (migration epoch)
    uint64_t exch[kMaxRanks];   // rank src's exchange slot is written (profile epoch)
    uint64_t exch_epoch;        // this rank's profile-exchange epoch counter
    unsigned int pull_ctr;      // last-block counter of k_pull
    int32_t err;                // sticky error (timeouts)
    // device-driven migration (dynmo_migrate_layers_dev): own flags/epochs
    uint64_t dready[kMaxRanksEpi];
    uint64_t ddone[kMaxRanksEpi];
    uint64_t mig_dev_epoch;
    unsigned int dpull_ctr;
    int32_t barrier;            // dynmo_ctx_barrier's all-reduce word (local use only)
    // migration overlapped with the backward pass (NEXT-3): per-layer
    // "payload final" words and per-rank "pulls done" words, written by the
    // owners / receivers into EVERY rank's window, polled locally by stream
    // memory operations (epochs from the host)
    uint64_t bwd_done[kMaxRanksEpi];
    uint64_t layer_ready[1024];
    unsigned long long bwd_claim[1024];  // per layer {epoch, chunks claimed} (local use)
    unsigned int bwd_finished[2];        // chunks copied, per epoch parity (local use)
    // profile-phase timing: k_profile's own span (ProfArgs::span), local use
    unsigned long long prof_span[4];
};
constexpr size_t kPeerWindowBytes = 32768;  // the window allocation
static_assert(sizeof(PeerWindow) <= kPeerWindowBytes, "peer window page");

struct DevBuf {
    void *ptr;
    int64_t bytes;
};

// Device-driven migration: boundaries and stage->rank maps on the device;
// every kernel derives the moves itself (no host round trip, graph-safe).
struct DevMigArgs {
    int32_t n_layers, n_bufs, me, nranks;
    int32_t n_old, n_new;
    const int32_t *bnd_old, *rank_old, *bnd_new, *rank_new;
    const DevBuf *src_tab;   // [nranks][n_layers * n_bufs], readable from this rank
    const DevBuf *recv_tab;  // [n_layers * n_bufs], this rank's receive buffers
    PeerWindow *win;
    PeerWindow *peer_win[kMaxRanksEpi];
    int64_t *bytes_sent, *bytes_recv;  // nullable
    int32_t hint;  // backward pulls: streaming cache hints (A/B knob DYNMO_PULL_HINT)
};
cudaError_t launch_mig_dev(const DevMigArgs &a, int grid, bool budget, cudaStream_t s);
// NEXT-3 backward-ordered variant: per-layer ready release into every
// window, one pull kernel per layer, the done release, the bytes sent
struct BwdPeers {
    PeerWindow *win[kMaxRanksEpi];
    int32_t nranks;
};
cudaError_t launch_layer_ready(const BwdPeers &p, int32_t layer, uint64_t epoch, cudaStream_t s);
cudaError_t launch_bwd_pull_layer(const DevMigArgs &a, int32_t layer, uint64_t epoch, int grid, cudaStream_t s);
cudaError_t launch_bwd_drain(const DevMigArgs &a, uint64_t epoch, int grid, cudaStream_t s);
cudaError_t launch_bwd_done(const DevMigArgs &a, const BwdPeers &p, uint64_t epoch, cudaStream_t s);
cudaError_t launch_bwd_sent(const DevMigArgs &a, cudaStream_t s);
// force-load every peer-path kernel (CUDA lazy loading; see k_p2p.cu)
cudaError_t preload_p2p_kernels();

struct P2PItem {
    const void *src;
    void *dst;
    uint64_t bytes;
};
// Host-driven migration epochs are kept per directed rank pair (sender ->
// receiver): both sides derive the same move set, so both count the calls in
// which the pair exchanges data and agree on the epoch, whichever other
// ranks take part in a call.
struct P2PSignal {
    int n;
    uint64_t epoch[kMaxRanks];       // per receiver: ++send_epoch[dst]
    uint64_t *remote[kMaxRanks];
};
struct P2PWait {
    int n;
    uint64_t epoch[kMaxRanks];       // per receiver: send_epoch[dst]
    const uint64_t *local;
    int idx[kMaxRanks];
    int32_t *err;
};
struct P2PPull {
    int n_items;
    P2PItem items[kP2PMaxItems];
    int n_src;
    int src_rank[kMaxRanks];
    const uint64_t *ready;           // local window ready[]
    uint64_t *done_remote[kMaxRanks];  // &peer_window[src].done[me] (written by the last block)
    int signal_done;
    uint64_t epoch[kMaxRanks];       // per sender: ++recv_epoch[src]
    unsigned int *ctr;
    int32_t *err;
};

cudaError_t launch_signal(const P2PSignal &s, cudaStream_t st);
cudaError_t launch_wait(const P2PWait &w, cudaStream_t st);
cudaError_t launch_pull(const P2PPull &p, int grid, cudaStream_t st);

cudaError_t launch_partition(const SolveArgs &a, cudaStream_t s);
cudaError_t launch_diffuse(const SolveArgs &a, cudaStream_t s);
cudaError_t launch_repack(const SolveArgs &a, cudaStream_t s);

}  // namespace dynmo
