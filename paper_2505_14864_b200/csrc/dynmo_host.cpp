// dynmo_host.cpp -- host side of the C-ABI declared in include/dynmo.h:
// argument validation, profile plans (tile decomposition), the NCCL context,
// kernel launches and layer migration.  No device compute happens here.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dynmo_internal.h"

using namespace dynmo;

namespace {
thread_local std::string g_err;

dynmo_status cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return DYNMO_E_CUDA;
}
dynmo_status invalid(const char *what) {
    g_err = what;
    return DYNMO_E_INVALID;
}
#define CUDA_TRY(call, what)                       \
    do {                                           \
        cudaError_t e_ = (call);                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
}  // namespace

struct PhaseTimer {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;     // eager launches
    size_t used = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> graph;  // baked into captured graphs
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> detached;  // of graphs no longer polled
    double acc_ms = 0.0;
    int64_t acc_n = 0;
};

struct dynmo_ctx_s {
    int device = 0, nranks = 1, rank = 0;
    ncclComm_t comm = nullptr;
    int num_sms = 148;
    int32_t timing = 0;  // bitmask of timed phases
    PhaseTimer ph[DYNMO_NUM_PHASES];
    // peer-memory window (nranks > 1): local flags + every peer's, mapped
    PeerWindow *d_win = nullptr;
    std::vector<PeerWindow *> peer_win;
    cudaStream_t aux = nullptr;  // setup collectives
    // host-driven peer migration: epochs per directed rank pair (P2PSignal)
    uint64_t send_epoch[kMaxRanks] = {}, recv_epoch[kMaxRanks] = {};
    long long *d_map_work = nullptr;  // [1 << kMaxMapRanks] DP table of dynmo_map_stages
    uint64_t bwd_epoch = 0;  // backward-overlapped migration: iterations begun (host epochs)
    bool memops = false;     // 64-bit stream memory operations available
};

namespace dynmo {
bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("DYNMO_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace dynmo

namespace {
// All-gather `n` bytes per rank over the ctx communicator (setup only:
// synchronous, through a temporary device buffer).
dynmo_status allgather_bytes(dynmo_ctx c, const void *mine, size_t n, std::vector<char> &all) {
    all.assign(n * c->nranks, 0);
    char *d = nullptr;
    CUDA_TRY(cudaMalloc(&d, n * c->nranks), "cudaMalloc (allgather)");
    cudaError_t e = cudaMemcpy(d + n * c->rank, mine, n, cudaMemcpyHostToDevice);
    ncclResult_t r = ncclSuccess;
    if (e == cudaSuccess) r = ncclAllGather(d + n * c->rank, d, n, ncclChar, c->comm, c->aux);
    if (e == cudaSuccess && r == ncclSuccess) e = cudaStreamSynchronize(c->aux);
    if (e == cudaSuccess && r == ncclSuccess) e = cudaMemcpy(all.data(), d, n * c->nranks, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (r != ncclSuccess) {
        g_err = std::string("ncclAllGather (setup): ") + ncclGetErrorString(r);
        return DYNMO_E_NCCL;
    }
    if (e != cudaSuccess) return cuda_fail(e, "allgather_bytes");
    return DYNMO_OK;
}

// Base and size of the cudaMalloc allocation containing p (driver API via
// the runtime's entry-point query; no link-time libcuda dependency).
dynmo_status alloc_range(const void *p, CUdeviceptr *base, size_t *size) {
    typedef CUresult (*Fn)(CUdeviceptr *, size_t *, CUdeviceptr);
    static Fn fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
            return invalid("cuMemGetAddressRange unavailable");
        fn = (Fn)f;
    }
    if (fn(base, size, (CUdeviceptr)p) != CUDA_SUCCESS) return invalid("pointer is not device memory");
    return DYNMO_OK;
}
}  // namespace

namespace {
// Records the start event of `phase` on `s`; returns the end event to record
// after the launch (nullptr when timing is off).
// During stream capture the pair becomes two external event-record nodes of
// the graph (re-recorded at every replay; read them with timing_poll after
// each replay).
cudaEvent_t phase_begin(dynmo_ctx c, int phase, cudaStream_t s) {
    if (!(c->timing & (1 << phase))) return nullptr;
    PhaseTimer &t = c->ph[phase];
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    const bool cap = cs == cudaStreamCaptureStatusActive;
    std::pair<cudaEvent_t, cudaEvent_t> pr;
    if (cap || t.used == t.ev.size()) {
        if (cudaEventCreate(&pr.first) != cudaSuccess || cudaEventCreate(&pr.second) != cudaSuccess)
            return nullptr;
        if (cap) t.graph.push_back(pr);
        else t.ev.push_back(pr);
    }
    if (!cap) pr = t.ev[t.used++];
    cudaEventRecordWithFlags(pr.first, s, cap ? cudaEventRecordExternal : cudaEventRecordDefault);
    return pr.second;
}
void phase_end(cudaEvent_t e, cudaStream_t s) {
    if (!e) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    cudaEventRecordWithFlags(e, s, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                       : cudaEventRecordDefault);
}
}  // namespace

struct dynmo_plan_s {
    dynmo_ctx ctx = nullptr;
    int32_t layer_begin = 0, n_local = 0, n_total = 0, exchange = 0, max_E = 0;
    bool has_hist = false;
    int32_t warp_words = 1;
    int32_t ops = 1;
    int64_t n_tiles = 0, bytes = 0;
    int grid = 1;
    void *dmem = nullptr;
    ProfTile *d_tiles = nullptr;
    LayerInfo *d_info = nullptr;
    unsigned long long *d_acc = nullptr, *d_hist = nullptr, *d_exit = nullptr;
    int32_t *d_ws_status = nullptr;
    unsigned int *d_ws_done = nullptr;
    unsigned long long *d_warm = nullptr;  // epilogue code warm-up scratch (EpiArgs::warm)
    int64_t *d_slot_send = nullptr, *d_slot_recv = nullptr;
    int64_t slot_elems = 0;
    // exchange over peer memory (exchange == 1): [2][nranks][slot_elems] here,
    // and every peer's area mapped
    int64_t *d_p2p_slots = nullptr;
    std::vector<int64_t *> peer_slots;
};

extern "C" {

const char *dynmo_strerror(dynmo_status s) {
    switch (s) {
        case DYNMO_OK: return "ok";
        case DYNMO_E_INVALID: return "invalid argument";
        case DYNMO_E_INFEASIBLE: return "infeasible under the memory cap";
        case DYNMO_E_OVERFLOW: return "int64 overflow";
        case DYNMO_E_CUDA: return "CUDA error";
        case DYNMO_E_NCCL: return "NCCL error";
        case DYNMO_E_NOMEM: return "out of device memory";
        case DYNMO_W_NOT_CONVERGED: return "diffusion not converged (max_rounds)";
        case DYNMO_W_BOUND_UNMET: return "repack bound/target unmet";
        default: return "unknown status";
    }
}

const char *dynmo_last_error(void) { return g_err.c_str(); }

const char *dynmo_version(void) { return "dynmo-b200 0.1 (sm_100a)"; }

dynmo_status dynmo_get_unique_id(uint8_t h_id_out[128]) {
    if (!h_id_out) return invalid("null id buffer");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        g_err = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
        return DYNMO_E_NCCL;
    }
    static_assert(sizeof(id.internal) == 128, "nccl id size");
    memcpy(h_id_out, id.internal, 128);
    return DYNMO_OK;
}

// 64-bit stream memory operations (CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS
// = 122) and the cuStreamWaitValue64 entry point: the backward-ordered
// migration's waits.
static bool memops_supported(int device) {
    typedef int (*AttrFn)(int *, int, int);
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
        return false;
    int v = 0;
    if (((AttrFn)f)(&v, 122, device) != 0 || !v) return false;
    void *w = nullptr;
    return cudaGetDriverEntryPoint("cuStreamWaitValue64", &w, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess && w;
}

// Peer window of a multi-rank ctx: a page of flags every peer can write,
// CUDA-IPC mapped by every rank (handles all-gathered over the ctx comm).
static dynmo_status setup_peer_window(dynmo_ctx c) {
    const int nranks = c->nranks, rank = c->rank;
    // peer window: flags every peer can write (CUDA IPC over NVLink)
    dynmo_status st = DYNMO_OK;
    if (cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc((void **)&c->d_win, kPeerWindowBytes) != cudaSuccess ||
        cudaMemset(c->d_win, 0, kPeerWindowBytes) != cudaSuccess)
        st = cuda_fail(cudaGetLastError(), "peer window");
    if (!st && preload_p2p_kernels() != cudaSuccess) st = cuda_fail(cudaGetLastError(), "peer kernels preload");
    cudaIpcMemHandle_t h;
    if (!st && cudaIpcGetMemHandle(&h, c->d_win) != cudaSuccess) st = cuda_fail(cudaGetLastError(), "cudaIpcGetMemHandle");
    std::vector<char> all;
    if (!st) st = allgather_bytes(c, &h, sizeof(h), all);
    c->peer_win.assign(nranks, nullptr);
    for (int rr = 0; !st && rr < nranks; ++rr) {
        if (rr == rank) {
            c->peer_win[rr] = c->d_win;
            continue;
        }
        cudaIpcMemHandle_t ph;
        memcpy(&ph, all.data() + rr * sizeof(ph), sizeof(ph));
        void *mp = nullptr;
        if (cudaIpcOpenMemHandle(&mp, ph, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
            st = cuda_fail(cudaGetLastError(), "cudaIpcOpenMemHandle (window)");
        c->peer_win[rr] = (PeerWindow *)mp;
    }
    return st;
}

// Single-rank ctx: the window is local (peer_win[0] = d_win), so the
// peer-memory exchange runs against itself; no NCCL communicator until a
// plan asks for the NCCL exchange (ensure_comm).
static dynmo_status setup_single_window(dynmo_ctx c) {
    if (cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc((void **)&c->d_win, kPeerWindowBytes) != cudaSuccess ||
        cudaMemset(c->d_win, 0, kPeerWindowBytes) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "peer window (single rank)");
    if (preload_p2p_kernels() != cudaSuccess) return cuda_fail(cudaGetLastError(), "peer kernels preload");
    c->peer_win.assign(1, c->d_win);
    return DYNMO_OK;
}

// A one-rank NCCL communicator (legal in NCCL) for the NCCL exchange of a
// single-rank ctx: the all-gather then degenerates to a local copy.
static dynmo_status ensure_comm(dynmo_ctx c) {
    if (c->comm) return DYNMO_OK;
    if (c->nranks != 1) return invalid("multi-rank ctx without a communicator");
    int dev = c->device;
    const ncclResult_t r = ncclCommInitAll(&c->comm, 1, &dev);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        g_err = std::string("ncclCommInitAll (single rank): ") + ncclGetErrorString(r);
        return DYNMO_E_NCCL;
    }
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_create(int32_t device, int32_t nranks, int32_t rank,
                              const uint8_t *h_nccl_id, dynmo_ctx *out) {
    if (!out) return invalid("null ctx out");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks || device < 0) return invalid("bad rank/device");
    if (nranks > 1 && !h_nccl_id) return invalid("nranks > 1 needs a NCCL unique id");
    if (nranks > kMaxRanks) return invalid("nranks > 16");
    DeviceGuard g(device);
    CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
    auto *c = new dynmo_ctx_s();
    c->device = device;
    c->nranks = nranks;
    c->rank = rank;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
        c->num_sms = sms;
    c->memops = memops_supported(device);
    if (cudaMalloc((void **)&c->d_map_work, sizeof(long long) << kMaxMapRanks) != cudaSuccess) {
        delete c;
        return cuda_fail(cudaGetLastError(), "ctx workspace");
    }
    if (nranks > 1) {
        ncclUniqueId id;
        memcpy(id.internal, h_nccl_id, 128);
        ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            g_err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
            c->comm = nullptr;
            dynmo_ctx_destroy(c);  // frees the workspace
            return DYNMO_E_NCCL;
        }
        const dynmo_status st = setup_peer_window(c);
        if (st) {
            dynmo_ctx_destroy(c);
            return st;
        }
    } else {
        const dynmo_status st = setup_single_window(c);
        if (st) {
            dynmo_ctx_destroy(c);
            return st;
        }
    }
    *out = c;
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_split(dynmo_ctx ctx, int32_t color, int32_t key, dynmo_ctx *out) {
    if (!ctx || !out) return invalid("null ctx/out");
    *out = nullptr;
    DeviceGuard g(ctx->device);
    auto *c = new dynmo_ctx_s();
    c->device = ctx->device;
    c->num_sms = ctx->num_sms;
    c->memops = ctx->memops;
    if (cudaMalloc((void **)&c->d_map_work, sizeof(long long) << kMaxMapRanks) != cudaSuccess) {
        delete c;
        return cuda_fail(cudaGetLastError(), "ctx workspace");
    }
    if (ctx->nranks == 1) {  // nothing to split: a fresh single-rank ctx (or none)
        if (color < 0) {
            dynmo_ctx_destroy(c);
            return DYNMO_OK;
        }
        const dynmo_status st = setup_single_window(c);
        if (st) {
            dynmo_ctx_destroy(c);
            return st;
        }
        *out = c;
        return DYNMO_OK;
    }
    ncclComm_t nc = nullptr;
    ncclResult_t r = ncclCommSplit(ctx->comm, color < 0 ? NCCL_SPLIT_NOCOLOR : color, key, &nc, nullptr);
    if (r != ncclSuccess) {
        g_err = std::string("ncclCommSplit: ") + ncclGetErrorString(r);
        dynmo_ctx_destroy(c);
        return DYNMO_E_NCCL;
    }
    if (color < 0 || !nc) {  // this rank is released (no communicator)
        dynmo_ctx_destroy(c);
        return DYNMO_OK;
    }
    int n = 1, rk = 0;
    ncclCommCount(nc, &n);
    ncclCommUserRank(nc, &rk);
    c->comm = nc;
    c->nranks = n;
    c->rank = rk;
    const dynmo_status st = n > 1 ? setup_peer_window(c) : setup_single_window(c);
    if (st) {
        dynmo_ctx_destroy(c);
        return st;
    }
    *out = c;
    return DYNMO_OK;
}

void dynmo_ctx_destroy(dynmo_ctx ctx) {
    if (!ctx) return;
    for (int r = 0; r < (int)ctx->peer_win.size(); ++r)
        if (r != ctx->rank && ctx->peer_win[r]) cudaIpcCloseMemHandle(ctx->peer_win[r]);
    if (ctx->d_win) cudaFree(ctx->d_win);
    if (ctx->d_map_work) cudaFree(ctx->d_map_work);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    // abort, not destroy: NCCL's destroy blocks while a CUDA graph still holds
    // captured work of the communicator (the caller has synchronised)
    if (ctx->comm) ncclCommAbort(ctx->comm);
    for (auto &t : ctx->ph) {
        for (auto &pr : t.ev) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
        for (auto &pr : t.graph) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
        for (auto &pr : t.detached) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
    }
    delete ctx;
}

dynmo_status dynmo_ctx_set_timing(dynmo_ctx ctx, int32_t enable) {
    if (!ctx) return invalid("null ctx");
    ctx->timing = enable == 1 ? -1 : enable;  // 1 (true) = every phase, else a bitmask
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_timing_poll(dynmo_ctx ctx) {
    if (!ctx) return invalid("null ctx");
    for (auto &t : ctx->ph) {
        for (size_t i = 0; i < t.used; ++i) {
            CUDA_TRY(cudaEventSynchronize(t.ev[i].second), "cudaEventSynchronize");
            float ms = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&ms, t.ev[i].first, t.ev[i].second), "cudaEventElapsedTime");
            t.acc_ms += ms;
            t.acc_n++;
        }
        t.used = 0;
        for (auto &pr : t.graph) {
            CUDA_TRY(cudaEventSynchronize(pr.second), "cudaEventSynchronize");
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, pr.first, pr.second) != cudaSuccess) {
                cudaGetLastError();  // not yet recorded by any replay
                continue;
            }
            t.acc_ms += ms;
            t.acc_n++;
        }
    }
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_barrier(dynmo_ctx ctx, dynmo_stream stream) {
    if (!ctx) return invalid("null ctx");
    if (ctx->nranks == 1) return DYNMO_OK;
    DeviceGuard g(ctx->device);
    // one int32 all-reduce on the window's own barrier word: completes on
    // every rank's stream only once every rank's stream has reached it
    const ncclResult_t r = ncclAllReduce(&ctx->d_win->barrier, &ctx->d_win->barrier, 1, ncclInt32, ncclSum,
                                         ctx->comm, (cudaStream_t)stream);
    if (r != ncclSuccess) {
        g_err = std::string("ncclAllReduce (barrier): ") + ncclGetErrorString(r);
        return DYNMO_E_NCCL;
    }
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_timing_detach(dynmo_ctx ctx) {
    if (!ctx) return invalid("null ctx");
    for (auto &t : ctx->ph) {
        t.detached.insert(t.detached.end(), t.graph.begin(), t.graph.end());
        t.graph.clear();
    }
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_timing_read(dynmo_ctx ctx, int32_t phase, double *h_total_ms, int64_t *h_count) {
    if (!ctx || phase < 0 || phase >= DYNMO_NUM_PHASES) return invalid("bad ctx/phase");
    PhaseTimer &t = ctx->ph[phase];
    if (t.used) {  // fold pending eager launches in (graph pairs need explicit polls)
        for (size_t i = 0; i < t.used; ++i) {
            CUDA_TRY(cudaEventSynchronize(t.ev[i].second), "cudaEventSynchronize");
            float ms = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&ms, t.ev[i].first, t.ev[i].second), "cudaEventElapsedTime");
            t.acc_ms += ms;
            t.acc_n++;
        }
        t.used = 0;
    }
    if (h_total_ms) *h_total_ms = t.acc_ms;
    if (h_count) *h_count = t.acc_n;
    t.acc_ms = 0.0;
    t.acc_n = 0;
    return DYNMO_OK;
}

int32_t dynmo_ctx_nranks(dynmo_ctx ctx) { return ctx ? ctx->nranks : 0; }
int32_t dynmo_ctx_rank(dynmo_ctx ctx) { return ctx ? ctx->rank : -1; }

// ------------------------------------------------------------------ plans
// The rank-local part of dynmo_profile_plan_create: validation, the tile
// decomposition and the device workspace (no collective).
static dynmo_status profile_plan_local(dynmo_ctx ctx, const dynmo_segment *h_segs, int32_t n_segs,
                                       int32_t layer_begin, int32_t n_local, int32_t n_total,
                                       int32_t exchange, dynmo_plan *out) {
    if (n_segs < 0 || (n_segs > 0 && !h_segs)) return invalid("bad segment array");
    if (layer_begin < 0 || n_local < 0 || n_total < 0) return invalid("negative layer range");
    if (exchange < 0 || exchange > 2) return invalid("exchange must be 0, 1 (peer memory) or 2 (NCCL)");
    if (exchange) {
        if ((int64_t)layer_begin + n_local > n_total) return invalid("local layers exceed n_total");
    } else if (n_total != n_local) {
        return invalid("without exchange n_total must equal n_local");
    }
    std::vector<LayerInfo> info(n_local, LayerInfo{0, 0});
    std::vector<ProfTile> vec, sca;
    // tile size: about two tiles per resident warp (small per-GPU inputs, e.g.
    // 75 MB at 8 GPUs, must still spread over every SM), 4 KiB .. 32 KiB
    uint32_t tile_bytes = kTileBytes;
    {
        int64_t total = 0;
        bool pre_exit = false;
        int pre_words = 0, pre_ops = 0;
        for (int32_t i = 0; i < n_segs; ++i) {
            const int k = h_segs[i].src_kind;
            if (k == DYNMO_SRC_EXIT_U8) pre_exit = true;
            if (k == DYNMO_SRC_EXPERT_I64 || k == DYNMO_SRC_EXPERT_I32)
                pre_words = std::max(pre_words, expert_words(std::min((int)h_segs[i].n_experts, kMaxExperts)));
            pre_ops |= k == DYNMO_SRC_EXIT_U8 ? 2 : (k == DYNMO_SRC_EXPERT_I64 || k == DYNMO_SRC_EXPERT_I32) ? 4 : 1;  // TIME: count family
            if ((k == DYNMO_SRC_EXPERT_I64 || k == DYNMO_SRC_EXPERT_I32) && h_segs[i].n_experts > 16) pre_ops |= 8;
            const int64_t ne = h_segs[i].n_elem < 0 ? 0 : h_segs[i].n_elem;
            const int es = k == DYNMO_SRC_NZ_BF16 ? 2 : (k == DYNMO_SRC_NZ_F32 || k == DYNMO_SRC_EXPERT_I32) ? 4
                           : k == DYNMO_SRC_EXPERT_I64 ? 8 : 1;
            total += (k == DYNMO_SRC_MASK_BITS || k == DYNMO_SRC_TOKMASK_BITS) ? ne / 8 : ne * es;
        }
        const int64_t warps = (int64_t)ctx->num_sms *
                              profile_blocks_per_sm(pre_ops ? pre_ops : 1, profile_warp_words(pre_exit, pre_words)) *
                              (kProfThreads / 32);
        int64_t want = total / std::max<int64_t>(1, 2 * warps);
        uint32_t t = 4096;
        while (t < kTileBytes && (int64_t)t * 2 <= want) t *= 2;
        tile_bytes = t;
        if (const char *e = getenv("DYNMO_TILE_BYTES")) {  // tuning knob (multiple of 16)
            const long v = atol(e);
            if (v >= 16 && v % 16 == 0 && v <= (1l << 30)) tile_bytes = (uint32_t)v;
        }
    }
    // Strided runs: consecutive bit-mask segments of one kind, back to back in
    // memory, one per consecutive local layer, all of one 16-byte-multiple
    // size in [512 B, 4 KiB] (config 5: 4096-bit token masks).  run[i] > 0:
    // a run of run[i] segments starts at i; -1: a member (tiles emitted by
    // the run's first segment).
    std::vector<int32_t> run(std::max(0, n_segs), 0);
    {
        auto seg_bytes = [](const dynmo_segment &g) -> int64_t {  // bit-mask kinds only
            switch (g.src_kind) {
                case DYNMO_SRC_MASK_BITS:
                case DYNMO_SRC_TOKMASK_BITS: return g.n_elem % 8 ? -1 : g.n_elem / 8;
                default: return -1;
            }
        };
        auto start_ok = [&](const dynmo_segment &g) {
            const int64_t nb = seg_bytes(g);
            const int q = g.layer - layer_begin;
            return g.n_elem > 0 && g.d_ptr && nb > 0 && nb % 16 == 0 && nb / 16 >= kStridedMinVec &&
                   nb / 16 <= kStridedMaxVec && ((uintptr_t)g.d_ptr & 15) == 0 && q >= 0 && q < n_local;
        };
        const char *e = getenv("DYNMO_STRIDED");  // 0: never merge (A/B knob)
        for (int32_t i = 0; i < n_segs && !(e && e[0] == '0');) {
            const dynmo_segment &a0 = h_segs[i];
            if (!start_ok(a0)) {
                ++i;
                continue;
            }
            const int64_t nb = seg_bytes(a0);
            int32_t j = i + 1;
            while (j < n_segs && h_segs[j].src_kind == a0.src_kind && h_segs[j].n_elem == a0.n_elem &&
                   (uintptr_t)h_segs[j].d_ptr == (uintptr_t)h_segs[j - 1].d_ptr + (uintptr_t)nb &&
                   h_segs[j].layer == h_segs[j - 1].layer + 1 && h_segs[j].layer - layer_begin < n_local)
                ++j;
            if (j - i >= kStridedMinRun) {
                run[i] = j - i;
                for (int32_t m = i + 1; m < j; ++m) run[m] = -1;
            }
            i = j;
        }
    }
    bool any_exit = false, has_hist = false;
    int max_E = 0;
    int64_t bytes = 0;
    for (int32_t i = 0; i < n_segs; ++i) {
        const dynmo_segment &sg = h_segs[i];
        if (sg.n_elem < 0) return invalid("negative n_elem");
        if (sg.src_kind < DYNMO_SRC_MASK_BITS || sg.src_kind > DYNMO_SRC_TIME_NS)
            return invalid("unknown src_kind");
        if (sg.src_kind == DYNMO_SRC_TIME_NS && sg.n_elem % 2)
            return invalid("TIME_NS segment with an odd number of stamps");
        const bool is_exit = sg.src_kind == DYNMO_SRC_EXIT_U8;
        const int q = sg.layer - layer_begin;
        if (!is_exit && (q < 0 || q >= n_local)) return invalid("segment layer outside local range");
        int op = 0, es = 1, slot = ACC_NNZ, E = 0;
        int64_t nb = 0, partial_bits = 0;
        switch (sg.src_kind) {
            case DYNMO_SRC_MASK_BITS:
            case DYNMO_SRC_TOKMASK_BITS:
                op = OP_POPC;
                slot = sg.src_kind == DYNMO_SRC_MASK_BITS ? ACC_NNZ : ACC_TOK;
                nb = sg.n_elem / 8;
                partial_bits = sg.n_elem % 8;
                es = 4;  // words are uint32: pointer must be 4-byte aligned
                break;
            case DYNMO_SRC_MASK_U8: op = OP_NZ8; nb = sg.n_elem; break;
            case DYNMO_SRC_NZ_BF16: op = OP_NZ16; es = 2; nb = sg.n_elem * 2; break;
            case DYNMO_SRC_NZ_F32: op = OP_NZ32; es = 4; nb = sg.n_elem * 4; break;
            case DYNMO_SRC_EXIT_U8: op = OP_EXIT; nb = sg.n_elem; break;
            case DYNMO_SRC_EXPERT_I64: op = OP_EXP64; es = 8; nb = sg.n_elem * 8; break;
            case DYNMO_SRC_EXPERT_I32: op = OP_EXP32; es = 4; nb = sg.n_elem * 4; break;
            case DYNMO_SRC_TIME_NS: op = OP_TIME; es = 8; nb = sg.n_elem * 8; slot = ACC_TIME; break;
        }
        if (sg.src_kind == DYNMO_SRC_EXPERT_I64 || sg.src_kind == DYNMO_SRC_EXPERT_I32) {
            E = sg.n_experts;
            if (E < 1 || E > kMaxExperts) return invalid("n_experts outside [1, 1024]");
            if (info[q].E != 0 && info[q].E != E) return invalid("inconsistent n_experts in a layer");
            info[q].E = E;
            info[q].flags |= SRC_HAS_MOE;
            max_E = std::max(max_E, E);
            has_hist = true;
        } else if (is_exit) {
            any_exit = true;
            has_hist = true;
        } else if (slot == ACC_TOK) {
            info[q].flags |= SRC_HAS_TOK;
        } else if (slot == ACC_TIME) {
            info[q].flags |= SRC_HAS_TIME;
        } else {
            info[q].flags |= SRC_HAS_NNZ;
        }
        if (sg.n_elem == 0) continue;
        if (!sg.d_ptr) return invalid("null segment pointer");
        const uintptr_t p = (uintptr_t)sg.d_ptr;
        if (p % es) return invalid("segment pointer misaligned for its element type");
        bytes += nb + (partial_bits ? 1 : 0);
        const int32_t lay = is_exit ? 0 : q;
        const uint16_t aux = (uint16_t)(E ? E : slot);
        if (run[i] != 0) {  // member of a strided run: whole layers per tile
            if (run[i] > 0) {
                const uint32_t S = (uint32_t)(nb / 16);
                const int32_t per = (int32_t)std::max<uint32_t>(1u, tile_bytes / (S * 16u));
                for (int32_t l0 = 0; l0 < run[i]; l0 += per) {
                    const int32_t k = std::min(per, run[i] - l0);
                    vec.push_back(ProfTile{(const void *)(p + (uintptr_t)l0 * S * 16u), k * S * 16u, lay + l0,
                                           (uint16_t)(op | OP_STRIDED), aux, S});
                }
            }
            continue;
        }
        if (op == OP_TIME) {  // pairs only need 8-byte alignment: tiles of <= 1024 pairs
            for (int64_t o = 0; o < nb; o += 16 * 1024) {
                const int64_t len = std::min<int64_t>(16 * 1024, nb - o);
                sca.push_back(ProfTile{(const void *)(p + o), (uint32_t)len, lay, (uint16_t)OP_TIME, aux, 0});
            }
            continue;
        }
        auto add_scalar = [&](uintptr_t a, int64_t n, uint32_t bits) {
            if (n <= 0) return;
            sca.push_back(ProfTile{(const void *)a, (uint32_t)n, lay, (uint16_t)(op | OP_SCALAR), aux, bits});
        };
        // head up to 16-byte alignment, aligned body in tile_bytes tiles, tail
        int64_t head = (int64_t)((16 - (p & 15)) & 15);
        if (head > nb) head = nb;
        const int64_t body = ((nb - head) / 16) * 16;
        const int64_t tail = nb - head - body;
        add_scalar(p, head, 0);
        for (int64_t o = 0; o < body; o += tile_bytes) {
            const int64_t len = std::min<int64_t>(tile_bytes, body - o);
            vec.push_back(ProfTile{(const void *)(p + head + o), (uint32_t)len, lay, (uint16_t)op, aux, 0});
        }
        add_scalar(p + head + body, tail, 0);
        if (partial_bits) add_scalar(p + nb, 1, (uint32_t)partial_bits);
    }
    if (any_exit)
        for (auto &li : info) li.flags |= SRC_HAS_TOK | SRC_HAS_EXIT;
    auto *pl = new dynmo_plan_s();
    pl->ctx = ctx;
    pl->layer_begin = layer_begin;
    pl->n_local = n_local;
    pl->n_total = n_total;
    pl->exchange = exchange;
    pl->max_E = max_E;
    pl->has_hist = has_hist;
    pl->bytes = bytes;
    std::vector<ProfTile> tiles;
    tiles.reserve(vec.size() + sca.size());
    tiles.insert(tiles.end(), vec.begin(), vec.end());
    tiles.insert(tiles.end(), sca.begin(), sca.end());
    pl->n_tiles = (int64_t)tiles.size();
    // one device block: tiles | info | acc | hist | exit | status,done | slots
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t sz_tiles = up(sizeof(ProfTile) * std::max<size_t>(1, tiles.size()));
    const size_t sz_info = up(sizeof(LayerInfo) * std::max(1, n_local));
    const size_t sz_acc = up(sizeof(unsigned long long) * ACC_N * std::max(1, n_local));
    const size_t sz_hist = up(sizeof(unsigned long long) * (size_t)std::max(1, n_local) * std::max(1, max_E));
    const size_t sz_exit = up(sizeof(unsigned long long) * kExitBins);
    const size_t sz_ws = up(16);
    const size_t sz_warm = up(sizeof(unsigned long long) * (3 + 3 * (size_t)std::max(1, max_E) + kExitBins + 8));
    pl->slot_elems = 3 + 2 * (int64_t)n_total;
    const size_t sz_send = exchange ? up(sizeof(int64_t) * pl->slot_elems) : 0;
    const size_t sz_recv = exchange ? up(sizeof(int64_t) * pl->slot_elems * ctx->nranks) : 0;
    const size_t total = sz_tiles + sz_info + sz_acc + sz_hist + sz_exit + sz_ws + sz_warm + sz_send + sz_recv;
    DeviceGuard g(ctx->device);
    cudaError_t e = cudaMalloc(&pl->dmem, total);
    if (e != cudaSuccess) {
        delete pl;
        g_err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
        return DYNMO_E_NOMEM;
    }
    char *b = (char *)pl->dmem;
    pl->d_tiles = (ProfTile *)b; b += sz_tiles;
    pl->d_info = (LayerInfo *)b; b += sz_info;
    pl->d_acc = (unsigned long long *)b; b += sz_acc;
    pl->d_hist = (unsigned long long *)b; b += sz_hist;
    pl->d_exit = (unsigned long long *)b; b += sz_exit;
    pl->d_ws_status = (int32_t *)b;
    pl->d_ws_done = (unsigned int *)(b + 4); b += sz_ws;
    pl->d_warm = (unsigned long long *)b; b += sz_warm;
    if (exchange) {
        pl->d_slot_send = (int64_t *)b; b += sz_send;
        pl->d_slot_recv = (int64_t *)b;
    }
    bool ok = cudaMemset(pl->dmem, 0, total) == cudaSuccess;
    if (ok && !tiles.empty())
        ok = cudaMemcpy(pl->d_tiles, tiles.data(), sizeof(ProfTile) * tiles.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok && n_local > 0)
        ok = cudaMemcpy(pl->d_info, info.data(), sizeof(LayerInfo) * n_local, cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) {
        e = cudaGetLastError();
        cudaFree(pl->dmem);
        delete pl;
        return cuda_fail(e, "plan upload");
    }
    const int warps_per_block = kProfThreads / 32;
    const int64_t want = (pl->n_tiles + warps_per_block - 1) / warps_per_block;
    int max_words = 0;
    for (const LayerInfo &li : info) max_words = std::max(max_words, expert_words(li.E));
    pl->warp_words = profile_warp_words(any_exit, max_words);
    pl->ops = 0;
    for (const ProfTile &t : tiles) {
        const int k = t.op & 0xF;
        pl->ops |= (k <= OP_NZ32 || k == OP_TIME) ? 1 : k == OP_EXIT ? 2 : 4;
        if ((k == OP_EXP64 || k == OP_EXP32) && t.aux > 16) pl->ops |= 8;  // smem expert histograms
    }
    if (!pl->ops) pl->ops = 1;
    const int64_t cap_blocks = (int64_t)ctx->num_sms * profile_blocks_per_sm(pl->ops, pl->warp_words);
    pl->grid = (int)std::max<int64_t>(1, std::min(want, cap_blocks));
    *out = pl;
    return DYNMO_OK;
}

// All ranks agree on a setup step: every rank contributes its status and
// every rank gets the worst one (a failure on any rank fails the call on
// every rank, so no rank is left waiting in a later collective).
static dynmo_status agree(dynmo_ctx ctx, dynmo_status mine, const char *what) {
    if (ctx->nranks < 2) return mine;
    const int32_t v = (int32_t)mine;
    std::vector<char> all;
    const dynmo_status st = allgather_bytes(ctx, &v, sizeof(v), all);
    if (st) return st;
    int32_t worst = DYNMO_OK;
    for (int r = 0; r < ctx->nranks; ++r) {
        int32_t x;
        memcpy(&x, all.data() + r * sizeof(x), sizeof(x));
        if (x < worst) worst = x;
    }
    if (mine == DYNMO_OK && worst != DYNMO_OK) g_err = std::string(what) + " failed on another rank";
    return mine != DYNMO_OK ? mine : (dynmo_status)worst;
}

dynmo_status dynmo_profile_plan_create(dynmo_ctx ctx, const dynmo_segment *h_segs, int32_t n_segs,
                                       int32_t layer_begin, int32_t n_local, int32_t n_total,
                                       int32_t exchange, dynmo_plan *out) {
    if (!out) return invalid("null plan out");
    *out = nullptr;
    if (!ctx) return invalid("null ctx");
    dynmo_plan pl = nullptr;
    dynmo_status st = profile_plan_local(ctx, h_segs, n_segs, layer_begin, n_local, n_total, exchange, &pl);
    if (exchange == 2 && !st && ctx->nranks == 1) st = ensure_comm(ctx);
    if (exchange != 1) {
        if (st && pl) dynmo_profile_plan_destroy(pl);
        if (!st) *out = pl;
        return st;
    }
    // exchange == 1 is collective: the receive slot area of every rank,
    // mapped by every peer.  Every rank takes part in both agreement steps
    // even after a local failure.
    DeviceGuard g(ctx->device);
    const size_t bytes = pl ? sizeof(int64_t) * 2 * ctx->nranks * pl->slot_elems * 2 : 0;  // LL: 2 words per value
    if (!st && (cudaMalloc((void **)&pl->d_p2p_slots, bytes) != cudaSuccess ||
                cudaMemset(pl->d_p2p_slots, 0, bytes) != cudaSuccess))
        st = cuda_fail(cudaGetLastError(), "p2p slots");
    if (ctx->nranks == 1) {  // the slot area of the only rank is local
        if (!st) pl->peer_slots.assign(1, pl->d_p2p_slots);
    } else {
        struct {
            int32_t st;
            cudaIpcMemHandle_t h;
        } mine{}, other{};
        if (!st && cudaIpcGetMemHandle(&mine.h, pl->d_p2p_slots) != cudaSuccess)
            st = cuda_fail(cudaGetLastError(), "cudaIpcGetMemHandle (slots)");
        mine.st = st;
        std::vector<char> all;
        const dynmo_status ag = allgather_bytes(ctx, &mine, sizeof(mine), all);
        if (!st) st = ag;
        for (int r = 0; !st && r < ctx->nranks; ++r) {
            memcpy(&other, all.data() + r * sizeof(other), sizeof(other));
            if (other.st) st = invalid("profile plan creation failed on another rank");
        }
        if (!st) pl->peer_slots.assign(ctx->nranks, nullptr);
        for (int r = 0; !st && r < ctx->nranks; ++r) {
            if (r == ctx->rank) {
                pl->peer_slots[r] = pl->d_p2p_slots;
                continue;
            }
            memcpy(&other, all.data() + r * sizeof(other), sizeof(other));
            void *mp = nullptr;
            if (cudaIpcOpenMemHandle(&mp, other.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
                st = cuda_fail(cudaGetLastError(), "cudaIpcOpenMemHandle (slots)");
            pl->peer_slots[r] = (int64_t *)mp;
        }
        if (ag == DYNMO_OK) st = agree(ctx, st, "profile plan (peer mapping)");
    }
    if (st) {
        if (pl) dynmo_profile_plan_destroy(pl);
        return st;
    }
    *out = pl;
    return DYNMO_OK;
}

void dynmo_profile_plan_destroy(dynmo_plan plan) {
    if (!plan) return;
    DeviceGuard g(plan->ctx->device);
    for (int r = 0; r < (int)plan->peer_slots.size(); ++r)
        if (r != plan->ctx->rank && plan->peer_slots[r]) cudaIpcCloseMemHandle(plan->peer_slots[r]);
    if (plan->d_p2p_slots) cudaFree(plan->d_p2p_slots);
    cudaFree(plan->dmem);
    delete plan;
}

int64_t dynmo_plan_num_tiles(dynmo_plan plan) { return plan ? plan->n_tiles : -1; }
int64_t dynmo_plan_bytes(dynmo_plan plan) { return plan ? plan->bytes : -1; }
int32_t dynmo_plan_max_experts(dynmo_plan plan) { return plan ? plan->max_E : -1; }

// ------------------------------------------------ global pruning (NEXT-2)
struct dynmo_pplan_s {
    dynmo_ctx ctx = nullptr;
    void *dmem = nullptr;
    PruneArgs args{};
    int grid[40] = {};  // per launch kind: persistent grid (SMs x resident blocks), capped by the tiles
};

dynmo_status dynmo_prune_plan_create(dynmo_ctx ctx, const dynmo_prune_segment *h_segs, int32_t n_segs,
                                     dynmo_pplan *out) {
    if (!out) return invalid("null plan out");
    *out = nullptr;
    if (!ctx) return invalid("null ctx");
    std::vector<PruneTile> tiles;
    bool any_f32 = false;
    const char *bad = nullptr;  // validated before the collective: every rank takes part in it
    if (n_segs < 0 || (n_segs > 0 && !h_segs)) bad = "bad segment list";
    for (int32_t i = 0; !bad && i < n_segs; ++i) {
        const dynmo_prune_segment &sg = h_segs[i];
        if (sg.n < 0) { bad = "negative segment length"; break; }
        if (sg.dtype != DYNMO_W_F32 && sg.dtype != DYNMO_W_BF16) { bad = "unknown weight dtype"; break; }
        if (sg.n == 0) continue;
        if (!sg.d_w || !sg.d_mask) { bad = "null segment pointer"; break; }
        if ((uintptr_t)sg.d_w % 16) { bad = "weights must be 16-byte aligned"; break; }
        any_f32 |= sg.dtype == DYNMO_W_F32;
        const int64_t esz = sg.dtype == DYNMO_W_F32 ? 4 : 2;
        for (int64_t o = 0; o < sg.n; o += kPruneTileElems) {
            const int64_t len = std::min<int64_t>(kPruneTileElems, sg.n - o);
            tiles.push_back(PruneTile{(const char *)sg.d_w + o * esz, sg.d_mask + o, (uint32_t)len, sg.dtype});
        }
    }
    // every rank must run the same passes (one NCCL all-reduce per pass): an
    // f32 segment on any rank adds passes 1 and 2 everywhere; an invalid
    // argument on any rank fails the call on every rank
    bool global_f32 = any_f32;
    if (ctx->nranks > 1) {
        const char mine = (char)((any_f32 ? 1 : 0) | (bad ? 2 : 0));
        std::vector<char> all;
        const dynmo_status st = allgather_bytes(ctx, &mine, 1, all);
        if (st != DYNMO_OK) return st;
        bool any_bad = false;
        for (char c : all) {
            global_f32 |= (c & 1) != 0;
            any_bad |= (c & 2) != 0;
        }
        if (any_bad && !bad) bad = "invalid segments on another rank";
    }
    if (bad) return invalid(bad);
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t nt = std::max<size_t>(1, tiles.size());
    const size_t sz_tiles = up(sizeof(PruneTile) * nt), sz_hist = up(sizeof(unsigned long long) * 32770);
    const size_t sz_sel = up(sizeof(PruneSel)), sz_tie = up(sizeof(long long) * std::max(1, ctx->nranks));
    // tie counts / offsets per (tile, warp range of the mask pass)
    const size_t sz_tt = up(sizeof(uint32_t) * nt * 8), sz_to = up(sizeof(unsigned long long) * nt * 8);
    // per-(tile, warp range) window-bin counts (bf16-only plans: ties on the first digit)
    const size_t sz_tw = any_f32 ? 0 : up(sizeof(uint16_t) * nt * 8 * kWinCnt);
    const size_t sz_tot = up(sizeof(uint32_t) * nt);
    const size_t sz_cw = up(sizeof(unsigned long long) * kPruneCw);
    const size_t total = sz_tiles + 2 * sz_hist + sz_sel + sz_tie + sz_tt + sz_to + sz_tw + sz_tot + 2 * sz_cw;
    DeviceGuard g(ctx->device);
    auto *pl = new dynmo_pplan_s();
    pl->ctx = ctx;
    cudaError_t e = cudaMalloc(&pl->dmem, total);
    if (e != cudaSuccess) {
        delete pl;
        g_err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
        return DYNMO_E_NOMEM;
    }
    char *b = (char *)pl->dmem;
    PruneArgs &a = pl->args;
    a.tiles = (const PruneTile *)b; b += sz_tiles;
    a.hist_local = (unsigned long long *)b; b += sz_hist;
    a.hist_global = (unsigned long long *)b; b += sz_hist;
    a.sel = (PruneSel *)b; b += sz_sel;
    a.tie_all = (const long long *)b; b += sz_tie;
    a.tile_ties = (uint32_t *)b; b += sz_tt;
    a.tile_off = (unsigned long long *)b; b += sz_to;
    a.tile_win = sz_tw ? (uint16_t *)b : nullptr;
    b += sz_tw;
    a.tile_tot = (uint32_t *)b; b += sz_tot;
    a.cw_local = (unsigned long long *)b; b += sz_cw;
    a.cw_global = (unsigned long long *)b;
    a.n_tiles = (int64_t)tiles.size();
    for (const PruneTile &t : tiles) a.n_elems += t.n;
    a.rank = ctx->rank;
    a.nranks = ctx->nranks;
    a.last_pass = global_f32 ? 2 : 0;  // bf16 keys have 16 zero low bits: the 15-bit first digit is exact
    bool ok = cudaMemset(pl->dmem, 0, total) == cudaSuccess;
    if (ok && !tiles.empty())
        ok = cudaMemcpy((void *)a.tiles, tiles.data(), sizeof(PruneTile) * tiles.size(), cudaMemcpyHostToDevice) ==
             cudaSuccess;
    if (!ok) {
        e = cudaGetLastError();
        cudaFree(pl->dmem);
        delete pl;
        return cuda_fail(e, "prune plan upload");
    }
    // persistent grids: every SM filled to its occupancy for each streaming kernel
    for (int kind : {0, 1, 2, 21, 23, 32})
        pl->grid[kind] = (int)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)ctx->num_sms * prune_blocks_per_sm(kind), a.n_tiles));
    pl->grid[30] = (int)std::max<int64_t>(  // the sample pass: every kPruneSampleStride-th tile
        1, std::min<int64_t>((int64_t)ctx->num_sms * prune_blocks_per_sm(30),
                             (a.n_tiles + kPruneSampleStride - 1) / kPruneSampleStride));
    *out = pl;
    return DYNMO_OK;
}

void dynmo_prune_plan_destroy(dynmo_pplan plan) {
    if (!plan) return;
    DeviceGuard g(plan->ctx->device);
    cudaFree(plan->dmem);
    delete plan;
}

dynmo_status dynmo_global_prune(dynmo_ctx ctx, dynmo_pplan plan, int64_t k, int64_t *d_info,
                                int32_t *d_status, dynmo_stream stream) {
    if (!ctx || !plan || plan->ctx != ctx) return invalid("bad ctx/plan");
    if (k < 0) return invalid("k < 0");
    const cudaStream_t s = (cudaStream_t)stream;
    DeviceGuard g(ctx->device);
    const PruneArgs &a = plan->args;
    const bool multi = ctx->nranks > 1;
    CUDA_TRY(launch_prune_begin(a.sel, (long long)k, s), "k_prune_begin");
    auto all_reduce = [&](int count, bool compact = false) -> dynmo_status {
        if (!multi) return DYNMO_OK;
        const ncclResult_t r = compact ? ncclAllReduce(a.cw_local, a.cw_global, count, ncclUint64, ncclSum, ctx->comm, s)
                                       : ncclAllReduce(a.hist_local, a.hist_global, count, ncclUint64, ncclSum, ctx->comm, s);
        if (r != ncclSuccess) {
            g_err = std::string("ncclAllReduce (prune): ") + ncclGetErrorString(r);
            return DYNMO_E_NCCL;
        }
        return DYNMO_OK;
    };
    dynmo_status st;
    // pass 0: sample histogram -> bin window -> windowed full pass -> select;
    // on a miss (the k-th key outside the window) the full histogram and a
    // second select run (both launched unconditionally: graph-capturable;
    // they return at once without a miss)
    CUDA_TRY(launch_prune(a, 30, plan->grid[30], s), "k_prune_hist0 (sample)");
    if ((st = all_reduce(32770)) != DYNMO_OK) return st;
    CUDA_TRY(launch_prune(a, 31, 1, s), "k_prune_window");
    CUDA_TRY(launch_prune(a, 0, plan->grid[0], s), "k_prune_hist0w");
    if ((st = all_reduce(kPruneCw, true)) != DYNMO_OK) return st;  // the compact window histogram
    CUDA_TRY(launch_prune(a, 10, 1, s), "k_prune_select_win");
    CUDA_TRY(launch_prune(a, 32, plan->grid[32], s), "k_prune_hist0 (on a miss)");
    if ((st = all_reduce(32769)) != DYNMO_OK) return st;
    CUDA_TRY(launch_prune(a, 13, 1, s), "k_prune_select (on a miss)");
    for (int pass = 1; pass <= a.last_pass; ++pass) {
        CUDA_TRY(launch_prune(a, pass, plan->grid[pass], s), "k_prune_hist");
        if ((st = all_reduce(32769)) != DYNMO_OK) return st;
        CUDA_TRY(launch_prune(a, 10 + pass, 1, s), "k_prune_select");
    }
    if (multi) {
        const ncclResult_t r = ncclAllGather(&a.sel->tie_local, (void *)a.tie_all, 1, ncclInt64, ctx->comm, s);
        if (r != ncclSuccess) {
            g_err = std::string("ncclAllGather (prune): ") + ncclGetErrorString(r);
            return DYNMO_E_NCCL;
        }
    }
    CUDA_TRY(launch_prune(a, 20, 1, s), "k_prune_ties");
    CUDA_TRY(launch_prune(a, 21, plan->grid[21], s), "k_prune_tiecount");
    CUDA_TRY(launch_prune(a, 22, 1, s), "k_prune_tiescan");
    CUDA_TRY(launch_prune(a, 23, plan->grid[23], s), "k_prune_mask");
    CUDA_TRY(launch_prune_info(a, (long long *)d_info, d_status, s), "k_prune_info");
    return DYNMO_OK;
}

// ----------------------------------------------------------- call 1 profile
dynmo_status dynmo_profile_layers(dynmo_ctx ctx, dynmo_plan plan, const uint8_t *d_frozen,
                                  const dynmo_cost_coef *d_coef, const int64_t *d_mem_local,
                                  int64_t *d_counters, int64_t *d_hist, int64_t *d_cost,
                                  int64_t *d_mem, int32_t *d_status, dynmo_stream stream) {
    if (!ctx || !plan || plan->ctx != ctx) return invalid("bad ctx/plan");
    if ((plan->n_local > 0 && !d_coef) || !d_cost || !d_status) return invalid("null required output");
    cudaStream_t s = (cudaStream_t)stream;
    DeviceGuard g(ctx->device);
    static const int64_t l2_max = [] {  // DYNMO_L2_PREFETCH_MAX=<bytes> (0: off), A/B knob
        const char *e = getenv("DYNMO_L2_PREFETCH_MAX");
        return e ? (int64_t)atoll(e) : kL2PrefetchMaxBytes;
    }();
    ProfArgs pa{plan->d_tiles, plan->n_tiles, plan->d_acc, plan->d_hist, plan->d_exit,
                std::max(1, plan->max_E), plan->d_ws_status, plan->warp_words, plan->n_local,
                plan->bytes <= l2_max ? 1 : 0, nullptr};
    // profile-phase timing also measures the kernel's own span on the device
    unsigned long long *span = (ctx->timing & (1 << DYNMO_PHASE_PROFILE)) ? ctx->d_win->prof_span : nullptr;
    pa.span = span;
    cudaEvent_t te = phase_begin(ctx, DYNMO_PHASE_PROFILE, s);
    CUDA_TRY(launch_profile(pa, plan->ops, plan->grid, s), "k_profile launch");
    phase_end(te, s);
    EpiArgs ea{};
    ea.span = span;
    ea.layer_begin = plan->layer_begin;
    ea.n_local = plan->n_local;
    ea.n_total = plan->n_total;
    ea.exchange = plan->exchange;
    ea.max_E = std::max(1, plan->max_E);
    ea.info = plan->d_info;
    ea.acc = plan->d_acc;
    ea.hist = plan->d_hist;
    ea.exit_hist = plan->d_exit;
    ea.frozen = d_frozen;
    ea.coef = d_coef;
    ea.mem_local = d_mem_local;
    ea.counters_out = d_counters;
    ea.hist_out = plan->max_E > 0 ? d_hist : nullptr;
    ea.cost_out = d_cost;
    ea.mem_out = d_mem;
    ea.slot_send = plan->d_slot_send;
    ea.ws_status = plan->d_ws_status;
    ea.ws_done = plan->d_ws_done;
    ea.status_out = d_status;
    static const bool epi_warm = [] {  // DYNMO_EPI_WARM=0: no code warm-up pass (A/B knob)
        const char *e = getenv("DYNMO_EPI_WARM");
        return !(e && e[0] == '0');
    }();
    ea.warm = epi_warm ? plan->d_warm : nullptr;
    static const bool fuse_exch = [] {  // DYNMO_EXCH_FUSED=0: separate k_unpack_p2p (A/B knob)
        const char *e = getenv("DYNMO_EXCH_FUSED");
        return !(e && e[0] == '0');
    }();
    if (plan->exchange == 1) {
        ea.p2p = 1;
        ea.rank = ctx->rank;
        ea.nranks = ctx->nranks;
        ea.win = ctx->d_win;
        for (int r = 0; r < ctx->nranks; ++r) {
            ea.peer_slots[r] = plan->peer_slots[r];
            ea.peer_win[r] = ctx->peer_win[r];
        }
        ea.fuse_unpack = fuse_exch;
        ea.p2p_slots = plan->d_p2p_slots;
        ea.decoded = plan->d_slot_recv;
        ea.x_cost = d_cost;
        ea.x_mem = d_mem;
        ea.x_status = d_status;
    }
    te = phase_begin(ctx, DYNMO_PHASE_EPILOGUE, s);
    CUDA_TRY(launch_epilogue(ea, s), "k_epilogue launch");
    phase_end(te, s);
    if (plan->exchange == 1 && !fuse_exch) {
        te = phase_begin(ctx, DYNMO_PHASE_EXCHANGE, s);
        CUDA_TRY(launch_unpack_p2p(plan->d_p2p_slots, ctx->d_win, ctx->nranks, plan->n_total, plan->d_slot_recv, d_cost, d_mem,
                                   d_status, s),
                 "k_unpack_p2p launch");
        phase_end(te, s);
    } else if (plan->exchange == 2) {
        te = phase_begin(ctx, DYNMO_PHASE_EXCHANGE, s);
        ncclResult_t r = ncclAllGather(plan->d_slot_send, plan->d_slot_recv, (size_t)plan->slot_elems,
                                       ncclInt64, ctx->comm, s);
        if (r != ncclSuccess) {
            g_err = std::string("ncclAllGather: ") + ncclGetErrorString(r);
            return DYNMO_E_NCCL;
        }
        CUDA_TRY(launch_unpack(plan->d_slot_recv, ctx->nranks, plan->n_total, d_cost, d_mem, d_status, s),
                 "k_unpack launch");
        phase_end(te, s);
    }
    return DYNMO_OK;
}

// ----------------------------------------------------------- calls 2 - 4
static dynmo_status check_solve(dynmo_ctx ctx, int32_t n_inst, int32_t max_layers, const void *cost,
                                const void *layer_off, const void *n_stages, const void *bnd_off,
                                const void *bnd_out, const void *status) {
    if (!ctx) return invalid("null ctx");
    if (n_inst < 1) return invalid("n_inst < 1");
    if (max_layers < 1 || max_layers > DYNMO_MAX_LAYERS) return invalid("max_layers outside [1, 1023]");
    if (!cost || !layer_off || !n_stages || !bnd_off || !bnd_out || !status)
        return invalid("null required pointer");
    return DYNMO_OK;
}

dynmo_status dynmo_timestamp(dynmo_ctx ctx, int64_t *d_slot, dynmo_stream stream) {
    if (!ctx || !d_slot) return invalid("null ctx/slot");
    DeviceGuard g(ctx->device);
    CUDA_TRY(launch_stamp(d_slot, (cudaStream_t)stream), "k_stamp launch");
    return DYNMO_OK;
}

constexpr int64_t kPublishKernelMax = 4096;  // larger results: the copy engine

// Diagnostic build only (-DDYNMO_STEP_STAMPS; not in dynmo.h): per step
// kernel [first warp start, last warp end] in %globaltimer ns, 2 x STAMP_N
// pairs (k_profile.cu's table, then k_solve.cu's); reset re-arms them.
int dynmo_diag_step_stamps(unsigned long long *h_out, int reset) {
#ifdef DYNMO_STEP_STAMPS
    diag_stamps_profile(h_out, reset != 0);
    diag_stamps_solve(h_out + 2 * STAMP_N, reset != 0);
    return STAMP_N;
#else
    (void)h_out;
    (void)reset;
    return 0;
#endif
}

dynmo_status dynmo_publish(dynmo_ctx ctx, const void *d_src, void *h_dst, int64_t bytes, dynmo_stream stream) {
    if (!ctx || !d_src || !h_dst) return invalid("null ctx/src/dst");
    if (bytes < 0) return invalid("bytes < 0");
    if (bytes == 0) return DYNMO_OK;
    DeviceGuard g(ctx->device);
    // h_dst: page-locked host memory mapped into the device address space
    // (cudaHostAlloc / cudaMallocHost / torch pin_memory under UVA); both
    // ends of the range must be, or nothing is enqueued
    void *d_dst = nullptr;
    for (int end = 0; end < 2; ++end) {
        cudaPointerAttributes at{};
        const char *q = (const char *)h_dst + (end ? bytes - 1 : 0);
        if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
            cudaGetLastError();
            return invalid("h_dst is not CUDA-registered host memory");
        }
        if (at.type != cudaMemoryTypeHost || !at.devicePointer)
            return invalid("h_dst is not page-locked, device-mapped host memory");
        if (!end) d_dst = at.devicePointer;
    }
    cudaPointerAttributes sa{};
    if (cudaPointerGetAttributes(&sa, d_src) != cudaSuccess || sa.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        return invalid("d_src is not device memory");
    }
    // GPU stores to host memory run at a few GB/s (tools/publish_bench.py:
    // 49 KB 15.4 us vs 11.4 us by the copy engine); the kernel wins only
    // for small results, where it saves the copy node's fixed latency
    if (bytes > kPublishKernelMax) {
        CUDA_TRY(cudaMemcpyAsync(h_dst, d_src, (size_t)bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream),
                 "publish copy");
        return DYNMO_OK;
    }
    CUDA_TRY(launch_publish(d_src, d_dst, bytes, (cudaStream_t)stream), "k_publish launch");
    return DYNMO_OK;
}

dynmo_status dynmo_map_stages(dynmo_ctx ctx, int32_t n_layers, int32_t n_old, const int32_t *d_bnd_old,
                              const int32_t *d_rank_old, int32_t n_new, const int32_t *d_bnd_new,
                              const int64_t *d_bytes, int32_t G, uint32_t allowed, const int32_t *d_slot_rank,
                              int32_t *d_rank_new, int64_t *d_kept, int32_t *d_status, dynmo_stream stream) {
    if (!ctx) return invalid("null ctx");
    if (n_layers < 1 || n_layers > 1023 || n_old < 1 || n_old > n_layers || n_new < 1 || n_new > n_layers)
        return invalid("n_layers in [1, 1023], stage counts in [1, n_layers]");
    if (G < 1 || G > kMaxMapRanks) return invalid("G outside [1, 16]");
    if (!d_bnd_old || !d_rank_old || !d_bnd_new || !d_bytes || !d_rank_new || !d_kept || !d_status)
        return invalid("null pointer");
    DeviceGuard g(ctx->device);
    MapArgs a{n_layers, n_old, n_new, G, allowed, d_bnd_old, d_rank_old, d_bnd_new, d_bytes,
              d_rank_new, d_kept, d_status, ctx->d_map_work, d_slot_rank};
    CUDA_TRY(launch_map_stages(a, (cudaStream_t)stream), "k_map_stages launch");
    return DYNMO_OK;
}

dynmo_status dynmo_partition_stages(dynmo_ctx ctx, int32_t n_inst, int32_t max_layers,
                                    const int64_t *d_cost, const int64_t *d_mem,
                                    const int32_t *d_layer_off, const int32_t *d_n_stages,
                                    const int64_t *d_cap, const int32_t *d_bnd_off, int32_t *d_bnd,
                                    int64_t *d_bottleneck, double *d_imbalance, int32_t *d_status,
                                    dynmo_stream stream) {
    dynmo_status st = check_solve(ctx, n_inst, max_layers, d_cost, d_layer_off, d_n_stages, d_bnd_off,
                                  d_bnd, d_status);
    if (st) return st;
    if (!d_bottleneck) return invalid("null bottleneck");
    if (d_mem && !d_cap) return invalid("mem without cap");
    SolveArgs a{};
    a.n_inst = n_inst;
    a.max_layers = max_layers;
    a.cost = d_cost;
    a.mem = d_mem;
    a.layer_off = d_layer_off;
    a.n_stages = d_n_stages;
    a.cap = d_cap;
    a.bnd_off = d_bnd_off;
    a.bnd_out = d_bnd;
    a.bottleneck = d_bottleneck;
    a.imbalance = d_imbalance;
    a.status = d_status;
    DeviceGuard g(ctx->device);
    cudaEvent_t te = phase_begin(ctx, DYNMO_PHASE_PARTITION, (cudaStream_t)stream);
    CUDA_TRY(launch_partition(a, (cudaStream_t)stream), "k_partition launch");
    phase_end(te, (cudaStream_t)stream);
    return DYNMO_OK;
}

dynmo_status dynmo_diffuse_balance(dynmo_ctx ctx, int32_t n_inst, int32_t max_layers,
                                   const int64_t *d_cost, const int64_t *d_mem,
                                   const int32_t *d_layer_off, const int32_t *d_n_stages,
                                   const int64_t *d_cap, const int32_t *d_bnd_off,
                                   const int32_t *d_bnd_in, const int64_t *d_gamma,
                                   const double *d_gamma_fluid, int32_t max_rounds,
                                   int32_t *d_bnd_out, int32_t *d_rounds, int64_t *d_phi,
                                   int64_t *d_phi0, double *d_fluid_x, int32_t *d_fluid_rounds,
                                   double *d_fluid_phi, int32_t *d_fluid_status, int32_t *d_status,
                                   dynmo_stream stream) {
    dynmo_status st = check_solve(ctx, n_inst, max_layers, d_cost, d_layer_off, d_n_stages, d_bnd_off,
                                  d_bnd_out, d_status);
    if (st) return st;
    if (!d_bnd_in) return invalid("null bnd_in");
    if (d_mem && !d_cap) return invalid("mem without cap");
    SolveArgs a{};
    a.n_inst = n_inst;
    a.max_layers = max_layers;
    a.cost = d_cost;
    a.mem = d_mem;
    a.layer_off = d_layer_off;
    a.n_stages = d_n_stages;
    a.cap = d_cap;
    a.bnd_off = d_bnd_off;
    a.bnd_in = d_bnd_in;
    a.bnd_out = d_bnd_out;
    a.status = d_status;
    a.gamma = d_gamma;
    a.gamma_fluid = d_gamma_fluid;
    a.max_rounds = max_rounds;
    a.rounds = d_rounds;
    a.phi = d_phi;
    a.phi0 = d_phi0;
    a.fluid_x = d_fluid_x;
    static const int spec = [] {  // DYNMO_FLUID_SPEC: 0 per-round chain, 1 speculative, 2 (default) + overlap for n <= 8
        const char *e = getenv("DYNMO_FLUID_SPEC");
        return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : 2;
    }();
    a.fluid_spec = spec;
    a.fluid_rounds = d_fluid_rounds;
    a.fluid_phi = d_fluid_phi;
    a.fluid_status = d_fluid_status;
    DeviceGuard g(ctx->device);
    cudaEvent_t te = phase_begin(ctx, DYNMO_PHASE_DIFFUSE, (cudaStream_t)stream);
    CUDA_TRY(launch_diffuse(a, (cudaStream_t)stream), "k_diffuse launch");
    phase_end(te, (cudaStream_t)stream);
    return DYNMO_OK;
}

dynmo_status dynmo_repack_workers(dynmo_ctx ctx, int32_t n_inst, int32_t max_layers,
                                  const int64_t *d_cost, const int64_t *d_mem,
                                  const int32_t *d_layer_off, const int32_t *d_n_cur,
                                  const int64_t *d_cap, const int32_t *d_bnd_off,
                                  const int32_t *d_bnd_in, const int64_t *d_bound,
                                  const int32_t *d_floor, int32_t mode, int32_t *d_n_new,
                                  int32_t *d_bnd, int64_t *d_bottleneck, int32_t *d_status,
                                  dynmo_stream stream) {
    dynmo_status st = check_solve(ctx, n_inst, max_layers, d_cost, d_layer_off, d_n_cur, d_bnd_off,
                                  d_bnd, d_status);
    if (st) return st;
    if (mode != DYNMO_REPACK_BOUND && mode != DYNMO_REPACK_ALG2) return invalid("bad repack mode");
    if (!d_floor || !d_n_new || !d_bottleneck) return invalid("null repack pointer");
    if (mode == DYNMO_REPACK_BOUND && !d_bound) return invalid("BOUND mode needs d_bound");
    if (mode == DYNMO_REPACK_ALG2 && !d_bnd_in) return invalid("ALG2 mode needs d_bnd_in");
    if (d_mem && !d_cap) return invalid("mem without cap");
    SolveArgs a{};
    a.n_inst = n_inst;
    a.max_layers = max_layers;
    a.cost = d_cost;
    a.mem = d_mem;
    a.layer_off = d_layer_off;
    a.n_stages = d_n_cur;
    a.cap = d_cap;
    a.bnd_off = d_bnd_off;
    a.bnd_in = d_bnd_in;
    a.bnd_out = d_bnd;
    a.bottleneck = d_bottleneck;
    a.status = d_status;
    a.bound = d_bound;
    a.floor_ = d_floor;
    a.mode = mode;
    a.n_new = d_n_new;
    DeviceGuard g(ctx->device);
    cudaEvent_t te = phase_begin(ctx, DYNMO_PHASE_REPACK, (cudaStream_t)stream);
    CUDA_TRY(launch_repack(a, (cudaStream_t)stream), "k_repack launch");
    phase_end(te, (cudaStream_t)stream);
    return DYNMO_OK;
}

// ------------------------------------------------------------ call 5 migrate
static bool valid_split(int32_t L, int32_t n, const int32_t *b) {
    if (n < 1 || !b || b[0] != 0 || b[n] != L) return false;
    for (int32_t s = 0; s < n; ++s)
        if (b[s + 1] <= b[s]) return false;
    return true;
}

int32_t dynmo_migration_plan(int32_t n_layers, int32_t n_old, const int32_t *h_bnd_old,
                             const int32_t *h_rank_old, int32_t n_new, const int32_t *h_bnd_new,
                             const int32_t *h_rank_new, int32_t *h_moves) {
    if (n_layers < 1 || !h_rank_old || !h_rank_new || !h_moves) return DYNMO_E_INVALID;
    if (!valid_split(n_layers, n_old, h_bnd_old) || !valid_split(n_layers, n_new, h_bnd_new))
        return DYNMO_E_INVALID;
    // merge walk over the two boundary vectors
    int32_t so = 0, sn = 0, m = 0;
    for (int32_t i = 0; i < n_layers; ++i) {
        while (i >= h_bnd_old[so + 1]) ++so;
        while (i >= h_bnd_new[sn + 1]) ++sn;
        const int32_t src = h_rank_old[so], dst = h_rank_new[sn];
        if (src != dst) {
            h_moves[3 * m + 0] = i;
            h_moves[3 * m + 1] = src;
            h_moves[3 * m + 2] = dst;
            ++m;
        }
    }
    return m;
}

dynmo_status dynmo_migrate_layers(dynmo_ctx ctx, int32_t n_layers, int32_t n_old,
                                  const int32_t *h_bnd_old, const int32_t *h_rank_old, int32_t n_new,
                                  const int32_t *h_bnd_new, const int32_t *h_rank_new,
                                  const dynmo_buf *h_send, const dynmo_buf *h_recv, int32_t n_bufs,
                                  int64_t *h_bytes_sent, int64_t *h_bytes_recv, dynmo_stream stream) {
    if (!ctx) return invalid("null ctx");
    if (n_bufs < 0 || (n_bufs > 0 && (!h_send || !h_recv))) return invalid("bad buffer tables");
    for (int32_t s = 0; s < n_old; ++s)
        if (!h_rank_old || h_rank_old[s] < 0 || h_rank_old[s] >= ctx->nranks) return invalid("bad old rank");
    for (int32_t s = 0; s < n_new; ++s)
        if (!h_rank_new || h_rank_new[s] < 0 || h_rank_new[s] >= ctx->nranks) return invalid("bad new rank");
    std::vector<int32_t> moves(3 * (size_t)std::max(1, n_layers));
    const int32_t m = dynmo_migration_plan(n_layers, n_old, h_bnd_old, h_rank_old, n_new, h_bnd_new,
                                           h_rank_new, moves.data());
    if (m < 0) return invalid("malformed boundary vector");
    const int me = ctx->rank;
    int64_t sent = 0, recvd = 0;
    // validate every buffer this rank needs before touching NCCL
    for (int32_t k = 0; k < m; ++k) {
        const int32_t i = moves[3 * k], src = moves[3 * k + 1], dst = moves[3 * k + 2];
        for (int32_t u = 0; u < n_bufs; ++u) {
            if (src == me) {
                const dynmo_buf &b = h_send[(int64_t)i * n_bufs + u];
                if (b.bytes < 0 || (b.bytes > 0 && !b.d_ptr)) return invalid("missing send buffer");
                sent += b.bytes;
            }
            if (dst == me) {
                const dynmo_buf &b = h_recv[(int64_t)i * n_bufs + u];
                if (b.bytes < 0 || (b.bytes > 0 && !b.d_ptr)) return invalid("missing recv buffer");
                recvd += b.bytes;
            }
        }
    }
    if (h_bytes_sent) *h_bytes_sent = sent;
    if (h_bytes_recv) *h_bytes_recv = recvd;
    if (m == 0 || (sent == 0 && recvd == 0)) return DYNMO_OK;
    if (ctx->nranks < 2 || !ctx->comm) return invalid("cross-rank move without a communicator");
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t te = phase_begin(ctx, DYNMO_PHASE_MIGRATE, s);
    ncclResult_t r = ncclGroupStart();
    for (int32_t k = 0; k < m && r == ncclSuccess; ++k) {
        const int32_t i = moves[3 * k], src = moves[3 * k + 1], dst = moves[3 * k + 2];
        for (int32_t u = 0; u < n_bufs && r == ncclSuccess; ++u) {
            if (src == me) {
                const dynmo_buf &b = h_send[(int64_t)i * n_bufs + u];
                if (b.bytes > 0) r = ncclSend(b.d_ptr, (size_t)b.bytes, ncclUint8, dst, ctx->comm, s);
            }
            if (dst == me && r == ncclSuccess) {
                const dynmo_buf &b = h_recv[(int64_t)i * n_bufs + u];
                if (b.bytes > 0) r = ncclRecv(b.d_ptr, (size_t)b.bytes, ncclUint8, src, ctx->comm, s);
            }
        }
    }
    ncclResult_t r2 = ncclGroupEnd();
    phase_end(te, s);
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) {
        g_err = std::string("NCCL send/recv: ") + ncclGetErrorString(r);
        return DYNMO_E_NCCL;
    }
    return DYNMO_OK;
}


// ---------------------------------------------- call 5, peer-memory variant
struct dynmo_mplan_s {
    dynmo_ctx ctx = nullptr;
    int32_t n_layers = 0, n_bufs = 0;
    std::vector<dynmo_buf> recv;                        // [n_layers * n_bufs] (this rank)
    std::map<std::pair<int, int64_t>, dynmo_buf> src;   // (rank, layer*n_bufs+k) -> readable ptr
    std::vector<void *> opened;                         // IPC mappings to close
    DevBuf *d_src_tab = nullptr;                        // [nranks][n_layers*n_bufs] (device path)
    DevBuf *d_recv_tab = nullptr;                       // [n_layers*n_bufs]
    int32_t max_ctas = 0;                               // device-driven pull: SM budget (0 = every SM)
};

namespace {
struct SendRec {
    int32_t idx;      // layer * n_bufs + k
    int32_t handle;   // index into the rank's handle list
    uint64_t offset;  // from the allocation base
    int64_t bytes;
};
}  // namespace

dynmo_status dynmo_migrate_plan_create(dynmo_ctx ctx, int32_t n_layers, int32_t n_bufs,
                                       const dynmo_buf *h_send, const dynmo_buf *h_recv,
                                       dynmo_mplan *out) {
    if (!out) return invalid("null mplan out");
    *out = nullptr;
    if (!ctx || ctx->nranks < 2) return invalid(!ctx ? "null ctx" : "the peer-memory migration needs nranks > 1");
    // collective: a local failure is recorded and every rank still takes
    // part in the first all-gather, which carries the status
    dynmo_status st = DYNMO_OK;
    if (n_layers < 1 || n_bufs < 1 || !h_send || !h_recv) st = invalid("bad migrate plan args");
    DeviceGuard g(ctx->device);
    const int64_t nb = st ? 0 : (int64_t)n_layers * n_bufs;
    // this rank's send buffers -> (allocation handle, offset)
    std::vector<CUdeviceptr> bases;
    std::vector<cudaIpcMemHandle_t> handles;
    std::vector<SendRec> recs;
    for (int64_t i = 0; !st && i < nb; ++i) {
        const dynmo_buf &b = h_send[i];
        if (b.bytes <= 0 || !b.d_ptr) continue;
        CUdeviceptr base;
        size_t size;
        st = alloc_range(b.d_ptr, &base, &size);
        if (st) break;
        if ((CUdeviceptr)b.d_ptr + (size_t)b.bytes > base + size) {
            st = invalid("send buffer crosses its allocation");
            break;
        }
        int hi = -1;
        for (size_t k = 0; k < bases.size(); ++k)
            if (bases[k] == base) hi = (int)k;
        if (hi < 0) {
            cudaIpcMemHandle_t h;
            if (cudaIpcGetMemHandle(&h, (void *)base) != cudaSuccess) {
                st = cuda_fail(cudaGetLastError(), "cudaIpcGetMemHandle (send buffer)");
                break;
            }
            hi = (int)bases.size();
            bases.push_back(base);
            handles.push_back(h);
        }
        recs.push_back(SendRec{(int32_t)i, hi, (uint64_t)((CUdeviceptr)b.d_ptr - base), b.bytes});
    }
    // gather every rank's tables (counts + status, then fixed-size padded arrays)
    int64_t cnt[3] = {(int64_t)handles.size(), (int64_t)recs.size(), (int64_t)st};
    std::vector<char> allc;
    const dynmo_status ag = allgather_bytes(ctx, cnt, sizeof(cnt), allc);
    if (st) return st;
    if (ag) return ag;
    int64_t mh = 1, mr = 1;
    for (int r = 0; r < ctx->nranks; ++r) {
        const int64_t *c = (const int64_t *)(allc.data() + r * sizeof(cnt));
        if (c[2] != DYNMO_OK) return invalid("migrate plan creation failed on another rank");
        mh = std::max(mh, c[0]);
        mr = std::max(mr, c[1]);
    }
    const size_t blk = mh * sizeof(cudaIpcMemHandle_t) + mr * sizeof(SendRec);
    std::vector<char> mine(blk, 0), all;
    if (!handles.empty()) memcpy(mine.data(), handles.data(), handles.size() * sizeof(cudaIpcMemHandle_t));
    if (!recs.empty()) memcpy(mine.data() + mh * sizeof(cudaIpcMemHandle_t), recs.data(), recs.size() * sizeof(SendRec));
    st = allgather_bytes(ctx, mine.data(), blk, all);
    if (st) return st;
    auto *mp = new dynmo_mplan_s();
    mp->ctx = ctx;
    mp->n_layers = n_layers;
    mp->n_bufs = n_bufs;
    mp->recv.assign(h_recv, h_recv + nb);
    for (int r = 0; r < ctx->nranks; ++r) {
        const int64_t *c = (const int64_t *)(allc.data() + r * sizeof(cnt));
        const char *b = all.data() + r * blk;
        std::vector<char *> mapped(c[0], nullptr);
        for (int64_t k = 0; k < c[0]; ++k) {
            if (r == ctx->rank) {
                mapped[k] = (char *)bases[k];
                continue;
            }
            cudaIpcMemHandle_t h;
            memcpy(&h, b + k * sizeof(h), sizeof(h));
            void *p = nullptr;
            if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                st = cuda_fail(cudaGetLastError(), "cudaIpcOpenMemHandle (send buffer)");
                break;
            }
            mp->opened.push_back(p);
            mapped[k] = (char *)p;
        }
        if (st) break;
        const SendRec *rr = (const SendRec *)(b + mh * sizeof(cudaIpcMemHandle_t));
        for (int64_t k = 0; k < c[1]; ++k)
            mp->src[{r, rr[k].idx}] = dynmo_buf{mapped[rr[k].handle] + rr[k].offset, rr[k].bytes};
    }
    // device tables for dynmo_migrate_layers_dev
    std::vector<DevBuf> st_h((size_t)ctx->nranks * nb, DevBuf{nullptr, 0}), rt_h(nb, DevBuf{nullptr, 0});
    for (auto &kv : mp->src)
        st_h[(size_t)kv.first.first * nb + kv.first.second] = DevBuf{kv.second.d_ptr, kv.second.bytes};
    for (int64_t i = 0; i < nb; ++i) rt_h[i] = DevBuf{h_recv[i].d_ptr, h_recv[i].bytes};
    if (!st && (cudaMalloc((void **)&mp->d_src_tab, sizeof(DevBuf) * st_h.size()) != cudaSuccess ||
                cudaMalloc((void **)&mp->d_recv_tab, sizeof(DevBuf) * rt_h.size()) != cudaSuccess ||
                cudaMemcpy(mp->d_src_tab, st_h.data(), sizeof(DevBuf) * st_h.size(), cudaMemcpyHostToDevice) !=
                    cudaSuccess ||
                cudaMemcpy(mp->d_recv_tab, rt_h.data(), sizeof(DevBuf) * rt_h.size(), cudaMemcpyHostToDevice) !=
                    cudaSuccess))
        st = cuda_fail(cudaGetLastError(), "migrate plan tables");
    st = agree(ctx, st, "migrate plan (peer mapping)");
    if (st) {
        dynmo_migrate_plan_destroy(mp);
        return st;
    }
    *out = mp;
    return DYNMO_OK;
}

void dynmo_migrate_plan_destroy(dynmo_mplan mp) {
    if (!mp) return;
    DeviceGuard g(mp->ctx->device);
    for (void *p : mp->opened) cudaIpcCloseMemHandle(p);
    if (mp->d_src_tab) cudaFree(mp->d_src_tab);
    if (mp->d_recv_tab) cudaFree(mp->d_recv_tab);
    delete mp;
}

dynmo_status dynmo_migrate_layers_dev(dynmo_ctx ctx, dynmo_mplan mp, int32_t n_old,
                                      const int32_t *d_bnd_old, const int32_t *d_rank_old,
                                      int32_t n_new, const int32_t *d_bnd_new,
                                      const int32_t *d_rank_new, int64_t *d_bytes_sent,
                                      int64_t *d_bytes_recv, dynmo_stream stream) {
    if (!ctx || !mp || mp->ctx != ctx) return invalid("bad ctx/mplan");
    if (!d_bnd_old || !d_rank_old || !d_bnd_new || !d_rank_new) return invalid("null boundary/rank array");
    if (n_old < 1 || n_new < 1 || n_old > mp->n_layers || n_new > mp->n_layers) return invalid("bad stage count");
    if (mp->n_layers > 1023) return invalid("n_layers > 1023");
    DevMigArgs a{};
    a.n_layers = mp->n_layers;
    a.n_bufs = mp->n_bufs;
    a.me = ctx->rank;
    a.nranks = ctx->nranks;
    a.n_old = n_old;
    a.n_new = n_new;
    a.bnd_old = d_bnd_old;
    a.rank_old = d_rank_old;
    a.bnd_new = d_bnd_new;
    a.rank_new = d_rank_new;
    a.src_tab = mp->d_src_tab;
    a.recv_tab = mp->d_recv_tab;
    a.win = ctx->d_win;
    for (int r = 0; r < ctx->nranks; ++r) a.peer_win[r] = ctx->peer_win[r];
    a.bytes_sent = d_bytes_sent;
    a.bytes_recv = d_bytes_recv;
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t te = phase_begin(ctx, DYNMO_PHASE_MIGRATE, s);
    const bool budget = mp->max_ctas > 0 && mp->max_ctas < ctx->num_sms;
    CUDA_TRY(launch_mig_dev(a, budget ? mp->max_ctas : ctx->num_sms, budget, s), "migration kernels launch");
    phase_end(te, s);
    return DYNMO_OK;
}

// ------------------------- NEXT-3: migration during the backward pass
namespace {
// cuStreamWaitValue64 through the runtime's driver entry point (no -lcuda).
typedef int (*WaitValue64Fn)(cudaStream_t, unsigned long long, unsigned long long, unsigned int);
WaitValue64Fn wait_value64() {
    static WaitValue64Fn fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return (WaitValue64Fn)f;
    }();
    return fn;
}

// Stream waits until *addr - value >= 0 as int64 (CU_STREAM_WAIT_VALUE_GEQ):
// the GPU front end polls; no kernel, no SM.
dynmo_status stream_wait_geq(dynmo_ctx ctx, cudaStream_t s, const uint64_t *addr, uint64_t value) {
    if (!ctx->memops) return DYNMO_E_CUDA;
    const int r = wait_value64()(s, (unsigned long long)(uintptr_t)addr, (unsigned long long)value, 0x0);
    if (r != 0) {
        g_err = "cuStreamWaitValue64 failed (CUresult " + std::to_string(r) + ")";
        return DYNMO_E_CUDA;
    }
    return DYNMO_OK;
}

BwdPeers bwd_peers(dynmo_ctx ctx) {
    BwdPeers p{};
    p.nranks = ctx->nranks;
    for (int r = 0; r < ctx->nranks; ++r) p.win[r] = ctx->peer_win[r];
    return p;
}

dynmo_status bwd_args(dynmo_ctx ctx, dynmo_mplan mp, int32_t n_old, const int32_t *d_bnd_old,
                      const int32_t *d_rank_old, int32_t n_new, const int32_t *d_bnd_new,
                      const int32_t *d_rank_new, DevMigArgs &a) {
    if (!d_bnd_old || !d_rank_old || !d_bnd_new || !d_rank_new) return invalid("null boundary/rank array");
    if (n_old < 1 || n_new < 1 || n_old > mp->n_layers || n_new > mp->n_layers) return invalid("bad stage count");
    if (mp->n_layers > 1024) return invalid("n_layers > 1024");
    a = DevMigArgs{};
    a.n_layers = mp->n_layers;
    a.n_bufs = mp->n_bufs;
    a.me = ctx->rank;
    a.nranks = ctx->nranks;
    a.n_old = n_old;
    a.n_new = n_new;
    a.bnd_old = d_bnd_old;
    a.rank_old = d_rank_old;
    a.bnd_new = d_bnd_new;
    a.rank_new = d_rank_new;
    a.src_tab = mp->d_src_tab;
    a.recv_tab = mp->d_recv_tab;
    a.win = ctx->d_win;
    for (int r = 0; r < ctx->nranks; ++r) a.peer_win[r] = ctx->peer_win[r];
    static const int hint = [] {
        const char *e = getenv("DYNMO_PULL_HINT");
        return e && e[0] == '1' ? 1 : 0;
    }();
    a.hint = hint;
    return DYNMO_OK;
}
}  // namespace

dynmo_status dynmo_migrate_bwd_begin(dynmo_ctx ctx, dynmo_mplan mp, dynmo_stream stream) {
    if (!ctx || !mp || mp->ctx != ctx) return invalid("bad ctx/mplan");
    if (!ctx->memops) {
        g_err = "backward migration: 64-bit stream memory operations unsupported on this device/driver";
        return DYNMO_E_CUDA;
    }
    (void)stream;
    ++ctx->bwd_epoch;  // host-side iteration epoch (every rank calls this once per iteration)
    return DYNMO_OK;
}

dynmo_status dynmo_migrate_layer_ready(dynmo_ctx ctx, dynmo_mplan mp, int32_t layer, dynmo_stream stream) {
    if (!ctx || !mp || mp->ctx != ctx) return invalid("bad ctx/mplan");
    if (layer < 0 || layer >= mp->n_layers || layer >= 1024) return invalid("layer outside [0, n_layers)");
    if (ctx->bwd_epoch == 0) return invalid("dynmo_migrate_layer_ready before dynmo_migrate_bwd_begin");
    DeviceGuard g(ctx->device);
    CUDA_TRY(launch_layer_ready(bwd_peers(ctx), layer, ctx->bwd_epoch, (cudaStream_t)stream), "k_layer_ready launch");
    return DYNMO_OK;
}

dynmo_status dynmo_migrate_layers_bwd(dynmo_ctx ctx, dynmo_mplan mp, int32_t n_old, const int32_t *d_bnd_old,
                                      const int32_t *d_rank_old, int32_t n_new, const int32_t *d_bnd_new,
                                      const int32_t *d_rank_new, int64_t *d_bytes_recv, dynmo_stream stream) {
    if (!ctx || !mp || mp->ctx != ctx) return invalid("bad ctx/mplan");
    if (ctx->bwd_epoch == 0) return invalid("dynmo_migrate_layers_bwd before dynmo_migrate_bwd_begin");
    DevMigArgs a;
    if (dynmo_status st = bwd_args(ctx, mp, n_old, d_bnd_old, d_rank_old, n_new, d_bnd_new, d_rank_new, a)) return st;
    a.bytes_recv = d_bytes_recv;
    // the pulls share the GPU with this rank's own backward pass
    if (!(mp->max_ctas > 0 && mp->max_ctas < ctx->num_sms))
        return invalid("backward migration needs an SM budget (dynmo_migrate_plan_set_ctas, < SM count)");
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    const uint64_t ep = ctx->bwd_epoch;
    cudaEvent_t te = phase_begin(ctx, DYNMO_PHASE_MIGRATE, s);
    for (int i = mp->n_layers - 1; i >= 0; --i) {  // the backward order: last layer first
        if (dynmo_status st = stream_wait_geq(ctx, s, &ctx->d_win->layer_ready[i], ep)) return st;
        CUDA_TRY(launch_bwd_pull_layer(a, i, ep, mp->max_ctas, s), "k_bwd_pull_layer launch");
    }
    CUDA_TRY(launch_bwd_done(a, bwd_peers(ctx), ep, s), "k_bwd_done launch");
    phase_end(te, s);
    return DYNMO_OK;
}

dynmo_status dynmo_migrate_bwd_end(dynmo_ctx ctx, dynmo_mplan mp, int32_t n_old, const int32_t *d_bnd_old,
                                   const int32_t *d_rank_old, int32_t n_new, const int32_t *d_bnd_new,
                                   const int32_t *d_rank_new, int64_t *d_bytes_sent, dynmo_stream stream) {
    if (!ctx || !mp || mp->ctx != ctx) return invalid("bad ctx/mplan");
    if (ctx->bwd_epoch == 0) return invalid("dynmo_migrate_bwd_end before dynmo_migrate_bwd_begin");
    DevMigArgs a;
    if (dynmo_status st = bwd_args(ctx, mp, n_old, d_bnd_old, d_rank_old, n_new, d_bnd_new, d_rank_new, a)) return st;
    a.bytes_sent = d_bytes_sent;
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    // the caller's backward is done: pull what is left with every SM
    static const bool drain = [] {  // DYNMO_BWD_DRAIN=0: no drain (A/B knob)
        const char *e = getenv("DYNMO_BWD_DRAIN");
        return !(e && e[0] == '0');
    }();
    if (drain) CUDA_TRY(launch_bwd_drain(a, ctx->bwd_epoch, ctx->num_sms, s), "k_bwd_drain launch");
    for (int r = 0; r < ctx->nranks; ++r)
        if (dynmo_status st = stream_wait_geq(ctx, s, &ctx->d_win->bwd_done[r], ctx->bwd_epoch)) return st;
    if (d_bytes_sent) CUDA_TRY(launch_bwd_sent(a, s), "k_bwd_sent launch");
    return DYNMO_OK;
}

// Escape hatch of the unbounded stream waits: releases, in this rank's OWN
// window, every layer word and every done word at the current epoch and sets
// the sticky error to E_NCCL, so this rank's streams waiting in
// dynmo_migrate_layers_bwd / dynmo_migrate_bwd_end complete.  Copies on a
// private non-blocking stream (no kernel, no SM).  The iteration's received
// payload is undefined afterwards; the next iteration starts clean.
dynmo_status dynmo_migrate_bwd_abort(dynmo_ctx ctx, dynmo_mplan mp) {
    if (!ctx || !mp || mp->ctx != ctx) return invalid("bad ctx/mplan");
    if (ctx->bwd_epoch == 0) return invalid("dynmo_migrate_bwd_abort before dynmo_migrate_bwd_begin");
    DeviceGuard g(ctx->device);
    const int n = std::min<int>(mp->n_layers, 1024);
    std::vector<uint64_t> ready(n, ctx->bwd_epoch), done(ctx->nranks, ctx->bwd_epoch);
    const int32_t err = DYNMO_E_NCCL;
    cudaStream_t s;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "abort stream");
    cudaError_t e = cudaMemcpyAsync(&ctx->d_win->err, &err, sizeof(err), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(ctx->d_win->layer_ready, ready.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(ctx->d_win->bwd_done, done.data(), sizeof(uint64_t) * done.size(),
                            cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) return cuda_fail(e, "backward migration abort");
    return DYNMO_OK;
}

dynmo_status dynmo_migrate_plan_set_ctas(dynmo_mplan plan, int32_t max_ctas) {
    if (!plan) return invalid("null plan");
    if (max_ctas < 0) return invalid("max_ctas < 0");
    plan->max_ctas = max_ctas;
    return DYNMO_OK;
}

dynmo_status dynmo_migrate_layers_p2p(dynmo_ctx ctx, dynmo_mplan mp, int32_t n_old,
                                      const int32_t *h_bnd_old, const int32_t *h_rank_old,
                                      int32_t n_new, const int32_t *h_bnd_new,
                                      const int32_t *h_rank_new, int64_t *h_bytes_sent,
                                      int64_t *h_bytes_recv, dynmo_stream stream) {
    if (!ctx || !mp || mp->ctx != ctx) return invalid("bad ctx/mplan");
    for (int32_t s = 0; s < n_old; ++s)
        if (!h_rank_old || h_rank_old[s] < 0 || h_rank_old[s] >= ctx->nranks) return invalid("bad old rank");
    for (int32_t s = 0; s < n_new; ++s)
        if (!h_rank_new || h_rank_new[s] < 0 || h_rank_new[s] >= ctx->nranks) return invalid("bad new rank");
    const int L = mp->n_layers, nb = mp->n_bufs, me = ctx->rank;
    std::vector<int32_t> moves(3 * (size_t)L);
    const int32_t m = dynmo_migration_plan(L, n_old, h_bnd_old, h_rank_old, n_new, h_bnd_new, h_rank_new,
                                           moves.data());
    if (m < 0) return invalid("malformed boundary vector");
    std::vector<int> srcs, dsts;
    std::vector<P2PItem> items;
    int64_t sent = 0, recvd = 0;
    for (int32_t k = 0; k < m; ++k) {
        const int32_t i = moves[3 * k], src = moves[3 * k + 1], dst = moves[3 * k + 2];
        for (int32_t u = 0; u < nb; ++u) {
            const int64_t idx = (int64_t)i * nb + u;
            auto it = mp->src.find({src, idx});
            const int64_t sb = it == mp->src.end() ? 0 : it->second.bytes;
            if (src == me) sent += sb;
            if (dst == me) {
                const dynmo_buf &r = mp->recv[idx];
                if (r.bytes != sb) return invalid("recv buffer size differs from the sender's");
                if (sb > 0 && !r.d_ptr) return invalid("missing recv buffer");
                if (sb > 0) items.push_back(P2PItem{it->second.d_ptr, r.d_ptr, (uint64_t)sb});
                recvd += sb;
            }
        }
        if (dst == me && std::find(srcs.begin(), srcs.end(), src) == srcs.end()) srcs.push_back(src);
        if (src == me && std::find(dsts.begin(), dsts.end(), dst) == dsts.end()) dsts.push_back(dst);
    }
    if (h_bytes_sent) *h_bytes_sent = sent;
    if (h_bytes_recv) *h_bytes_recv = recvd;
    if (srcs.empty() && dsts.empty()) return DYNMO_OK;
    DeviceGuard g(ctx->device);
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t te = phase_begin(ctx, DYNMO_PHASE_MIGRATE, s);
    // epochs per directed pair: both ends count the calls in which the pair
    // moves data (identical move sets on every rank), so they agree whatever
    // the other ranks do (one ctx-wide epoch drifted between
    // ranks that skip calls)
    for (int d : dsts) ++ctx->send_epoch[d];
    for (int r : srcs) ++ctx->recv_epoch[r];
    // 1. tell my receivers that my buffers are ready (stream order = after my prior work)
    P2PSignal sig{};
    for (int d : dsts) {
        sig.epoch[sig.n] = ctx->send_epoch[d];
        sig.remote[sig.n++] = &ctx->peer_win[d]->ready[me];
    }
    CUDA_TRY(launch_signal(sig, s), "k_signal launch");
    // 2. pull every incoming buffer over NVLink, then tell the senders
    if (!srcs.empty()) {
        P2PPull pl{};
        pl.n_src = (int)srcs.size();
        for (int i = 0; i < pl.n_src; ++i) {
            pl.src_rank[i] = srcs[i];
            pl.done_remote[i] = &ctx->peer_win[srcs[i]]->done[me];
            pl.epoch[i] = ctx->recv_epoch[srcs[i]];
        }
        pl.ready = ctx->d_win->ready;
        pl.ctr = &ctx->d_win->pull_ctr;
        pl.err = &ctx->d_win->err;
        size_t pos = 0;
        do {
            pl.n_items = (int)std::min<size_t>(kP2PMaxItems, items.size() - pos);
            for (int i = 0; i < pl.n_items; ++i) pl.items[i] = items[pos + i];
            pos += pl.n_items;
            pl.signal_done = pos == items.size();
            CUDA_TRY(launch_pull(pl, ctx->num_sms, s), "k_pull launch");
        } while (pos < items.size());
    }
    // 3. my receivers have finished reading my buffers
    P2PWait wt{};
    wt.local = ctx->d_win->done;
    wt.err = &ctx->d_win->err;
    for (int d : dsts) {
        wt.epoch[wt.n] = ctx->send_epoch[d];
        wt.idx[wt.n++] = d;
    }
    CUDA_TRY(launch_wait(wt, s), "k_wait launch");
    phase_end(te, s);
    return DYNMO_OK;
}

// Diagnostics: a snapshot of this rank's peer window (hang analysis).  Copies
// on a private non-blocking stream, so it completes while other streams of
// the ctx wait.  Words: [0] err, [1] mig_dev_epoch, [2] exch_epoch,
// [3..3+16) bwd_done, [19..21) bwd_finished, [21..21+n) layer_ready,
// then n claim words (n = min(n_layers, 1024)).
dynmo_status dynmo_ctx_window_snapshot(dynmo_ctx ctx, int32_t n_layers, uint64_t *h_out, int64_t n_words) {
    if (!ctx || !h_out || n_layers < 0) return invalid("null ctx/out");
    const int n = std::min(n_layers, 1024);
    if (n_words < 21 + 2 * (int64_t)n) return invalid("snapshot buffer too small");
    DeviceGuard g(ctx->device);
    std::vector<char> w(sizeof(PeerWindow));
    cudaStream_t s;
    CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "snapshot stream");
    cudaError_t e = cudaMemcpyAsync(w.data(), ctx->d_win, sizeof(PeerWindow), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) return cuda_fail(e, "window snapshot");
    const PeerWindow *pw = (const PeerWindow *)w.data();
    h_out[0] = (uint64_t)(int64_t)pw->err;
    h_out[1] = pw->mig_dev_epoch;
    h_out[2] = pw->exch_epoch;
    for (int r = 0; r < 16; ++r) h_out[3 + r] = pw->bwd_done[r];
    h_out[19] = pw->bwd_finished[0];
    h_out[20] = pw->bwd_finished[1];
    for (int i = 0; i < n; ++i) h_out[21 + i] = pw->layer_ready[i];
    for (int i = 0; i < n; ++i) h_out[21 + n + i] = pw->bwd_claim[i];
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_profile_span(dynmo_ctx ctx, double *h_total_ms, int64_t *h_count) {
    if (!ctx || !h_total_ms || !h_count) return invalid("null ctx/out");
    DeviceGuard g(ctx->device);
    unsigned long long h[4];
    CUDA_TRY(cudaMemcpy(h, ctx->d_win->prof_span, sizeof(h), cudaMemcpyDeviceToHost), "read profile span");
    *h_total_ms = (double)h[2] * 1e-6;
    *h_count = (int64_t)h[3];
    CUDA_TRY(cudaMemset(ctx->d_win->prof_span + 2, 0, 2 * sizeof(unsigned long long)), "reset profile span");
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_p2p_error(dynmo_ctx ctx, int32_t *h_err) {
    if (!ctx || !h_err) return invalid("bad args");
    *h_err = 0;
    if (!ctx->d_win) return DYNMO_OK;
    DeviceGuard g(ctx->device);
    CUDA_TRY(cudaMemcpy(h_err, &ctx->d_win->err, sizeof(int32_t), cudaMemcpyDeviceToHost), "read p2p error");
    return DYNMO_OK;
}

dynmo_status dynmo_ctx_p2p_error_clear(dynmo_ctx ctx) {
    if (!ctx) return invalid("null ctx");
    if (!ctx->d_win) return DYNMO_OK;
    DeviceGuard g(ctx->device);
    CUDA_TRY(cudaDeviceSynchronize(), "p2p error clear (drain)");
    CUDA_TRY(cudaMemset(&ctx->d_win->err, 0, sizeof(int32_t)), "p2p error clear");
    return DYNMO_OK;
}

}  // extern "C"
