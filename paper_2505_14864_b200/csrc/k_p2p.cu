// k_p2p.cu -- layer migration over NVLink peer memory (
// P:L636 "When a layer is migrated from GPU A to GPU B ...").
//
// Receivers PULL: every moved layer buffer of the sender is mapped into the
// receiver's address space (CUDA IPC, exchanged once by the migration plan),
// and one kernel on the receiver copies all incoming buffers with 128-bit
// loads over NVLink (4 in flight per thread), grid-striding over each item.
// Cross-GPU ordering uses per-rank flag words in a peer-mapped window:
//   sender:   k_signal  -> READY[me] on each receiver      (release, system scope)
//   receiver: k_pull waits READY[src] >= epoch, copies, then writes DONE[me]
//             on each sender
//   sender:   k_wait    -> DONE[dst] >= epoch before its stream moves on
// All waits are bounded (10 s of %globaltimer) and report DYNMO_E_NCCL-like
// failure through an error word instead of hanging the GPU.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "dynmo_internal.h"

namespace dynmo {
namespace {

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Spin until *flag >= epoch (bounded): returns false on timeout.
__device__ bool wait_flag(const uint64_t *flag, uint64_t epoch) {
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(flag) < epoch) {
        if (globaltimer() - t0 > 10ull * 1000 * 1000 * 1000) return false;
        __nanosleep(200);
    }
    return true;
}

__global__ void k_signal(P2PSignal s) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int i = 0; i < s.n; ++i) st_release_sys(s.remote[i], s.epoch[i]);
}

__global__ void k_wait(P2PWait w) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int i = 0; i < w.n; ++i)
            if (!wait_flag(w.local + w.idx[i], w.epoch[i])) atomicExch(w.err, (int)DYNMO_E_NCCL);
}

__global__ void __launch_bounds__(kP2PThreads) k_pull(P2PPull p) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        int ok = 1;
        for (int i = 0; i < p.n_src; ++i) ok &= wait_flag(p.ready + p.src_rank[i], p.epoch[i]);
        s_ok = ok;
        if (!ok) atomicExch(p.err, (int)DYNMO_E_NCCL);
    }
    __syncthreads();
    if (s_ok) {
        const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
        for (int it = 0; it < p.n_items; ++it) {
            const P2PItem t = p.items[it];
            const uint8_t *src = (const uint8_t *)t.src;
            uint8_t *dst = (uint8_t *)t.dst;
            const bool vec = (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
            const uint64_t nvec = vec ? t.bytes >> 4 : 0;
            const uint4 *s4 = (const uint4 *)src;
            uint4 *d4 = (uint4 *)dst;
            uint64_t v = gt;
            for (; v + 3 * gs < nvec; v += 4 * gs) {  // 4 x 16 B in flight per thread
                const uint4 a = s4[v], b = s4[v + gs], c = s4[v + 2 * gs], d = s4[v + 3 * gs];
                d4[v] = a;
                d4[v + gs] = b;
                d4[v + 2 * gs] = c;
                d4[v + 3 * gs] = d;
            }
            for (; v < nvec; v += gs) d4[v] = s4[v];
            for (uint64_t b = nvec * 16 + gt; b < t.bytes; b += gs) dst[b] = src[b];
        }
    }
    // completion: the last block to finish tells every sender it may move on
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(p.ctr, 1u);
        if (prev == gridDim.x - 1) {
            *p.ctr = 0u;
            __threadfence_system();
            if (p.signal_done)
                for (int i = 0; i < p.n_src; ++i) st_release_sys(p.done_remote[i], p.epoch[i]);
        }
    }
}

// ------------------------------------------------ device-driven migration
// Stage of layer i under boundaries b[0..n] (binary search).
__device__ __forceinline__ int stage_of(const int32_t *b, int n, int i) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ bool valid_split(const int32_t *b, int n, int L) {
    if (n < 1 || b[0] != 0 || b[n] != L) return false;
    for (int s = 0; s < n; ++s)
        if (b[s + 1] <= b[s]) return false;
    return true;
}

// Block-local view of the migration: the layers this rank receives (and
// from whom), the set of its senders and of its receivers.  ok = 0 when a
// split is malformed or a stage -> rank entry lies outside [0, nranks) (e.g.
// the -1 k_map_stages writes on failure): then nothing moves anywhere and
// every rank reports DYNMO_E_INVALID in its window's error word.
struct MigView {
    int n_in;
    unsigned senders, receivers;
    int ok;
};

__device__ __forceinline__ bool ranks_ok(const int32_t *rk, int n, int nranks) {
    for (int s = 0; s < n; ++s)
        if (rk[s] < 0 || rk[s] >= nranks) return false;
    return true;
}

__device__ void mig_view(const DevMigArgs &a, MigView &v, int16_t *in_layers, int8_t *in_src) {
    if (threadIdx.x == 0) {
        v.n_in = 0;
        v.senders = v.receivers = 0u;
        v.ok = valid_split(a.bnd_old, a.n_old, a.n_layers) && valid_split(a.bnd_new, a.n_new, a.n_layers) &&
               ranks_ok(a.rank_old, a.n_old, a.nranks) && ranks_ok(a.rank_new, a.n_new, a.nranks);
    }
    __syncthreads();
    if (v.ok) {
        for (int i = threadIdx.x; i < a.n_layers; i += blockDim.x) {
            const int src = a.rank_old[stage_of(a.bnd_old, a.n_old, i)];
            const int dst = a.rank_new[stage_of(a.bnd_new, a.n_new, i)];
            if (src == dst) continue;
            if (dst == a.me) {
                const int k = atomicAdd(&v.n_in, 1);
                in_layers[k] = (int16_t)i;
                in_src[k] = (int8_t)src;
                atomicOr(&v.senders, 1u << src);
            }
            if (src == a.me) atomicOr(&v.receivers, 1u << dst);
        }
    }
    __syncthreads();
}

// Sender side: advance the device epoch, release ready[me] at every receiver.
__global__ void k_mig_signal(DevMigArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ unsigned s_recv;
    __shared__ int s_ok;
    __shared__ unsigned long long s_sent;
    if (threadIdx.x == 0) {
        s_recv = 0u;
        s_sent = 0ull;
        s_ok = valid_split(a.bnd_old, a.n_old, a.n_layers) && valid_split(a.bnd_new, a.n_new, a.n_layers) &&
               ranks_ok(a.rank_old, a.n_old, a.nranks) && ranks_ok(a.rank_new, a.n_new, a.nranks);
    }
    __syncthreads();
    if (s_ok)
        for (int i = threadIdx.x; i < a.n_layers; i += blockDim.x) {
            const int src = a.rank_old[stage_of(a.bnd_old, a.n_old, i)];
            const int dst = a.rank_new[stage_of(a.bnd_new, a.n_new, i)];
            if (src == a.me && dst != a.me) {
                atomicOr(&s_recv, 1u << dst);
                unsigned long long b = 0;
                const DevBuf *row = a.src_tab + ((int64_t)a.me * a.n_layers + i) * a.n_bufs;
                for (int k = 0; k < a.n_bufs; ++k) b += (unsigned long long)row[k].bytes;
                atomicAdd(&s_sent, b);
            }
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint64_t epoch = a.win->mig_dev_epoch + 1;
        a.win->mig_dev_epoch = epoch;
        if (!s_ok) atomicExch(&a.win->err, (int)DYNMO_E_INVALID);
        for (int r = 0; r < a.nranks; ++r)
            if (s_recv & (1u << r)) st_release_sys(&a.peer_win[r]->dready[a.me], epoch);
        if (a.bytes_sent) *a.bytes_sent = (int64_t)s_sent;
    }
}

// Receiver side: every block derives the incoming set, waits for the senders,
// copies its grid-stride share of every incoming buffer; the last block
// releases ddone[me] at every sender.
// U = 16-byte NVLink loads in flight per thread: 4 with one CTA per SM (the
// full-GPU migration: finer tail), 16 under an SM budget (the migration
// overlapped with compute: 128 KB per CTA, so 16-32 CTAs cover the peer
// latency; bench_overlap.py)
template <int U>
__global__ void __launch_bounds__(kP2PThreads) k_mig_pull(DevMigArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ MigView v;
    __shared__ int16_t in_layers[1024];
    __shared__ int8_t in_src[1024];
    __shared__ int s_ok;
    mig_view(a, v, in_layers, in_src);
    const uint64_t epoch = a.win->mig_dev_epoch;
    if (threadIdx.x == 0) {
        int ok = v.ok;
        for (int r = 0; ok && r < a.nranks; ++r)
            if (v.senders & (1u << r)) ok &= wait_flag(&a.win->dready[r], epoch);
        if (!ok) atomicExch(&a.win->err, v.ok ? (int)DYNMO_E_NCCL : (int)DYNMO_E_INVALID);
        s_ok = ok;
    }
    __syncthreads();
    const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long recvd = 0;
    if (s_ok) {
        for (int it = 0; it < v.n_in; ++it) {
            const int i = in_layers[it], src = in_src[it];
            for (int k = 0; k < a.n_bufs; ++k) {
                const int64_t idx = (int64_t)i * a.n_bufs + k;
                const DevBuf sb = a.src_tab[((int64_t)src * a.n_layers) * a.n_bufs + idx];
                const DevBuf rb = a.recv_tab[idx];
                if (sb.bytes != rb.bytes || (sb.bytes > 0 && (!sb.ptr || !rb.ptr))) {
                    // the receive buffer does not match the sender's: reported,
                    // never silently truncated
                    if (gt == 0) atomicExch(&a.win->err, (int)DYNMO_E_INVALID);
                    continue;
                }
                const uint64_t bytes = (uint64_t)sb.bytes;
                recvd += bytes;
                const uint8_t *sp = (const uint8_t *)sb.ptr;
                uint8_t *dp = (uint8_t *)rb.ptr;
                const bool vec = (((uintptr_t)sp | (uintptr_t)dp) & 15) == 0;
                const uint64_t nvec = vec ? bytes >> 4 : 0;
                const uint4 *s4 = (const uint4 *)sp;
                uint4 *d4 = (uint4 *)dp;
                uint64_t x = gt;
                for (; x + (U - 1) * gs < nvec; x += U * gs) {
                    uint4 q[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) q[u] = s4[x + u * gs];
#pragma unroll
                    for (int u = 0; u < U; ++u) d4[x + u * gs] = q[u];
                }
                for (; x < nvec; x += gs) d4[x] = s4[x];
                for (uint64_t b = nvec * 16 + gt; b < bytes; b += gs) dp[b] = sp[b];
            }
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0 && a.bytes_recv) *a.bytes_recv = (int64_t)recvd;
        const unsigned prev = atomicAdd(&a.win->dpull_ctr, 1u);
        if (prev == gridDim.x - 1) {
            a.win->dpull_ctr = 0u;
            __threadfence_system();
            for (int r = 0; r < a.nranks; ++r)
                if (v.senders & (1u << r)) st_release_sys(&a.peer_win[r]->ddone[a.me], epoch);
        }
    }
}

// Sender side again: wait until every receiver has finished reading.
__global__ void k_mig_wait(DevMigArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ MigView v;
    __shared__ int16_t in_layers[1024];
    __shared__ int8_t in_src[1024];
    mig_view(a, v, in_layers, in_src);
    if (threadIdx.x == 0 && v.ok) {
        const uint64_t epoch = a.win->mig_dev_epoch;
        for (int r = 0; r < a.nranks; ++r)
            if (v.receivers & (1u << r))
                if (!wait_flag(&a.win->ddone[r], epoch)) atomicExch(&a.win->err, (int)DYNMO_E_NCCL);
    }
}

// One-kernel device-driven migration (the three kernels above fused: one
// launch on the step's critical path instead of three).  Every block derives
// the moves from the device boundaries; block 0 releases dready[me] at this
// rank's receivers (this call's epoch = the window's + 1, written back by the
// last block); every block waits for its senders and copies its grid-stride
// share; the last block to finish releases ddone[me] at the senders, then
// waits (bounded) for every receiver's ddone -- releases always precede
// waits in every rank's last block, so the ranks cannot wait on each other
// in a cycle -- and only then lets the stream reuse the sent buffers.
template <int U>
__global__ void __launch_bounds__(kP2PThreads) k_mig_fused(DevMigArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ MigView v;
    __shared__ int16_t in_layers[1024];
    __shared__ int8_t in_src[1024];
    __shared__ int s_ok;
    __shared__ bool s_last;
    mig_view(a, v, in_layers, in_src);
    const uint64_t epoch = a.win->mig_dev_epoch + 1;
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0) {
            if (!v.ok) atomicExch(&a.win->err, (int)DYNMO_E_INVALID);
            else if (v.receivers) {
                __threadfence_system();  // the payload written by earlier stream work
                for (int r = 0; r < a.nranks; ++r)
                    if (v.receivers & (1u << r)) st_release_sys(&a.peer_win[r]->dready[a.me], epoch);
            }
        }
        int ok = v.ok;
        for (int r = 0; ok && r < a.nranks; ++r)
            if (v.senders & (1u << r)) ok &= wait_flag(&a.win->dready[r], epoch);
        if (!ok && v.ok) atomicExch(&a.win->err, (int)DYNMO_E_NCCL);
        s_ok = ok;
    }
    __syncthreads();
    const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    unsigned long long recvd = 0;
    if (s_ok) {
        for (int it = 0; it < v.n_in; ++it) {
            const int i = in_layers[it], src = in_src[it];
            for (int k = 0; k < a.n_bufs; ++k) {
                const int64_t idx = (int64_t)i * a.n_bufs + k;
                const DevBuf sb = a.src_tab[((int64_t)src * a.n_layers) * a.n_bufs + idx];
                const DevBuf rb = a.recv_tab[idx];
                if (sb.bytes != rb.bytes || (sb.bytes > 0 && (!sb.ptr || !rb.ptr))) {
                    if (gt == 0) atomicExch(&a.win->err, (int)DYNMO_E_INVALID);
                    continue;
                }
                const uint64_t bytes = (uint64_t)sb.bytes;
                recvd += bytes;
                const uint8_t *sp = (const uint8_t *)sb.ptr;
                uint8_t *dp = (uint8_t *)rb.ptr;
                const bool vec = (((uintptr_t)sp | (uintptr_t)dp) & 15) == 0;
                const uint64_t nvec = vec ? bytes >> 4 : 0;
                const uint4 *s4 = (const uint4 *)sp;
                uint4 *d4 = (uint4 *)dp;
                uint64_t x = gt;
                for (; x + (U - 1) * gs < nvec; x += U * gs) {
                    uint4 q[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) q[u] = s4[x + u * gs];
#pragma unroll
                    for (int u = 0; u < U; ++u) d4[x + u * gs] = q[u];
                }
                for (; x < nvec; x += gs) d4[x] = s4[x];
                for (uint64_t b = nvec * 16 + gt; b < bytes; b += gs) dp[b] = sp[b];
            }
        }
    }
    if (v.n_in > 0) __threadfence_system();  // (a step that moves nothing skips the system fences)
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockIdx.x == 0 && a.bytes_recv) *a.bytes_recv = (int64_t)recvd;
        const unsigned prev = atomicAdd(&a.win->dpull_ctr, 1u);
        s_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    // the last block: done at the senders, then this rank's receivers, then
    // the bytes this rank sent and the epoch for the next call
    __shared__ unsigned long long s_sent;
    if (threadIdx.x == 0) {
        a.win->dpull_ctr = 0u;
        s_sent = 0ull;
        if (v.senders) __threadfence_system();
        for (int r = 0; r < a.nranks; ++r)
            if (v.senders & (1u << r)) st_release_sys(&a.peer_win[r]->ddone[a.me], epoch);
        if (v.ok)
            for (int r = 0; r < a.nranks; ++r)
                if (v.receivers & (1u << r))
                    if (!wait_flag(&a.win->ddone[r], epoch)) atomicExch(&a.win->err, (int)DYNMO_E_NCCL);
    }
    __syncthreads();
    if (v.ok)
        for (int i = threadIdx.x; i < a.n_layers; i += blockDim.x) {
            const int src = a.rank_old[stage_of(a.bnd_old, a.n_old, i)];
            const int dst = a.rank_new[stage_of(a.bnd_new, a.n_new, i)];
            if (src == a.me && dst != a.me) {
                unsigned long long b = 0;
                const DevBuf *row = a.src_tab + ((int64_t)a.me * a.n_layers + i) * a.n_bufs;
                for (int k = 0; k < a.n_bufs; ++k) b += (unsigned long long)row[k].bytes;
                atomicAdd(&s_sent, b);
            }
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.bytes_sent) *a.bytes_sent = (int64_t)s_sent;
        a.win->mig_dev_epoch = epoch;
    }
}

// ------------------- NEXT-3: migration during the backward pass
// "moving layers while the gradients calculation take place, from the last
// to the first layer".  While the backward runs, no kernel waits on the GPU:
// the backward stream releases layer i (k_layer_ready: its payload is final)
// into EVERY rank's window; each rank's side stream waits for the layers in
// descending order with stream memory operations (the GPU front end polls,
// no SM is held) and runs one pull kernel per layer under the SM budget.  A
// layer's payload is cut into 256 KiB chunks claimed by CTAs through an
// epoch-tagged counter, so a DRAIN kernel with every SM, launched by
// dynmo_migrate_bwd_end once the caller's backward is done, can take over
// the chunks not yet pulled (the last layers are released when there is no
// compute left to hide them).  k_bwd_done waits until every incoming chunk
// is copied, then releases done[me] everywhere; the senders' streams wait
// for every rank's done before reusing the sent buffers.
constexpr uint64_t kBwdChunk = 256u << 10;

__global__ void k_layer_ready(BwdPeers p, int32_t layer, uint64_t epoch) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        // the stream's earlier kernels wrote the layer's buffers: make them
        // visible at system scope, then release the layer on every rank
        __threadfence_system();
        for (int r = 0; r < p.nranks; ++r) st_release_sys(&p.win[r]->layer_ready[layer], epoch);
    }
}

__device__ __forceinline__ bool mig_args_ok(const DevMigArgs &a) {
    return valid_split(a.bnd_old, a.n_old, a.n_layers) && valid_split(a.bnd_new, a.n_new, a.n_layers) &&
           ranks_ok(a.rank_old, a.n_old, a.nranks) && ranks_ok(a.rank_new, a.n_new, a.nranks);
}

// Sender of layer i if it moves to this rank, else -1.
__device__ __forceinline__ int incoming_src(const DevMigArgs &a, int i) {
    const int src = a.rank_old[stage_of(a.bnd_old, a.n_old, i)];
    const int dst = a.rank_new[stage_of(a.bnd_new, a.n_new, i)];
    return (dst == a.me && src != a.me) ? src : -1;
}

// Chunks of layer i from src (every buffer cut at kBwdChunk); 0 and an error
// if a receive buffer does not match its send buffer.
__device__ uint32_t layer_chunks(const DevMigArgs &a, int i, int src, bool &bad) {
    uint32_t nc = 0;
    for (int k = 0; k < a.n_bufs; ++k) {
        const int64_t idx = (int64_t)i * a.n_bufs + k;
        const DevBuf sb = a.src_tab[((int64_t)src * a.n_layers) * a.n_bufs + idx];
        const DevBuf rb = a.recv_tab[idx];
        if (sb.bytes != rb.bytes || (sb.bytes > 0 && (!sb.ptr || !rb.ptr))) {
            bad = true;
            return 0;
        }
        nc += (uint32_t)(((uint64_t)sb.bytes + kBwdChunk - 1) / kBwdChunk);
    }
    return nc;
}

// Claim the next chunk of layer i in iteration `ep` (thread 0).  The word is
// {epoch low 32 bits, claims}: a stale epoch restarts at 0, a newer one means
// this launch's iteration is over (nothing to claim).  Returns the chunk
// index, or UINT32_MAX.
__device__ uint32_t claim_chunk(unsigned long long *w, uint64_t ep, uint32_t nc) {
    const unsigned long long e = (unsigned long long)(uint32_t)ep;
    unsigned long long cur = *(volatile unsigned long long *)w;
    for (;;) {
        const unsigned long long we = cur >> 32;
        unsigned long long nxt;
        uint32_t got;
        if (we == e) {
            got = (uint32_t)cur;
            if (got >= nc) return UINT32_MAX;
            nxt = cur + 1;
        } else if ((uint32_t)(we - e) > 0x7FFFFFFFu) {  // stale (older) epoch
            got = 0;
            nxt = (e << 32) | 1ull;
        } else {
            return UINT32_MAX;  // a newer iteration owns the word
        }
        const unsigned long long prev = atomicCAS(w, cur, nxt);
        if (prev == cur) return got;
        cur = prev;
    }
}

__device__ __forceinline__ uint4 ld_evict_first(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_evict_first(uint4 *p, const uint4 &v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// Copy chunk c of layer i (whole CTA, 16 x 16-byte NVLink loads in flight
// per thread), then count it finished (after a fence: the copy is visible
// before the counter that k_bwd_done waits on).
__device__ void copy_chunk(const DevMigArgs &a, int i, int src, uint32_t c, unsigned int *finished) {
    constexpr int U = 16;
    for (int k = 0; k < a.n_bufs; ++k) {
        const int64_t idx = (int64_t)i * a.n_bufs + k;
        const DevBuf sb = a.src_tab[((int64_t)src * a.n_layers) * a.n_bufs + idx];
        const DevBuf rb = a.recv_tab[idx];
        const uint32_t nck = (uint32_t)(((uint64_t)sb.bytes + kBwdChunk - 1) / kBwdChunk);
        if (c >= nck) {
            c -= nck;
            continue;
        }
        const uint64_t off = (uint64_t)c * kBwdChunk;
        const uint64_t rem = (uint64_t)sb.bytes - off;
        const uint64_t bytes = rem < kBwdChunk ? rem : kBwdChunk;
        const uint8_t *sp = (const uint8_t *)sb.ptr + off;
        uint8_t *dp = (uint8_t *)rb.ptr + off;
        const bool vec = (((uintptr_t)sp | (uintptr_t)dp) & 15) == 0;
        const uint64_t nvec = vec ? bytes >> 4 : 0;
        const uint4 *s4 = (const uint4 *)sp;
        uint4 *d4 = (uint4 *)dp;
        const uint64_t gs = blockDim.x;
        uint64_t x = threadIdx.x;
        if (a.hint) {  // streaming (.cs: evict-first) loads and stores
            for (; x + (U - 1) * gs < nvec; x += U * gs) {
                uint4 q[U];
#pragma unroll
                for (int u = 0; u < U; ++u) q[u] = ld_evict_first(s4 + x + u * gs);
#pragma unroll
                for (int u = 0; u < U; ++u) st_evict_first(d4 + x + u * gs, q[u]);
            }
        } else {
            for (; x + (U - 1) * gs < nvec; x += U * gs) {
                uint4 q[U];
#pragma unroll
                for (int u = 0; u < U; ++u) q[u] = s4[x + u * gs];
#pragma unroll
                for (int u = 0; u < U; ++u) d4[x + u * gs] = q[u];
            }
        }
        for (; x < nvec; x += gs) d4[x] = s4[x];
        for (uint64_t b = nvec * 16 + threadIdx.x; b < bytes; b += gs) dp[b] = sp[b];
        break;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(finished, 1u);
}

// Claim-and-copy loop of one CTA over layer i.
__device__ void pull_chunks(const DevMigArgs &a, int i, int src, uint32_t nc, uint64_t ep) {
    __shared__ uint32_t s_c;
    unsigned int *finished = &a.win->bwd_finished[ep & 1];
    for (;;) {
        if (threadIdx.x == 0) s_c = claim_chunk(&a.win->bwd_claim[i], ep, nc);
        __syncthreads();
        const uint32_t c = s_c;
        __syncthreads();
        if (c == UINT32_MAX) return;
        copy_chunk(a, i, src, c, finished);
    }
}

// One layer of the backward-ordered pull (side stream, SM budget).
__global__ void __launch_bounds__(kP2PThreads) k_bwd_pull_layer(DevMigArgs a, int32_t i, uint64_t ep) {
    __shared__ int s_ok;
    __shared__ uint32_t s_nc;
    if (threadIdx.x == 0) {
        int ok = mig_args_ok(a);
        s_nc = 0;
        if (ok) {
            const int src = incoming_src(a, i);
            bool bad = false;
            if (src >= 0) s_nc = layer_chunks(a, i, src, bad);
            ok = !bad;
        }
        s_ok = ok;
    }
    __syncthreads();
    if (!s_ok || s_nc == 0) return;  // errors are reported by k_bwd_done
    pull_chunks(a, i, incoming_src(a, i), s_nc, ep);
}

// Drain (dynmo_migrate_bwd_end, every SM): the incoming layers in descending
// order, each once its release has arrived (bounded wait), sharing the
// chunk claims with the per-layer pulls still queued on the side stream.
__global__ void __launch_bounds__(kP2PThreads) k_bwd_drain(DevMigArgs a, uint64_t ep) {
    __shared__ int s_go;
    __shared__ uint32_t s_nc;
    __shared__ int s_src;
    if (!mig_args_ok(a)) return;
    for (int i = a.n_layers - 1; i >= 0; --i) {
        if (threadIdx.x == 0) {
            s_src = incoming_src(a, i);
            bool bad = false;
            s_nc = s_src >= 0 ? layer_chunks(a, i, s_src, bad) : 0u;
            s_go = s_nc > 0 && !bad;
            if (s_go && !wait_flag(&a.win->layer_ready[i], ep)) {
                atomicExch(&a.win->err, (int)DYNMO_E_NCCL);
                s_go = -1;
            }
        }
        __syncthreads();
        const int go = s_go;
        const uint32_t nc = s_nc;
        const int src = s_src;
        __syncthreads();
        if (go < 0) return;
        if (go) pull_chunks(a, i, src, nc, ep);
    }
}

// After the side stream's pulls: wait until every incoming chunk is copied
// (by a pull or the drain; bounded), report the bytes and errors, reset the
// finished counter of this epoch's parity, release done[me] everywhere.
__global__ void k_bwd_done(DevMigArgs a, BwdPeers p, uint64_t ep) {
    __shared__ unsigned long long s_bytes;
    __shared__ unsigned s_total;
    __shared__ int s_bad;
    if (threadIdx.x == 0) {
        s_bytes = 0ull;
        s_total = 0u;
        s_bad = !mig_args_ok(a);
    }
    __syncthreads();
    if (!s_bad)
        for (int i = threadIdx.x; i < a.n_layers; i += blockDim.x) {
            const int src = incoming_src(a, i);
            if (src < 0) continue;
            bool bad = false;
            const uint32_t nc = layer_chunks(a, i, src, bad);
            if (bad) {
                atomicExch(&s_bad, 1);
                continue;
            }
            atomicAdd(&s_total, nc);
            unsigned long long b = 0;
            for (int k = 0; k < a.n_bufs; ++k)
                b += (unsigned long long)a.recv_tab[(int64_t)i * a.n_bufs + k].bytes;
            atomicAdd(&s_bytes, b);
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_bad) atomicExch(&a.win->err, (int)DYNMO_E_INVALID);
        unsigned int *fin = &a.win->bwd_finished[ep & 1];
        const uint64_t t0 = globaltimer();
        while (*(volatile unsigned int *)fin < s_total) {
            if (globaltimer() - t0 > 10ull * 1000 * 1000 * 1000) {
                atomicExch(&a.win->err, (int)DYNMO_E_NCCL);
                break;
            }
            __nanosleep(200);
        }
        __threadfence();
        *fin = 0u;
        if (a.bytes_recv) *a.bytes_recv = s_bad ? 0 : (int64_t)s_bytes;
        __threadfence_system();
        for (int r = 0; r < p.nranks; ++r) st_release_sys(&p.win[r]->bwd_done[a.me], ep);
    }
}

// Sender side (at dynmo_migrate_bwd_end, after the done waits): bytes sent.
__global__ void k_bwd_sent(DevMigArgs a) {
    __shared__ unsigned long long s_sent;
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        s_sent = 0ull;
        s_ok = mig_args_ok(a);
    }
    __syncthreads();
    if (s_ok)
        for (int i = threadIdx.x; i < a.n_layers; i += blockDim.x) {
            const int src = a.rank_old[stage_of(a.bnd_old, a.n_old, i)];
            const int dst = a.rank_new[stage_of(a.bnd_new, a.n_new, i)];
            if (src == a.me && dst != a.me) {
                unsigned long long b = 0;
                const DevBuf *row = a.src_tab + ((int64_t)a.me * a.n_layers + i) * a.n_bufs;
                for (int k = 0; k < a.n_bufs; ++k) b += (unsigned long long)row[k].bytes;
                atomicAdd(&s_sent, b);
            }
        }
    __syncthreads();
    if (threadIdx.x == 0 && a.bytes_sent) *a.bytes_sent = s_ok ? (int64_t)s_sent : 0;
}

}  // namespace

cudaError_t launch_layer_ready(const BwdPeers &p, int32_t layer, uint64_t epoch, cudaStream_t s) {
    k_layer_ready<<<1, 32, 0, s>>>(p, layer, epoch);
    return cudaGetLastError();
}

cudaError_t launch_bwd_pull_layer(const DevMigArgs &a, int32_t layer, uint64_t epoch, int grid, cudaStream_t s) {
    k_bwd_pull_layer<<<grid, kP2PThreads, 0, s>>>(a, layer, epoch);
    return cudaGetLastError();
}

cudaError_t launch_bwd_drain(const DevMigArgs &a, uint64_t epoch, int grid, cudaStream_t s) {
    k_bwd_drain<<<grid, kP2PThreads, 0, s>>>(a, epoch);
    return cudaGetLastError();
}

cudaError_t launch_bwd_done(const DevMigArgs &a, const BwdPeers &p, uint64_t epoch, cudaStream_t s) {
    k_bwd_done<<<1, 256, 0, s>>>(a, p, epoch);
    return cudaGetLastError();
}

cudaError_t launch_bwd_sent(const DevMigArgs &a, cudaStream_t s) {
    k_bwd_sent<<<1, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_mig_dev(const DevMigArgs &a, int grid, bool budget, cudaStream_t s) {
    static const bool fused = [] {  // DYNMO_MIG_FUSED=0: the three-kernel path (A/B knob)
        const char *e = getenv("DYNMO_MIG_FUSED");
        return !(e && e[0] == '0');
    }();
    if (fused) {
        const cudaError_t f = budget ? launch_pdl(k_mig_fused<16>, grid, kP2PThreads, 0, s, a)
                                     : launch_pdl(k_mig_fused<4>, grid, kP2PThreads, 0, s, a);
        return f != cudaSuccess ? f : cudaGetLastError();
    }
    cudaError_t e = launch_pdl(k_mig_signal, 1, 256, 0, s, a);
    if (e == cudaSuccess)
        e = budget ? launch_pdl(k_mig_pull<16>, grid, kP2PThreads, 0, s, a)
                   : launch_pdl(k_mig_pull<4>, grid, kP2PThreads, 0, s, a);
    if (e == cudaSuccess) e = launch_pdl(k_mig_wait, 1, 256, 0, s, a);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// CUDA lazy loading (the default module loading mode) loads a kernel at its
// first launch, and that load may synchronise the context.  A kernel that
// spins on a flag released by a LATER launch in another stream (the
// backward-ordered pull waits on k_layer_ready; the pulls wait on the
// signals) would then deadlock until its bounded wait times out: load every
// peer-path kernel once when the window is created.
cudaError_t preload_p2p_kernels() {
    cudaFuncAttributes fa;
    const void *ks[] = {(const void *)k_signal,           (const void *)k_wait,
                        (const void *)k_pull,             (const void *)k_mig_signal,
                        (const void *)k_mig_pull<4>,      (const void *)k_mig_pull<16>,
                        (const void *)k_mig_wait,         (const void *)k_layer_ready,
                        (const void *)k_bwd_done,         (const void *)k_bwd_pull_layer,
                        (const void *)k_bwd_drain,        (const void *)k_bwd_sent,
                        (const void *)k_mig_fused<4>,     (const void *)k_mig_fused<16>};
    for (const void *k : ks) {
        const cudaError_t e = cudaFuncGetAttributes(&fa, k);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_signal(const P2PSignal &s, cudaStream_t st) {
    if (s.n == 0) return cudaSuccess;
    k_signal<<<1, 32, 0, st>>>(s);
    return cudaGetLastError();
}
cudaError_t launch_wait(const P2PWait &w, cudaStream_t st) {
    if (w.n == 0) return cudaSuccess;
    k_wait<<<1, 32, 0, st>>>(w);
    return cudaGetLastError();
}
cudaError_t launch_pull(const P2PPull &p, int grid, cudaStream_t st) {
    k_pull<<<grid, kP2PThreads, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace dynmo
