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
        for (int i = 0; i < s.n; ++i) st_release_sys(s.remote[i], s.epoch);
}

__global__ void k_wait(P2PWait w) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int i = 0; i < w.n; ++i)
            if (!wait_flag(w.local + w.idx[i], w.epoch)) atomicExch(w.err, (int)DYNMO_E_NCCL);
}

__global__ void __launch_bounds__(kP2PThreads) k_pull(P2PPull p) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        int ok = 1;
        for (int i = 0; i < p.n_src; ++i) ok &= wait_flag(p.ready + p.src_rank[i], p.epoch);
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
                for (int i = 0; i < p.n_src; ++i) st_release_sys(p.done_remote[i], p.epoch);
        }
    }
}

}  // namespace

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
