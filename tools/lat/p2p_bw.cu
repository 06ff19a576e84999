// Peer-memory bandwidth on B200 over NVLink 5: receiver-pull (remote 128-bit
// loads) vs sender-push (remote 128-bit stores), one process, 2 GPUs with
// peer access.  Prints GB/s per variant at the migration's transfer size.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a p2p_bw.cu -o p2p_bw
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U>
__global__ void copy16(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
    const size_t bytes = 141ull << 20;
    const size_t n = bytes / 16;
    void *a0, *b0, *a1, *b1;
    CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); CK(cudaMalloc(&a0, bytes)); CK(cudaMalloc(&b0, bytes));
    CK(cudaMemset(a0, 1, bytes));
    CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMalloc(&a1, bytes)); CK(cudaMalloc(&b1, bytes));
    CK(cudaMemset(a1, 2, bytes));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 1));
    cudaEvent_t e0, e1;
    for (int variant = 0; variant < 3; ++variant) {
        // 0: pull (kernel on GPU1 reads GPU0, writes local); 1: push (kernel on GPU0 reads local, writes GPU1);
        // 2: cudaMemcpyPeerAsync GPU0 -> GPU1 (copy engines)
        const int dev = variant == 0 ? 1 : 0;
        CK(cudaSetDevice(dev));
        CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
        const uint4 *src = (const uint4 *)(variant == 0 ? a0 : a0);
        uint4 *dst = (uint4 *)(variant == 0 ? b1 : b1);
        for (int threads : {256, 512, 1024}) {
            for (int bps : {1, 2, 4}) {
                if (variant == 2 && (threads != 256 || bps != 1)) continue;
                float best = 1e9;
                for (int rep = 0; rep < 6; ++rep) {
                    CK(cudaEventRecord(e0));
                    if (variant == 2) CK(cudaMemcpyPeerAsync(dst, 1, src, 0, bytes));
                    else copy16<4><<<sms * bps, threads>>>(src, dst, n);
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
                    if (rep >= 1 && ms < best) best = ms;
                }
                printf("%-6s threads=%4d blocks/SM=%d  %.1f GB/s  (%.1f us)\n",
                       variant == 0 ? "pull" : variant == 1 ? "push" : "memcpy", threads, bps,
                       bytes / (best * 1e-3) / 1e9, best * 1e3);
            }
        }
    }
    return 0;
}
