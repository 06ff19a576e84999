// NVLink GPU0 -> GPU1 transfer of 141 MiB split between a receiver pull
// (kernel on GPU1 loading GPU0 memory) and a sender push (kernel on GPU0
// storing into GPU1 memory), run concurrently: does driving one link
// direction from both ends beat the pull alone?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a p2p_split.cu -o p2p_split
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void copy16(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint4 v0 = src[i], v1 = src[i + stride], v2 = src[i + 2 * stride], v3 = src[i + 3 * stride];
        dst[i] = v0; dst[i + stride] = v1; dst[i + 2 * stride] = v2; dst[i + 3 * stride] = v3;
    }
    for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
    const size_t bytes = 141ull << 20, n = bytes / 16;
    void *src0, *dst1;
    CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); CK(cudaMalloc(&src0, bytes)); CK(cudaMemset(src0, 1, bytes));
    CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMalloc(&dst1, bytes));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaStream_t s0, s1;
    CK(cudaSetDevice(0)); CK(cudaStreamCreate(&s0));
    CK(cudaSetDevice(1)); CK(cudaStreamCreate(&s1));
    for (int pct : {100, 70, 60, 50, 0}) {  // share pulled by GPU1
        const size_t n_pull = n * pct / 100, n_push = n - n_pull;
        double best = 1e9;
        for (int rep = 0; rep < 8; ++rep) {
            CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
            CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
            const auto t0 = std::chrono::high_resolution_clock::now();
            if (n_pull) {
                CK(cudaSetDevice(1));
                copy16<<<sms * 2, 512, 0, s1>>>((const uint4 *)src0, (uint4 *)dst1, n_pull);
            }
            if (n_push) {
                CK(cudaSetDevice(0));
                copy16<<<sms * 2, 512, 0, s0>>>((const uint4 *)src0 + n_pull, (uint4 *)dst1 + n_pull, n_push);
            }
            CK(cudaStreamSynchronize(s0));
            CK(cudaStreamSynchronize(s1));
            const double us = std::chrono::duration<double, std::micro>(std::chrono::high_resolution_clock::now() - t0).count();
            if (rep >= 2 && us < best) best = us;
        }
        printf("pull %3d%% / push %3d%%: %.1f us  %.1f GB/s (host-timed, incl. launch)\n", pct, 100 - pct, best, bytes / (best * 1e-6) / 1e9);
    }
    return 0;
}
