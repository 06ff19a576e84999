// Streaming read ceiling with TMA bulk copies (cp.async.bulk global->shared,
// mbarrier completion) vs the plain 16-byte-load kernel: a persistent CTA per
// SM keeps STAGES chunks of CHUNK bytes in flight and reduces each chunk from
// shared memory (popcount) once its mbarrier completes.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tma_read.cu -o tma_read
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *b, uint32_t parity) {
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(saddr(b)), "r"(parity) : "memory");
    return ok != 0;
}

template <int STAGES, int CHUNK>
__global__ void tma_read(const uint8_t *p, size_t nbytes, unsigned *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const size_t nch = nbytes / CHUNK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s) {
            const size_t c = blockIdx.x + (size_t)s * gridDim.x;
            if (c < nch) {
                mbar_expect(&full[s], CHUNK);
                bulk_g2s(sm + s * CHUNK, p + c * CHUNK, CHUNK, &full[s]);
            }
        }
    unsigned acc = 0;
    for (size_t it = 0;; ++it) {
        const size_t c = blockIdx.x + it * gridDim.x;
        if (c >= nch) break;
        const int s = (int)(it % STAGES);
        const uint32_t par = (uint32_t)((it / STAGES) & 1);
        while (!mbar_try(&full[s], par)) {
        }
        const uint4 *v = (const uint4 *)(sm + s * CHUNK);
#pragma unroll 4
        for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) {
            const uint4 x = v[i];
            acc += __popc(x.x ^ x.y) + __popc(x.z ^ x.w);
        }
        __syncthreads();  // slot s consumed by every thread
        if (threadIdx.x == 0) {
            const size_t c2 = blockIdx.x + (it + STAGES) * gridDim.x;
            if (c2 < nch) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect(&full[s], CHUNK);
                bulk_g2s(sm + s * CHUNK, p + c2 * CHUNK, CHUNK, &full[s]);
            }
        }
    }
    if (acc == 0xFFFFFFFFu) *out = acc;
}

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__global__ void ldg_read(const uint4 *__restrict__ p, size_t n, unsigned *out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (; i + 7 * stride < n; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_stream(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __popc(v[u].x ^ v[u].y) + __popc(v[u].z ^ v[u].w);
    }
    for (; i < n; i += stride) acc += ld_stream(p + i).x;
    if (acc == 0xFFFFFFFFu) *out = acc;
}

int main(int argc, char **argv) {
    const size_t bytes = argc > 1 ? (size_t)atoll(argv[1]) : 603979776ull;
    uint8_t *p; unsigned *o; char *fl, *fr;
    cudaMalloc(&p, bytes); cudaMalloc(&o, 4); cudaMalloc(&fl, 256u << 20); cudaMalloc(&fr, 256u << 20);
    cudaMemset(p, 0x5a, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char *name, auto launch) {
        float best = 1e9, sum = 0; int cnt = 0;
        for (int r = 0; r < 12; ++r) {
            cudaMemset(fl, r, 256u << 20);  // evict (write) ...
            cudaMemcpy(fr, fl, 256u << 20, cudaMemcpyDeviceToDevice);  // ... and read
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (r >= 2) { best = ms < best ? ms : best; sum += ms; cnt++; }
        }
        cudaError_t e = cudaGetLastError();
        printf("%-26s best %.1f us (%.0f GB/s)  mean %.1f us  %s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
               sum / cnt * 1e3, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    run("ldg grid 592x256 U8", [&] { ldg_read<<<sms * 4, 256>>>((const uint4 *)p, bytes / 16, o); });
#define TMA(ST, CH, TH, BPS)                                                                              \
    {                                                                                                    \
        cudaFuncSetAttribute(tma_read<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * CH);   \
        char nm[64]; snprintf(nm, 64, "tma %dx%dK thr%d bps%d", ST, CH / 1024, TH, BPS);                  \
        run(nm, [&] { tma_read<ST, CH><<<sms * BPS, TH, ST * CH>>>(p, bytes, o); });                   \
    }
    TMA(6, 32768, 256, 1)
    TMA(12, 16384, 256, 1)
    TMA(3, 65536, 256, 1)
    TMA(6, 32768, 512, 1)
    TMA(3, 32768, 256, 2)
    TMA(6, 16384, 256, 2)
    return 0;
}
