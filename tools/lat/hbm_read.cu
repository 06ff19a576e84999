// Practical HBM3e read ceiling on B200: a minimal streaming reduction over
// 604 MB (config 2's mask bytes) with the same load flavour as k_profile
// (ld.global.nc.L1::no_allocate.L2::256B.v4), several grid shapes / loads in
// flight.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a hbm_read.cu -o hbm_read
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int U>
__global__ void rd(const uint4 *__restrict__ p, size_t n, unsigned *out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += __popc(v[u].x ^ v[u].y) + __popc(v[u].z ^ v[u].w);
    }
    for (; i < n; i += stride) acc += ld_stream(p + i).x;
    if (acc == 0xFFFFFFFFu) *out = acc;
}

// 256-bit loads (ld.global...v8.b32, LDG.256 on sm_100): U loads of 32 B per thread
struct u8x32 { unsigned a[8]; };
__device__ __forceinline__ u8x32 ld_stream256(const uint4 *p) {
    u8x32 v;
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.a[0]), "=r"(v.a[1]), "=r"(v.a[2]), "=r"(v.a[3]), "=r"(v.a[4]), "=r"(v.a[5]),
                   "=r"(v.a[6]), "=r"(v.a[7]) : "l"(p));
    return v;
}
template <int U>
__global__ void rd256(const uint4 *__restrict__ p, size_t n, unsigned *out) {
    const size_t n2 = n / 2;  // 32-byte elements
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
        u8x32 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream256(p + 2 * (i + u * stride));
#pragma unroll
        for (int u = 0; u < U; ++u)
            acc += __popc(v[u].a[0] ^ v[u].a[1]) + __popc(v[u].a[2] ^ v[u].a[3]) + __popc(v[u].a[4] ^ v[u].a[5]) +
                   __popc(v[u].a[6] ^ v[u].a[7]);
    }
    for (; i < n2; i += stride) acc += ld_stream256(p + 2 * i).a[0];
    if (acc == 0xFFFFFFFFu) *out = acc;
}

// contiguous chunk per warp (k_profile's layout): each warp streams its own range
template <int U>
__global__ void rd_chunk(const uint4 *__restrict__ p, size_t n, unsigned *out) {
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const size_t per = (n + nw - 1) / nw;
    const size_t b = w * per, e = b + per < n ? b + per : n;
    unsigned acc = 0;
    for (size_t i = b + lane; i < e; i += 32 * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = i + 32 * u < e ? ld_stream(p + i + 32 * u) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += __popc(v[u].x ^ v[u].y) + __popc(v[u].z ^ v[u].w);
    }
    if (acc == 0xFFFFFFFFu) *out = acc;
}

// fixed-size tiles dealt round-robin to warps (tile j -> warp j % nwarps,
// or chunks of C consecutive tiles); a warp streams its tile with 8 loads
// in flight per lane, like k_profile's count path
template <int C>
__global__ void rd_tiles(const uint4 *__restrict__ p, size_t n, unsigned *out) {
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const size_t T = 2048;  // 32 KiB tiles
    const size_t ntiles = (n + T - 1) / T;
    unsigned acc = 0;
    for (size_t c0 = w * C; c0 < ntiles; c0 += nw * C) {
        for (size_t t = c0; t < c0 + C && t < ntiles; ++t) {
            const size_t b = t * T, e = b + T < n ? b + T : n;
            for (size_t i = b + lane; i < e; i += 32 * 8) {
                uint4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = i + 32 * u < e ? ld_stream(p + i + 32 * u) : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += __popc(v[u].x ^ v[u].y) + __popc(v[u].z ^ v[u].w);
            }
        }
    }
    if (acc == 0xFFFFFFFFu) *out = acc;
}

int main(int argc, char **argv) {
    const size_t bytes = argc > 1 ? (size_t)atoll(argv[1]) : 603979776ull, n = bytes / 16;
    uint4 *p; unsigned *o; char *fl;
    cudaMalloc(&p, bytes); cudaMalloc(&o, 4); cudaMalloc(&fl, 256u << 20);
    cudaMemset(p, 0x5a, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char *name, auto kern, int blocks, int threads) {
        float best = 1e9, sum = 0; int cnt = 0;
        for (int r = 0; r < 12; ++r) {
            cudaMemset(fl, r, 256u << 20);  // evict
            cudaEventRecord(a);
            kern<<<blocks, threads>>>(p, n, o);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (r >= 2) { best = ms < best ? ms : best; sum += ms; cnt++; }
        }
        printf("%-10s blocks=%5d threads=%4d  best %.1f us (%.0f GB/s)  mean %.1f us (%.0f GB/s)\n", name, blocks,
               threads, best * 1e3, bytes / (best * 1e-3) / 1e9, sum / cnt * 1e3, bytes / (sum / cnt * 1e-3) / 1e9);
    };
    for (int bps : {4}) {
        run("grid-U8", rd<8>, sms * bps, 256);
        run("g256-U4", rd256<4>, sms * bps, 256);
        run("g256-U8", rd256<8>, sms * bps, 256);
        run("g256-U4x2", rd256<4>, sms * bps * 2, 256);
        run("chunk-U8", rd_chunk<8>, sms * bps, 256);
        run("tiles-C1", rd_tiles<1>, sms * bps, 256);
        run("tiles-C2", rd_tiles<2>, sms * bps, 256);
        run("tiles-C4", rd_tiles<4>, sms * bps, 256);
    }
    // flush by READ (clean L2), as bench.py does: rerun with a read flush
    return 0;
}
