// Where the fixed cost of a short HBM read goes (the G = 8 profile share is
// 75.5 MB: ~11 us of transfer at 7 TB/s, ~18 us measured).  One streaming
// read kernel (k_profile's load flavour, 8 x 16 B in flight per lane,
// grid = 148 x 4 CTAs of 256 threads) instrumented with %globaltimer: per
// warp the time of its first instruction, of its first data (first batch of
// loads consumed) and of its end.  Conditions before the timed read:
//   cold   : a 2 GiB read of another buffer (L2 and TLBs hold other pages)
//   touch  : cold, then one 4-byte load per 64 KiB of the buffer (TLB warm,
//            L2 holds only the touched sectors)
//   warm   : cold, then the same read once (TLB warm; L2 holds its tail)
// Per condition: CUDA-event time of the read, and from the stamps the
// launch-to-first-warp, first-warp-to-first-data, and the end spread.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a ramp.cu -o ramp && ./ramp [bytes]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

struct Stamp {
    unsigned long long t0, t1, t2;
};

// contiguous range per warp (k_profile's layout)
__global__ void rd(const uint4 *__restrict__ p, size_t n, Stamp *st, unsigned *out) {
    const unsigned long long t0 = gtime();
    const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const size_t per = (n + nw - 1) / nw;
    const size_t b = w * per, e = b + per < n ? b + per : n;
    unsigned acc = 0;
    unsigned long long t1 = 0;
    for (size_t i = b + lane; i < e; i += 32 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = i + 32 * u < e ? ld_stream(p + i + 32 * u) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __popc(v[u].x ^ v[u].y) + __popc(v[u].z ^ v[u].w);
        if (!t1) t1 = gtime() | (acc & 0);  // after the first batch is consumed
    }
    acc = __reduce_add_sync(0xFFFFFFFFu, acc);
    if (lane == 0) {
        st[w] = Stamp{t0, t1, gtime()};
        if (acc == 0xFFFFFFFFu) *out = acc;
    }
}

__global__ void big_read(const uint4 *__restrict__ p, size_t n, unsigned *out) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t s = (size_t)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (; i < n; i += s) acc += ld_stream(p + i).x;
    if (acc == 0xFFFFFFFFu) *out = acc;
}

__global__ void touch(const unsigned *__restrict__ p, size_t n_words, size_t step, unsigned *out) {
    size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * step;
    unsigned acc = 0;
    if (i < n_words) acc = p[i];
    if (acc == 0xFFFFFFFFu) *out = acc;
}

int main(int argc, char **argv) {
    const size_t bytes = argc > 1 ? strtoull(argv[1], nullptr, 10) : 75497472ull;
    const size_t other = 2ull << 30;
    uint4 *a, *o;
    unsigned *out;
    Stamp *st;
    cudaMalloc(&a, bytes);
    cudaMalloc(&o, other);
    cudaMalloc(&out, 4);
    cudaMemset(a, 0x5a, bytes);
    cudaMemset(o, 0x33, other);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 4, thr = 256, nw = grid * thr / 32;
    cudaMalloc(&st, sizeof(Stamp) * nw);
    std::vector<Stamp> h(nw);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[] = {"cold", "touch", "warm"};
    for (int cond = 0; cond < 3; ++cond) {
        std::vector<double> ev, launch_first, first_data, span, end_spread;
        for (int rep = 0; rep < 12; ++rep) {
            big_read<<<grid, 512>>>(o, other / 16, out);
            if (cond == 1) touch<<<(unsigned)((bytes / 65536 + 255) / 256), 256>>>((const unsigned *)a, bytes / 4, 16384, out);
            if (cond == 2) rd<<<grid, thr>>>(a, bytes / 16, st, out);
            cudaEventRecord(e0);
            rd<<<grid, thr>>>(a, bytes / 16, st, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(h.data(), st, sizeof(Stamp) * nw, cudaMemcpyDeviceToHost);
            unsigned long long s0 = ~0ull, s0max = 0, d0 = ~0ull, dmed, end_max = 0, end_min = ~0ull;
            std::vector<unsigned long long> fd;
            for (auto &x : h) {
                s0 = std::min(s0, x.t0);
                s0max = std::max(s0max, x.t0);
                d0 = std::min(d0, x.t1);
                fd.push_back(x.t1);
                end_max = std::max(end_max, x.t2);
                end_min = std::min(end_min, x.t2);
            }
            std::sort(fd.begin(), fd.end());
            dmed = fd[fd.size() / 2];
            if (rep < 2) continue;
            ev.push_back(ms * 1e3);
            launch_first.push_back((s0max - s0) * 1e-3);
            first_data.push_back((dmed - s0) * 1e-3);
            span.push_back((end_max - s0) * 1e-3);
            end_spread.push_back((end_max - end_min) * 1e-3);
        }
        auto med = [](std::vector<double> v) {
            std::sort(v.begin(), v.end());
            return v[v.size() / 2];
        };
        printf("%-6s bytes=%zu event %.2f us | warp starts spread %.2f us | median first data %.2f us | "
               "first start->last end %.2f us | end spread %.2f us | %.0f GB/s (event)\n",
               names[cond], bytes, med(ev), med(launch_first), med(first_data), med(span), med(end_spread),
               bytes / (med(ev) * 1e-6) / 1e9);
    }
    return 0;
}
