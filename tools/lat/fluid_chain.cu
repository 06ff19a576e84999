// Latency of the fluid process's dependent chain on one warp (lane = stage):
//   A  one round = fp64 shuffle of the partner + fma(y, 0.5, x * 0.5)
//   B  A + the history-row store (STS.64) per round (fluid_spec's loop)
//   C  two rounds per exchange: three fp64 shuffles (partner, partner's
//      partner under the other matching, ...) then two dependent fmas
//   D  raw SHFL.IDX (32-bit) chain, E raw DFMA chain
// Cycles per round from clock64 over 4096 rounds.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a fluid_chain.cu -o fc && ./fc
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k(double *out, long long *cyc, int mode) {
    __shared__ double hist[64 * 33];
    const int lane = threadIdx.x;
    double x = 1.0 + lane;
    const int pa = (lane & 1) ? lane - 1 : lane + 1;                    // pairs (0,1)(2,3)...
    const int pb = (lane & 1) ? (lane + 1 < 32 ? lane + 1 : lane) : (lane ? lane - 1 : lane);
    const int pab = __shfl_sync(~0u, pa, pb);                           // partner of pb under pa
    unsigned u = lane;
    __syncwarp();
    const long long t0 = clock64();
    if (mode == 0 || mode == 1) {
        for (int r = 0; r < N; r += 2) {
            if (mode == 1) hist[(r & 63) * 33 + lane] = x;
            double y = __shfl_sync(~0u, x, pa);
            x = fma(y, 0.5, x * 0.5);
            if (mode == 1) hist[((r + 1) & 63) * 33 + lane] = x;
            y = __shfl_sync(~0u, x, pb);
            x = fma(y, 0.5, x * 0.5);
        }
    } else if (mode == 2) {
        for (int r = 0; r < N; r += 2) {
            const double ya = __shfl_sync(~0u, x, pa);   // x at pa(s)
            const double yb = __shfl_sync(~0u, x, pb);   // x at pb(s)
            const double yab = __shfl_sync(~0u, x, pab); // x at pa(pb(s))
            const double x1 = fma(ya, 0.5, x * 0.5);     // round 1 at s
            const double x1b = fma(yab, 0.5, yb * 0.5);  // round 1 at pb(s)
            x = fma(x1b, 0.5, x1 * 0.5);                 // round 2 at s
        }
    } else if (mode == 3) {
        for (int r = 0; r < N; ++r) u = __shfl_sync(~0u, u, (u + 1) & 31);
        x = u;
    } else {
        for (int r = 0; r < N; ++r) x = fma(x, 0.5, 0.25);
    }
    const long long t1 = clock64();
    out[lane] = x + hist[lane];
    if (lane == 0) *cyc = t1 - t0;
}

int main() {
    double *o;
    long long *c, h;
    cudaMalloc(&o, 32 * 8);
    cudaMalloc(&c, 8);
    const char *name[] = {"A shfl+fma", "B shfl+fma+sts", "C 2 rounds/exchange", "D SHFL.IDX chain",
                          "E DFMA chain"};
    for (int m = 0; m < 5; ++m) {
        for (int rep = 0; rep < 3; ++rep) k<<<1, 32>>>(o, c, m);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-22s %.1f cycles per round\n", name[m], (double)h / N);
    }
    return 0;
}
