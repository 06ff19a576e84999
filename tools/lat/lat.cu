// Dependent-latency microbenchmark (one warp): cycles per op for chains of
// DADD, DMUL, SHFL (32/64-bit), LDS.64, BALLOT+POPC, IADD64, ISETP64+SEL.
#include <cstdio>
#include <cstdint>
#define N 4096
__global__ void k(double *out, long long *cyc, const double *in) {
    __shared__ long long sm[64];
    const int lane = threadIdx.x;
    sm[lane] = lane; sm[lane + 32] = lane;
    __syncwarp();
    double x = in[lane], y = in[lane + 32];
    long long t0, t1;
    // DADD
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __dadd_rn(x, y);
    t1 = clock64(); if (lane == 0) cyc[0] = t1 - t0;
    // DMUL
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __dmul_rn(x, 1.0000001);
    t1 = clock64(); if (lane == 0) cyc[1] = t1 - t0;
    // SHFL 64-bit
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_down_sync(0xffffffffu, x, 1);
    t1 = clock64(); if (lane == 0) cyc[2] = t1 - t0;
    // SHFL 32-bit
    int v = lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
    t1 = clock64(); if (lane == 0) cyc[3] = t1 - t0;
    // LDS.64 chain (pointer chase in smem)
    long long p = lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) p = sm[p & 63];
    t1 = clock64(); if (lane == 0) cyc[4] = t1 - t0;
    // BALLOT+POPC chain
    int c = lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) c = __popc(__ballot_sync(0xffffffffu, c > i % 32)) ;
    t1 = clock64(); if (lane == 0) cyc[5] = t1 - t0;
    // 64-bit compare+select chain
    long long a = lane, b = 7;
    t0 = clock64();
    for (int i = 0; i < N; ++i) a = (a > b) ? a - b : a + b;
    t1 = clock64(); if (lane == 0) cyc[6] = t1 - t0;
    // FABS(DSUB) + DSETP + SEL chain
    double g = x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) g = (fabs(__dsub_rn(g, y)) > 1.0) ? g * 0.5 : g + 1.0;
    t1 = clock64(); if (lane == 0) cyc[7] = t1 - t0;
    out[lane] = x + v + p + c + a + g;
}
int main() {
    double *o, *in; long long *c;
    cudaMalloc(&o, 64 * 8); cudaMalloc(&in, 64 * 8); cudaMalloc(&c, 64 * 8);
    cudaMemset(in, 0, 64 * 8);
    k<<<1, 32>>>(o, c, in);
    k<<<1, 32>>>(o, c, in);
    long long h[8];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    const char *nm[8] = {"DADD", "DMUL", "SHFL64", "SHFL32+IADD", "LDS64 chase", "BALLOT+POPC", "I64 cmp+sel+add", "DSUB/FABS/DSETP/SEL/DMUL|DADD"};
    for (int i = 0; i < 8; ++i) printf("%-32s %.1f cycles/op\n", nm[i], (double)h[i] / N);
    return 0;
}
