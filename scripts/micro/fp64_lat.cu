// FP64 / shared-memory / shuffle latency and throughput on one warp (dev tool).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double *out, long long *cyc, double a, double b, int n) {
    __shared__ double sm[64];
    sm[threadIdx.x & 63] = a;
    __syncthreads();
    double x = a, y = b;
    long long t0, t1;
    // dependent DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x = fma(x, b, a);
    }
    t1 = clock64();
    cyc[0] = t1 - t0;
    // dependent DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) y = y + x;
    }
    t1 = clock64();
    cyc[1] = t1 - t0;
    // 8 independent DFMA chains (throughput for one warp)
    double z[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = a + k;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
#pragma unroll
            for (int m = 0; m < 8; ++m) z[m] = fma(z[m], b, a);
    }
    t1 = clock64();
    cyc[2] = t1 - t0;
    // dependent shared-memory load chain (address from loaded value)
    volatile double *vs = sm;
    int idx = threadIdx.x & 1;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) idx = (int)vs[idx] & 1;
    }
    t1 = clock64();
    cyc[3] = t1 - t0;
    // dependent shuffle chain
    double s = x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) s = __shfl_sync(0xffffffff, s, (threadIdx.x + 1) & 31);
    }
    t1 = clock64();
    cyc[4] = t1 - t0;
    // FP32 FMA chain for comparison
    float f = a, fb = b;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) f = fmaf(f, fb, 1.0f);
    }
    t1 = clock64();
    cyc[5] = t1 - t0;
    double zz = 0;
    for (int k = 0; k < 8; ++k) zz += z[k];
    out[threadIdx.x] = x + y + zz + s + idx + f;
}

int main() {
    double *out;
    long long *cyc, h[6];
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 6 * 8);
    const int n = 1000;
    lat<<<1, 32>>>(out, cyc, 0.999, 1.0000001, n);
    lat<<<1, 32>>>(out, cyc, 0.999, 1.0000001, n);
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    const double ops = 16.0 * n;
    printf("DFMA dependent latency     %.1f cycles\n", h[0] / ops);
    printf("DADD dependent latency     %.1f cycles\n", h[1] / ops);
    printf("DFMA 8 chains, per instr   %.2f cycles (one warp)\n", h[2] / (ops * 8));
    printf("LDS dependent latency      %.1f cycles\n", h[3] / ops);
    printf("SHFL dependent latency     %.1f cycles\n", h[4] / ops);
    printf("FFMA dependent latency     %.1f cycles\n", h[5] / ops);
    return 0;
}
