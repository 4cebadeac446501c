// Latency of one ILU pivot application (apply_pivot) on one warp (dev tool).
#include <cstdio>
#include <cuda_runtime.h>

template <bool FULL, int MODE>
__device__ __forceinline__ double apply_pivot(double *row, const unsigned *colmask, const double *uk,
                                              int s, int ox, int oy, int r, int W, int S, int c, int lane) {
    constexpr int MJ = 16;
    const double l = MODE == 1 ? row[s] * (1.0 / uk[c]) : __ddiv_rn(row[s], uk[c]);
    const int txlo = max(-r, ox - r), txhi = min(r, ox + r);
    const int tx = txlo + lane;
    const int nty = min(r, oy + r) - oy + 1;
    unsigned jm = (1u << nty) - 1u;
    if (tx <= ox) jm &= ~1u;
    if (tx > txhi) jm = 0;
    else if (!FULL) jm &= colmask[tx + r] >> (oy + r);
    const int t0 = (tx > txhi ? r : tx + r) + W * (oy + r);
    const int d = c - s;
    if (MODE == 2) return l;
    double u[MJ], v[MJ];
#pragma unroll
    for (int j = 0; j < MJ; ++j) {
        const int t = min(t0 + W * j, S - 1);
        u[j] = uk[min(t + d, S - 1)];
        v[j] = row[t];
    }
#pragma unroll
    for (int j = 0; j < MJ; ++j)
        if ((jm >> j) & 1u) row[t0 + W * j] = __dsub_rn(v[j], __dmul_rn(l, u[j]));
    __syncwarp();
    return l;
}

template <int MODE>
__global__ void k(double *out, long long *cyc, int n) {
    extern __shared__ double sm[];
    const int r = 12, W = 25, S = 625, c = 312;
    double *row = sm, *uk = sm + 640;
    unsigned *cm = (unsigned *)(sm + 1280);
    const int lane = threadIdx.x;
    for (int i = lane; i < 640; i += 32) { row[i] = 1.0 + i * 1e-3; uk[i] = 2.0 + i * 1e-3; }
    if (lane < 32) cm[lane] = ~0u;
    __syncwarp();
    long long t0 = clock64();
    double acc = 0;
    for (int it = 0; it < n; ++it) {
        const int m = 1 + (it % 12);
        const int s = (r - m) + W * r;
        acc += apply_pivot<true, MODE>(row, cm, uk, s, -m, 0, r, W, S, c, lane);
        if (lane == 0) row[s] = 1.0 + 1e-9 * it;
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) { cyc[MODE] = t1 - t0; out[0] = acc; }
}

int main() {
    double *out; long long *cyc, h[4];
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
    const int n = 2000;
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 32, 16384>>>(out, cyc, n);
        k<1><<<1, 32, 16384>>>(out, cyc, n);
        k<2><<<1, 32, 16384>>>(out, cyc, n);
    }
    cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("apply (ddiv_rn)      %.0f cycles\napply (mul by rcp)   %.0f cycles\ndivide only          %.0f cycles\n",
           (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
    return 0;
}
