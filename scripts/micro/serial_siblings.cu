// Microbenchmark (dev tool): serial-recurrence step cost with 15 sibling warps
// in the CTA polling in different ways.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long bits(double v) { return (unsigned long long)__double_as_longlong(v); }
__device__ __forceinline__ double ld_poll_nc(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_poll(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
template <int MODE>
__global__ void kern(int K, int r, double *out, double *gflag, long long *cyc) {
    __shared__ double s_c[64];
    __shared__ double s_band[128 * 40];
    __shared__ volatile int s_stop;
    __shared__ double s_y[16];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64; i += blockDim.x) s_c[i] = 1.0 + i;
    for (int i = threadIdx.x; i < 128 * 40; i += blockDim.x) s_band[i] = 1e-3 * (i % 7);
    if (threadIdx.x == 0) s_stop = 0;
    __syncthreads();
    volatile double *v_c = s_c;
    if (warp == 15) {
        double acc = 0.0, yprev = 0.0, cn = v_c[0];
        double ynext = ld_poll(gflag);
        if (MODE == 14 && lane == 0) {
            for (int d = 0; d < 8; ++d) {
                unsigned dst = (unsigned)__cvta_generic_to_shared(s_y + (d & 15));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(dst), "l"(gflag + (d & 7)) : "memory");
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
        }
        long long t0 = clock64();
        for (int t = 0; t < K; ++t) {
            const int slot = t & 63;
            const double qi = (lane < r) ? s_band[((t + lane) & 127) * 38 + lane] : 0.0;
            const double qg = (lane <= 2 * r) ? s_band[((t + lane) & 127) * 38 + r + lane] : 0.0;
            double yn = ynext;
            if (MODE == 10) { while (bits(yn) == 0x7ff0dead00000000ull) yn = ld_poll(gflag + (t & 7)); ynext = ld_poll(gflag + ((t + 1) & 7)); }
            else if (MODE == 11) { while (bits(yn) == 0x7ff0dead00000000ull) yn = ld_poll(gflag + (t & 7)); ynext = ld_poll_nc(gflag + ((t + 1) & 7)); }
            else if (MODE == 12) { while (bits(yn) == 0x7ff0dead00000000ull) yn = ld_poll(gflag + (t & 7)); ynext = __ldcg(gflag + ((t + 1) & 7)); }
            else if (MODE == 13) { yn = 0.5; }
            else if (MODE == 14) {
                if (lane == 0) {
                    unsigned dst = (unsigned)__cvta_generic_to_shared(s_y + ((t + 8) & 15));
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(dst), "l"(gflag + ((t + 8) & 7)) : "memory");
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    asm volatile("cp.async.wait_group 8;" ::: "memory");
                }
                __syncwarp();
                yn = ((volatile double *)s_y)[t & 15];
                while (bits(yn) == 0x7ff0dead00000000ull) yn = ld_poll(gflag + (t & 7));
            }
            else yn = ld_poll(gflag + (t & 7));
            const double yb = __shfl_sync(0xffffffff, yprev, 0);
            acc = fma(qg, yn, acc);
            if (lane != 0) acc = fma(qi, yb, acc);
            double cc = cn;
            if (bits(cc) == 0x7ff0dead00000000ull) { do { cc = v_c[slot]; } while (bits(cc) == 0x7ff0dead00000000ull); }
            double y = fma(-qi, yprev, cc - acc);
            y = isnan(y) ? 0.0 : y;
            if (lane == 0) { v_c[slot] = cc + 1.0; __stcg(out + t, y); }
            cn = v_c[(t + 1) & 63];
            yprev = y;
            acc = __shfl_down_sync(0xffffffff, acc, 1);
            if (lane >= 2 * r) acc = 0.0;
        }
        long long t1 = clock64();
        if (lane == 0) { cyc[0] = t1 - t0; out[K] = yprev; s_stop = 1; }
    } else {
        if (MODE == 0 || MODE >= 10) return;
        if (MODE == 1) { if (lane == 0) while (!s_stop) __nanosleep(20); __syncwarp(); }        // ring-wait style
        if (MODE == 2) { if (lane == 0) while (!s_stop) { double v = ld_poll(gflag + 64 + warp); (void)v; __nanosleep(20); } __syncwarp(); }
        if (MODE == 3) { while (!s_stop) {} }                                                    // tight smem spin, all lanes
        if (MODE == 4) { while (!s_stop) __nanosleep(1000); }
    }
}
int main() {
    double *out, *g; long long *cyc, h;
    int K = 4096, r = 12;
    cudaMalloc(&out, (K + 1) * 8); cudaMalloc(&g, 8 * 256); cudaMemset(g, 0, 8 * 256); cudaMalloc(&cyc, 8);
    const char *names[] = {"siblings exit", "lane0 smem poll+sleep20", "lane0 global poll+sleep20", "tight smem spin (all lanes)", "sleep 1us loop", "", "", "", "", "", "prefetched, siblings exit", "prefetch no clobber", "prefetch ldcg", "no poll at all", "cp.async prefetch 8 ahead"};
#define RUN(M) kern<M><<<1, 512>>>(K, r, out, g, cyc); kern<M><<<1, 512>>>(K, r, out, g, cyc); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-30s %.1f cycles/step\n", names[M], (double)h / K);
    RUN(0) RUN(1) RUN(3)
    printf("prefetched poll:\n");
    RUN(10) RUN(13) RUN(14)
    return 0;
}
