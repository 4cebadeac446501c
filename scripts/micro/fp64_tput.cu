// Vector-pipe FP64 throughput per SM (dev tool): independent DFMA, DMUL+DADD chains.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) tput(double *out, double a, double b, int n) {
    double z[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) z[k] = a + k + threadIdx.x;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            if (MODE == 0) z[m] = fma(z[m], b, a);
            else if (MODE == 1) z[m] = __dsub_rn(z[m], __dmul_rn(a, b + z[(m + 1) & 15] * 0.0));
            else z[m] = __dsub_rn(z[m], __dmul_rn(a, b));
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += z[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char *name, int threads, double ops_per_iter, int n = 20000) {
    double *out;
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    tput<MODE><<<148, threads>>>(out, 0.999, 1.0000001, n);
    cudaEventRecord(e0);
    tput<MODE><<<148, threads>>>(out, 0.999, 1.0000001, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double insts = 148.0 * threads * 16.0 * n * ops_per_iter;
    printf("%s threads=%d: %.3f ms, %.2f T DP-inst-lanes/s, %.1f lanes/clk/SM @1.965GHz\n", name, threads, ms,
           insts / ms / 1e9, insts / (ms * 1e-3) / 148 / 1.965e9);
    cudaFree(out);
}

int main() {
    run<0>("DFMA", 512, 1);
    run<0>("DFMA", 128, 1);
    run<2>("DMUL(hoisted)+DADD", 512, 1);
    run<1>("DMUL+DADD", 512, 3);
    // sustained: seconds, not milliseconds (power / clock behaviour under a long FP64 load)
    run<0>("DFMA sustained", 512, 1, 4000000);
    run<2>("DADD sustained", 512, 1, 4000000);
    run<0>("DFMA sustained", 512, 1, 20000000);
    return 0;
}
