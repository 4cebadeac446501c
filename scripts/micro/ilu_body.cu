// The arithmetic step of the 3-D row-block ILU in isolation (dev tool): B rows x (R+1)
// planes of separately rounded multiply-subtract per thread, operands from shared memory.
#include <cstdio>
#include <cuda_runtime.h>

template <int B, int RP, int TPB, bool BRANCHY>
__global__ void __launch_bounds__(TPB, 1) body(double *out, int nsteps, unsigned zm) {
    extern __shared__ double sm[];
    double *stage = sm;                 // [4][RP][TPB]
    double *ls = sm + 4 * RP * TPB;     // [64][B]
    for (int q = threadIdx.x; q < 4 * RP * TPB; q += TPB) stage[q] = 1e-3 * (q % 97);
    for (int q = threadIdx.x; q < 64 * B; q += TPB) ls[q] = 1e-4 * (q % 13);
    __syncthreads();
    double v[B][RP];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int j = 0; j < RP; ++j) v[b][j] = 1.0 + b + j + threadIdx.x;
    const int tid = threadIdx.x;
    for (int e = 0; e < nsteps; ++e) {
        const double *src = stage + (size_t)(e & 3) * RP * TPB + tid;
        double l[B];
#pragma unroll
        for (int b = 0; b < B; ++b) l[b] = ls[(e & 63) * B + b];
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            if (!BRANCHY || ((zm >> j) & 1u)) {
                const double u = src[j * TPB];
#pragma unroll
                for (int b = 0; b < B; ++b) v[b][j] = __dsub_rn(v[b][j], __dmul_rn(l[b], u));
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int j = 0; j < RP; ++j) s += v[b][j];
    out[blockIdx.x * TPB + tid] = s;
}

template <int B, int RP, int TPB, bool BR>
void run(const char *name) {
    double *out;
    cudaMalloc(&out, 148 * TPB * 8);
    const size_t smem = (4 * RP * TPB + 64 * B) * 8;
    cudaFuncSetAttribute(body<B, RP, TPB, BR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int n = 200000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    body<B, RP, TPB, BR><<<148, TPB, smem>>>(out, 1000, 0xFFFFFFFFu);
    cudaEventRecord(e0);
    body<B, RP, TPB, BR><<<148, TPB, smem>>>(out, n, 0xFFFFFFFFu);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double clk = ms * 1e-3 * 1.965e9 / n;
    printf("%s: B=%d threads=%d: %.0f clk/step, %.1f FP64 lanes/clk/SM (err %s)\n", name, B, TPB, clk,
           2.0 * B * RP * TPB / clk, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run<4, 11, 512, false>("plain");
    run<4, 11, 512, true>("uniform branch per plane");
    run<3, 11, 512, false>("plain");
    run<2, 11, 512, false>("plain");
    run<4, 11, 256, false>("plain");
    return 0;
}
