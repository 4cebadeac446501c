// Microbenchmark (dev tool): latency of a dependent SHFL chain in warp 0 while
// the other 15 warps of the CTA do different kinds of polling.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long ld_relaxed(const long long *p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int MODE>
__global__ void kern(long long *flag, long long *out, int rounds) {
    __shared__ volatile long long s_flag;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_flag = 0;
    __syncthreads();
    if (warp == 0) {
        double v = lane;
        long long t0 = clock64();
        for (int i = 0; i < rounds; ++i) {
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
        }
        long long t1 = clock64();
        if (lane == 0) { out[0] = (t1 - t0) / (rounds * 5); out[1] = (long long)v; }
        if (lane == 0) { s_flag = 1; *(volatile long long *)flag = 1; }
    } else {
        if (MODE == 0) return;                         // idle siblings
        if (MODE == 1) { while (s_flag == 0) {} }      // tight smem poll (one lane group per warp, all lanes)
        if (MODE == 2) { while (lane == 0 && s_flag == 0) {} }   // divergent single-lane smem poll
        if (MODE == 3) { while (ld_relaxed(flag) == 0) {} }      // global relaxed poll, all lanes
        if (MODE == 4) { while (ld_relaxed(flag) == 0) __nanosleep(20); }
        if (MODE == 5) { if (lane == 0) while (ld_relaxed(flag) == 0) __nanosleep(20); __syncwarp(); }
    }
}

int main() {
    long long *flag, *out, h[2];
    cudaMalloc(&flag, 8); cudaMalloc(&out, 16);
    const char *names[] = {"idle", "smem poll all lanes", "smem poll lane0 (divergent)",
                           "global relaxed poll all lanes", "global poll + nanosleep", "lane0 global poll + nanosleep"};
#define RUN(M) cudaMemset(flag, 0, 8); kern<M><<<1, 512>>>(flag, out, 2000); cudaDeviceSynchronize(); cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost); printf("%-32s %lld cycles per dependent SHFL round\n", names[M], h[0]);
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5)
    return 0;
}
