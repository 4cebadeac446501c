// Microbenchmark (dev tool): cross-SM flag ping-pong latency on B200 for
// several publish/poll flavours.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long ld_relaxed(const long long *p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ long long ld_acquire(const long long *p) {
    long long v;
    asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ long long ld_volatile(const long long *p) { return *(volatile const long long *)p; }

template <int PUB, int POLL>
__global__ void pingpong(long long *a, long long *b, int iters, long long *out) {
    // block 0 and block 1 land on different SMs (grid of 2, 1 warp each)
    if (threadIdx.x != 0) return;
    long long *mine = blockIdx.x == 0 ? a : b;
    long long *theirs = blockIdx.x == 0 ? b : a;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (blockIdx.x == 0) {
            // publish i, wait for the echo
            if (PUB == 0) __stcg(mine, (long long)i);
            else if (PUB == 1) asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(mine), "l"((long long)i) : "memory");
            else if (PUB == 2) atomicExch((unsigned long long *)mine, (unsigned long long)i);
            else *(volatile long long *)mine = i;
            while ((POLL == 0 ? ld_relaxed(theirs) : POLL == 1 ? ld_acquire(theirs) : ld_volatile(theirs)) != i) {}
        } else {
            while ((POLL == 0 ? ld_relaxed(theirs) : POLL == 1 ? ld_acquire(theirs) : ld_volatile(theirs)) != i) {}
            if (PUB == 0) __stcg(mine, (long long)i);
            else if (PUB == 1) asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(mine), "l"((long long)i) : "memory");
            else if (PUB == 2) atomicExch((unsigned long long *)mine, (unsigned long long)i);
            else *(volatile long long *)mine = i;
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
}

int main() {
    long long *a, *b, *out, h;
    cudaMalloc(&a, 4096); cudaMalloc(&b, 4096); cudaMalloc(&out, 8);
    int iters = 2000;
    const char *pub[] = {"st.cg", "st.release", "atom.exch", "st.volatile"};
    const char *poll[] = {"ld.relaxed", "ld.acquire", "ld.volatile"};
#define RUN(P, Q) cudaMemset(a, 0, 8); cudaMemset(b, 0, 8); pingpong<P, Q><<<2, 32>>>(a, b, iters, out); cudaDeviceSynchronize(); cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost); printf("%-12s %-12s round trip %.0f cycles = %.2f us @1.965GHz\n", pub[P], poll[Q], (double)h / iters, (double)h / iters / 1965.0);
    RUN(0, 0) RUN(0, 2) RUN(1, 0) RUN(1, 1) RUN(2, 0) RUN(3, 2)
    return 0;
}
