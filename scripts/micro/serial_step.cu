// Microbenchmark (dev tool): cost per step of the sweep's serial-warp recurrence
// variants.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 serial_step.cu -o serial_step
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long bits(double v) { return (unsigned long long)__double_as_longlong(v); }

template <int VAR>
__global__ void kern(int K, int r, double *out, const double *band, long long *cyc) {
    __shared__ double s_c[64];
    __shared__ double s_band[128 * 32];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64; i += 32) s_c[i] = 1.0 + i;
    for (int i = threadIdx.x; i < 128 * 32; i += 32) s_band[i] = 1e-3 * (i % 7);
    __syncwarp();
    volatile double *v_c = s_c;
    double acc = 0.0, yprev = 0.0;
    long long t0 = clock64();
    double cn = v_c[0];
    for (int t = 0; t < K; ++t) {
        const int slot = t & 63;
        const double qv = (lane < r && t + lane < K) ? s_band[((t + lane) & 127) * 32 + lane] : 0.0;
        const double yb = __shfl_sync(0xffffffff, yprev, 0);
        if (lane != 0) acc = fma(qv, yb, acc);
        if (VAR & 64) {
            double cc = cn;
            if (bits(cc) == 0x7ff0dead00000000ull) {
                do { cc = v_c[slot]; } while (bits(cc) == 0x7ff0dead00000000ull);
            }
            double y = fma(-qv, yprev, cc - acc);
            y = isnan(y) ? 0.0 : y;
            if (lane == 0) { v_c[slot] = cc + 1.0; __stcg(out + t, y); }
            cn = v_c[(t + 1) & 63];
            yprev = y;
        } else if (VAR & 32) {
            double cc;
            do { cc = v_c[slot]; } while (bits(cc) == 0x7ff0dead00000000ull);
            double y = fma(-qv, yprev, cc - acc);
            y = isnan(y) ? 0.0 : y;
            if (lane == 0) { v_c[slot] = cc + 1.0; __stcg(out + t, y); }
            yprev = y;
        } else if (lane == 0) {
            double cc;
            if (VAR & 1) { while (bits(cc = v_c[slot]) == 0x7ff0dead00000000ull) {} }
            else cc = s_c[slot];
            if (VAR & 2) v_c[slot] = cc + 1.0;
            double y = fma(-qv, yprev, cc - acc);
            if (VAR & 4) y = isnan(y) ? 0.0 : y;
            if (VAR & 8) __stcg(out + t, y);
            if (VAR & 16) out[t] = y;
            yprev = y;
        }
        acc = __shfl_down_sync(0xffffffff, acc, 1);
        if (lane >= r - 1) acc = 0.0;
    }
    long long t1 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; out[K] = yprev; }
}

int main() {
    int K = 4096, r = 12;
    double *out, *band; long long *cyc;
    cudaMalloc(&out, (K + 1) * 8); cudaMalloc(&band, 8 * 1024); cudaMalloc(&cyc, 8);
    long long h;
#define RUN(V) kern<V><<<1, 32>>>(K, r, out, band, cyc); kern<V><<<1, 32>>>(K, r, out, band, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("variant %2d: %.1f cycles/step\n", V, (double)h / K);
    RUN(64) RUN(32) RUN(0) RUN(1) RUN(3) RUN(7) RUN(15) RUN(23) RUN(8) RUN(16)
    return 0;
}
