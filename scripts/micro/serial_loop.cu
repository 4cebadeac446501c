// Cycles per step of the sweep's serial recurrence, with pieces removed (dev tool).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_addr(const void *p) {
    unsigned a;
    asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(p));
    return a;
}
__device__ __forceinline__ double lds(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds2(unsigned a, double &x, double &y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ double lds_v(unsigned a) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_v(unsigned a, double v) {
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

constexpr int NQ = 16, BRING = 128, RING = 64;

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ void mbar_init(unsigned a, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned a, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void *src, unsigned bytes, unsigned mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 ::"r"(a), "r"(parity) : "memory");
}

template <int V>
__global__ void serial(double *out, long long *cyc, int K, const double *band, int bs) {
    __shared__ __align__(16) double s_in[BRING * NQ];
    __shared__ double s_d[RING];
    const int lane = threadIdx.x & 31;
    out += (size_t)blockIdx.x * (K + 64);
    if (threadIdx.x < blockDim.x - 32) {   // idle warps wait at a barrier, as in the sweep kernel
        __syncthreads();
        return;
    }
    for (int i = lane; i < BRING * NQ; i += 32) s_in[i] = 1e-3 * (i % 7);
    for (int i = lane; i < RING; i += 32) s_d[i] = 1.0;
    __syncwarp();
    constexpr unsigned RB = BRING * NQ * 8;
    const unsigned in0 = smem_addr(s_in), d0 = smem_addr(s_d);
    unsigned roff = 0, doff = 0, jl = lane;
    double sp = 0.0, yprev = 0.0, e1 = 0.0, e1n, rdn;
    lds2(in0, e1n, rdn);
    double qn = (jl >= 2 && jl < NQ) ? lds(in0 + 8 * jl) : 0.0;
    double spn = 0.0, dn = lds_v(d0);
    double *outp = out;
    long long t0 = clock64();
    auto stage = [&](int u0) {
        if (V & 32) {
            for (int e = lane; e < 32 * (NQ / 2); e += 32) {
                const int rr = e / (NQ / 2), q = e % (NQ / 2);
                const int ix = u0 + rr;
                if (ix < K) cp_async16(s_in + (size_t)(ix & (BRING - 1)) * NQ + 2 * q, band + (size_t)ix * bs + 2 * q);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    };
    __shared__ __align__(8) unsigned long long mbar[4];
    const unsigned mb0 = smem_addr(mbar);
    if (V & 128) {
        if (lane == 0) for (int i = 0; i < 4; ++i) mbar_init(mb0 + 8 * i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
    }
    auto tstage = [&](int c) {   // chunk c = rows [32c, 32c+32), contiguous [K][NQ]
        if (lane == 0 && 32 * c < K) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect(mb0 + 8 * (c & 3), 32 * NQ * 8);
            bulk_g2s(in0 + (c & 3) * 32 * NQ * 8, band + (size_t)32 * c * NQ, 32 * NQ * 8, mb0 + 8 * (c & 3));
        }
    };
    if (V & 128) { tstage(0); tstage(1); tstage(2); }
    else { stage(0); stage(32); stage(64); }
    if (V & 32) asm volatile("cp.async.wait_group 2;" ::: "memory");
    for (int t = 0; t < K; ++t) {
        if ((V & 128) && (t & 31) == 0) {
            const int c = t >> 5;
            tstage(c + 3);
            if (32 * (c + 1) < K) mbar_wait(mb0 + 8 * ((c + 1) & 3), ((c + 1) >> 2) & 1);
            if (c == 0) mbar_wait(mb0, 0);
        }
        if ((V & 32) && (t & 31) == 0) {
            stage(t + 96);
            if (!(V & 64)) asm volatile("cp.async.wait_group 2;" ::: "memory");
            __syncwarp();
        }
        const double q = qn, e1c = e1n, rd = rdn, spt = spn;
        double d = (V & 16) ? 1.0 : dn;
        const double y = fma(-e1, yprev, fma(rd, d, -spt));
        if (!(V & 1)) sts_v(d0 + doff, 2.0);
        if (!(V & 2)) __stcg(outp, y);
        outp += 1;
        doff = (doff + 8) & (RING * 8 - 1);
        if (!(V & 1)) dn = lds_v(d0 + doff);
        if (!(V & 4)) spn = __shfl_sync(0xffffffff, sp, (t + 1) & 31);
        else spn = sp;
        roff = (roff + NQ * 8) & (RB - 1);
        jl = (jl - 1) & 31;
        if (!(V & 8)) {
            lds2(in0 + roff, e1n, rdn);
            qn = (jl >= 2 && jl < NQ) ? lds(in0 + roff + 8 * jl) : 0.0;
        }
        sp = ((unsigned)lane == ((unsigned)t & 31)) ? 0.0 : fma(q, y, sp);
        e1 = e1c;
        yprev = y;
    }
    long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) cyc[V & 63] = t1 - t0;
    out[K + lane] = sp + yprev;
    if (blockDim.x > 32) __syncthreads();
}

template <int V>
double run(double *out, long long *cyc, int K, const double *band, int nb = 1, int nt = 32) {
    long long h = 0;
    serial<V><<<nb, nt>>>(out, cyc, K, band, 42);
    serial<V><<<nb, nt>>>(out, cyc, K, band, 42);
    cudaMemcpy(&h, cyc + (V & 63), 8, cudaMemcpyDeviceToHost);
    return (double)h / K;
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    const int K = 4096;
    double *out, *band;
    long long *cyc;
    cudaMalloc(&out, (size_t)148 * (K + 64) * 8);
    cudaMalloc(&cyc, 64 * 8);
    cudaMalloc(&band, (size_t)K * 42 * 8);
    cudaMemset(band, 0, (size_t)K * 42 * 8);
    printf("%-28s %.1f\n", "full", run<0>(out, cyc, K, band));
    printf("%-28s %.1f\n", "no v_d sts/lds", run<1>(out, cyc, K, band));
    printf("%-28s %.1f\n", "no STG", run<2>(out, cyc, K, band));
    printf("%-28s %.1f\n", "no shfl", run<4>(out, cyc, K, band));
    printf("%-28s %.1f\n", "no coef LDS", run<8>(out, cyc, K, band));
    printf("%-28s %.1f\n", "chain only", run<31>(out, cyc, K, band));
    printf("%-28s %.1f\n", "full + staging", run<32>(out, cyc, K, band));
    printf("%-28s %.1f\n", "full + staging, no wait", run<96>(out, cyc, K, band));
    printf("%-28s %.1f\n", "staging no wait, no STG", run<98>(out, cyc, K, band));
    printf("%-28s %.1f\n", "full + TMA bulk staging", run<128>(out, cyc, K, band));
    printf("%-28s %.1f\n", "TMA, 148 CTAs", run<128>(out, cyc, K, band, 148, 32));
    printf("%-28s %.1f\n", "TMA, 1 CTA x 512 thr", run<128>(out, cyc, K, band, 1, 512));
    printf("%-28s %.1f\n", "TMA, 148 CTAs x 512 thr", run<128>(out, cyc, K, band, 148, 512));
    printf("%-28s %.1f\n", "no staging, 148 x 512", run<0>(out, cyc, K, band, 148, 512));
    return 0;
}
