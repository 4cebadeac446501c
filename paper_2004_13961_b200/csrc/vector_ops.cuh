// Deterministic double-double reductions and the fused PCG vector updates.
#pragma once

#include "lp_common.cuh"

namespace lp {

struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd dd_two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}

__device__ __forceinline__ dd dd_quick(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}

__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = dd_two_sum(a.hi, b.hi);
    dd t = dd_two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = dd_quick(s.hi, s.lo);
    s.lo += t.lo;
    return dd_quick(s.hi, s.lo);
}

__device__ __forceinline__ dd dd_add_prod(dd acc, double x, double y) {
    const double p = x * y;
    const double e = fma(x, y, -p);
    return dd_add(acc, {p, e});
}

// Fixed reduction geometry: results are bitwise reproducible for a given n.
constexpr int RED_BLOCKS = 296;   // 2 x 148 SMs
constexpr int RED_THREADS = 256;

// Block-wide dd sum in a fixed order; result valid in thread 0.
__device__ __forceinline__ dd block_reduce_dd(dd v) {
    __shared__ double sh_hi[32], sh_lo[32];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        dd w{__shfl_down_sync(0xffffffff, v.hi, o), __shfl_down_sync(0xffffffff, v.lo, o)};
        v = dd_add(v, w);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sh_hi[warp] = v.hi;
        sh_lo[warp] = v.lo;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        v = lane < nw ? dd{sh_hi[lane], sh_lo[lane]} : dd{0.0, 0.0};
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            dd w{__shfl_down_sync(0xffffffff, v.hi, o), __shfl_down_sync(0xffffffff, v.lo, o)};
            v = dd_add(v, w);
        }
    }
    return v;
}

// partial[RED_BLOCKS] (dd pairs) -> out (dd pair); out may be device scalars.
int dot_dd(int64_t n, const double *a, const double *b, double *partial, double *out,
           cudaStream_t st);
int finalize_dd(const double *partial, double *out, cudaStream_t st);
// out (dd pair) = sum of v[0..n) in double-double, fixed order (one block)
int sum_lines_dd(const double *v, int64_t n, double *out, cudaStream_t st);

// p = first ? z : z + (rho_new / rho_old) * p   (pcg.py:150-155)
int pcg_update_p(int64_t n, const double *z, double *p, const double *rho_new,
                 const double *rho_old, int first, cudaStream_t st);
// x += alpha p; r -= alpha w with alpha = rho / curv; partial <- r.r  (pcg.py:160-162)
int pcg_update_xr(int64_t n, double *x, double *r, const double *p, const double *w,
                  const double *rho, const double *curv, double *partial, cudaStream_t st);
// r = f - w (initial residual for a nonzero x0)
int vec_sub(int64_t n, const double *f, const double *w, double *r, cudaStream_t st);

}  // namespace lp
