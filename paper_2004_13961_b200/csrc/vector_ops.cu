// PCG vector kernels: deterministic double-double dots and fused updates.
// Reference: pcg.py:77-79 (_dot in 80-bit long double), pcg.py:150-164.
#include "vector_ops.cuh"

namespace lp {
namespace {

__global__ void __launch_bounds__(RED_THREADS)
dot_kernel(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
           double *__restrict__ partial) {
    dd acc{0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < n;
         i += (int64_t)RED_BLOCKS * RED_THREADS)
        acc = dd_add_prod(acc, a[i], b[i]);
    acc = block_reduce_dd(acc);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = acc.hi;
        partial[2 * blockIdx.x + 1] = acc.lo;
    }
}

__global__ void finalize_kernel(const double *__restrict__ partial, double *__restrict__ out) {
    dd acc{0.0, 0.0};
    for (int i = threadIdx.x; i < RED_BLOCKS; i += blockDim.x)
        acc = dd_add(acc, dd{partial[2 * i], partial[2 * i + 1]});
    acc = block_reduce_dd(acc);
    if (threadIdx.x == 0) {
        out[0] = acc.hi;
        out[1] = acc.lo;
    }
}

__global__ void sum_lines_kernel(const double *__restrict__ v, int64_t n, double *__restrict__ out) {
    dd acc{0.0, 0.0};
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = dd_add(acc, dd{v[i], 0.0});
    acc = block_reduce_dd(acc);
    if (threadIdx.x == 0) {
        out[0] = acc.hi;
        out[1] = acc.lo;
    }
}

__global__ void update_p_kernel(int64_t n, const double *__restrict__ z, double *__restrict__ p,
                                const double *__restrict__ rho_new,
                                const double *__restrict__ rho_old, int first) {
    const double beta = first ? 0.0 : __ddiv_rn(rho_new[0], rho_old[0]);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = first ? z[i] : __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

__global__ void __launch_bounds__(RED_THREADS)
update_xr_kernel(int64_t n, double *__restrict__ x, double *__restrict__ r,
                 const double *__restrict__ p, const double *__restrict__ w,
                 const double *__restrict__ rho, const double *__restrict__ curv,
                 double *__restrict__ partial) {
    const double alpha = __ddiv_rn(rho[0], curv[0]);
    dd acc{0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < n;
         i += (int64_t)RED_BLOCKS * RED_THREADS) {
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
        const double ri = __dsub_rn(r[i], __dmul_rn(alpha, w[i]));
        r[i] = ri;
        acc = dd_add_prod(acc, ri, ri);
    }
    acc = block_reduce_dd(acc);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = acc.hi;
        partial[2 * blockIdx.x + 1] = acc.lo;
    }
}

__global__ void sub_kernel(int64_t n, const double *__restrict__ f, const double *__restrict__ w,
                           double *__restrict__ r) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        r[i] = f[i] - w[i];
}

unsigned grid_for(int64_t n) {
    int64_t b = ceil_div(n, 256);
    const int64_t cap = 4 * (int64_t)num_sms();
    return (unsigned)(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

int finalize_dd(const double *partial, double *out, cudaStream_t st) {
    finalize_kernel<<<1, 256, 0, st>>>(partial, out);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int sum_lines_dd(const double *v, int64_t n, double *out, cudaStream_t st) {
    sum_lines_kernel<<<1, 1024, 0, st>>>(v, n, out);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int dot_dd(int64_t n, const double *a, const double *b, double *partial, double *out,
           cudaStream_t st) {
    dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, a, b, partial);
    count_launch();
    LP_CHECK_LAUNCH();
    return finalize_dd(partial, out, st);
}

int pcg_update_p(int64_t n, const double *z, double *p, const double *rho_new,
                 const double *rho_old, int first, cudaStream_t st) {
    update_p_kernel<<<grid_for(n), 256, 0, st>>>(n, z, p, rho_new, rho_old, first);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int pcg_update_xr(int64_t n, double *x, double *r, const double *p, const double *w,
                  const double *rho, const double *curv, double *partial, cudaStream_t st) {
    update_xr_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, x, r, p, w, rho, curv, partial);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int vec_sub(int64_t n, const double *f, const double *w, double *r, cudaStream_t st) {
    sub_kernel<<<grid_for(n), 256, 0, st>>>(n, f, w, r);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

}  // namespace lp

extern "C" int lp_dot(int64_t n, const double *a, const double *b, double *out2, void *stream) {
    cudaStream_t st = lp::as_stream(stream);
    double *partial;
    LP_CUDA(cudaMallocAsync((void **)&partial, 2 * lp::RED_BLOCKS * sizeof(double), st));
    int rc = lp::dot_dd(n, a, b, partial, out2, st);
    cudaFreeAsync(partial, st);
    return rc;
}

// ---- host-scalar variants for the sharded PCG driver (sharded.py): the
// scalars come from rank-ordered double-double reductions on the host.
namespace lp {
namespace {

__global__ void axpby_p_kernel(int64_t n, const double *__restrict__ z, double *__restrict__ p,
                               double beta, int first) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = first ? z[i] : __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

__global__ void __launch_bounds__(RED_THREADS)
update_xr_host_kernel(int64_t n, double *__restrict__ x, double *__restrict__ r,
                      const double *__restrict__ p, const double *__restrict__ w, double alpha,
                      double *__restrict__ partial) {
    dd acc{0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < n;
         i += (int64_t)RED_BLOCKS * RED_THREADS) {
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
        const double ri = __dsub_rn(r[i], __dmul_rn(alpha, w[i]));
        r[i] = ri;
        acc = dd_add_prod(acc, ri, ri);
    }
    acc = block_reduce_dd(acc);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = acc.hi;
        partial[2 * blockIdx.x + 1] = acc.lo;
    }
}

}  // namespace
}  // namespace lp

// p = z (first) or z + beta p  (pcg.py:150-155 with beta = rho / rho_old)
extern "C" int lp_update_p(int64_t n, const double *z, double *p, double beta, int first,
                           void *stream) {
    cudaStream_t st = lp::as_stream(stream);
    lp::axpby_p_kernel<<<lp::grid_for(n), 256, 0, st>>>(n, z, p, beta, first);
    lp::count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

// x += alpha p, r -= alpha w (pcg.py:161-162); out2 = double-double r'r of this slab
extern "C" int lp_update_xr(int64_t n, double *x, double *r, const double *p, const double *w,
                            double alpha, double *out2, void *stream) {
    cudaStream_t st = lp::as_stream(stream);
    double *partial;
    LP_CUDA(cudaMallocAsync((void **)&partial, 2 * lp::RED_BLOCKS * sizeof(double), st));
    lp::update_xr_host_kernel<<<lp::RED_BLOCKS, lp::RED_THREADS, 0, st>>>(n, x, r, p, w, alpha,
                                                                         partial);
    lp::count_launch();
    int rc = lp::finalize_dd(partial, out2, st);
    cudaFreeAsync(partial, st);
    return rc;
}
