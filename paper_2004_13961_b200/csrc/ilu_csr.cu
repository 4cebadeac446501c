// General-pattern CSR matrices: ILU(0) factorisation, sweeps and SpMV.
//
// Reference: sparse.py:116-221.  Used for SparseMatrix objects that do not
// come from assemble_M (from_dense / from_scipy / Matrix Market).  Matrices
// assembled by assemble_M use the implicit-offset box kernels (ilu_box.cu).
//
// All three triangular kernels are "sync-free": one warp per row, rows handed
// out in increasing (decreasing for the backward sweep) order through an
// atomic ticket, and per-row completion flags published with release fences.
// A warp only ever waits on rows handed out before its own, which are held
// by resident warps, so the schedule cannot deadlock.  The factorisation
// keeps the reference's per-row k-ascending order and separately rounded
// multiply/subtract, so its factors are bit-identical to sparse.py:116-139.
#include <stdlib.h>

#include <vector>

#include <string.h>

#include "ilu.cuh"
#include "vector_ops.cuh"

namespace lp {
namespace {

constexpr int WARPS_PER_BLOCK = 8;

__device__ __forceinline__ int next_ticket(int *ticket) {
    int t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(ticket, 1);
    return __shfl_sync(0xffffffff, t, 0);
}

__device__ __forceinline__ void wait_flag(const int *flags, int64_t k, int epoch) {
    const volatile int *f = flags + k;
    while (*f != epoch) {
    }
    __threadfence();
}

__device__ __forceinline__ void publish(int *flags, int64_t row, int epoch) {
    __threadfence();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        __threadfence();
        *((volatile int *)(flags + row)) = epoch;
    }
}

__device__ __forceinline__ int64_t find_col(const int32_t *__restrict__ idx, int64_t lo,
                                            int64_t hi, int32_t col) {
    int64_t a = lo, b = hi;
    while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (__ldg(idx + mid) < col) a = mid + 1;
        else b = mid;
    }
    return (a < hi && __ldg(idx + a) == col) ? a : -1;
}

__global__ void diag_kernel(int64_t n, const int64_t *__restrict__ indptr,
                            const int32_t *__restrict__ idx, int64_t *__restrict__ diag,
                            unsigned long long *__restrict__ missing) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t lo = indptr[i], hi = indptr[i + 1];
    int64_t a = lo, b = hi;
    while (a < b) {
        const int64_t m = (a + b) >> 1;
        if (idx[m] < i) a = m + 1;
        else b = m;
    }
    if (a < hi && idx[a] == i) diag[i] = a;
    else {
        diag[i] = -1;
        atomicMin(missing, (unsigned long long)i);
    }
}

__global__ void ilu0_csr_kernel(int64_t n, const int64_t *__restrict__ indptr,
                                const int32_t *__restrict__ idx, const int64_t *__restrict__ diag,
                                double *lu, int *flags, int epoch, int *ticket, double tol,
                                unsigned long long *bad) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int64_t row = next_ticket(ticket);
        if (row >= n) return;
        const int64_t lo = indptr[row], hi = indptr[row + 1], dr = diag[row];
        for (int64_t e = lo; e < dr; ++e) {
            const int64_t k = __ldg(idx + e);
            if (lane == 0) wait_flag(flags, k, epoch);
            __syncwarp();
            const int64_t dk = __ldg(diag + k);
            const double piv = __ldcg(lu + dk);
            if (fabs(piv) < tol && lane == 0)
                atomicMin(bad, (unsigned long long)(row * n + k));
            const double lik = __ddiv_rn(__ldcg(lu + e), piv);
            __syncwarp();
            if (lane == 0) __stcg(lu + e, lik);
            const int64_t kend = indptr[k + 1];
            for (int64_t f = dk + 1 + lane; f < kend; f += 32) {
                const int64_t pos = find_col(idx, lo, hi, __ldg(idx + f));
                if (pos >= 0) {
                    const double u = __ldcg(lu + f);
                    __stcg(lu + pos, __dsub_rn(__ldcg(lu + pos), __dmul_rn(lik, u)));
                }
            }
            __threadfence_block();
            __syncwarp();
        }
        publish(flags, row, epoch);
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    return v;
}

__global__ void fwd_csr_kernel(int64_t n, const int64_t *__restrict__ indptr,
                               const int32_t *__restrict__ idx, const int64_t *__restrict__ diag,
                               const double *__restrict__ lu, const double *__restrict__ r,
                               double *y, int *flags, int epoch, int *ticket) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int64_t row = next_ticket(ticket);
        if (row >= n) return;
        const int64_t lo = indptr[row], dr = diag[row];
        double acc = 0.0;
        for (int64_t e = lo + lane; e < dr; e += 32) {
            const int64_t k = __ldg(idx + e);
            wait_flag(flags, k, epoch);
            acc = fma(__ldg(lu + e), __ldcg(y + k), acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) __stcg(y + row, r[row] - acc);
        publish(flags, row, epoch);
    }
}

__global__ void bwd_csr_kernel(int64_t n, const int64_t *__restrict__ indptr,
                               const int32_t *__restrict__ idx, const int64_t *__restrict__ diag,
                               const double *__restrict__ lu, const double *__restrict__ y,
                               double *z, int *flags, int epoch, int *ticket) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        const int64_t t = next_ticket(ticket);
        if (t >= n) return;
        const int64_t row = n - 1 - t;
        const int64_t hi = indptr[row + 1], dr = diag[row];
        double acc = 0.0;
        for (int64_t e = dr + 1 + lane; e < hi; e += 32) {
            const int64_t k = __ldg(idx + e);
            wait_flag(flags, k, epoch);
            acc = fma(__ldg(lu + e), __ldcg(z + k), acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) __stcg(z + row, (y[row] - acc) / __ldg(lu + dr));
        publish(flags, row, epoch);
    }
}

__global__ void spmv_csr_kernel(int64_t n, const int64_t *__restrict__ indptr,
                                const int32_t *__restrict__ idx, const double *__restrict__ v,
                                const double *__restrict__ x, double *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (row >= n) return;
    double acc = 0.0;
    for (int64_t e = indptr[row] + lane; e < indptr[row + 1]; e += 32)
        acc = fma(v[e], x[idx[e]], acc);
    acc = warp_sum(acc);
    if (lane == 0) y[row] = acc;
}

unsigned syncfree_blocks(int64_t n) {
    int64_t b = ceil_div(n, WARPS_PER_BLOCK);
    const int64_t cap = (int64_t)num_sms() * 8;
    return (unsigned)(b < cap ? b : cap);
}

// per-call progress flags (zeroed, epoch 1) and ticket
int csr_fwd(lp_ilu *m, const double *r, double *y, int *flags, int *ticket, cudaStream_t st) {
    LP_CUDA(cudaMemsetAsync(flags, 0, m->n * sizeof(int), st));
    LP_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    fwd_csr_kernel<<<syncfree_blocks(m->n), 32 * WARPS_PER_BLOCK, 0, st>>>(
        m->n, m->indptr, m->indices, m->diag, m->lu, r, y, flags, 1, ticket);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int csr_bwd(lp_ilu *m, const double *y, double *z, int *flags, int *ticket, cudaStream_t st) {
    LP_CUDA(cudaMemsetAsync(flags, 0, m->n * sizeof(int), st));
    LP_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    bwd_csr_kernel<<<syncfree_blocks(m->n), 32 * WARPS_PER_BLOCK, 0, st>>>(
        m->n, m->indptr, m->indices, m->diag, m->lu, y, z, flags, 1, ticket);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

}  // namespace

int scratch_alloc(const lp_ilu *m, SweepScratch &s, cudaStream_t st) {
    int rc;
    if ((rc = salloc(&s.ytmp, (size_t)m->n, "sweep vector", st)) ||
        (rc = salloc(&s.tickets, 2, "sweep tickets", st)))
        return rc;
    if (m->kind != MAT_BOX && (rc = salloc(&s.flags, (size_t)m->n, "sweep flags", st))) return rc;
    // fused r'z: one part per x-line (box sweeps) or the dd block partials of dot_dd
    size_t nd = 2 * RED_BLOCKS;
    if (m->kind == MAT_BOX && (size_t)(m->n / m->box.K) > nd) nd = (size_t)(m->n / m->box.K);
    return salloc(&s.dotpart, nd, "dot partials", st);
}

void scratch_free(SweepScratch &s, cudaStream_t st) {
    sfree(s.ytmp, st);
    sfree(s.tickets, st);
    sfree(s.flags, st);
    sfree(s.dotpart, st);
    s = SweepScratch{};
}

int ilu_apply(lp_ilu *m, const double *r, double *z, const SweepScratch &s, cudaStream_t st) {
    int rc;
    if (m->kind == MAT_BOX) return box_apply(m, r, z, s, st);
    if ((rc = csr_fwd(m, r, s.ytmp, s.flags, s.tickets, st))) return rc;
    return csr_bwd(m, s.ytmp, z, s.flags, s.tickets + 1, st);
}

int ilu_apply_dot(lp_ilu *m, const double *r, double *z, const SweepScratch &s, double *rz, cudaStream_t st) {
    if (m->kind == MAT_BOX && box_apply_dot_fused(m)) return box_apply_dot(m, r, z, s, rz, st);
    const int rc = ilu_apply(m, r, z, s, st);
    return rc ? rc : dot_dd(m->n, r, z, s.dotpart, rz, st);
}

int ilu_forward(lp_ilu *m, const double *r, double *y, const SweepScratch &s, cudaStream_t st) {
    if (m->kind == MAT_BOX) return box_forward(m, r, y, s.tickets, st);
    return csr_fwd(m, r, y, s.flags, s.tickets, st);
}

int ilu_backward(lp_ilu *m, const double *y, double *z, const SweepScratch &s, cudaStream_t st) {
    if (m->kind == MAT_BOX) return box_backward(m, y, z, s.tickets + 1, st);
    return csr_bwd(m, y, z, s.flags, s.tickets + 1, st);
}

}  // namespace lp

using namespace lp;

static int alloc_sweep_state(lp_ilu *m) {
    int rc;
    if ((rc = dalloc(&m->flags, m->n, "row flags")) || (rc = dalloc(&m->ticket, 4, "tickets")) ||
        (rc = dalloc(&m->bad, 1, "pivot key")))
        return rc;
    LP_CUDA(cudaMemset(m->flags, 0, m->n * sizeof(int)));
    return LP_OK;
}

extern "C" int lp_csr_create(int64_t n, int64_t nnz, const int64_t *indptr,
                             const int32_t *indices, const double *values, lp_ilu **out) {
    *out = nullptr;
    LP_ARG(n > 0, "empty matrix");
    LP_ARG(nnz >= 0, "negative nnz");
    lp_ilu *m = new lp_ilu();
    m->kind = MAT_CSR;
    m->n = n;
    m->nnz = nnz;
    int rc;
    if ((rc = dalloc(&m->indptr, n + 1, "indptr")) || (rc = dalloc(&m->indices, nnz, "indices")) ||
        (rc = dalloc(&m->values, nnz, "values")) || (rc = dalloc(&m->lu, nnz, "factors")) ||
        (rc = dalloc(&m->diag, n, "diag")) || (rc = alloc_sweep_state(m))) {
        lp_ilu_destroy(m);
        return rc;
    }
    cudaError_t e = cudaMemcpy(m->indptr, indptr, (n + 1) * sizeof(int64_t), cudaMemcpyDefault);
    if (e == cudaSuccess && nnz)
        e = cudaMemcpy(m->indices, indices, nnz * sizeof(int32_t), cudaMemcpyDefault);
    if (e == cudaSuccess && nnz)
        e = cudaMemcpy(m->values, values, nnz * sizeof(double), cudaMemcpyDefault);
    if (e != cudaSuccess) {
        lp_ilu_destroy(m);
        return cuda_fail(e, "csr upload", __FILE__, __LINE__);
    }
    *out = m;
    return LP_OK;
}

extern "C" int lp_ilu_destroy(lp_ilu *m) {
    if (!m) return LP_OK;
    cudaDeviceSynchronize();
    void *ptrs[] = {m->indptr, m->indices, m->values, m->lu, m->diag, m->flags, m->ticket,
                    m->bad, m->box.values, m->box.lu, m->box.mask,
                    m->box.band_lo, m->box.band_up, m->box.diag, m->box.line_order,
                    m->box.line_groups, m->box.full, m->box.ilu_tasks, m->box.rdiag, m->box.even};
    for (void *p : ptrs)
        if (p) dfree(p);
    for (auto &ro : m->box.rank_order) {
        dfree(ro.order);
        dfree(ro.groups);
    }
    delete m;
    return LP_OK;
}

extern "C" int lp_matrix_nnz(const lp_ilu *m, int64_t *nnz) {
    *nnz = m->kind == MAT_BOX ? m->box.nnz : m->nnz;
    return LP_OK;
}

extern "C" int lp_ilu0(lp_ilu *m, double tol, int64_t *bad_row, void *stream) {
    cudaStream_t st = as_stream(stream);
    *bad_row = -1;
    if (m->kind == MAT_BOX) return box_ilu0(m, tol, bad_row, st);
    const int64_t n = m->n;
    unsigned long long *key = reinterpret_cast<unsigned long long *>(m->bad);
    const unsigned long long none = ~0ull;
    LP_CUDA(cudaMemcpyAsync(key, &none, sizeof none, cudaMemcpyHostToDevice, st));
    diag_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, m->indptr, m->indices, m->diag, key);
    count_launch();
    unsigned long long hk;
    LP_CUDA(cudaMemcpyAsync(&hk, key, sizeof hk, cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaStreamSynchronize(st));
    if (hk != none) {
        *bad_row = (int64_t)hk;
        set_error("zero pivot at elimination step %lld", (long long)hk);
        return LP_ERR_ZERO_PIVOT;
    }
    LP_CUDA(cudaMemcpyAsync(m->lu, m->values, m->nnz * sizeof(double), cudaMemcpyDeviceToDevice, st));
    const int ep = ++m->epoch;
    LP_CUDA(cudaMemsetAsync(m->ticket, 0, sizeof(int), st));
    ilu0_csr_kernel<<<syncfree_blocks(n), 32 * WARPS_PER_BLOCK, 0, st>>>(
        n, m->indptr, m->indices, m->diag, m->lu, m->flags, ep, m->ticket, tol, key);
    count_launch();
    LP_CHECK_LAUNCH();
    int64_t dlast;
    double plast;
    LP_CUDA(cudaMemcpyAsync(&hk, key, sizeof hk, cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaMemcpyAsync(&dlast, m->diag + (n - 1), sizeof dlast, cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaStreamSynchronize(st));
    LP_CUDA(cudaMemcpy(&plast, m->lu + dlast, sizeof plast, cudaMemcpyDeviceToHost));
    if (hk != none) *bad_row = (int64_t)(hk % (unsigned long long)n);
    else if (fabs(plast) < tol) *bad_row = n - 1;
    if (*bad_row >= 0) {
        set_error("zero pivot at elimination step %lld", (long long)*bad_row);
        return LP_ERR_ZERO_PIVOT;
    }
    m->factored = true;
    return LP_OK;
}

// The sweeps run on per-call stream-ordered scratch (reentrant: concurrent
// calls on one set of factors from different streams or threads are safe).
template <class F>
static int with_scratch(lp_ilu *m, cudaStream_t st, F &&body) {
    SweepScratch s;
    int rc = scratch_alloc(m, s, st);
    if (!rc) rc = body(s);
    scratch_free(s, st);
    return rc;
}

extern "C" int lp_ilu0_ranks(lp_ilu *const *ms, int nranks, const int *ys, double tol, int64_t *bad_row,
                             void *stream) {
    return box_ilu0_ranks(ms, nranks, ys, -1, nullptr, nullptr, tol, bad_row, as_stream(stream));
}

extern "C" int lp_ilu0_rank(lp_ilu *m, int nranks, const int *ys, int rank, double *const *peer_lu,
                            int *const *peer_flags, double tol, int64_t *bad_row, void *stream) {
    LP_ARG(rank >= 0 && rank < nranks, "rank out of range");
    lp_ilu *ms[1] = {m};
    return box_ilu0_ranks(ms, nranks, ys, rank, peer_lu, peer_flags, tol, bad_row, as_stream(stream));
}

extern "C" int lp_ilu_rank_arrays(lp_ilu *m, double **lu, int **flags, unsigned char *handle_lu64,
                                  unsigned char *handle_flags64) {
    LP_ARG(m->kind == MAT_BOX, "box matrices only");
    lp::BoxLayout &b = m->box;
    LP_ARG(b.lu == nullptr, "call before the matrix is factored");
    // plain cudaMalloc memory: stream-ordered pool allocations cannot be exported over CUDA IPC
    double *nlu = nullptr;
    int *nfl = nullptr;
    LP_CUDA(cudaMalloc(&nlu, ((size_t)b.n * b.S + 2) * sizeof(double)));
    cudaError_t e = cudaMalloc(&nfl, (size_t)b.n * sizeof(int));
    if (e != cudaSuccess) {
        cudaFree(nlu);
        return cuda_fail(e, "rank flag array", __FILE__, __LINE__);
    }
    cudaIpcMemHandle_t h1, h2;
    if ((e = cudaIpcGetMemHandle(&h1, nlu)) != cudaSuccess || (e = cudaIpcGetMemHandle(&h2, nfl)) != cudaSuccess) {
        cudaFree(nlu);
        cudaFree(nfl);
        return cuda_fail(e, "IPC export of the rank arrays", __FILE__, __LINE__);
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    memcpy(handle_lu64, &h1, 64);
    memcpy(handle_flags64, &h2, 64);
    dfree(m->flags);
    m->flags = nfl;
    b.lu = nlu;
    *lu = nlu;
    *flags = nfl;
    return LP_OK;
}

extern "C" int lp_ilu0_rank_prepare(lp_ilu *m, int64_t *bad_row, void *stream) {
    LP_ARG(m->kind == MAT_BOX, "box matrices only");
    *bad_row = -1;
    return box_ilu0_prepare(m, bad_row, as_stream(stream));
}

extern "C" int lp_forward_sub(lp_ilu *m, const double *r, double *y, void *stream) {
    LP_ARG(m->factored, "matrix has not been factored (call lp_ilu0)");
    cudaStream_t st = as_stream(stream);
    return with_scratch(m, st, [&](const SweepScratch &s) { return ilu_forward(m, r, y, s, st); });
}

extern "C" int lp_backward_sub(lp_ilu *m, const double *y, double *z, void *stream) {
    LP_ARG(m->factored, "matrix has not been factored (call lp_ilu0)");
    cudaStream_t st = as_stream(stream);
    return with_scratch(m, st, [&](const SweepScratch &s) { return ilu_backward(m, y, z, s, st); });
}

extern "C" int lp_precond_apply(lp_ilu *m, const double *r, double *z, void *stream) {
    LP_ARG(m->factored, "matrix has not been factored (call lp_ilu0)");
    cudaStream_t st = as_stream(stream);
    return with_scratch(m, st, [&](const SweepScratch &s) { return ilu_apply(m, r, z, s, st); });
}

extern "C" int lp_precond_apply_rz(lp_ilu *m, const double *r, double *z, double *rz, void *stream) {
    LP_ARG(m->factored, "matrix has not been factored (call lp_ilu0)");
    LP_ARG(rz != nullptr, "rz must point to two device doubles");
    cudaStream_t st = as_stream(stream);
    return with_scratch(m, st, [&](const SweepScratch &s) { return ilu_apply_dot(m, r, z, s, rz, st); });
}

extern "C" int lp_spmv(lp_ilu *m, const double *x, double *y, void *stream) {
    cudaStream_t st = as_stream(stream);
    if (m->kind == MAT_BOX) return box_spmv(m, x, y, st);
    spmv_csr_kernel<<<(unsigned)ceil_div(m->n * 32, 256), 256, 0, st>>>(m->n, m->indptr,
                                                                       m->indices, m->values, x, y);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

extern "C" int lp_matrix_export(const lp_ilu *m, int which, int64_t *indptr, int32_t *indices,
                                double *values) {
    LP_ARG(which >= 0 && which <= 2, "which must be 0 (M), 1 (L) or 2 (U)");
    LP_ARG(which == 0 || m->factored, "matrix has not been factored");
    if (m->kind == MAT_BOX) return box_export(m, which, indptr, indices, values);
    const int64_t n = m->n, nnz = m->nnz;
    std::vector<int64_t> ip(n + 1), dg(n);
    std::vector<int32_t> ix(nnz);
    std::vector<double> v(nnz);
    LP_CUDA(cudaMemcpy(ip.data(), m->indptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    LP_CUDA(cudaMemcpy(ix.data(), m->indices, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
    LP_CUDA(cudaMemcpy(v.data(), which == 0 ? m->values : m->lu, nnz * sizeof(double),
                       cudaMemcpyDeviceToHost));
    if (which) LP_CUDA(cudaMemcpy(dg.data(), m->diag, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
    int64_t out = 0;
    indptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t a = ip[i], b = ip[i + 1];
        if (which == 1) b = dg[i];
        if (which == 2) a = dg[i];
        for (int64_t e = a; e < b; ++e, ++out) {
            if (indices) indices[out] = ix[e];
            if (values) values[out] = v[e];
        }
        indptr[i + 1] = out;
    }
    return LP_OK;
}
