// Device-resident PCG loop (Algorithm 1; reference pcg.py:111-179).
//
// All vectors stay on the device; the scalars rho, p'Ap and r'r are
// double-double device values consumed directly by the update kernels.  The
// host reads back one 32-byte status block per iteration (r'r and p'Ap) to
// evaluate the stopping test and the curvature check, exactly where the
// reference evaluates them.
#include <math.h>

#include <chrono>

#include "ilu.cuh"
#include "operator.cuh"
#include "vector_ops.cuh"

using namespace lp;

namespace {

// device scalar slots (dd pairs)
enum { S_RR = 0, S_RHO0 = 2, S_RHO1 = 4, S_CURV = 6, S_FF = 8, S_NSLOTS = 10 };

struct Workspace {
    double *r = nullptr, *z = nullptr, *p = nullptr, *w = nullptr;
    double *partial = nullptr, *scal = nullptr;
    ~Workspace() {
        double *ps[] = {r, z, p, w, partial, scal};
        for (double *q : ps)
            if (q) dfree(q);
    }
};

// Pinned status block, allocated once per host thread: cudaMallocHost /
// cudaFreeHost per solve cost milliseconds (and cudaFreeHost synchronises the
// device).
double *status_block() {
    static thread_local double *blk = nullptr;
    if (!blk && cudaMallocHost((void **)&blk, 4 * sizeof(double)) != cudaSuccess) blk = nullptr;
    return blk;
}

}  // namespace

extern "C" int lp_pcg_solve(lp_operator *op, lp_ilu *pre, const double *F, double *x, int has_x0,
                            double epsilon, int64_t k_max, double *history, lp_report *rep,
                            void *stream) {
    cudaStream_t st = as_stream(stream);
    LP_ARG(epsilon > 0, "epsilon must be positive");
    LP_ARG(k_max >= 1, "k_max must be at least 1");
    const int64_t n = (int64_t)pow((double)op->K, op->d) + 0.5;
    if (pre) {
        LP_ARG(pre->n == n, "preconditioner size %lld does not match the problem (%lld)",
               (long long)pre->n, (long long)n);
        LP_ARG(pre->factored, "preconditioner has not been factored");
    }
    *rep = lp_report{};
    const int64_t launches0 = g_launches;
    Workspace ws;
    int rc;
    if ((rc = dalloc(&ws.r, n, "r")) || (rc = dalloc(&ws.p, n, "p")) || (rc = dalloc(&ws.w, n, "w")) ||
        (rc = dalloc(&ws.partial, 2 * RED_BLOCKS, "partials")) ||
        (rc = dalloc(&ws.scal, S_NSLOTS, "scalars")))
        return rc;
    if (pre && (rc = dalloc(&ws.z, n, "z"))) return rc;
    double *const host = status_block();
    LP_ARG(host != nullptr, "cannot allocate the pinned status block");
    double *sc = ws.scal;

    // ||f|| and the initial residual
    if ((rc = dot_dd(n, F, F, ws.partial, sc + S_FF, st))) return rc;
    bool x_nonzero = false;
    if (has_x0) {
        if ((rc = dot_dd(n, x, x, ws.partial, sc + S_RR, st))) return rc;
        LP_CUDA(cudaMemcpyAsync(host, sc + S_RR, sizeof(double), cudaMemcpyDeviceToHost, st));
        LP_CUDA(cudaStreamSynchronize(st));
        x_nonzero = host[0] != 0.0;
    } else {
        LP_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
    }
    if (x_nonzero) {
        if ((rc = operator_apply(op, 3, x, ws.w, st))) return rc;
        if ((rc = vec_sub(n, F, ws.w, ws.r, st))) return rc;
    } else {
        LP_CUDA(cudaMemcpyAsync(ws.r, F, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    if ((rc = dot_dd(n, ws.r, ws.r, ws.partial, sc + S_RR, st))) return rc;
    LP_CUDA(cudaMemcpyAsync(host, sc + S_RR, sizeof(double), cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaMemcpyAsync(host + 2, sc + S_FF, sizeof(double), cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaStreamSynchronize(st));
    const double fnorm = sqrt(host[2]);
    double rr = host[0];
    if (history) history[0] = sqrt(rr);

    int64_t it = 0;
    const double tol = epsilon * fnorm;
    const auto t0 = std::chrono::steady_clock::now();
    while (sqrt(rr) > tol && it < k_max) {
        const double *zz = ws.r;
        if (pre) {
            if ((rc = ilu_apply(pre, ws.r, ws.z, st))) return rc;
            zz = ws.z;
        }
        ++it;
        double *rho_new = sc + ((it & 1) ? S_RHO1 : S_RHO0);
        double *rho_old = sc + ((it & 1) ? S_RHO0 : S_RHO1);
        if ((rc = dot_dd(n, ws.r, zz, ws.partial, rho_new, st))) return rc;
        if ((rc = pcg_update_p(n, zz, ws.p, rho_new, rho_old, it == 1, st))) return rc;
        if ((rc = operator_apply(op, 3, ws.p, ws.w, st))) return rc;
        if ((rc = dot_dd(n, ws.p, ws.w, ws.partial, sc + S_CURV, st))) return rc;
        if ((rc = pcg_update_xr(n, x, ws.r, ws.p, ws.w, rho_new, sc + S_CURV, ws.partial, st)))
            return rc;
        if ((rc = finalize_dd(ws.partial, sc + S_RR, st))) return rc;
        LP_CUDA(cudaMemcpyAsync(host, sc + S_RR, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        LP_CUDA(cudaMemcpyAsync(host + 2, sc + S_CURV, sizeof(double), cudaMemcpyDeviceToHost, st));
        LP_CUDA(cudaStreamSynchronize(st));
        const double curv = host[2];
        if (curv <= 0.0) {
            rep->iterations = it;
            rep->indefinite_value = curv;
            set_error("non-positive curvature p'Ap = %.3e at iteration %lld", curv, (long long)it);
            return LP_ERR_INDEFINITE;
        }
        rr = host[0];
        if (history) history[it] = sqrt(rr);
    }
    const auto t1 = std::chrono::steady_clock::now();
    rep->iterations = it;
    rep->converged = sqrt(rr) <= tol;
    rep->final_relative_residual = fnorm > 0 ? sqrt(rr) / fnorm : 0.0;
    rep->loop_seconds = std::chrono::duration<double>(t1 - t0).count();
    rep->kernel_launches = g_launches - launches0;
    return LP_OK;
}
