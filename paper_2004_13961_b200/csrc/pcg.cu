// Device-resident PCG loop (Algorithm 1; reference pcg.py:111-179).
//
// All vectors stay on the device; the scalars rho, p'Ap and r'r are
// double-double device values consumed directly by the update kernels.  The
// host reads back one small status block per iteration (r'r and p'Ap) to
// evaluate the stopping test and the curvature check, exactly where the
// reference evaluates them.
//
// Host work per iteration: one graph launch (the whole iteration -- both
// sweeps, the dots, the p update, the matvec passes, the x/r update and the
// status copy -- captured once per solve, one graph per parity of the
// iteration number because rho_new / rho_old alternate), one stream
// synchronisation, and the host-side test.  Workspaces are stream-ordered
// allocations from the device pool (no device synchronisation), so a solve
// never writes to the operator or factor handles and concurrent solves on
// different streams are independent.
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
    cudaStream_t st = nullptr;
    double *r = nullptr, *z = nullptr, *p = nullptr, *w = nullptr;
    double *partial = nullptr, *scal = nullptr, *opws = nullptr;
    SweepScratch sweep;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    ~Workspace() {
        for (auto &e : exec)
            if (e) cudaGraphExecDestroy(e);
        double *ps[] = {r, z, p, w, partial, scal, opws};
        for (double *q : ps) sfree(q, st);
        scratch_free(sweep, st);
    }
};

// Per-thread non-blocking stream for solves issued on the legacy stream (which
// cannot be captured into a graph); forked from / joined to the caller's
// stream with events, so the caller's stream order is kept.
struct LoopStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
LoopStream *loop_stream() {
    static thread_local LoopStream ls;
    if (!ls.s) {
        if (cudaStreamCreateWithFlags(&ls.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ls.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ls.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            ls.s = nullptr;
            return nullptr;
        }
    }
    return &ls;
}

// Pinned status block, allocated once per host thread: cudaMallocHost /
// cudaFreeHost per solve cost milliseconds (and cudaFreeHost synchronises the
// device).
double *status_block() {
    static thread_local double *blk = nullptr;
    if (!blk && cudaMallocHost((void **)&blk, 4 * sizeof(double)) != cudaSuccess) blk = nullptr;
    return blk;
}

struct Loop {
    lp_operator *op;
    lp_ilu *pre;
    int64_t n;
    double *x;
    Workspace *ws;
    double *host;
};

// One iteration (pcg.py:147-162), all stream-ordered on st: z = M^-1 r;
// rho = r'z; p = z + (rho/rho_old) p; w = (A+B) p; curv = p'w; x += alpha p,
// r -= alpha w with r'r; status (r'r, p'w) to the pinned host block.
int iteration(const Loop &L, int64_t it, cudaStream_t st) {
    Workspace &ws = *L.ws;
    double *sc = ws.scal;
    int rc;
    const double *zz = ws.r;
    double *rho_new = sc + ((it & 1) ? S_RHO1 : S_RHO0);
    double *rho_old = sc + ((it & 1) ? S_RHO0 : S_RHO1);
    if (L.pre) {
        // z = M^-1 r with rho = r'z carried by the backward sweep (pcg.py:147-151)
        if ((rc = ilu_apply_dot(L.pre, ws.r, ws.z, ws.sweep, rho_new, st))) return rc;
        zz = ws.z;
    } else if ((rc = dot_dd(L.n, ws.r, zz, ws.partial, rho_new, st))) {
        return rc;
    }
    if ((rc = pcg_update_p(L.n, zz, ws.p, rho_new, rho_old, it == 1, st))) return rc;
    // w = (A + B) p with the curvature p'w carried by the last pass (pcg.py:156-157)
    if ((rc = operator_apply(L.op, 3, ws.p, ws.w, st, ws.opws, sc + S_CURV))) return rc;
    if ((rc = pcg_update_xr(L.n, L.x, ws.r, ws.p, ws.w, rho_new, sc + S_CURV, ws.partial, st)))
        return rc;
    if ((rc = finalize_dd(ws.partial, sc + S_RR, st))) return rc;
    LP_CUDA(cudaMemcpyAsync(L.host, sc + S_RR, sizeof(double), cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaMemcpyAsync(L.host + 2, sc + S_CURV, sizeof(double), cudaMemcpyDeviceToHost, st));
    return LP_OK;
}

// Capture iteration `it` (its parity) into an executable graph; nullptr and
// LP_OK when capture is not possible (the loop then runs the iteration eagerly).
int capture(const Loop &L, int64_t it, cudaStream_t st, cudaGraphExec_t *out) {
    *out = nullptr;
    if (!st) return LP_OK;   // the legacy stream cannot be captured
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return LP_OK;
    }
    const int64_t l0 = g_launches;
    const int rc = iteration(L, it, st);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &graph);
    g_launches = l0;   // counted when the graph runs
    if (rc != LP_OK || e != cudaSuccess || !graph) {
        cudaGetLastError();
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    const cudaError_t ei = cudaGraphInstantiate(out, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
    }
    return LP_OK;
}

}  // namespace

static int pcg_solve_on(lp_operator *op, lp_ilu *pre, const double *F, double *x, int has_x0,
                        double epsilon, int64_t k_max, double *history, lp_report *rep,
                        cudaStream_t st);

extern "C" int lp_pcg_solve(lp_operator *op, lp_ilu *pre, const double *F, double *x, int has_x0,
                            double epsilon, int64_t k_max, double *history, lp_report *rep,
                            void *stream) {
    cudaStream_t st = as_stream(stream);
    LoopStream *ls = st ? nullptr : loop_stream();
    if (!ls) return pcg_solve_on(op, pre, F, x, has_x0, epsilon, k_max, history, rep, st);
    LP_CUDA(cudaEventRecord(ls->fork, st));
    LP_CUDA(cudaStreamWaitEvent(ls->s, ls->fork, 0));
    const int rc = pcg_solve_on(op, pre, F, x, has_x0, epsilon, k_max, history, rep, ls->s);
    LP_CUDA(cudaEventRecord(ls->join, ls->s));
    LP_CUDA(cudaStreamWaitEvent(st, ls->join, 0));
    return rc;
}

static int pcg_solve_on(lp_operator *op, lp_ilu *pre, const double *F, double *x, int has_x0,
                        double epsilon, int64_t k_max, double *history, lp_report *rep,
                        cudaStream_t st) {
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
    ws.st = st;
    int rc;
    if ((rc = salloc(&ws.r, n, "r", st)) || (rc = salloc(&ws.p, n, "p", st)) ||
        (rc = salloc(&ws.w, n, "w", st)) || (rc = salloc(&ws.partial, 2 * RED_BLOCKS, "partials", st)) ||
        (rc = salloc(&ws.scal, S_NSLOTS, "scalars", st)) ||
        (rc = salloc(&ws.opws, operator_ws_doubles(op), "operator workspace", st)))
        return rc;
    if (pre && ((rc = salloc(&ws.z, n, "z", st)) || (rc = scratch_alloc(pre, ws.sweep, st)))) return rc;
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
        if ((rc = operator_apply(op, 3, x, ws.w, st, ws.opws))) return rc;
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

    const Loop L{op, pre, n, x, &ws, host};
    int64_t it = 0, per_iter = 0;
    const double tol = epsilon * fnorm;
    const auto t0 = std::chrono::steady_clock::now();
    while (sqrt(rr) > tol && it < k_max) {
        ++it;
        cudaGraphExec_t &ge = ws.exec[it & 1];
        if (it >= 2 && !ge && (rc = capture(L, it, st, &ge))) return rc;
        if (ge) {
            LP_CUDA(cudaGraphLaunch(ge, st));
            g_launches += per_iter;
        } else {
            const int64_t l0 = g_launches;
            if ((rc = iteration(L, it, st))) return rc;
            per_iter = g_launches - l0;
        }
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
