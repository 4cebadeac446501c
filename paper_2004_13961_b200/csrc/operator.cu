// TransformPlan, tensor transforms and the sum-factorised operator A + B.
//
// Reference: transforms.py:289-375 (plan, BDLT/FDLT), operator.py:95-210
// (apply_A / apply_B / apply_system), legendre.py:86-95,176-215 (tables).
//
// The reference applies 2d+2 full tensor transforms per matvec (phi->Legendre
// conversion, BDLT, x beta, FDLT, closed-form contraction, per direction).
// Composing those pieces gives exactly
//   (A+B)u = sum_i (C_i)^T diag(beta w^d) C_i u + Phi^T diag(alpha w^d) Phi u,
//   C_i = dPhi on axis i and Phi elsewhere,  Phi[j,m] = phi_m(x_j),
// which this file evaluates with 2d parity-split line-transform passes that
// share intermediate fields: 3-D x:1->2, y:2->3,
// z:3->4 (x beta w^3, alpha w^3 in the epilogue), then x:4->3, y:3->2, z:2->1.
#include <math.h>

#include "line_transform.cuh"
#include "operator.cuh"
#include "vector_ops.cuh"

namespace lp {
namespace {

// V[j][n] = L_n(x_j) with the reference recurrence, every operation
// separately rounded (legendre.py:86-95: ((2k+1) * x * L_k - k * L_{k-1}) / (k+1)).
__global__ void vandermonde_kernel(int P, const double *__restrict__ x, double *__restrict__ V) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= P) return;
    const double xj = x[j];
    double *row = V + (size_t)j * P;
    double lm1 = 1.0, l = xj;
    row[0] = 1.0;
    if (P > 1) row[1] = xj;
    for (int k = 1; k + 1 < P; ++k) {
        const double t = __dmul_rn(__dmul_rn((double)(2 * k + 1), xj), l);
        const double nxt = __ddiv_rn(__dsub_rn(t, __dmul_rn((double)k, lm1)), (double)(k + 1));
        row[k + 1] = nxt;
        lm1 = l;
        l = nxt;
    }
}

// Phi[j][m] = L_m - L_{m+2}, dPhi[j][m] = -(2m+3) L_{m+1} (legendre.py:176-215),
// Tf[j][n] = V[j][n] w_j (2n+1)/2 (the FDLT of transforms.py:319-325 as a table).
__global__ void derived_tables_kernel(int P, const double *__restrict__ V,
                                      const double *__restrict__ w, double *__restrict__ Phi,
                                      double *__restrict__ DPhi, double *__restrict__ Tf) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)P * P) return;
    const int j = (int)(i / P), n = (int)(i % P);
    const int K = P - 2;
    const double *row = V + (size_t)j * P;
    Tf[i] = __dmul_rn(__dmul_rn(row[n], w[j]), 0.5 * (2.0 * n + 1.0));
    if (n < K) {
        Phi[(size_t)j * K + n] = __dsub_rn(row[n], row[n + 2]);
        DPhi[(size_t)j * K + n] = __dmul_rn(-(2.0 * n + 3.0), row[n + 1]);
    }
}

// gw[z][y][x] = base(x,y,z) * w_x w_y w_z.  base is a full P^d grid
// (axis1d < 0) or a 1-D array along axis `axis1d` broadcast over the rest.
__global__ void weighted_grid_kernel(int d, int P, const double *__restrict__ base, int axis1d,
                                     const double *__restrict__ w, double *__restrict__ gw) {
    const int64_t n = (d == 1) ? P : (d == 2 ? (int64_t)P * P : (int64_t)P * P * P);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ix = (int)(i % P);
    const int iy = d > 1 ? (int)((i / P) % P) : 0;
    const int iz = d > 2 ? (int)(i / ((int64_t)P * P)) : 0;
    double wt = w[ix];
    if (d > 1) wt *= w[iy];
    if (d > 2) wt *= w[iz];
    double b;
    if (axis1d < 0) b = base[i];
    else b = base[axis1d == 0 ? ix : (axis1d == 1 ? iy : iz)];
    gw[i] = b * wt;
}

__global__ void min_kernel(int64_t n, const double *__restrict__ v, double *__restrict__ out) {
    __shared__ double sh[32];
    double m = INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = fmin(m, v[i]);
    for (int o = 16; o; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffff, m, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : INFINITY;
        for (int o = 16; o; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffff, m, o));
        if (threadIdx.x == 0) out[blockIdx.x] = m;
    }
}

int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    while (e-- > 0) r *= b;
    return r;
}

int device_min(const double *v, int64_t n, double *result, cudaStream_t st) {
    const int blocks = 256;
    double *part;
    int rc = dalloc(&part, blocks, "min partials");
    if (rc) return rc;
    min_kernel<<<blocks, 256, 0, st>>>(n, v, part);
    count_launch();
    double hostp[blocks];
    cudaError_t e = cudaMemcpyAsync(hostp, part, sizeof hostp, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    dfree(part);
    LP_CUDA(e);
    double m = INFINITY;
    for (int i = 0; i < blocks; ++i) m = fmin(m, hostp[i]);
    *result = m;
    return LP_OK;
}

}  // namespace
}  // namespace lp

using namespace lp;

// ------------------------------------------------------------------ plans

extern "C" int lp_plan_create(int P, const double *nodes, const double *weights, lp_plan **out) {
    *out = nullptr;
    LP_ARG(P >= 2, "plan order %d too small (need P >= 2)", P);
    lp_plan *p = new lp_plan();
    p->P = P;
    int rc;
    double *V = nullptr, *Phi = nullptr, *DPhi = nullptr, *Tf = nullptr;
    const size_t PP = (size_t)P * P;
    if ((rc = dalloc(&p->nodes, P, "nodes")) || (rc = dalloc(&p->weights, P, "weights")) ||
        (rc = dalloc(&V, PP, "V")) || (rc = dalloc(&Phi, PP, "Phi")) ||
        (rc = dalloc(&DPhi, PP, "dPhi")) || (rc = dalloc(&Tf, PP, "Tf"))) {
        lp_plan_destroy(p);
        return rc;
    }
    p->V = V;
    cudaStream_t st = 0;
    cudaError_t e = cudaMemcpy(p->nodes, nodes, P * sizeof(double), cudaMemcpyDefault);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->weights, weights, P * sizeof(double), cudaMemcpyDefault);
    if (e != cudaSuccess) {
        lp_plan_destroy(p);
        dfree(Phi); dfree(DPhi); dfree(Tf);
        return cuda_fail(e, "plan upload", __FILE__, __LINE__);
    }
    vandermonde_kernel<<<(P + 127) / 128, 128, 0, st>>>(P, p->nodes, V);
    derived_tables_kernel<<<(unsigned)ceil_div((int64_t)PP, 256), 256, 0, st>>>(P, V, p->weights,
                                                                            Phi, DPhi, Tf);
    count_launch(2);
    if ((rc = line_table_build(p->tV, V, P, P, 0, st)) ||
        (rc = line_table_build(p->tF, Tf, P, P, 0, st)) ||
        (P >= 4 && (rc = line_table_build(p->tPhi, Phi, P, P - 2, 0, st))) ||
        (P >= 4 && (rc = line_table_build(p->tDPhi, DPhi, P, P - 2, 1, st)))) {
        dfree(Phi); dfree(DPhi); dfree(Tf);
        lp_plan_destroy(p);
        return rc;
    }
    e = cudaDeviceSynchronize();
    dfree(Phi);
    dfree(DPhi);
    dfree(Tf);
    if (e != cudaSuccess) {
        lp_plan_destroy(p);
        return cuda_fail(e, "plan tables", __FILE__, __LINE__);
    }
    *out = p;
    return LP_OK;
}

extern "C" int lp_plan_destroy(lp_plan *p) {
    if (!p) return LP_OK;
    cudaDeviceSynchronize();
    line_table_free(p->tV);
    line_table_free(p->tF);
    line_table_free(p->tPhi);
    line_table_free(p->tDPhi);
    if (p->nodes) dfree(p->nodes);
    if (p->weights) dfree(p->weights);
    if (p->V) dfree(p->V);
    delete p;
    return LP_OK;
}

extern "C" int lp_plan_table(const lp_plan *p, double *dst) {
    LP_CUDA(cudaMemcpy(dst, p->V, sizeof(double) * p->P * p->P, cudaMemcpyDefault));
    return LP_OK;
}

static int tensor_transform(lp_plan *p, const LineTable &t, int fold, int d, const double *in,
                            double *out, cudaStream_t st) {
    LP_ARG(d >= 1 && d <= 3, "tensor transforms support d = 1, 2, 3");
    const int64_t n = ipow(p->P, d);
    double *tmp = nullptr;
    if (d > 1) LP_CUDA(cudaMallocAsync((void **)&tmp, n * sizeof(double), st));
    // d passes; pass a reads src, writes dst, ending in `out`
    const double *src = in;
    for (int a = 0; a < d; ++a) {
        double *dst = ((d - a) % 2 == 1) ? out : tmp;
        LtArgs args = fold ? lt_fold(t, (int)(n / p->P)) : lt_unfold(t, (int)(n / p->P));
        lt_add_term(args, 0, t, src);
        lt_set_out(args, 0, dst);
        int rc = line_transform(args, st);
        if (rc) {
            if (tmp) cudaFreeAsync(tmp, st);
            return rc;
        }
        src = dst;
    }
    if (tmp) LP_CUDA(cudaFreeAsync(tmp, st));
    return LP_OK;
}

extern "C" int lp_tensor_bdlt(lp_plan *p, int d, const double *in, double *out, void *stream) {
    return tensor_transform(p, p->tV, 0, d, in, out, as_stream(stream));
}

extern "C" int lp_tensor_fdlt(lp_plan *p, int d, const double *in, double *out, void *stream) {
    return tensor_transform(p, p->tF, 1, d, in, out, as_stream(stream));
}

// --------------------------------------------------------------- operator

extern "C" int lp_operator_create(lp_plan *plan, int d, const double *beta_grid,
                                  int n_axis_betas, const double *const *axis_betas,
                                  const double *alpha_grid, lp_operator **out) {
    *out = nullptr;
    LP_ARG(d >= 1 && d <= 3, "dim must be 1, 2 or 3");
    LP_ARG(n_axis_betas == 0 || n_axis_betas == d, "axis_betas must supply one field per axis");
    LP_ARG((n_axis_betas == 0) == (beta_grid != nullptr),
           "exactly one of beta / axis_betas is required");
    const int P = plan->P;
    LP_ARG(P >= 4, "plan order %d too small for an operator (N >= 3)", P);
    const int64_t nP = ipow(P, d);
    lp_operator *op = new lp_operator();
    op->plan = plan;
    op->d = d;
    op->P = P;
    op->K = P - 2;
    op->nP = nP;
    int rc;
    const int ngrids = n_axis_betas ? d : 1;
    double *stage = nullptr;
    if ((rc = dalloc(&stage, nP, "grid staging"))) { delete op; return rc; }
    cudaStream_t st = 0;
    auto fail = [&](int code) { dfree(stage); lp_operator_destroy(op); return code; };
    for (int g = 0; g < ngrids; ++g) {
        if ((rc = dalloc(&op->beta_w[g], nP, "weighted beta grid"))) return fail(rc);
        const double *src = n_axis_betas ? axis_betas[g] : beta_grid;
        const int64_t cnt = n_axis_betas ? P : nP;
        cudaError_t e = cudaMemcpy(stage, src, cnt * sizeof(double), cudaMemcpyDefault);
        if (e != cudaSuccess) return fail(cuda_fail(e, "beta upload", __FILE__, __LINE__));
        double mn;
        if ((rc = device_min(stage, cnt, &mn, st))) return fail(rc);
        if (!(mn > 0.0)) {
            set_error("diffusion coefficient is not positive on the grid (min %.3e)", mn);
            return fail(LP_ERR_NONPOSITIVE);
        }
        weighted_grid_kernel<<<(unsigned)ceil_div(nP, 256), 256, 0, st>>>(
            d, P, stage, n_axis_betas ? g : -1, plan->weights, op->beta_w[g]);
        count_launch();
    }
    for (int g = ngrids; g < d; ++g) op->beta_w[g] = op->beta_w[0];
    op->n_beta_grids = ngrids;
    if (alpha_grid) {
        if ((rc = dalloc(&op->alpha_w, nP, "weighted alpha grid"))) return fail(rc);
        cudaError_t e = cudaMemcpy(stage, alpha_grid, nP * sizeof(double), cudaMemcpyDefault);
        if (e != cudaSuccess) return fail(cuda_fail(e, "alpha upload", __FILE__, __LINE__));
        weighted_grid_kernel<<<(unsigned)ceil_div(nP, 256), 256, 0, st>>>(d, P, stage, -1,
                                                                         plan->weights, op->alpha_w);
        count_launch();
    }
    cudaError_t e = cudaDeviceSynchronize();
    dfree(stage);
    if (e != cudaSuccess) {
        lp_operator_destroy(op);
        return cuda_fail(e, "operator setup", __FILE__, __LINE__);
    }
    *out = op;
    return LP_OK;
}

extern "C" int lp_operator_destroy(lp_operator *op) {
    if (!op) return LP_OK;
    cudaDeviceSynchronize();
    for (int g = 0; g < op->n_beta_grids; ++g)
        if (op->beta_w[g]) dfree(op->beta_w[g]);
    if (op->alpha_w) dfree(op->alpha_w);
    for (int i = 0; i < op->nslabs; ++i) dfree(op->slabs[i].grid);
    delete op;
    return LP_OK;
}

namespace lp {

// 7 fields of P^d plus the per-CTA parts of the fused p'w (last fold pass: at most
// ceil(K^(d-1) / 64) * ceil(K / 128) CTAs)
static int64_t dot_parts(const lp_operator *op) {
    const int64_t lines = ipow(op->K, op->d - 1);
    return ((lines + LT_BN - 1) / LT_BN) * ((op->K / 2 + 1 + LT_BM - 1) / LT_BM + 1);
}
int64_t operator_ws_doubles(const lp_operator *op) { return 7 * op->nP + dot_parts(op); }

static int operator_apply_ws(lp_operator *op, int which, const double *u, double *out,
                             cudaStream_t st, double *ws, double *uw);

int operator_apply(lp_operator *op, int which, const double *u, double *out, cudaStream_t st,
                   double *ws, double *uw) {
    if (ws) return operator_apply_ws(op, which, u, out, st, ws, uw);
    double *tmp = nullptr;
    int rc = salloc(&tmp, (size_t)operator_ws_doubles(op), "operator workspace", st);
    if (rc) return rc;
    rc = operator_apply_ws(op, which, u, out, st, tmp, uw);
    sfree(tmp, st);
    return rc;
}

// uw (optional, device double-double pair): u' out, accumulated by the last fold
// pass (a part per CTA, summed in double-double in a fixed order).
static int operator_apply_ws(lp_operator *op, int which, const double *u, double *out,
                             cudaStream_t st, double *ws, double *uw) {
    const lp_plan *pl = op->plan;
    const LineTable &F = pl->tPhi, &D = pl->tDPhi;
    const int K = op->K, P = op->P, d = op->d;
    const bool hasA = (which & 1) != 0;
    const bool hasB = (which & 2) != 0 && op->alpha_w != nullptr;
    const int64_t nP = op->nP;
    double *A[4], *B[3];
    for (int i = 0; i < 4; ++i) A[i] = ws + i * nP;
    for (int i = 0; i < 3; ++i) B[i] = ws + (4 + i) * nP;
    const int64_t nK = ipow(K, d);
    if (!hasA && !hasB) {
        LP_CUDA(cudaMemsetAsync(out, 0, nK * sizeof(double), st));
        if (uw) LP_CUDA(cudaMemsetAsync(uw, 0, 2 * sizeof(double), st));
        return LP_OK;
    }
    int rc;
    double *parts = ws + 7 * nP;
    int64_t nparts = 0;
#define LAST(args)                                                    \
    do {                                                              \
        if (uw) {                                                     \
            (args).dotv = u;                                          \
            (args).dotpart = parts;                                   \
            nparts = line_transform_ctas(args);                       \
        }                                                             \
        if ((rc = line_transform((args), st))) return rc;             \
    } while (0)
#define RUN(args)                                   \
    do {                                            \
        if ((rc = line_transform((args), st))) return rc; \
    } while (0)
    if (d == 1) {
        LtArgs s = lt_unfold(F, 1);
        int o = 0;
        if (hasA) { lt_add_term(s, o, D, u); lt_set_out(s, o, A[0], op->beta_w[0]); ++o; }
        if (hasB) { lt_add_term(s, o, F, u); lt_set_out(s, o, A[1], op->alpha_w); ++o; }
        RUN(s);
        LtArgs f = lt_fold(F, 1);
        if (hasA) lt_add_term(f, 0, D, A[0]);
        if (hasB) lt_add_term(f, 0, F, A[1]);
        lt_set_out(f, 0, out);
        LAST(f);
    } else if (d == 2) {
        // S1 along x: G0 = Phi u (A[0]), G1 = dPhi u (A[1]) -> [x'][y]
        LtArgs s1 = lt_unfold(F, K);
        lt_add_term(s1, 0, F, u);
        lt_set_out(s1, 0, A[0]);
        if (hasA) { lt_add_term(s1, 1, D, u); lt_set_out(s1, 1, A[1]); }
        RUN(s1);
        // S2 along y: Q0 = Phi G1 (bw0), Q1 = dPhi G0 (bw1), Q2 = Phi G0 (aw) -> [y'][x']
        LtArgs s2 = lt_unfold(F, P);
        int o = 0;
        int q0 = -1, q1 = -1, q2 = -1;
        if (hasA) {
            q0 = o; lt_add_term(s2, o, F, A[1]); lt_set_out(s2, o, B[o], op->beta_w[0]); ++o;
            q1 = o; lt_add_term(s2, o, D, A[0]); lt_set_out(s2, o, B[o], op->beta_w[1]); ++o;
        }
        if (hasB) { q2 = o; lt_add_term(s2, o, F, A[0]); lt_set_out(s2, o, B[o], op->alpha_w); ++o; }
        RUN(s2);
        // S3 along x (fold): T02 = dPhi^T Q0 + Phi^T Q2 (A[0]); T1 = Phi^T Q1 (A[1]) -> [kx][y']
        LtArgs s3 = lt_fold(F, P);
        if (hasA) lt_add_term(s3, 0, D, B[q0]);
        if (hasB) lt_add_term(s3, 0, F, B[q2]);
        lt_set_out(s3, 0, A[0]);
        if (hasA) { lt_add_term(s3, 1, F, B[q1]); lt_set_out(s3, 1, A[1]); }
        RUN(s3);
        // S4 along y (fold): out = Phi^T T02 + dPhi^T T1 -> [ky][kx]
        LtArgs s4 = lt_fold(F, K);
        lt_add_term(s4, 0, F, A[0]);
        if (hasA) lt_add_term(s4, 0, D, A[1]);
        lt_set_out(s4, 0, out);
        LAST(s4);
    } else {
        // S1 along x: Gx0 = Phi u (A0), Gx1 = dPhi u (A1) -> [x'][z][y]
        LtArgs s1 = lt_unfold(F, K * K);
        lt_add_term(s1, 0, F, u);
        lt_set_out(s1, 0, A[0]);
        if (hasA) { lt_add_term(s1, 1, D, u); lt_set_out(s1, 1, A[1]); }
        RUN(s1);
        // S2 along y: (dx) Phi Gx1, (dy) dPhi Gx0, (dz + mass) Phi Gx0 -> [y'][x'][z]
        LtArgs s2 = lt_unfold(F, P * K);
        int o = 0, a0 = -1, a1 = -1, a2;
        if (hasA) {
            a0 = o; lt_add_term(s2, o, F, A[1]); lt_set_out(s2, o, B[o]); ++o;
            a1 = o; lt_add_term(s2, o, D, A[0]); lt_set_out(s2, o, B[o]); ++o;
        }
        a2 = o; lt_add_term(s2, o, F, A[0]); lt_set_out(s2, o, B[o]); ++o;
        RUN(s2);
        // S3 along z with the coefficient products: Q0..Q2 (beta), Q3 (alpha) -> [z'][y'][x']
        LtArgs s3 = lt_unfold(F, P * P);
        o = 0;
        int q0 = -1, q1 = -1, q2 = -1, q3 = -1;
        if (hasA) {
            q0 = o; lt_add_term(s3, o, F, B[a0]); lt_set_out(s3, o, A[o], op->beta_w[0]); ++o;
            q1 = o; lt_add_term(s3, o, F, B[a1]); lt_set_out(s3, o, A[o], op->beta_w[1]); ++o;
            q2 = o; lt_add_term(s3, o, D, B[a2]); lt_set_out(s3, o, A[o], op->beta_w[2]); ++o;
        }
        if (hasB) { q3 = o; lt_add_term(s3, o, F, B[a2]); lt_set_out(s3, o, A[o], op->alpha_w); ++o; }
        RUN(s3);
        // B1 along x (fold): W03 = dPhi^T Q0 + Phi^T Q3; W1 = Phi^T Q1; W2 = Phi^T Q2 -> [kx][z'][y']
        LtArgs b1 = lt_fold(F, P * P);
        if (hasA) lt_add_term(b1, 0, D, A[q0]);
        if (hasB) lt_add_term(b1, 0, F, A[q3]);
        lt_set_out(b1, 0, B[0]);
        if (hasA) {
            lt_add_term(b1, 1, F, A[q1]); lt_set_out(b1, 1, B[1]);
            lt_add_term(b1, 2, F, A[q2]); lt_set_out(b1, 2, B[2]);
        }
        RUN(b1);
        // B2 along y (fold): V0 = Phi^T W03 + dPhi^T W1; V1 = Phi^T W2 -> [ky][kx][z']
        LtArgs b2 = lt_fold(F, K * P);
        lt_add_term(b2, 0, F, B[0]);
        if (hasA) lt_add_term(b2, 0, D, B[1]);
        lt_set_out(b2, 0, A[0]);
        if (hasA) { lt_add_term(b2, 1, F, B[2]); lt_set_out(b2, 1, A[1]); }
        RUN(b2);
        // B3 along z (fold): out = Phi^T V0 + dPhi^T V1 -> [kz][ky][kx]
        LtArgs b3 = lt_fold(F, K * K);
        lt_add_term(b3, 0, F, A[0]);
        if (hasA) lt_add_term(b3, 0, D, A[1]);
        lt_set_out(b3, 0, out);
        LAST(b3);
    }
#undef RUN
#undef LAST
    if (uw) {
        if (nparts > dot_parts(op)) {
            set_error("internal: %lld dot parts exceed the workspace", (long long)nparts);
            return LP_ERR_ARG;
        }
        return sum_lines_dd(parts, nparts, uw, st);
    }
    return LP_OK;
}

}  // namespace lp

extern "C" int lp_apply_dot(lp_operator *op, int which, const double *u, double *out, double *uw,
                            void *stream) {
    LP_ARG(which >= 1 && which <= 3, "which must be 1 (A), 2 (B) or 3 (A+B)");
    LP_ARG(u != out, "output may not alias the input");
    LP_ARG(uw != nullptr, "uw must point to two device doubles");
    return lp::operator_apply(op, which, u, out, as_stream(stream), nullptr, uw);
}

extern "C" int lp_apply(lp_operator *op, int which, const double *u, double *out, void *stream) {
    LP_ARG(which >= 1 && which <= 3, "which must be 1 (A), 2 (B) or 3 (A+B)");
    LP_ARG(u != out, "output may not alias the input");
    return lp::operator_apply(op, which, u, out, as_stream(stream));
}
