// Slab-sharded 3-D matvec stages.
//
// The single-GPU operator (operator.cu) runs six line passes with a rotating
// layout: a pass transforms the fastest axis of its input and writes it as the
// slowest axis of its output, so the passes go x, y, z (unfold, coefficient
// products in the z epilogue) then x, y, z (fold).  Sharded over G ranks, each
// pass needs its axis local, which fixes the schedule:
//
//   vectors z-slab [z_g][y][x]  --S1(x) S2(y)-->  3 fields [y'][x'][z_g]
//   exchange E1 (y' slabs)      --S3(z)+grids, B1(x)-->  3 fields [kx][z'][y'_g]
//   exchange E2 (kx slabs)      --B2(y) B3(z)-->  [kz][ky][kx_g]
//   exchange E3 (kz slabs)      -->  w = (A+B) u on the z-slab [kz_g][ky][kx]
//
// The stages below are the compute between the exchanges; every line is the
// same line the single-GPU operator computes, with the same kernels, so the
// sharded result is bit-identical.  The exchanges are NCCL all-to-alls issued
// by the host (paper_2004_13961_b200/sharded.py); the chunk each rank sends to
// rank h is contiguous in these layouts (the distributed axis is the slowest),
// and lp_copy2d places received chunks (one strided copy per source rank).
#include "line_transform.cuh"
#include "lp_common.cuh"
#include "operator.cuh"

namespace lp {
namespace {

__global__ void copy2d_kernel(int64_t rows, int cols, const double *__restrict__ src, int64_t lds,
                              double *__restrict__ dst, int64_t ldd) {
    const int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / cols;
        const int c = (int)(e - r * cols);
        dst[r * ldd + c] = src[r * lds + c];
    }
}

int copy2d(int64_t rows, int cols, const double *src, int64_t lds, double *dst, int64_t ldd,
           cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return LP_OK;
    int64_t blocks = ceil_div(rows * cols, 256);
    if (blocks > num_sms() * 16) blocks = num_sms() * 16;
    copy2d_kernel<<<(unsigned)blocks, 256, 0, st>>>(rows, cols, src, lds, dst, ldd);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

#define RUN(args)                                         \
    do {                                                  \
        if ((rc = line_transform((args), st))) return rc; \
    } while (0)

}  // namespace
}  // namespace lp

using namespace lp;

extern "C" int lp_copy2d(int64_t rows, int cols, const double *src, int64_t lds, double *dst,
                         int64_t ldd, void *stream) {
    LP_ARG(cols >= 0 && rows >= 0 && lds >= cols && ldd >= cols, "copy2d: bad extents");
    return copy2d(rows, cols, src, lds, dst, ldd, as_stream(stream));
}

// Stage 1: S1 (x) and S2 (y) on nz planes of the z-slab.  u: [nz][K][K];
// f0, f1, f2: [P][P][nz] = Phi G1, dPhi G0, Phi G0 with G0 = Phi u, G1 = dPhi u
// along x (f0, f1 are left untouched when the operator has no A part).
extern "C" int lp_slab_forward(lp_operator *op, int which, int nz, const double *u, double *f0,
                               double *f1, double *f2, void *stream) {
    LP_ARG(op->d == 3, "slab stages are for 3-D operators");
    LP_ARG(which >= 1 && which <= 3, "which must be 1 (A), 2 (B) or 3 (A+B)");
    cudaStream_t st = as_stream(stream);
    const lp_plan *pl = op->plan;
    const LineTable &F = pl->tPhi, &D = pl->tDPhi;
    const int K = op->K, P = op->P;
    const bool hasA = (which & 1) != 0;
    if (nz <= 0) return LP_OK;
    double *g0 = nullptr, *g1 = nullptr;
    const size_t nf = (size_t)P * nz * K;
    LP_CUDA(cudaMallocAsync((void **)&g0, 2 * nf * sizeof(double), st));
    g1 = g0 + nf;
    int rc;
    auto body = [&]() -> int {
        LtArgs s1 = lt_unfold(F, K * nz);
        lt_add_term(s1, 0, F, u);
        lt_set_out(s1, 0, g0);
        if (hasA) { lt_add_term(s1, 1, D, u); lt_set_out(s1, 1, g1); }
        RUN(s1);
        LtArgs s2 = lt_unfold(F, P * nz);
        int o = 0;
        if (hasA) {
            lt_add_term(s2, o, F, g1); lt_set_out(s2, o, f0); ++o;
            lt_add_term(s2, o, D, g0); lt_set_out(s2, o, f1); ++o;
        }
        lt_add_term(s2, o, F, g0); lt_set_out(s2, o, f2);
        RUN(s2);
        return LP_OK;
    };
    rc = body();
    cudaFreeAsync(g0, st);
    return rc;
}

// Stage 2: S3 (z, with the coefficient products) and B1 (x, fold) on the
// y'-slab [y0, y0 + ny).  f0..f2: [ny][P][K] (z fastest, all K modes);
// w0, w1, w2: [K][P][ny] = dPhi^T Q0 + Phi^T Q3, Phi^T Q1, Phi^T Q2.
extern "C" int lp_slab_middle(lp_operator *op, int which, int y0, int ny, const double *f0,
                              const double *f1, const double *f2, double *w0, double *w1,
                              double *w2, void *stream) {
    LP_ARG(op->d == 3, "slab stages are for 3-D operators");
    LP_ARG(which >= 1 && which <= 3, "which must be 1 (A), 2 (B) or 3 (A+B)");
    const int K = op->K, P = op->P;
    LP_ARG(y0 >= 0 && ny >= 0 && y0 + ny <= P, "y' slab [%d, %d) outside [0, %d)", y0, y0 + ny, P);
    cudaStream_t st = as_stream(stream);
    if (ny <= 0) return LP_OK;
    const lp_plan *pl = op->plan;
    const LineTable &F = pl->tPhi, &D = pl->tDPhi;
    const bool hasA = (which & 1) != 0;
    const bool hasB = (which & 2) != 0 && op->alpha_w != nullptr;
    const size_t nq = (size_t)P * ny * P;   // [z'][ny][x']
    // the coefficient grids of the slab, in the S3 output layout [z'][y' - y0][x'],
    // extracted once per (operator, slab) and kept with the operator
    lp_operator::SlabGrid *sg = nullptr;
    for (int i = 0; i < op->nslabs; ++i)
        if (op->slabs[i].y0 == y0 && op->slabs[i].ny == ny) sg = &op->slabs[i];
    if (!sg) {
        if (op->nslabs < lp_operator::MAX_SLABS) {
            sg = &op->slabs[op->nslabs++];
        } else {
            // evict the oldest, stream-ordered after the work already queued on `st`
            sg = &op->slabs[0];
            dfree(sg->grid, st);
            for (int i = 1; i < op->nslabs; ++i) op->slabs[i - 1] = op->slabs[i];
            sg = &op->slabs[op->nslabs - 1];
        }
        sg->grid = nullptr;
        sg->y0 = sg->ny = -1;
        int rcg = salloc(&sg->grid, 4 * nq, "slab grids", st);
        if (rcg) {
            --op->nslabs;
            return rcg;
        }
        const double *src[4] = {op->beta_w[0], op->beta_w[1], op->beta_w[2], op->alpha_w};
        for (int g = 0; g < 4; ++g) {
            if (!src[g]) continue;
            // P planes z', each a block of ny rows of P at row offset y0
            for (int z = 0; z < P; ++z)
                if ((rcg = copy2d(ny, P, src[g] + ((size_t)z * P + y0) * P, P,
                                  sg->grid + g * nq + (size_t)z * ny * P, P, st)))
                    return rcg;
        }
        sg->y0 = y0;
        sg->ny = ny;
    }
    double *buf = nullptr;
    LP_CUDA(cudaMallocAsync((void **)&buf, 4 * nq * sizeof(double), st));
    double *q[4] = {buf, buf + nq, buf + 2 * nq, buf + 3 * nq};
    double *gr[4] = {sg->grid, sg->grid + nq, sg->grid + 2 * nq, sg->grid + 3 * nq};
    int rc = LP_OK;
    auto body = [&]() -> int {
        LtArgs s3 = lt_unfold(F, P * ny);
        int o = 0, iq0 = -1, iq1 = -1, iq2 = -1, iq3 = -1;
        if (hasA) {
            iq0 = o; lt_add_term(s3, o, F, f0); lt_set_out(s3, o, q[o], gr[0]); ++o;
            iq1 = o; lt_add_term(s3, o, F, f1); lt_set_out(s3, o, q[o], gr[1]); ++o;
            iq2 = o; lt_add_term(s3, o, D, f2); lt_set_out(s3, o, q[o], gr[2]); ++o;
        }
        if (hasB) { iq3 = o; lt_add_term(s3, o, F, f2); lt_set_out(s3, o, q[o], gr[3]); ++o; }
        RUN(s3);
        LtArgs b1 = lt_fold(F, P * ny);
        if (hasA) lt_add_term(b1, 0, D, q[iq0]);
        if (hasB) lt_add_term(b1, 0, F, q[iq3]);
        lt_set_out(b1, 0, w0);
        if (hasA) {
            lt_add_term(b1, 1, F, q[iq1]); lt_set_out(b1, 1, w1);
            lt_add_term(b1, 2, F, q[iq2]); lt_set_out(b1, 2, w2);
        }
        RUN(b1);
        return LP_OK;
    };
    rc = body();
    cudaFreeAsync(buf, st);
    (void)K;
    return rc;
}

// Stage 3: B2 (y, fold) and B3 (z, fold) on the kx-slab of nkx modes.
// w0, w1, w2: [nkx][P][P] (y' fastest, all P nodes); out: [K][K][nkx].
extern "C" int lp_slab_backward(lp_operator *op, int which, int nkx, const double *w0,
                                const double *w1, const double *w2, double *out, void *stream) {
    LP_ARG(op->d == 3, "slab stages are for 3-D operators");
    LP_ARG(which >= 1 && which <= 3, "which must be 1 (A), 2 (B) or 3 (A+B)");
    cudaStream_t st = as_stream(stream);
    if (nkx <= 0) return LP_OK;
    const lp_plan *pl = op->plan;
    const LineTable &F = pl->tPhi, &D = pl->tDPhi;
    const int K = op->K, P = op->P;
    const bool hasA = (which & 1) != 0;
    const size_t nv = (size_t)K * nkx * P;   // [ky][nkx][z']
    double *v0 = nullptr;
    LP_CUDA(cudaMallocAsync((void **)&v0, 2 * nv * sizeof(double), st));
    double *v1 = v0 + nv;
    int rc;
    auto body = [&]() -> int {
        LtArgs b2 = lt_fold(F, nkx * P);
        lt_add_term(b2, 0, F, w0);
        if (hasA) lt_add_term(b2, 0, D, w1);
        lt_set_out(b2, 0, v0);
        if (hasA) { lt_add_term(b2, 1, F, w2); lt_set_out(b2, 1, v1); }
        RUN(b2);
        LtArgs b3 = lt_fold(F, K * nkx);
        lt_add_term(b3, 0, F, v0);
        if (hasA) lt_add_term(b3, 0, D, v1);
        lt_set_out(b3, 0, out);
        RUN(b3);
        return LP_OK;
    };
    rc = body();
    cudaFreeAsync(v0, st);
    return rc;
}
