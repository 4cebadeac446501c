// Coefficient / right-hand-side front end on the GPU:
//
//   lp_blocks_1d      the exact-quadrature diagonals of the 1-D blocks
//                     S^(t) = (L_t phi', phi'), M^(t) = (L_t phi, phi)
//                     (building_blocks_1d, precond.py:118-161);
//   lp_mass_contract  the closed-form mass contraction of a Legendre
//                     coefficient tensor on every axis, P^d -> K^d
//                     (_mass_contract, operator.py:131-143; the last step of
//                     assemble_rhs, operator.py:213-222).
//
// Both reproduce the reference's arithmetic operation for operation (every
// product, sum and quotient separately rounded, the quadrature sum in node
// order in chunks of 512 nodes), so the outputs are bit-identical to the host
// restatement they replace.
#include <vector>

#include "lp_common.cuh"

namespace lp {

namespace {

// tab[p][k] = L_k(x_p), k = 0..ncol-1, with the reference recurrence
// (legendre.py:86-95), every operation separately rounded.
__global__ void legendre_rows_kernel(int Q, int ncol, const double *__restrict__ x, double *__restrict__ tab) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= Q) return;
    const double xp = x[p];
    double *row = tab + (size_t)p * ncol;
    double lm1 = 1.0, l = xp;
    row[0] = 1.0;
    if (ncol > 1) row[1] = xp;
    for (int k = 1; k + 1 < ncol; ++k) {
        const double t = __dmul_rn(__dmul_rn((double)(2 * k + 1), xp), l);
        const double nxt = __ddiv_rn(__dsub_rn(t, __dmul_rn((double)k, lm1)), (double)(k + 1));
        row[k + 1] = nxt;
        lm1 = l;
        l = nxt;
    }
}

// basis[kind][p][i]: stiff -(2i+3) L_{i+1}(x_p), mass L_i - L_{i+2} (precond.py:137-139)
__global__ void basis_kernel(int Q, int K, const double *__restrict__ tab, double *__restrict__ basis) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= (int64_t)Q * K) return;
    const int p = (int)(q / K), i = (int)(q % K);
    const double *row = tab + (size_t)p * (K + 2);
    basis[q] = __dmul_rn(-(2.0 * i + 3.0), row[i + 1]);
    basis[(size_t)Q * K + q] = __dsub_rn(row[i], row[i + 2]);
}

struct Combo {
    int kind, t, o;
};

// One (kind, t, o >= 0) diagonal per blockIdx.y, one entry i per thread:
// sum_p (w_p L_t(x_p) b_i(x_p)) b_{i+o}(x_p), nodes in order, a partial sum
// per chunk of 512 nodes added to the running total (precond.py:128-150).
__global__ void blocks_kernel(int Q, int K, int T, const Combo *__restrict__ combos,
                              const double *__restrict__ tab, const double *__restrict__ w,
                              const double *__restrict__ basis, double *__restrict__ blocks) {
    const Combo c = combos[blockIdx.y];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K - c.o) return;
    const int R = T + 2;
    const double *b = basis + (size_t)c.kind * Q * K;
    double acc = 0.0;
    for (int lo = 0; lo < Q; lo += 512) {
        const int hi = min(lo + 512, Q);
        double s = 0.0;
        for (int p = lo; p < hi; ++p) {
            const double wt = __dmul_rn(w[p], tab[(size_t)p * (K + 2) + c.t]);
            const double *bp = b + (size_t)p * K;
            s = __dadd_rn(s, __dmul_rn(__dmul_rn(wt, bp[i]), bp[i + c.o]));
        }
        acc = __dadd_rn(acc, s);
    }
    double *blk = blocks + ((size_t)c.kind * (T + 1) + c.t) * (2 * R + 1) * K;
    blk[(size_t)(R + c.o) * K + i] = acc;
    if (c.o > 0) blk[(size_t)(R - c.o) * K + i + c.o] = acc;   // the block is symmetric
}

// out[lo + nlo (k + K hi)] = c1(k) in[lo + nlo (k + P hi)] - c2(k) in[lo + nlo (k + 2 + P hi)]
__global__ void contract_axis_kernel(int64_t nlo, int P, int64_t nhi, const double *__restrict__ in,
                                     double *__restrict__ out) {
    const int K = P - 2;
    const int64_t total = nlo * K * nhi;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = q % nlo, r = q / nlo;
        const int k = (int)(r % K);
        const int64_t hi = r / K;
        const double *src = in + lo + nlo * (k + (int64_t)P * hi);
        const double c1 = __ddiv_rn(2.0, 2.0 * k + 1.0), c2 = __ddiv_rn(2.0, 2.0 * k + 5.0);
        out[q] = __dsub_rn(__dmul_rn(c1, src[0]), __dmul_rn(c2, src[2 * nlo]));
    }
}

}  // namespace

}  // namespace lp

using namespace lp;

extern "C" int lp_blocks_1d(int T, int K, int Q, const double *nodes, const double *weights, double *blocks) {
    LP_ARG(T >= 0 && K >= 1, "need T >= 0 and K >= 1");
    LP_ARG(Q >= K + T / 2 + 2, "quadrature order %d is insufficient for exact blocks with T=%d, K=%d", Q, T, K);
    LP_ARG(nodes && weights && blocks, "null argument");
    const int R = T + 2;
    const size_t nblk = (size_t)2 * (T + 1) * (2 * R + 1) * K;
    std::vector<Combo> combos;
    for (int kind = 0; kind < 2; ++kind)
        for (int t = 0; t <= T; ++t) {
            const int reach = kind == 0 ? t : t + 2;
            for (int o = 0; o <= reach && o < K; ++o)
                if ((o - t) % 2 == 0) combos.push_back({kind, t, o});
        }
    double *dx = nullptr, *dw = nullptr, *tab = nullptr, *basis = nullptr, *dblk = nullptr;
    Combo *dc = nullptr;
    int rc;
    auto done = [&](int code) {
        dfree(dx); dfree(dw); dfree(tab); dfree(basis); dfree(dblk); dfree(dc);
        return code;
    };
    if ((rc = dalloc(&dx, (size_t)Q, "quadrature nodes")) || (rc = dalloc(&dw, (size_t)Q, "quadrature weights")) ||
        (rc = dalloc(&tab, (size_t)Q * (K + 2), "Legendre table")) ||
        (rc = dalloc(&basis, (size_t)2 * Q * K, "basis table")) || (rc = dalloc(&dblk, nblk, "1-D blocks")) ||
        (rc = dalloc(&dc, combos.size(), "block list")))
        return done(rc);
    cudaError_t e;
    if ((e = cudaMemcpy(dx, nodes, (size_t)Q * sizeof(double), cudaMemcpyDefault)) != cudaSuccess ||
        (e = cudaMemcpy(dw, weights, (size_t)Q * sizeof(double), cudaMemcpyDefault)) != cudaSuccess ||
        (e = cudaMemcpy(dc, combos.data(), combos.size() * sizeof(Combo), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemset(dblk, 0, nblk * sizeof(double))) != cudaSuccess)
        return done(cuda_fail(e, "1-D block upload", __FILE__, __LINE__));
    legendre_rows_kernel<<<(Q + 127) / 128, 128>>>(Q, K + 2, dx, tab);
    basis_kernel<<<(unsigned)ceil_div((int64_t)Q * K, 256), 256>>>(Q, K, tab, basis);
    blocks_kernel<<<dim3((unsigned)ceil_div(K, 128), (unsigned)combos.size()), 128>>>(Q, K, T, dc, tab, dw, basis,
                                                                                      dblk);
    count_launch(3);
    if ((e = cudaGetLastError()) != cudaSuccess ||
        (e = cudaMemcpy(blocks, dblk, nblk * sizeof(double), cudaMemcpyDefault)) != cudaSuccess)
        return done(cuda_fail(e, "1-D blocks", __FILE__, __LINE__));
    return done(LP_OK);
}

extern "C" int lp_mass_contract(int d, int P, const double *in, double *out, void *stream) {
    LP_ARG(d >= 1 && d <= 3, "dimension must be 1, 2 or 3");
    LP_ARG(P >= 3, "need at least 3 Legendre coefficients per axis");
    LP_ARG(in && out, "null argument");
    cudaStream_t st = as_stream(stream);
    const int K = P - 2;
    // axis a: nlo = K^a (axes already contracted), nhi = P^(d-1-a)
    double *tmp[2] = {nullptr, nullptr};
    int rc;
    if (d > 1) {
        size_t big = (size_t)K;
        for (int a = 1; a < d; ++a) big *= (size_t)P;
        if ((rc = salloc(&tmp[0], big, "contraction workspace", st))) return rc;
        if (d > 2 && (rc = salloc(&tmp[1], big, "contraction workspace", st))) {
            sfree(tmp[0], st);
            return rc;
        }
    }
    const double *src = in;
    for (int a = 0; a < d; ++a) {
        int64_t nlo = 1, nhi = 1;
        for (int q = 0; q < a; ++q) nlo *= K;
        for (int q = a + 1; q < d; ++q) nhi *= P;
        double *dst = a == d - 1 ? out : tmp[a & 1];
        const int64_t total = nlo * K * nhi;
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(total, 256), (int64_t)num_sms() * 16);
        contract_axis_kernel<<<grid, 256, 0, st>>>(nlo, P, nhi, src, dst);
        count_launch();
        src = dst;
    }
    LP_CHECK_LAUNCH();
    sfree(tmp[0], st);
    sfree(tmp[1], st);
    return LP_OK;
}
