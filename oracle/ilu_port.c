/*
 * ORACLE -- test infrastructure only.  Not part of the product path.
 *
 * Plain-C restatement of the reference's sequential sparse kernels
 * (reference: pkg/src/legpcg/sparse.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Built with -ffp-contract=off so every a - l*u is a separately rounded
 * multiply and subtract, exactly as the numba kernels compile (SURVEY 8(a) a11:
 * the numba IR has no FMA contraction).  The ILU(0) factors are therefore
 * bit-identical to the reference's for the same CSR input.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

/* _ilu0_kernel, sparse.py:116-139.  IKJ elimination restricted to the
 * pattern, rows in natural order, a dense row marker for the pattern test.
 * Returns -1 on success or the pivot row k whose |u_kk| < pivot_tol. */
int64_t oracle_ilu0(int64_t n, const int64_t *indptr, const int64_t *indices,
                    double *data, const int64_t *diag_ptr, double pivot_tol)
{
    int64_t *marker = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) marker[i] = -1;
    int64_t bad = -1;
    for (int64_t i = 0; i < n && bad < 0; ++i) {
        const int64_t lo = indptr[i], hi = indptr[i + 1];
        for (int64_t e = lo; e < hi; ++e) marker[indices[e]] = e;
        for (int64_t e = lo; e < hi; ++e) {
            const int64_t k = indices[e];
            if (k >= i) break;
            const double piv = data[diag_ptr[k]];
            if (fabs(piv) < pivot_tol) { bad = k; break; }
            const double lik = data[e] / piv;
            data[e] = lik;
            for (int64_t f = diag_ptr[k] + 1; f < indptr[k + 1]; ++f) {
                const int64_t pos = marker[indices[f]];
                if (pos >= 0) {
                    data[pos] = data[pos] - lik * data[f];
                }
            }
        }
        for (int64_t e = lo; e < hi; ++e) marker[indices[e]] = -1;
    }
    free(marker);
    return bad;
}

/* _forward_kernel, sparse.py:175-181: y_i = r_i - sum_{j<i} L_ij y_j, the
 * sum accumulated left to right over the stored (strictly lower) entries. */
void oracle_forward(int64_t n, const int64_t *indptr, const int64_t *indices,
                    const double *values, const double *r, double *y)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            acc = acc + values[e] * y[indices[e]];
        }
        y[i] = r[i] - acc;
    }
}

/* _backward_kernel, sparse.py:184-196: z_i = (y_i - sum_{j>i} U_ij z_j)/U_ii,
 * rows from last to first, the diagonal read out of the row. */
void oracle_backward(int64_t n, const int64_t *indptr, const int64_t *indices,
                     const double *values, const double *y, double *z)
{
    for (int64_t i = n - 1; i >= 0; --i) {
        double acc = 0.0, diag = 0.0;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            const int64_t j = indices[e];
            if (j == i) {
                diag = values[e];
            } else {
                acc = acc + values[e] * z[j];
            }
        }
        z[i] = (y[i] - acc) / diag;
    }
}

/* _spmv_kernel, sparse.py:97-113 (used by the oracle's residual checks). */
void oracle_spmv(int64_t n, const int64_t *indptr, const int64_t *indices,
                 const double *values, const double *x, double *y)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            acc = acc + values[e] * x[indices[e]];
        }
        y[i] = acc;
    }
}
