// Internal definition of the sparse-matrix / ILU(0) handle.
#pragma once

#include "lp_common.cuh"

namespace lp {

enum { MAT_CSR = 0, MAT_BOX = 1 };

// Implicit-offset ("box") storage of a Kronecker-banded matrix: every row has
// S = (2r+1)^d slots, slot s <-> offset (ox, oy, oz) in [-r, r]^d with ox
// fastest; values[row * S + s] holds entry (row, row + ox + K oy + K^2 oz) or
// 0 where that column is outside the grid.  Slot order equals column order for
// the valid slots of every row (|ox| < K), so "lower" = s < S/2, "diag" = S/2.
struct BoxLayout {
    int d = 0, K = 0, r = 0, W = 0;   // W = 2r + 1
    int S = 0;                        // W^d slots
    int64_t n = 0;
    double *values = nullptr;         // original M            [n][S]
    double *lu = nullptr;             // ILU(0) factors         [n][S]
    uint32_t *mask = nullptr;         // in-pattern bits        [n][ceil(S/32)] (null: all valid slots)
    unsigned char *full = nullptr;    // [n]: every slot of the row is in the pattern
    int mask_words = 0;
    int64_t nnz = 0;
    // compact in-line bands of the factors for the sweeps' serial recurrence:
    // band_lo[row][q] = L(row, row-1-q), band_up[row][q] = U(row, row+1+q), q < r
    double *band_lo = nullptr, *band_up = nullptr, *diag = nullptr;
    // 3-D sweeps: x-lines in wavefront order (see box_sweep3d.cu)
    int *line_order = nullptr;
    int *line_groups = nullptr;   // small reach: starts of same-key groups in line_order
    int n_line_groups = 0;
    // one rank's lines of a y-slab split (multi-GPU sweeps): forward / backward
    // wavefront orders filtered to the rank's lines, and their same-key groups
    struct RankOrder {
        int sig[11] = {-1};       // nranks, own, ys[0..nranks]
        int *order = nullptr, *groups = nullptr;
        int norder = 0, ngroups = 0;
    } rank_order[2];
    // even-offset pattern (T = 0: every in-pattern offset even in each axis): the
    // factors compacted to the 27 even slots of the r = 2 box, [n][27] (3-D sweeps)
    double *even = nullptr;
    // 2-D factorisation (ilu_box2d.cu): block tasks in key order, RN(1/u_ii) per row
    int *ilu_tasks = nullptr;
    int ilu_ntask = 0, ilu_nb = 0;
    double *rdiag = nullptr;          // [n][2]
};

}  // namespace lp

struct lp_ilu {
    int kind = lp::MAT_CSR;
    int64_t n = 0, nnz = 0;
    // CSR (kind == MAT_CSR)
    int64_t *indptr = nullptr;
    int32_t *indices = nullptr;
    double *values = nullptr;   // original M
    double *lu = nullptr;       // factors in the pattern of M (L strictly lower, U upper)
    int64_t *diag = nullptr;
    // box layout (kind == MAT_BOX)
    lp::BoxLayout box;
    // sweep state
    bool factored = false;
    int *flags = nullptr;       // per-row progress, compared against `epoch`
    int epoch = 0;
    int *ticket = nullptr;      // dynamic row tickets (2 counters)
    int64_t *bad = nullptr;     // zero-pivot key (device)
    int64_t missing_diag = -1;  // first row without a stored diagonal (box assembly)
};

namespace lp {
// Per-call sweep state (stream-ordered scratch): the sweeps never write to the
// handle, so concurrent precond_apply / pcg_solve calls on one set of factors
// (different streams or threads) are independent.
struct SweepScratch {
    double *ytmp = nullptr;   // [n] forward-sweep result of precond_apply
    int *tickets = nullptr;   // [2] line / row tickets (forward, backward)
    int *flags = nullptr;     // [n] CSR sweeps: per-row progress
    double *dotpart = nullptr;   // fused r'z: per-line parts (box) / dd block partials (others)
};
int scratch_alloc(const lp_ilu *m, SweepScratch &s, cudaStream_t st);
void scratch_free(SweepScratch &s, cudaStream_t st);
// 3-D sweeps with the vector distributed over y-slab ranks: own = -1 is the
// one-launch emulation of every rank (replicas at out + v n, lp_sweep_ranks);
// own >= 0 is one rank of a multi-GPU run (lp_sweep_rank): only its lines, its
// replica `out`, the neighbours' replicas in peers[v] (IPC-mapped).
struct RankLayout {
    int nranks = 1;
    int ys[9] = {0};
    bool rhs_replicated = false;
    int own = -1;
    double *peers[8] = {nullptr};
};
int ilu_apply(lp_ilu *m, const double *r, double *z, const SweepScratch &s, cudaStream_t st);
// z = M^-1 r and rz = r'z (device double-double pair): fused into the backward
// sweep where the kernel supports it, a deterministic dot on the same stream otherwise
int ilu_apply_dot(lp_ilu *m, const double *r, double *z, const SweepScratch &s, double *rz, cudaStream_t st);
bool box_apply_dot_fused(const lp_ilu *m);
int box_apply_dot(lp_ilu *m, const double *r, double *z, const SweepScratch &s, double *rz, cudaStream_t st);
int ilu_forward(lp_ilu *m, const double *r, double *y, const SweepScratch &s, cudaStream_t st);
int ilu_backward(lp_ilu *m, const double *y, double *z, const SweepScratch &s, cudaStream_t st);
int box_forward(lp_ilu *m, const double *r, double *y, int *ticket, cudaStream_t st);
int box_backward(lp_ilu *m, const double *y, double *z, int *ticket, cudaStream_t st);
int box_ilu0(lp_ilu *m, double tol, int64_t *bad_row, cudaStream_t st);
int box_spmv(lp_ilu *m, const double *x, double *y, cudaStream_t st);
int box_export(const lp_ilu *m, int which, int64_t *indptr, int32_t *indices, double *values);
int box_build_bands(lp_ilu *m, cudaStream_t st);
int box_build_even(lp_ilu *m, cudaStream_t st);
int box_apply(lp_ilu *m, const double *r, double *z, const SweepScratch &s, cudaStream_t st);
int box_ilu0_2d_tasks(lp_ilu *m, const double *src, double tol, unsigned long long *key, int *done,
                      cudaStream_t st);
// y-slab rank layout of a multi-GPU ILU(0) (see ilu_box3d.cu): rank v factors the
// x-lines with y in [ys[v], ys[v+1]) in lu[v]; own = -1 runs every rank in one
// launch (emulation), own >= 0 one rank with its neighbours' arrays in lu/flags.
struct IluRanks {
    int nranks = 1, own = -1;
    int ys[9] = {0};
    double *lu[8] = {nullptr};
    int *flags[8] = {nullptr};
};
int box_ilu0_3d_rows(lp_ilu *m, double tol, unsigned long long *key, cudaStream_t st,
                     const IluRanks *ranks = nullptr);
int box_ilu0_prepare(lp_ilu *m, int64_t *bad_row, cudaStream_t st);
int box_ilu0_ranks(lp_ilu *const *ms, int nranks, const int *ys, int own, double *const *peer_lu,
                   int *const *peer_flags, double tol, int64_t *bad_row, cudaStream_t st);
int box_ilu0_3d_blocks(lp_ilu *m, double tol, unsigned long long *key, cudaStream_t st);
struct Geom;
bool box_sweep3d_applies(const Geom &g);
int ensure_line_order(BoxLayout &b, cudaStream_t st);
int box_sweep3d(lp_ilu *m, bool fwd, const double *rhs, double *out, int *ticket, cudaStream_t st,
                const RankLayout *ranks = nullptr);
}  // namespace lp
