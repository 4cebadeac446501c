/*
 * legpcg_b200 -- C ABI of the B200-native (sm_100a, fp64) hot path of the
 * preconditioned Legendre-Galerkin PCG solver (arXiv:2004.13961).
 *
 * The reference (/root/reference/pkg, Python package `legpcg`) has no FFI;
 * its boundary is the Python module API that `pcg_solve` calls.  Each entry
 * point below replaces one reference function and cites it (file:line
 * relative to /root/reference).  The Python shim `paper_2004_13961_b200`
 * binds these with ctypes and re-exports the reference names.
 *
 * Conventions
 *  - Plain C types only.  Handles are opaque, library-owned objects.
 *  - Vectors are caller-owned DEVICE pointers, x-fastest ("Fortran") order,
 *    exactly the PCG vectors of pcg.py:132-135.  Arrays documented as
 *    "host or device" are copied with cudaMemcpyDefault (UVA).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *  - Every call returns 0 on success or a negative LP_ERR_* code;
 *    lp_last_error() returns a human-readable message for the calling thread.
 *  - Not thread-safe per handle: one handle per stream.
 */
#ifndef LEGPCG_B200_H
#define LEGPCG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    LP_OK = 0,
    LP_ERR_CUDA = -1,          /* CUDA runtime error (message in lp_last_error) */
    LP_ERR_ARG = -2,           /* bad size / shape      -> ValueError            */
    LP_ERR_NONPOSITIVE = -3,   /* beta <= 0 on the grid -> ValueError (operator.py:116-119) */
    LP_ERR_ZERO_PIVOT = -4,    /* ILU(0) pivot          -> IluZeroPivotError (sparse.py:30-35) */
    LP_ERR_INDEFINITE = -5,    /* p'Ap <= 0             -> IndefiniteOperatorError (pcg.py:34-42) */
    LP_ERR_NODEVICE = -6,      /* no sm_100 device      -> RuntimeError          */
    LP_ERR_OOM = -7            /* device allocation failed                        */
};

typedef struct lp_plan lp_plan;         /* TransformPlan (transforms.py:289-325)     */
typedef struct lp_operator lp_operator; /* ProblemSpec + plan bound for A+B          */
typedef struct lp_ilu lp_ilu;           /* SparseMatrix M and/or IluFactors          */

const char *lp_last_error(void);
const char *lp_version(void);
/* Number of this library's kernels launched so far by the process (diagnostics). */
int64_t lp_kernel_launches(void);
/* Checks that device `device` is an sm_100 part and makes it current. */
int lp_init(int device);

/* ---------------------------------------------------------------- plans --
 * TransformPlan(order, "reference") (transforms.py:298-310).  nodes/weights
 * are the P-point Gauss rule (legendre.py:109-145) computed on the host, host
 * or device pointers.  The library builds, on the device, the Vandermonde
 * table V[k,n] = L_n(x_k) with the reference's recurrence (legendre.py:86-95)
 * evaluated with separately rounded operations (bit-identical to the
 * reference table), the Shen-basis tables Phi[k,m] = phi_m(x_k),
 * dPhi[k,m] = phi_m'(x_k) (m < K = P-2), and their parity-split
 * unfold/fold forms. */
int lp_plan_create(int P, const double *nodes, const double *weights, lp_plan **out);
int lp_plan_destroy(lp_plan *plan);
/* Copies the P x P table V (row-major, V[k*P+n]) to `dst` (host or device). */
int lp_plan_table(const lp_plan *plan, double *dst);

/* tensor_bdlt / tensor_fdlt (transforms.py:368-375) of a P^d tensor.  The
 * transform is applied to every axis; in/out are device, length P^d, any
 * axis order (all axes are transformed identically). */
int lp_tensor_bdlt(lp_plan *plan, int d, const double *in, double *out, void *stream);
int lp_tensor_fdlt(lp_plan *plan, int d, const double *in, double *out, void *stream);

/* ------------------------------------------------------------ operator --
 * apply_A / apply_B / apply_system (operator.py:161-210).
 * beta_grid: P^d values of beta on the Gauss grid, x fastest (host or
 *   device), used when n_axis_betas == 0;
 * axis_betas: n_axis_betas == d arrays of P values beta_i(x_i) for the
 *   per-axis diffusion form (operator.py:155-158);
 * alpha_grid: P^d values of alpha, or NULL when alpha is None / is_zero.
 * The positivity test of operator.py:116-119 runs once, at creation. */
int lp_operator_create(lp_plan *plan, int d, const double *beta_grid,
                       int n_axis_betas, const double *const *axis_betas,
                       const double *alpha_grid, lp_operator **out);
int lp_operator_destroy(lp_operator *op);
/* which: 1 = A (apply_A), 2 = B (apply_B), 3 = A + B (apply_system).
 * u, out: device, K^d, x fastest.  out may not alias u. */
int lp_apply(lp_operator *op, int which, const double *u, double *out, void *stream);
/* The same with the scalar u'(Op u) as a second output (the curvature p'w of
 * pcg.py:156-157): uw points to two device doubles (a double-double pair).
 * The last line pass of the matvec accumulates it in its epilogue, one part
 * per CTA, summed in double-double in a fixed order (deterministic). */
int lp_apply_dot(lp_operator *op, int which, const double *u, double *out, double *uw,
                 void *stream);

/* ------------------------------------------------ slab-sharded 3-D matvec --
 * apply_system (operator.py:204-210) split into the compute stages of a
 * z-slab sharded schedule; the host runs the three
 * all-to-alls between them (paper_2004_13961_b200/sharded.py).  All arrays
 * are device, row-major in the listed axis order (last axis fastest).
 *   forward:  u [nz][K][K]                      -> f0, f1, f2 [P][P][nz]
 *   middle:   f0..f2 [ny][P][K] (y' slab y0..)  -> w0, w1, w2 [K][P][ny]
 *   backward: w0..w2 [nkx][P][P]                -> out [K][K][nkx]
 * Each line is computed exactly as by lp_apply, so the sharded product is
 * bit-identical.  lp_copy2d copies a rows x cols block between leading
 * dimensions lds and ldd (placement of received all-to-all chunks). */
int lp_slab_forward(lp_operator *op, int which, int nz, const double *u, double *f0,
                    double *f1, double *f2, void *stream);
int lp_slab_middle(lp_operator *op, int which, int y0, int ny, const double *f0,
                   const double *f1, const double *f2, double *w0, double *w1, double *w2,
                   void *stream);
int lp_slab_backward(lp_operator *op, int which, int nkx, const double *w0, const double *w1,
                     const double *w2, double *out, void *stream);
int lp_copy2d(int64_t rows, int cols, const double *src, int64_t lds, double *dst, int64_t ldd,
              void *stream);

/* forward_sub (dir 0) / backward_sub (dir 1) of 3-D box factors with the vector
 * distributed over nranks y-slab ranks (rank v owns the x-lines with y in
 * [ys[v], ys[v+1])), emulated on one device in one launch: `out` holds nranks
 * replicas of n values (replica v at out + v*n); each line is computed from its
 * owner's replica and stored to the owner and to every rank whose stencil halo
 * [ys[u] - r, ys[u+1] + r) contains it -- the stores a multi-GPU run makes into
 * its neighbours' memory.  rhs: one vector, or nranks replicas when
 * rhs_replicated != 0.  Results equal lp_forward_sub / lp_backward_sub. */
int lp_sweep_ranks(lp_ilu *f, int nranks, const int *ys, int dir, const double *rhs,
                   int rhs_replicated, double *out, void *stream);

/* One rank of the same sweep in a multi-GPU run (one process per GPU, every
 * rank launching concurrently): only this rank's lines, in the global
 * wavefront order.  out: this rank's replica (n values: the rank's own lines
 * and the halo lines its neighbours store into it), pre-filled with
 * lp_sweep_prefill BEFORE the ranks synchronise for the sweep (a neighbour's
 * halo stores must land after the fill); rhs: this rank's replica of the
 * right-hand side; peers[v]: rank v's
 * replica mapped with lp_ipc_open (required for the slab neighbours rank-1 and
 * rank+1; halo values are stored into it over NVLink with .sys-scope stores).
 * Replaces, per rank, the forward_sub / backward_sub of sparse.py:199-216. */
int lp_sweep_rank(lp_ilu *f, int nranks, const int *ys, int rank, int dir, const double *rhs,
                  double *out, double *const *peers, void *stream);
int lp_sweep_prefill(int64_t n, double *out, void *stream);

/* CUDA IPC for the replicas: a cudaMalloc'd buffer and its 64-byte handle;
 * mapping / unmapping a peer's handle. */
int lp_ipc_alloc(int64_t bytes, void **ptr, unsigned char *handle64);
int lp_ipc_free(void *ptr);
int lp_ipc_open(const unsigned char *handle64, void **ptr);
int lp_ipc_close(void *ptr);

/* ----------------------------------------------------- preconditioner --
 * General CSR matrix (SparseMatrix, sparse.py:38-86): upload and hold.
 * indptr[n+1], indices[nnz] (sorted per row), values[nnz]; host or device. */
int lp_csr_create(int64_t n, int64_t nnz, const int64_t *indptr,
                  const int32_t *indices, const double *values, lp_ilu **out);

/* assemble_M (precond.py:207-297) into the implicit-offset "box" layout:
 * M[row][slot], slot <-> offset (o_x, o_y, o_z) in [-r, r]^d, x fastest.
 * n_groups terms; group g has a hat tensor of shape lens[g][0..d-1]
 * (C order, axis 0 = x), stiff_axis[g] in {-1, 0..d-1}.  The 1-D blocks
 * S^(t), M^(t) (building_blocks_1d, precond.py:118-161) are passed as
 * diagonal stacks: blocks[kind][t][o + R][i] = entry (i, i+o) of block t
 * (kind 0 = stiff, 1 = mass), for t <= tmax, |o| <= R = tmax + 2, i < K.
 * Entries |v| < 1e-300 are dropped from the pattern (precond.py:272-297). */
int lp_box_assemble(int d, int K, int n_groups, const int *lens,
                    const int *stiff_axis, const double *const *hats,
                    int tmax, const double *blocks, lp_ilu **out);

/* building_blocks_1d (precond.py:118-161) on the GPU: the diagonals of the
 * exact-quadrature 1-D blocks for t = 0..T on the Q-point Gauss rule
 * (nodes, weights: host or device, Q >= K + T/2 + 2), written to `blocks`
 * (host or device) in the layout lp_box_assemble takes:
 * blocks[kind][t][o + R][i], R = T + 2.  Same operation order as the
 * reference (node order, chunks of 512 nodes): bit-identical diagonals. */
int lp_blocks_1d(int T, int K, int Q, const double *nodes, const double *weights,
                 double *blocks);

/* _mass_contract (operator.py:131-143) on every axis of a P^d Legendre
 * coefficient tensor: out_k = 2 v_k/(2k+1) - 2 v_{k+2}/(2k+5), P^d -> K^d,
 * K = P - 2 (the last step of assemble_rhs, operator.py:213-222).  in/out
 * are device vectors, x fastest; axis 0 first, each operation separately
 * rounded (bit-identical to the reference's numpy expression). */
int lp_mass_contract(int d, int P, const double *in, double *out, void *stream);

/* Number of stored entries (SparseMatrix.nnz) and CSR export (host arrays
 * sized by nnz; indices/values may be NULL to fetch only indptr). */
int lp_matrix_nnz(const lp_ilu *m, int64_t *nnz);
int lp_matrix_export(const lp_ilu *m, int which /*0=M,1=L,2=U*/, int64_t *indptr,
                     int32_t *indices, double *values);

/* ilu0 (sparse.py:142-172): factor in place, keeping the original M.  On a
 * zero pivot returns LP_ERR_ZERO_PIVOT with *bad_row set to the row the
 * reference would report (missing diagonal, |u_kk| < pivot_tol). */
int lp_ilu0(lp_ilu *m, double pivot_tol, int64_t *bad_row, void *stream);

/* ILU(0) of a 3-D box matrix distributed over nranks y-slab ranks (rank v owns
 * the x-lines with y in [ys[v], ys[v+1]); the factorisation uses
 * the sweeps' wavefront and the neighbours' U rows of the r halo lines).  A
 * finished row goes to its owner's factor array and, its diagonal and upper
 * planes, to every rank whose halo [ys[u] - r, ys[u+1] + r) contains its
 * line, followed by that replica's line flag.  Every row's arithmetic is that
 * of lp_ilu0 (sparse.py:116-139), so a rank's rows equal the single-GPU
 * factors bit for bit.
 *   lp_ilu0_ranks: one-device emulation, f[v] = rank v's matrix (each assembled
 *     from the same problem), every rank in one launch, each reading only its
 *     own array.
 *   lp_ilu0_rank: one rank of a multi-GPU run (one process per GPU, launched
 *     concurrently); peer_lu[v] / peer_flags[v]: rank v's factor and flag
 *     arrays (lp_ilu_rank_arrays) mapped with lp_ipc_open -- required for the
 *     slab neighbours; system-scope publication over NVLink. */
int lp_ilu0_ranks(lp_ilu *const *f, int nranks, const int *ys, double pivot_tol,
                  int64_t *bad_row, void *stream);
int lp_ilu0_rank(lp_ilu *f, int nranks, const int *ys, int rank, double *const *peer_lu,
                 int *const *peer_flags, double pivot_tol, int64_t *bad_row, void *stream);
/* Multi-GPU set-up of lp_ilu0_rank, per rank: lp_ilu_rank_arrays gives the
 * matrix IPC-exportable factor and flag arrays (before any factorisation) and
 * their 64-byte CUDA IPC handles, which the ranks exchange and map with
 * lp_ipc_open; lp_ilu0_rank_prepare copies M into the factor array and clears
 * the flags; the ranks then synchronise (a barrier: a neighbour stores halo
 * rows and flags into these arrays as soon as it starts) and call lp_ilu0_rank. */
int lp_ilu_rank_arrays(lp_ilu *f, double **lu, int **flags, unsigned char *handle_lu64,
                       unsigned char *handle_flags64);
int lp_ilu0_rank_prepare(lp_ilu *f, int64_t *bad_row, void *stream);

/* forward_sub / backward_sub / precond_apply (sparse.py:199-221). */
int lp_forward_sub(lp_ilu *f, const double *r, double *y, void *stream);
int lp_backward_sub(lp_ilu *f, const double *y, double *z, void *stream);
int lp_precond_apply(lp_ilu *f, const double *r, double *z, void *stream);
/* precond_apply with the PCG scalar rho = r'z (pcg.py:147-151) as a second
 * output: rz points to two device doubles (a double-double pair, hi then lo).
 * The 1-D / 2-D line-wavefront sweeps accumulate r'z inside the backward sweep
 * (a part per x-line, summed in double-double in a fixed order: deterministic);
 * the other sweep kernels follow with a deterministic dot on the same stream. */
int lp_precond_apply_rz(lp_ilu *f, const double *r, double *z, double *rz, void *stream);
/* y = M x with the ORIGINAL matrix (spmv, sparse.py:97-113). */
int lp_spmv(lp_ilu *m, const double *x, double *y, void *stream);
int lp_ilu_destroy(lp_ilu *m);

/* ------------------------------------------------------------------ PCG --
 * pcg_solve loop (pcg.py:111-179): x (device, n) holds x0 on entry when
 * has_x0 != 0 and the solution on exit.  precond may be NULL (plain CG).
 * history (host, k_max + 1 doubles, may be NULL) receives ||r_k||_2.
 * Dots are deterministic double-double reductions (the reference accumulates
 * in 80-bit long double, pcg.py:77-79). */
typedef struct lp_report {
    int64_t iterations;
    int32_t converged;
    int32_t pad_;
    double final_relative_residual;
    double loop_seconds;
    double indefinite_value;   /* p'Ap at the failing iteration */
    int64_t kernel_launches;   /* this library's kernels launched by the loop */
} lp_report;

int lp_pcg_solve(lp_operator *op, lp_ilu *precond, const double *F, double *x,
                 int has_x0, double epsilon, int64_t k_max, double *history,
                 lp_report *report, void *stream);

/* --------------------------------------------------------- vector ops --
 * Building blocks exposed for tests and for host-driven loops. */
/* _dot (pcg.py:77-79): out2[0..1] (device) = double-double sum_i a_i b_i in a
 * fixed order (bitwise reproducible for a given n). */
int lp_dot(int64_t n, const double *a, const double *b, double *out2, void *stream);
/* PCG vector updates (pcg.py:150-155,161-162) with host scalars (sharded driver,
 * sharded.py): p = z (first != 0) or z + beta p;  x += alpha p, r -= alpha w
 * with the double-double r'r of the slab in out2[0..1] (device). */
int lp_update_p(int64_t n, const double *z, double *p, double beta, int first, void *stream);
int lp_update_xr(int64_t n, double *x, double *r, const double *p, const double *w, double alpha,
                 double *out2, void *stream);

/* ------------------------------------------------------------ multi-GPU --
 * Collectives of the distributed solve on the caller's NCCL communicator
 * (one process per GPU).  nccl_comm is an ncclComm_t; NCCL is
 * resolved at run time from the libnccl.so.2 the process already uses, the
 * library does not link it.  slab_axis: the axis the vectors are split along
 * (2 = z-slabs, the layout of the sharded matvec).  The communicator stays
 * the caller's.
 *   lp_comm_allreduce_dd: the PCG scalars r'z, p'w, r'r (pcg.py:150-159) --
 *     dd_inout (device, a double-double pair) is all-gathered and summed in
 *     rank order, so every rank holds the same bits.
 *   lp_comm_dot: this rank's deterministic double-double dot (lp_dot) followed
 *     by lp_comm_allreduce_dd.
 *   lp_comm_alltoall: the transposes of the slab-sharded apply_system
 *     (operator.py:204-210 across ranks): chunk v of `send` (send_counts[v]
 *     doubles, chunks in rank order) goes to rank v, chunk v of `recv` comes
 *     from rank v; counts are host arrays of `size` entries. */
typedef struct lp_comm lp_comm;
int lp_comm_init(void *nccl_comm, int rank, int size, int slab_axis, lp_comm **out);
int lp_comm_destroy(lp_comm *comm);
int lp_comm_allreduce_dd(lp_comm *comm, double *dd_inout, void *stream);
int lp_comm_dot(lp_comm *comm, int64_t n, const double *a, const double *b, double *out2,
                void *stream);
int lp_comm_alltoall(lp_comm *comm, const double *send, const int64_t *send_counts, double *recv,
                     const int64_t *recv_counts, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LEGPCG_B200_H */
