// Parity-split fp64 line transforms on DMMA (mma.sync.m16n8k8.f64).
//
// Every axis pass of the sum-factorised operator and of tensor_bdlt/fdlt is
// one "line transform": with the input viewed as In[b][k] (b = line, k = the
// fastest axis) it computes Out[j][b] = sum_k T[j][k] In[b][k], i.e. the
// transformed axis moves from fastest to slowest ("rotating layout", so after
// d passes the tensor is back in x-fastest order and no explicit transposes
// are ever needed).  The table T is a P x nk Legendre-type table whose
// columns are even or odd functions of the Gauss node, and the nodes are
// exactly antisymmetric (legendre.py:140-141).  The pass therefore splits
// into two half-size GEMMs:
//
//   UNFOLD (modes -> nodes):  E[jh][b] = sum_kk Tsym[jh][kk] In[b][2kk+ps]
//                             O[jh][b] = sum_kk Tanti[jh][kk] In[b][2kk+1-ps]
//                             Out[jh] = E + O,  Out[P-1-jh] = E - O
//   FOLD   (nodes -> modes):  s = In[b][jh] + In[b][P-1-jh], d = In[b][jh] - In[b][P-1-jh]
//                             Out[2kk]   = sum_jh Te[kk][jh] (ps==0 ? s : d)
//                             Out[2kk+1] = sum_jh To[kk][jh] (ps==0 ? d : s)
//
// where ps is the parity of k whose column is an even function.  For odd P
// the middle node x = 0 is a rank-1 correction (its antisymmetric table
// entries are exactly zero).  Up to two (table, input) terms are summed into
// each output and up to four outputs share one launch; the UNFOLD epilogue
// can multiply by a coefficient grid laid out like the output.
#pragma once

#include "lp_common.cuh"

namespace lp {

constexpr int LT_BM = 64;   // CTA tile rows (table side)
constexpr int LT_BN = 64;   // CTA tile columns (lines)
constexpr int LT_BK = 16;   // reduction step

// One Legendre-type table in both parity-split forms (device memory).
struct LineTable {
    int P = 0, nk = 0;      // nodes x modes
    int ps = 0;             // parity of k whose column is an even function of x
    int Hm = 0;             // number of mirror pairs = P / 2
    int KE = 0, KO = 0;     // counts of even / odd k in [0, nk)
    int u_ld = 0, u_rows = 0;   // unfold form: [u_rows][u_ld]
    int f_ld = 0, f_rows = 0;   // fold form:   [f_rows][f_ld]
    double *u_sym = nullptr, *u_anti = nullptr, *u_mid = nullptr;
    double *f_even = nullptr, *f_odd = nullptr, *f_mid_e = nullptr, *f_mid_o = nullptr;
};

struct LtTerm {
    const double *A0, *A1;          // table halves (sym/anti or even/odd)
    const double *mid0, *mid1;      // middle-node row/column (may be null)
    const double *in;
    int ps;
};

struct LtOut {
    LtTerm term[2];
    int nterms;
    double *out;
    const double *grid;             // UNFOLD only: multiply by grid[j*B + b]
};

struct LtArgs {
    int mode;          // 0 = UNFOLD, 1 = FOLD
    int P, nk, B;      // nodes, modes, lines
    int Hm, mid;       // mirror pairs, middle node index or -1
    int lda;           // leading dimension of the table halves
    int Mdim, Kdim;    // GEMM extents (unpadded): UNFOLD Hm x max(KE,KO); FOLD max(KE,KO) x Hm
    int nouts;
    LtOut outs[4];
    // FOLD passes with one output: dotpart[cta] = sum over the CTA's output tile of
    // out * dotv (same indexing as out) -- the p'w of pcg.py:157 inside the last
    // pass of the matvec; one value per CTA in a fixed order.  Null: no dot.
    const double *dotv;
    double *dotpart;
};

int line_table_build(LineTable &t, const double *Tdev, int P, int nk, int ps,
                     cudaStream_t st);
void line_table_free(LineTable &t);

// Launch one pass.  Terms must all share the table shape of `shape`.
int line_transform(const LtArgs &a, cudaStream_t st);
// CTAs of that launch (the length of dotpart)
int64_t line_transform_ctas(const LtArgs &a);

// Helpers to fill LtArgs from tables.
LtArgs lt_unfold(const LineTable &shape, int B);
LtArgs lt_fold(const LineTable &shape, int B);
void lt_add_term(LtArgs &a, int out_idx, const LineTable &t, const double *in);
void lt_set_out(LtArgs &a, int out_idx, double *out, const double *grid = nullptr);

}  // namespace lp
