// Internal definitions of the plan and operator handles.
#pragma once

#include "line_transform.cuh"

struct lp_plan {
    int P = 0;
    double *nodes = nullptr, *weights = nullptr;
    double *V = nullptr;            // P x P Vandermonde table (bit-identical to the reference)
    lp::LineTable tV;               // BDLT:  V                 (P x P, unfold)
    lp::LineTable tF;               // FDLT:  V w (2n+1)/2      (P x P, fold)
    lp::LineTable tPhi, tDPhi;      // Shen-basis tables        (P x K)
};

struct lp_operator {
    lp_plan *plan = nullptr;
    int d = 0, P = 0, K = 0;
    int64_t nP = 0;
    int n_beta_grids = 0;
    double *beta_w[3] = {nullptr, nullptr, nullptr};   // beta(x) w^d per diffusion direction
    double *alpha_w = nullptr;                         // alpha(x) w^d or null (B skipped)
    double *wsA = nullptr, *wsB = nullptr;             // 4 and 3 fields of P^d
    // slab-sharded middle stage (slab.cu): the coefficient grids of one y' slab,
    // [4][P][ny][P], extracted on first use
    double *slab_grid = nullptr;
    int slab_y0 = -1, slab_ny = -1;
};

namespace lp {
int operator_apply(lp_operator *op, int which, const double *u, double *out, cudaStream_t st);
}
