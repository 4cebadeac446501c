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
    // slab-sharded middle stage (slab.cu): the coefficient grids of y' slabs,
    // [4][P][ny][P] each, extracted on first use and kept (up to MAX_SLABS slabs,
    // so a one-device emulation over several ranks does not re-extract)
    static constexpr int MAX_SLABS = 8;
    struct SlabGrid {
        int y0 = -1, ny = -1;
        double *grid = nullptr;
    } slabs[MAX_SLABS];
    int nslabs = 0;
};

namespace lp {
// Doubles of workspace one apply needs (7 fields of P^d).
int64_t operator_ws_doubles(const lp_operator *op);
// apply_A / apply_B / apply_system.  ws: operator_ws_doubles(op) doubles of
// device workspace, or null to take stream-ordered scratch for this call (the
// handle is never written, so concurrent applies on different streams are safe).
// uw (optional): device double-double pair receiving u' out (the p'w of pcg.py:157),
// accumulated inside the last pass.
int operator_apply(lp_operator *op, int which, const double *u, double *out, cudaStream_t st,
                   double *ws = nullptr, double *uw = nullptr);
}
