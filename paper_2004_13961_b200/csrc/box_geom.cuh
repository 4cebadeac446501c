// Geometry helpers of the implicit-offset ("box") matrix layout (see ilu_box.cu).
#pragma once

#include "ilu.cuh"

namespace lp {

struct Geom {
    int d, K, r, W, S, c, mw;   // mw = mask words per row
    int64_t n;
    int nlines;
};

inline Geom geom_of(const BoxLayout &b) {
    Geom g;
    g.d = b.d;
    g.K = b.K;
    g.r = b.r;
    g.W = b.W;
    g.S = b.S;
    g.c = (b.S - 1) / 2;
    g.mw = b.mask_words;
    g.n = b.n;
    g.nlines = (int)(b.n / b.K);
    return g;
}

__device__ __forceinline__ void slot_axes(const Geom &g, int s, int &sx, int &sy, int &sz) {
    sx = s % g.W;
    const int q = s / g.W;
    sy = g.d > 1 ? q % g.W : g.r;
    sz = g.d > 2 ? q / g.W : g.r;
}

__device__ __forceinline__ void row_pos(const Geom &g, int64_t i, int &ix, int &iy, int &iz) {
    ix = (int)(i % g.K);
    const int64_t q = i / g.K;
    iy = g.d > 1 ? (int)(q % g.K) : 0;
    iz = g.d > 2 ? (int)(q / g.K) : 0;
}

// Column of slot s for row i, or -1 if it leaves the grid.
__device__ __forceinline__ int64_t slot_col(const Geom &g, int64_t i, int ix, int iy, int iz,
                                            int s) {
    int sx, sy, sz;
    slot_axes(g, s, sx, sy, sz);
    const int ox = sx - g.r, oy = sy - g.r, oz = sz - g.r;
    if (ix + ox < 0 || ix + ox >= g.K) return -1;
    if (g.d > 1 && (iy + oy < 0 || iy + oy >= g.K)) return -1;
    if (g.d > 2 && (iz + oz < 0 || iz + oz >= g.K)) return -1;
    return i + ox + (int64_t)g.K * (oy + (int64_t)g.K * oz);
}

}  // namespace lp
