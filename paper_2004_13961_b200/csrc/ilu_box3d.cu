// ILU(0) of a 3-D box matrix: one CTA per row, the row resident in registers.
//
// IKJ elimination (sparse.py:116-139) of row i = (x, y, z) visits its lower
// slots in column order: pivot planes pz = -r..0, pivot lines py, x fastest,
// the in-line pivots x-r..x-1 last.  The targets of pivot p = (px, py, pz) are
// the offsets t > p of the box with t - p in the box:
//
//     tz in [pz, pz + r],  |tx - px| <= r,  |ty - py| <= r,
//
// and the pivot-row entry of target t is slot t - s_p + c (offsets subtract
// slot-linearly).  A 3-D row has (2r+1)^3 slots (9,261 at r = 10), so one row
// is one CTA's working set: thread q = (ty, tx) owns the column of 2r+1
// entries (all tz) in registers; a pivot step is
//
//   owner of slot p:  l = v[pz] / u_kk, v[pz] = l, broadcast l (shared, 1 barrier)
//   every thread:     v[pz + j] -= l * u_k[t - s_p + c],  j = 0..r (its active planes)
//
// with pz a compile-time constant inside the unrolled plane loop, so the
// register file is indexed statically.  The pivot-row entries of the next D
// pivots are staged by per-thread cp.async copies into a shared ring (each
// thread reads only what it copied itself, so the ring needs no barrier).
// Every entry receives its updates in the reference's k order, each a
// separately rounded multiply and subtract: the factors are the reference's
// bit for bit.
//
// Rows are taken in natural order by an atomic ticket; a row only waits on
// smaller rows, which are resident or done, so the grid cannot deadlock.
// Completion is published per x-line as a contiguous row prefix
// (flags[line] = rows done): one acquire poll per pivot line (per pivot for the
// in-line ones); rows of a line finish in order because row x eliminates x - 1 last.
#include <math.h>

#include <algorithm>
#include <vector>

#include "box_geom.cuh"
#include "ilu.cuh"

#ifndef LP_ILU3_LEVEL_MAX_R
#define LP_ILU3_LEVEL_MAX_R 8   // level order for reach <= this; natural order above (measured, barrier-free kernel: r=2 11x faster, r=4 1.3x, r=7 1.24x, r=10 1.19x slower)
#endif

#ifndef LP_ILU3_BLK_MIN_R
#define LP_ILU3_BLK_MIN_R 9     // row-block kernel from this reach on
#endif

namespace lp {


namespace {

template <int R>
struct Cfg {
    static constexpr int W = 2 * R + 1;
    static constexpr int W2 = W * W;
    static constexpr int S = W2 * W;
    static constexpr int C = (S - 1) / 2;
    static constexpr int TPB = (W2 + 31) / 32 * 32;     // one thread per (tx, ty) column
    static constexpr int STAGE = (R + 1) * TPB;         // doubles per staged pivot
    static constexpr int D = STAGE * 8 * 5 <= 200 * 1024 ? 5 : 4;   // pivots in flight (r <= 10: 5)
};

__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void cp_async8(unsigned dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct Ilu3Args {
    Geom g;
    double *lu;
    const uint32_t *mask;
    int *lineflags;   // [nlines] rows of the line that are final
    int *ticket;
    double tol;
    unsigned long long *bad;
    // level order (null: natural order): ticket t -> level l with
    // lvl_start[l] <= t < lvl_start[l+1]; its o-th row lies on x-line
    // line_order[lvl_first[l] + o] at x = l - (r+1) key(line)
    const int *line_order;
    const int *lvl_first;
    const long long *lvl_start;
    // y-slab ranks (multi-GPU factorisation): rank v owns the x-lines
    // with y in [ys[v], ys[v+1]) and factors them in ITS factor array lu_r[v]
    // (global row indexing; only its own rows and the halo lines
    // [ys[v] - r, ys[v+1] + r) are ever valid there).  A finished row is stored
    // to its owner and -- its diagonal/upper planes, the part pivots read -- to
    // every rank whose halo contains its line, followed by that replica's
    // line flag.  nranks = 1: lu_r[0] = lu, flags_r[0] = lineflags.
    // own = -1: every rank in this launch (one-device emulation); own >= 0: this
    // launch factors rank `own` only, the other entries are its neighbours'
    // arrays mapped over CUDA IPC (system-scope publication).
    int nranks, own;
    int ys[9];
    double *lu_r[8];
    int *flags_r[8];
};

__device__ __forceinline__ void st_release_sys(int *p, int v) {
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int *p) {
    int v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ bool bit_of(const uint32_t *bits, int t) {
    return (bits[t >> 5] >> (t & 31)) & 1u;
}

// First in-pattern slot in [from, end).
__device__ __forceinline__ int next_slot(const uint32_t *bits, int from, int end) {
    if (from >= end) return end;
    int w = from >> 5;
    uint32_t m = bits[w] & (0xFFFFFFFFu << (from & 31));
    const int wlast = (end - 1) >> 5;
    while (!m) {
        if (++w > wlast) return end;
        m = bits[w];
    }
    const int s = (w << 5) + __ffs(m) - 1;
    return s < end ? s : end;
}

// IEEE quotient a / b from y = RN(1 / b) (Markstein: q0 = RN(a y) is within one
// ulp, r = a - b q0 is exact, RN(q0 + r y) = RN(a / b)); with y computed ahead,
// only three dependent operations remain on a pivot step's critical path.
__device__ __forceinline__ double div_by_recip(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-b, q0, a);
    return __fma_rn(r, y, q0);
}

#define LSTORE(idx, val)                                                                   \
    do {                                                                                   \
        const double _v = (val);                                                           \
        *(volatile double *)(sh_l + ((idx) & 63)) = isnan(_v) ? __longlong_as_double(0x7FF8000000000000ll) : _v; \
    } while (0)

template <int R>
__global__ void __launch_bounds__(Cfg<R>::TPB, 1) box_ilu0_3d_kernel(const __grid_constant__ Ilu3Args a) {
    using G = Cfg<R>;
    constexpr int W = G::W, W2 = G::W2, S = G::S, C = G::C, TPB = G::TPB, D = G::D;
    static_assert(D >= 3, "the next pivot's data must land one step early");
    extern __shared__ __align__(16) double sm[];
    double *stage = sm;                                                 // [D][R+1][TPB]
    double *spiv = stage + (size_t)D * G::STAGE;                        // [D]
    uint32_t *bits = reinterpret_cast<uint32_t *>(spiv + D);            // [mw]
    int *plist = reinterpret_cast<int *>(bits + a.g.mw);                // [C] packed pivots
    __shared__ double sh_l[64];   // l of pivot en at en % 64; sentinel = not yet published
    __shared__ long long sh_i;
    __shared__ int sh_wcount[(C + 31) / 32 + 1];
    const int tid = threadIdx.x;
    const bool col = tid < W2;
    const int tx = col ? tid % W - R : 0, ty = col ? tid / W - R : 0;
    const int K = a.g.K;
    const int mw = a.g.mw;
    const int64_t n = a.g.n;
    const unsigned stage_s = (unsigned)__cvta_generic_to_shared(stage);
    const unsigned spiv_s = (unsigned)__cvta_generic_to_shared(spiv);
    constexpr int NWL = (C + 31) / 32;   // mask words of the lower half
    int lvl = 0;   // level of this CTA's last ticket (tickets only grow)
    for (;;) {
        __syncthreads();
        if (tid == 0) {
            const long long t = atomicAdd(a.ticket, 1);
            if (a.line_order == nullptr || t >= n) {
                sh_i = t;
            } else {
                while (__ldg(a.lvl_start + lvl + 1) <= t) ++lvl;
                const int line = __ldg(a.line_order + __ldg(a.lvl_first + lvl) + (int)(t - __ldg(a.lvl_start + lvl)));
                const int key = line % K + (R + 1) * (line / K);
                sh_i = (long long)line * K + (lvl - (R + 1) * key);
            }
        }
        __syncthreads();
        const int64_t i = sh_i;
        if (i >= n) return;
        const int ix = (int)(i % K);
        const int64_t L = i / K;
        // the row's owner among the y-slab ranks, and that rank's arrays
        const int iyr = (int)(L % K);
        int rk = 0;
        while (rk + 1 < a.nranks && iyr >= a.ys[rk + 1]) ++rk;
        if (a.own >= 0 && rk != a.own) continue;   // another rank's row (uniform)
        double *const lu = a.lu_r[rk];
        int *const lineflags = a.flags_r[rk];
        double *gi = lu + (size_t)i * S;
        for (int q = tid; q < mw; q += TPB) bits[q] = a.mask[(size_t)i * mw + q];
        double v[W];
#pragma unroll
        for (int z = 0; z < W; ++z) v[z] = col ? __ldcg(gi + tid + z * W2) : 0.0;
        __syncthreads();
        // pivot list: the in-pattern lower slots in order, packed
        // s | (px + R) << 14 | (py + R) << 19 | (pz + R) << 24
        for (int w = tid; w < NWL; w += TPB) {
            uint32_t m = bits[w];
            if (w == NWL - 1 && (C & 31)) m &= (1u << (C & 31)) - 1u;
            sh_wcount[w] = __popc(m);
        }
        __syncthreads();
        if (tid < 32) {
            int run = 0;
            for (int w0 = 0; w0 < NWL; w0 += 32) {
                const int w = w0 + tid;
                const int cnt = w < NWL ? sh_wcount[w] : 0;
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += t;
                }
                if (w < NWL) sh_wcount[w] = run + incl - cnt;
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (tid == 0) sh_wcount[NWL] = run;
        }
        __syncthreads();
        for (int w = tid; w < NWL; w += TPB) {
            uint32_t m = bits[w];
            if (w == NWL - 1 && (C & 31)) m &= (1u << (C & 31)) - 1u;
            int o = sh_wcount[w];
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int s = w * 32 + b;
                plist[o++] = s | ((s % W) << 14) | (((s / W) % W) << 19) | ((s / W2) << 24);
            }
        }
        unsigned colbits = 0;
        if (col) {
#pragma unroll
            for (int z = 0; z < W; ++z) colbits |= (unsigned)bit_of(bits, tid + z * W2) << z;
        }
        if (tid < 64) sh_l[tid] = __longlong_as_double(0x7FF4000000000ABCll);
        __syncthreads();
        const int npiv = sh_wcount[NWL];

        // ---- prefetch: stages pivot pn into ring slot pn % D
        int pn = 0;
        int ready_line = -1 << 20;
        auto prefetch = [&]() {
            if (pn < npiv) {
                const int e = plist[pn];
                const int ps = e & 0x3FFF;
                const int px = ((e >> 14) & 31) - R, py = ((e >> 19) & 31) - R, pz = (e >> 24) - R;
                const int64_t Lk = L + py + (int64_t)K * pz;
                const int lid = pz * W + py;
                if (lid == 0) {
                    while ((a.own >= 0 ? ld_acquire_sys(lineflags + Lk) : ld_acquire(lineflags + Lk)) < ix + px + 1) {
                    }
                } else if (lid != ready_line) {
                    const int need = min(K, ix + R + 1);
                    while ((a.own >= 0 ? ld_acquire_sys(lineflags + Lk) : ld_acquire(lineflags + Lk)) < need) {
                    }
                    ready_line = lid;
                }
                const double *uk = lu + (size_t)(i + px + (int64_t)K * (py + (int64_t)K * pz)) * S;
                const int slot = pn % D;
                if (tid == (py + R) * W + (px + R)) cp_async8(spiv_s + slot * 8, uk + C);
                if (col && abs(tx - px) <= R && abs(ty - py) <= R) {
                    unsigned m = (colbits >> (pz + R)) & ((1u << (R + 1)) - 1u);
                    if (!(ty > py || (ty == py && tx > px))) m &= ~1u;
                    const double *src = uk + (C - ps) + tid + (pz + R) * W2;
                    const unsigned dst = stage_s + (unsigned)((slot * (R + 1)) * TPB + tid) * 8;
#pragma unroll
                    for (int j = 0; j <= R; ++j)
                        if ((m >> j) & 1u) cp_async8(dst + j * TPB * 8, src + j * W2);
                }
            }
            cp_commit();
            ++pn;
        };
#pragma unroll 1
        for (int q = 0; q < D; ++q) prefetch();

        // ---- pivot steps, plane by plane (pz static inside the unrolled loop).
        // Step en: barrier; every thread applies l_en to its targets; the owner of
        // the next pivot (same plane) then finishes that pivot's l at once, so the
        // critical path of a step is barrier -> one update -> one division.
        int en = 0;
        bool have_l = false;   // l of pivot en already computed and published
#pragma unroll
        for (int pzi = 0; pzi <= R; ++pzi) {
#pragma unroll 1
            while (en < npiv) {
                const int e = plist[en];
                if ((e >> 24) != pzi) break;
                const int px = ((e >> 14) & 31) - R, py = ((e >> 19) & 31) - R;
                const int slot = en % D;
                cp_wait<D - 2>();   // this pivot's and the next pivot's data have landed
                if (!have_l && tid == (py + R) * W + (px + R)) {
                    const double piv = spiv[slot];
                    const double l = __ddiv_rn(v[pzi], piv);
                    v[pzi] = l;
                    LSTORE(en, l);
                    if (fabs(piv) < a.tol) {
                        const int64_t k = i + px + (int64_t)K * (py + (int64_t)K * (pzi - R));
                        atomicMin(a.bad, (unsigned long long)(i * n + k));
                    }
                }
                // next pivot of this plane and its owner
                const int e1 = en + 1 < npiv ? plist[en + 1] : -1;
                const bool next_here = e1 >= 0 && (e1 >> 24) == pzi;
                const int own1 = ((e1 >> 19) & 31) * W + ((e1 >> 14) & 31);
                double y1 = 0.0, piv1 = 0.0;
                if (next_here && tid == own1) {
                    piv1 = spiv[(en + 1) % D];
                    y1 = __drcp_rn(piv1);
                }
                // no barrier per pivot: l is its own flag (sentinel-initialised
                // ring), a barrier every 32 pivots bounds the warps' drift and
                // recycles the half of the ring that every warp has consumed
                if ((en & 31) == 0 && en > 0) {
                    __syncthreads();
                    if (tid < 32) sh_l[((en & 63) ^ 32) + tid] = __longlong_as_double(0x7FF4000000000ABCll);
                    __syncthreads();
                }
                double l;
                {
                    const volatile double *lp = sh_l + (en & 63);
                    do {
                        l = *lp;
                    } while (__double_as_longlong(l) == 0x7FF4000000000ABCll);
                }
                if (col && abs(tx - px) <= R && abs(ty - py) <= R) {
                    unsigned m = (colbits >> pzi) & ((1u << (R + 1)) - 1u);
                    if (!(ty > py || (ty == py && tx > px))) m &= ~1u;
                    const double *src = stage + (size_t)slot * (R + 1) * TPB + tid;
                    // the next pivot's entry (plane pzi, j = 0) first
                    if (m & 1u) v[pzi] = __dsub_rn(v[pzi], __dmul_rn(l, src[0]));
                    if (next_here && tid == own1) {
                        const double l1 = div_by_recip(v[pzi], piv1, y1);
                        v[pzi] = l1;
                        LSTORE(en + 1, l1);
                        if (fabs(piv1) < a.tol) {
                            const int px1 = ((e1 >> 14) & 31) - R, py1 = ((e1 >> 19) & 31) - R;
                            const int64_t k = i + px1 + (int64_t)K * (py1 + (int64_t)K * (pzi - R));
                            atomicMin(a.bad, (unsigned long long)(i * n + k));
                        }
                    }
#pragma unroll
                    for (int j = 1; j <= R; ++j)
                        if (pzi + j < W && ((m >> j) & 1u))
                            v[pzi + j] = __dsub_rn(v[pzi + j], __dmul_rn(l, src[j * TPB]));
                } else if (next_here && tid == own1) {
                    const double l1 = div_by_recip(v[pzi], piv1, y1);
                    v[pzi] = l1;
                    LSTORE(en + 1, l1);
                    if (fabs(piv1) < a.tol) {
                        const int px1 = ((e1 >> 14) & 31) - R, py1 = ((e1 >> 19) & 31) - R;
                        const int64_t k = i + px1 + (int64_t)K * (py1 + (int64_t)K * (pzi - R));
                        atomicMin(a.bad, (unsigned long long)(i * n + k));
                    }
                }
                have_l = next_here;
                ++en;
                prefetch();
            }
        }
        cp_wait<0>();
        if (col) {
#pragma unroll
            for (int z = 0; z < W; ++z) __stcg(gi + tid + z * W2, v[z]);
        }
        // halo: the planes pivots read (diagonal and above) into the neighbours' arrays
        unsigned halo = 0;
        for (int u = 0; u < a.nranks; ++u)
            if (u != rk && iyr >= a.ys[u] - R && iyr < a.ys[u + 1] + R) halo |= 1u << u;
        for (int u = 0; u < a.nranks; ++u)
            if ((halo >> u) & 1u) {
                double *gu = a.lu_r[u] + (size_t)i * S;
                if (col) {
#pragma unroll
                    for (int z = R; z < W; ++z) __stcg(gu + tid + z * W2, v[z]);
                }
            }
        if (halo && a.own >= 0) __threadfence_system();
        else __threadfence();
        __syncthreads();
        if (tid == 0) {
            // publish the line's contiguous prefix (row x - 1 publishes first): the
            // neighbours' replicas before the owner's flag, which is what releases
            // row x + 1 -- so every replica's prefix grows in order too
            while (ld_acquire(lineflags + L) != ix) {
            }
            for (int u = 0; u < a.nranks; ++u)
                if ((halo >> u) & 1u) {
                    if (a.own >= 0) st_release_sys(a.flags_r[u] + L, ix + 1);
                    else st_release(a.flags_r[u] + L, ix + 1);
                }
            st_release(lineflags + L, ix + 1);
        }
    }
}

template <int R>
int launch3(const Ilu3Args &a, cudaStream_t st) {
    using G = Cfg<R>;
    const size_t smem = ((size_t)G::D * G::STAGE + G::D) * sizeof(double) +
                        (size_t)a.g.mw * sizeof(uint32_t) + (size_t)G::C * sizeof(int) + 16;
    LP_CUDA(cudaFuncSetAttribute(box_ilu0_3d_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int dev = 0, nsm = 0, occ = 1;
    LP_CUDA(cudaGetDevice(&dev));
    LP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, box_ilu0_3d_kernel<R>, G::TPB, smem));
    if (occ < 1) return LP_ERR_ARG;
    int64_t blocks = (int64_t)occ * nsm;
    if (blocks > a.g.n) blocks = a.g.n;
    box_ilu0_3d_kernel<R><<<(unsigned)blocks, G::TPB, smem, st>>>(a);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

}  // namespace

// Launches the 3-D row kernel; returns a negative code when it does not apply
// (r outside 1..10), in which case the caller uses the generic kernel.
int box_ilu0_3d_rows(lp_ilu *m, double tol, unsigned long long *key, cudaStream_t st, const IluRanks *ranks) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    if (g.d != 3) return LP_ERR_ARG;
    // large reach: blocks of x-adjacent rows share their pivot rows (ilu_box3d_blk.cu)
    if (!ranks && g.r >= LP_ILU3_BLK_MIN_R && box_ilu0_3d_blocks(m, tol, key, st) == LP_OK) return LP_OK;
    Ilu3Args a;
    a.g = g;
    a.lu = b.lu;
    a.mask = b.mask;
    a.lineflags = m->flags;
    a.ticket = m->ticket;
    a.tol = tol;
    a.bad = key;
    a.line_order = nullptr;
    a.lvl_first = nullptr;
    a.lvl_start = nullptr;
    a.nranks = 1;
    a.own = -1;
    a.ys[0] = 0;
    a.ys[1] = g.K;
    a.lu_r[0] = b.lu;
    a.flags_r[0] = m->flags;
    if (ranks) {
        a.nranks = ranks->nranks;
        a.own = ranks->own;
        for (int v = 0; v <= ranks->nranks; ++v) a.ys[v] = ranks->ys[v];
        for (int v = 0; v < ranks->nranks; ++v) {
            a.lu_r[v] = ranks->lu[v];
            a.flags_r[v] = ranks->flags[v];
        }
    }
    // Level order: row (x, y, z) can run at level x + (r+1)(y + (r+1)z) and every
    // row it depends on has a smaller level, so handing rows out by level is
    // deadlock-free while spreading the rows in flight over many x-lines (natural
    // order holds them to ~(rows in flight)/K lines, whose in-line chains then
    // bound the factorisation when rows are cheap, as at small r).
    int *lvl_first = nullptr;
    long long *lvl_start = nullptr;
    if (LP_ILU3_LEVEL_MAX_R >= g.r) {
        int rc = ensure_line_order(b, st);
        if (rc) return rc;
        const int K = g.K, A = g.r + 1;
        const int mmax = (K - 1) + A * (K - 1);
        std::vector<long long> key_start(mmax + 2, 0);
        for (int z = 0; z < K; ++z)
            for (int y = 0; y < K; ++y) key_start[y + A * z + 1] += 1;
        for (int m = 0; m <= mmax; ++m) key_start[m + 1] += key_start[m];
        const int nlev = (K - 1) + A * mmax + 1;
        std::vector<int> first(nlev);
        std::vector<long long> start(nlev + 2);
        start[0] = 0;
        for (int l = 0; l < nlev; ++l) {
            const int mlo = l - (K - 1) > 0 ? (l - (K - 1) + A - 1) / A : 0;
            const int mhi = std::min(mmax, l / A);
            first[l] = (int)key_start[mlo];
            start[l + 1] = start[l] + (mhi >= mlo ? key_start[mhi + 1] - key_start[mlo] : 0);
        }
        start[nlev + 1] = start[nlev] + 1;   // sentinel for the forward scan
        if ((rc = dalloc(&lvl_first, first.size(), "ILU level table")) ||
            (rc = dalloc(&lvl_start, start.size(), "ILU level table")))
            return rc;
        LP_CUDA(cudaMemcpyAsync(lvl_first, first.data(), first.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        LP_CUDA(cudaMemcpyAsync(lvl_start, start.data(), start.size() * sizeof(long long), cudaMemcpyHostToDevice, st));
        a.line_order = b.line_order;
        a.lvl_first = lvl_first;
        a.lvl_start = lvl_start;
    }
    int rc;
    switch (g.r) {
        case 1: rc = launch3<1>(a, st); break;
        case 2: rc = launch3<2>(a, st); break;
        case 3: rc = launch3<3>(a, st); break;
        case 4: rc = launch3<4>(a, st); break;
        case 5: rc = launch3<5>(a, st); break;
        case 6: rc = launch3<6>(a, st); break;
        case 7: rc = launch3<7>(a, st); break;
        case 8: rc = launch3<8>(a, st); break;
        case 9: rc = launch3<9>(a, st); break;
        case 10: rc = launch3<10>(a, st); break;
        default: rc = LP_ERR_ARG;
    }
    if (lvl_first) {
        cudaStreamSynchronize(st);
        dfree(lvl_first);
        dfree(lvl_start);
    }
    return rc;
}

}  // namespace lp
