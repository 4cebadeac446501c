// ILU(0) of a 3-D box matrix, large reach: B x-adjacent rows of a line per CTA.
//
// The row-per-CTA kernel (ilu_box3d.cu) streams every pivot row once per
// target row: (r+1)(2r+1)^2 doubles per pivot, 98 MB per row at r = 10 -- it
// runs at the L2/HBM bandwidth (ncu: 127x the factor bytes).  Rows x0..x0+B-1
// of one x-line share their pivot rows: row (x, y, z) eliminates against rows
// (x', y', z') with |x' - x| <= r of the lower lines, so a block of B rows
// needs B + 2r pivot rows per pivot line instead of B (2r + 1).
//
// Threads are the ABSOLUTE columns (X, Y) of the block's union box,
// X in [x0 - r, x0 + B - 1 + r], Y in [y - r, y + r]; thread (X, Y) keeps, for
// each of the B rows, the entries of that column in the r + 1 live planes
// (registers, a sliding window over z: pivot plane pz only touches the target
// planes pz..pz + r, so a plane is stored and the next one loaded when its
// pivot plane is finished; the plane loop is unrolled, the window is indexed
// statically).  In absolute columns an elimination step is a plain axpy,
// row_b -= l_bk row_k: a thread fetches its r + 1 pivot-row entries once
// (per-thread cp.async ring, no barrier) and applies them to all B rows --
// 2 B FP64 operations per staged double instead of 2.
//
// One step = one pivot row k; its multipliers l_bk (one per row b that has k in
// its pattern) are computed by the thread that owns column k, published
// through a sentinel-flagged shared ring (no barrier per step), and the owner
// of the next pivot of the same line updates its own entries first and
// finishes that step's multipliers at once.  Every entry receives its updates
// in the reference's k order (planes, lines, x ascending), each a separately
// rounded multiply and subtract: the factors are the reference's bit for bit
// (sparse.py:116-139).  The last B - 1 pivots of a row are rows of the block
// itself and are applied from registers.
//
// Blocks are taken in natural (line-major) order by an atomic ticket; a block
// waits only on rows with smaller tickets (the lower lines up to x0 + B + r,
// its own line up to x0), so the grid cannot deadlock.  Completion is the
// per-line row prefix of the row kernel.
#include <math.h>
#include <stdio.h>

#include "box_geom.cuh"
#include "ilu.cuh"

#ifndef LP_BLK_B
#define LP_BLK_B 4   // rows per block
#endif

namespace lp {

namespace {

template <int R, int B>
struct BlkCfg {
    static constexpr int W = 2 * R + 1;
    static constexpr int W2 = W * W;
    static constexpr int S = W2 * W;
    static constexpr int C = (S - 1) / 2;
    static constexpr int RP = R + 1;                 // live planes
    static constexpr int NX = B + 2 * R;             // absolute columns along x
    static constexpr int NT = NX * W;                // threads with a column
    static constexpr int TPB = (NT + 31) / 32 * 32;
    static constexpr int STAGE = RP * TPB;           // doubles per staged pivot row
    static constexpr int D = 4;                      // pivot rows in flight
    static constexpr int NLN = R * W + R + 1;        // pivot lines: planes -R..-1 in full, plane 0 up to the own line
};

struct BlkArgs {
    Geom g;
    double *lu;
    const uint32_t *mask;
    const unsigned char *full;
    int *lineflags;   // [nlines] rows of the line that are final
    int *ticket;
    double tol;
    unsigned long long *bad;
};

__device__ __forceinline__ int ld_acquire_i(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_i(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void cpa8(unsigned dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ bool bit_at(const uint32_t *bits, int t) { return (bits[t >> 5] >> (t & 31)) & 1u; }

constexpr long long kSentinel = 0x7FF4000000000ABCll;   // "not yet published"

template <int R, int B>
__global__ void __launch_bounds__(BlkCfg<R, B>::TPB, 1) box_ilu0_3d_blk_kernel(const __grid_constant__ BlkArgs a) {
    using G = BlkCfg<R, B>;
    constexpr int W = G::W, W2 = G::W2, S = G::S, RP = G::RP, NX = G::NX, NT = G::NT, TPB = G::TPB, D = G::D;
    constexpr int NLN = G::NLN, NTAB = NLN * NX;
    constexpr unsigned WIN = (1u << RP) - 1u;          // the live planes of a window
    static_assert((D & (D - 1)) == 0, "ring slots are taken modulo D");
    extern __shared__ __align__(16) double sm[];
    double *stage = sm;                                          // [D][RP][TPB]
    double *sh_l = stage + (size_t)D * G::STAGE;                 // [64][B] multipliers of step e at e % 64
    double *sh_lb = sh_l + 64 * B;                               // [B][B] in-block multipliers
    uint32_t *bits = reinterpret_cast<uint32_t *>(sh_lb + B * B);   // [B][mw]
    unsigned char *tab = reinterpret_cast<unsigned char *>(bits + B * a.g.mw);   // [NLN][NX] rows b with the pivot
    __shared__ long long sh_t;
    const int tid = threadIdx.x;
    const bool act = tid < NT;
    const int cx = act ? tid % NX : -4 * R - 8, cy = act ? tid / NX : -4 * R - 8;
    const int K = a.g.K, mw = a.g.mw;
    const int64_t n = a.g.n;
    const int nblk = (K + B - 1) / B;
    const long long total = (long long)a.g.nlines * nblk;
    const unsigned stage_s = (unsigned)__cvta_generic_to_shared(stage);
    const double sentinel = __longlong_as_double(kSentinel);
    // lanes outside a pivot row's box multiply stale ring entries by a zero
    // multiplier: the ring must never hold a non-finite bit pattern
    for (int q = tid; q < D * G::STAGE; q += TPB) stage[q] = 0.0;

    for (;;) {
        __syncthreads();
        if (tid == 0) sh_t = atomicAdd(a.ticket, 1);
        __syncthreads();
        const long long t = sh_t;
        if (t >= total) return;
        const int64_t L = t / nblk;
        const int x0 = (int)(t - L * nblk) * B;
        const int nb = min(B, K - x0);
        const int iy = (int)(L % K), iz = (int)(L / K);
        const int64_t i0 = L * K + x0;
        for (int q = tid; q < B * mw; q += TPB) {
            const int b = q / mw;
            bits[q] = b < nb ? a.mask[(size_t)(i0 + b) * mw + (q - b * mw)] : 0u;
        }
        for (int q = tid; q < 64 * B; q += TPB) sh_l[q] = sentinel;
        __syncthreads();
        // step table: rows b of the block that have pivot row (cxp, line) in their pattern
        for (int q = tid; q < NTAB; q += TPB) {
            const int ln = q / NX, cxp = q - ln * NX;
            const int pzi = ln / W, pyi = ln - pzi * W;
            const int X1 = x0 - R + cxp, y1 = iy + pyi - R, z1 = iz + pzi - R;
            unsigned bm = 0;
            if (X1 >= 0 && X1 < K && y1 >= 0 && y1 < K && z1 >= 0 && !(ln == NLN - 1 && cxp >= R)) {
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int d = cxp - b;
                    if (b < nb && d >= 0 && d <= 2 * R && bit_at(bits + b * mw, d + W * pyi + W2 * pzi)) bm |= 1u << b;
                }
            }
            tab[q] = (unsigned char)bm;
        }
        // planes of the box inside the grid (uniform)
        unsigned zm = 0;
#pragma unroll
        for (int z = 0; z < W; ++z) zm |= (unsigned)(iz + z - R >= 0 && iz + z - R < K) << z;

        // ---- this thread's column in each row: in-pattern planes, live window
        unsigned tb[B];
        bool gv[B];
        double v[B][RP];
        bool reg_ok = true;
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int d = cx - b;
            gv[b] = b < nb && d >= 0 && d <= 2 * R;
            tb[b] = 0;
            if (gv[b]) {
#pragma unroll 1
                for (int z = 0; z < W; ++z) tb[b] |= (unsigned)bit_at(bits + b * mw, d + W * cy + W2 * z) << z;
            }
            reg_ok = reg_ok && (tb[b] == 0u || tb[b] == zm);
            const double *gi = a.lu + (size_t)(i0 + b) * S + d + W * cy;
#pragma unroll
            for (int z = 0; z < RP; ++z) v[b][z] = gv[b] ? __ldcg(gi + z * W2) : 0.0;
        }
        // regular block: every column of every row is either absent or holds all
        // the planes inside the grid (no pattern holes): a lane's validity is then
        // folded into its multipliers and the arithmetic needs no per-entry tests
        const bool regular = __syncthreads_and(reg_ok) != 0;
        const int cxlo = max(0, R - x0);
        const int cxall = min(NX, K - x0 + R);

        // ---- prefetch iterator: the steps in order, D ahead of the arithmetic
        int pn = 0, q_q = 0, q_ln = -1;
        bool q_uyv = false, q_up = false, q_eq = false;
        const double *q_base = a.lu;
        auto prefetch = [&]() {
            while (q_q < NTAB && tab[q_q] == 0) ++q_q;
            if (q_q < NTAB) {
                const int ln = q_q / NX, cxp = q_q - ln * NX;
                if (ln != q_ln) {
                    const int pzi = ln / W, pyi = ln - pzi * W;
                    const int64_t Lk = L + (pyi - R) + (int64_t)K * (pzi - R);
                    const int need = ln == NLN - 1 ? x0 : min(K, x0 + B + R);
                    while (ld_acquire_i(a.lineflags + Lk) < need) {
                    }
                    const int uy = cy - pyi;
                    q_uyv = abs(uy) <= R;
                    q_up = uy > 0;
                    q_eq = uy == 0;
                    q_base = a.lu + (size_t)(Lk * K + (x0 - R)) * S + (cx + R) + W * (uy + R) + W2 * R;
                    q_ln = ln;
                }
                const int dx = cx - cxp;
                if (q_uyv && abs(dx) <= R) {
                    const double *src = q_base + (int64_t)cxp * (S - 1);
                    const unsigned dst = stage_s + (unsigned)((pn & (D - 1)) * G::STAGE + tid) * 8u;
                    // plane 0 of the pivot row: the diagonal (for the owner) and the strict upper part
                    if (q_up || (q_eq && dx >= 0)) cpa8(dst, src);
#pragma unroll
                    for (int j = 1; j <= R; ++j) cpa8(dst + j * TPB * 8, src + j * W2);
                }
                ++q_q;
            }
            cpa_commit();
            ++pn;
        };
#pragma unroll 1
        for (int q = 0; q < D; ++q) prefetch();

#define LP_LSTORE(step, b_, val)                                                                  \
    do {                                                                                          \
        const double _v = (val);                                                                  \
        *(volatile double *)(sh_l + ((step) & 63) * B + (b_)) =                                   \
            isnan(_v) ? __longlong_as_double(0x7FF8000000000000ll) : _v;                          \
    } while (0)

        // ---- the steps, plane by plane (window slots static inside the unrolled loop)
        int e = 0;
        bool have_l = false;   // the multipliers of step e are already published
#pragma unroll
        for (int pzi = 0; pzi <= R; ++pzi) {
            if (iz + pzi - R >= 0) {
                const int npy = pzi == R ? R + 1 : W;
#pragma unroll 1
                for (int pyi = 0; pyi < npy; ++pyi) {
                    if (iy + pyi - R < 0 || iy + pyi - R >= K) continue;
                    const int uy = cy - pyi;
                    const bool uyv = abs(uy) <= R;
                    const unsigned char *trow = tab + (pzi * W + pyi) * NX;
                    unsigned bmn = trow[cxlo];
#pragma unroll 1
                    for (int cxp = cxlo; cxp < cxall; ++cxp) {
                        const unsigned bm = bmn;
                        bmn = cxp + 1 < cxall ? trow[cxp + 1] : 0u;   // the next pivot of this line
                        if (!bm) continue;
                        const unsigned bm1 = bmn;
                        {
                            cpa_wait<D - 2>();   // this step's and the next step's entries have landed
                        }
                        const double *src = stage + (size_t)(e & (D - 1)) * G::STAGE + tid;
                        const int own = pyi * NX + cxp;
                        if ((e & 31) == 0 && e > 0) {
                            // every thread has consumed the older half of the ring
                            __syncthreads();
                            for (int q = tid; q < 32 * B; q += TPB) sh_l[(((e & 63) ^ 32)) * B + q] = sentinel;
                            __syncthreads();
                        }
                        if (!have_l && tid == own) {
                            const double piv = src[0];
#pragma unroll
                            for (int b = 0; b < B; ++b)
                                if ((bm >> b) & 1u) {
                                    const double l = __ddiv_rn(v[b][pzi % RP], piv);
                                    v[b][pzi % RP] = l;
                                    LP_LSTORE(e, b, l);
                                }
                            if (fabs(piv) < a.tol) {
                                const int64_t k = L * K + (x0 - R + cxp) + (int64_t)K * ((pyi - R) + (int64_t)K * (pzi - R));
                                atomicMin(a.bad, (unsigned long long)((i0 + __ffs(bm) - 1) * n + k));
                            }
                        }
                        double l[B];
                        {
#pragma unroll
                            for (int b = 0; b < B; ++b) {
                                l[b] = 0.0;
                                if ((bm >> b) & 1u) {
                                    const volatile double *lp = sh_l + (e & 63) * B + b;
                                    do {
                                        l[b] = *lp;
                                    } while (__double_as_longlong(l[b]) == kSentinel);
                                }
                            }
                        }
                        const int dx = cx - cxp;
                        const bool vs = uyv && abs(dx) <= R;
                        const bool up0 = uy > 0 || (uy == 0 && dx > 0);
                        if (regular) {
                            // lanes without the column in row b carry a zero multiplier
                            if (vs) {
#pragma unroll
                                for (int b = 0; b < B; ++b) l[b] = tb[b] ? l[b] : 0.0;
                                if (up0) {
                                    const double u0 = src[0];
#pragma unroll
                                    for (int b = 0; b < B; ++b)
                                        v[b][pzi % RP] = __dsub_rn(v[b][pzi % RP], __dmul_rn(l[b], u0));
                                }
                            }
                        } else if (vs && up0) {
                            const double u0 = src[0];
#pragma unroll
                            for (int b = 0; b < B; ++b)
                                if (((bm >> b) & 1u) && ((tb[b] >> pzi) & 1u))
                                    v[b][pzi % RP] = __dsub_rn(v[b][pzi % RP], __dmul_rn(l[b], u0));
                        }
                        if (bm1 && tid == own + 1) {
                            // owner of the next pivot: its entries are up to date, finish that step's multipliers
                            const double piv1 = stage[(size_t)((e + 1) & (D - 1)) * G::STAGE + tid];
                            const double y1 = __drcp_rn(piv1);
#pragma unroll
                            for (int b = 0; b < B; ++b)
                                if ((bm1 >> b) & 1u) {
                                    // IEEE quotient from y1 = RN(1 / piv1) (Markstein)
                                    const double q0 = __dmul_rn(v[b][pzi % RP], y1);
                                    const double rr = __fma_rn(-piv1, q0, v[b][pzi % RP]);
                                    const double l1 = __fma_rn(rr, y1, q0);
                                    v[b][pzi % RP] = l1;
                                    LP_LSTORE(e + 1, b, l1);
                                }
                            if (fabs(piv1) < a.tol) {
                                const int64_t k = L * K + (x0 - R + cxp + 1) + (int64_t)K * ((pyi - R) + (int64_t)K * (pzi - R));
                                atomicMin(a.bad, (unsigned long long)((i0 + __ffs(bm1) - 1) * n + k));
                            }
                        }
                        if (regular) {
                            if (vs) {
#pragma unroll
                                for (int j = 1; j <= R; ++j)
                                    if ((zm >> (pzi + j)) & 1u) {   // uniform: the plane is inside the grid
                                        const double u = src[j * TPB];
#pragma unroll
                                        for (int b = 0; b < B; ++b)
                                            v[b][(pzi + j) % RP] = __dsub_rn(v[b][(pzi + j) % RP], __dmul_rn(l[b], u));
                                    }
                            }
                        } else if (vs) {
                            unsigned mb[B];
#pragma unroll
                            for (int b = 0; b < B; ++b) mb[b] = ((bm >> b) & 1u) ? ((tb[b] >> pzi) & WIN) : 0u;
#pragma unroll
                            for (int j = 1; j <= R; ++j) {
                                const double u = src[j * TPB];
#pragma unroll
                                for (int b = 0; b < B; ++b)
                                    if ((mb[b] >> j) & 1u)
                                        v[b][(pzi + j) % RP] = __dsub_rn(v[b][(pzi + j) % RP], __dmul_rn(l[b], u));
                            }
                        }
                        have_l = bm1 != 0u;
                        ++e;
                        {
                            prefetch();
                        }
                    }
                }
            }
            if (pzi < R) {
                // plane pzi is final: store it, load plane pzi + R + 1 into its window slot
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    double *gi = a.lu + (size_t)(i0 + b) * S + (cx - b) + W * cy;
                    if ((tb[b] >> pzi) & 1u) __stcg(gi + pzi * W2, v[b][pzi % RP]);
                    v[b][pzi % RP] = gv[b] ? __ldcg(gi + (pzi + RP) * W2) : 0.0;
                }
            }
        }
        cpa_wait<0>();

        // ---- the pivots inside the block (rows x0..x0+B-2), from registers:
        // window slot of plane R + j is (R + j) % RP
#pragma unroll
        for (int bp = 0; bp + 1 < B; ++bp) {
            if (bp + 1 < nb) {
                const int own = R * NX + R + bp;   // column (x0 + bp, y), plane 0
                if (tid == own) {
                    const double piv = v[bp][R % RP];
                    bool anyb = false;
#pragma unroll
                    for (int b = bp + 1; b < B; ++b) {
                        double l = sentinel;
                        if (b < nb && ((tb[b] >> R) & 1u)) {
                            l = __ddiv_rn(v[b][R % RP], piv);
                            v[b][R % RP] = l;
                            if (isnan(l)) l = __longlong_as_double(0x7FF8000000000000ll);
                            if (!anyb && fabs(piv) < a.tol)
                                atomicMin(a.bad, (unsigned long long)((i0 + b) * n + (i0 + bp)));
                            anyb = true;
                        }
                        sh_lb[bp * B + b] = l;
                    }
                }
                __syncthreads();
                const bool up0 = cy > R || (cy == R && cx > R + bp);
#pragma unroll
                for (int b = bp + 1; b < B; ++b) {
                    const double l = sh_lb[bp * B + b];
                    if (__double_as_longlong(l) != kSentinel && gv[bp]) {
#pragma unroll
                        for (int j = 0; j <= R; ++j)
                            if (((tb[b] >> (R + j)) & 1u) && (j > 0 || up0))
                                v[b][(R + j) % RP] = __dsub_rn(v[b][(R + j) % RP], __dmul_rn(l, v[bp][(R + j) % RP]));
                    }
                }
            }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            double *gi = a.lu + (size_t)(i0 + b) * S + (cx - b) + W * cy;
#pragma unroll
            for (int j = 0; j <= R; ++j)
                if ((tb[b] >> (R + j)) & 1u) __stcg(gi + (R + j) * W2, v[b][(R + j) % RP]);
        }
        __threadfence();
        __syncthreads();
        // the previous block of the line was waited for before the in-line pivots
        if (tid == 0) st_release_i(a.lineflags + L, x0 + nb);
    }
#undef LP_LSTORE
}

template <int R, int B>
int launch_blk(const BlkArgs &a, cudaStream_t st) {
    using G = BlkCfg<R, B>;
    const size_t smem = ((size_t)G::D * G::STAGE + 64 * B + B * B) * sizeof(double) +
                        (size_t)B * a.g.mw * sizeof(uint32_t) + (size_t)G::NLN * G::NX + 16;
    LP_CUDA(cudaFuncSetAttribute(box_ilu0_3d_blk_kernel<R, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int dev = 0, nsm = 0, occ = 1;
    LP_CUDA(cudaGetDevice(&dev));
    LP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, box_ilu0_3d_blk_kernel<R, B>, G::TPB, smem));
    if (occ < 1) return LP_ERR_ARG;
    const int64_t total = (int64_t)a.g.nlines * ((a.g.K + B - 1) / B);
    int64_t blocks = (int64_t)occ * nsm;
    if (blocks > total) blocks = total;
    box_ilu0_3d_blk_kernel<R, B><<<(unsigned)blocks, G::TPB, smem, st>>>(a);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

}  // namespace

// Row-block kernel for the large reaches; LP_ERR_ARG when it does not apply.
int box_ilu0_3d_blocks(lp_ilu *m, double tol, unsigned long long *key, cudaStream_t st) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    if (g.d != 3 || !b.mask || !b.full) return LP_ERR_ARG;
    BlkArgs a;
    a.g = g;
    a.lu = b.lu;
    a.mask = b.mask;
    a.full = b.full;
    a.lineflags = m->flags;
    a.ticket = m->ticket;
    a.tol = tol;
    a.bad = key;
    switch (g.r) {
        case 9: return launch_blk<9, LP_BLK_B>(a, st);
        case 10: return launch_blk<10, LP_BLK_B>(a, st);
        default: return LP_ERR_ARG;
    }
}

}  // namespace lp
