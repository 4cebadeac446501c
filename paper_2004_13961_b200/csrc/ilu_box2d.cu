// ILU(0) of a 2-D box matrix (sparse.py:116-139) as a key-ordered block
// wavefront with register-resident rows.
//
// IKJ elimination of row i = (x, y) visits its lower slots in column order:
// the rows of lines y-r .. y-1 (x-r .. x+r each), then the in-line rows
// x-r .. x-1.  Every entry receives its updates in that order, each a
// separately rounded multiply and subtract, and every multiplier is the
// correctly rounded quotient, so any schedule that keeps the per-entry k order
// gives the reference's factors bit for bit.
//
// Task = block (y, b): rows x in [14 b, 14 b + 14) of line y, one CTA, 7
// consumer warps with two adjacent rows each plus one loader warp.
//  * A warp keeps its rows A = (x, y), B = (x+1, y) in registers: lane L owns
//    the absolute column x - r + L, and holds that column's 2r+1 entries (all
//    lines) of both rows.  A pivot row's entry at that column is then used by
//    both rows from one shared-memory load, and the targets need no loads or
//    stores at all: per update one DMUL + one DSUB.
//  * E part: the pivots of lines y-r .. y-1 (x0-r .. x0+13+r each) stream
//    through a 16-slot shared-memory ring by TMA bulk copies (the pivot row's
//    diagonal and upper half, plus RN(1/u_kk)), issued by the loader warp; the
//    consumers wait on the slot's mbarrier and report progress so the loader
//    can reuse the slot.
//  * In-line part: rows x-r .. x-1 of the same line, from the previous block
//    (loaded into a line buffer by the loader once that block is published) or
//    from the sibling warps (written to the line buffer as soon as final).
//    Row B applies row A straight from registers (same lane = same column).
//  * Quotients: Markstein's correction q = RN(q0 + RN(a - b q0) y) with
//    y = RN(1/b) and q0 = RN(a y) is the correctly rounded a / b (no overflow
//    or underflow); y is computed once per row by the row's owner and published
//    with it.
//  * Tasks go out by one ticket in key order key = b + 2y.  Block (y, b) needs
//    blocks (y, b-1) (in-line rows) and (y-d, b-1 .. b+1), d = 1..r (pivot
//    rows, r <= 14 = rows per block), all of smaller key: a task only waits on
//    tasks held by resident CTAs, so the grid cannot deadlock, and the
//    resident tasks of one key span many lines.  A block is published (row
//    values stored, fence, release flag) when all its rows are final.
#include <math.h>

#include <vector>

#include "box_geom.cuh"
#include "ilu.cuh"
#include "smem_tma.cuh"

namespace lp {

unsigned long long *g_ilu2d_trace = nullptr;   // LP_ILU2D_TRACE builds
size_t g_ilu2d_trace_n = 0;

namespace {

constexpr int NWC = 7;                 // consumer warps, two rows each (8 warps: 255 registers)
constexpr int RB = 2 * NWC;            // rows per block task
constexpr int NRING = 32;              // pivot-row ring slots
constexpr int NLR = 16;                // line-buffer slots (>= r + 2): row x in slot x mod 16
constexpr int LB = 8;                  // pivots issued per loader batch (one per lane)
constexpr int NTHR = 32 * (NWC + 1);   // + the loader warp
constexpr unsigned FULLM = 0xffffffffu;


struct Args {
    int K, nlines, nb, ntask, epoch, mw;
    int64_t n;
    const double *src;            // M (each row read once by its owner; may equal lu)
    double *lu;                   // factors [n][S]
    double *rd;                   // [n][2]: RN(1/u_ii), 0
    const uint32_t *mask;
    const unsigned char *full;
    const int *tasks;             // [ntask]: y * nb + b in key order
    int *done;                    // [nlines][nb]: block published (== epoch)
    int *ticket;
    double tol;
    unsigned long long *bad;
    unsigned long long *trace;    // LP_ILU2D_TRACE builds: [ntask][8] globaltimer stamps
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#ifdef LP_ILU2D_TRACE
#define TSTAMP(task, slot) atomicMax(a.trace + (size_t)(task) * 8 + (slot), gtime())
#else
#define TSTAMP(task, slot) ((void)0)
#endif

__device__ __forceinline__ int ld_acq_gpu(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_gpu(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acq_cta(const int *p) {
    int v;
    asm volatile("ld.acquire.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_cta(int *p, int v) {
    asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_vol_cta(const int *p) {
    int v;
    asm volatile("ld.volatile.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_vol_cta(int *p, int v) {
    asm volatile("st.volatile.shared::cta.s32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
// line-buffer tag of row x0 + dx (-r <= dx < 14) of a task: unique across the
// slot's reuses (a slot is reused only after every reader of its row is done)
__device__ __forceinline__ int ltag(int task, int dx) { return (task * 32 + dx + 16) & 0x7fffffff; }

__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }

// correctly rounded a / b from y = RN(1/b) (Markstein)
__device__ __forceinline__ double qdiv(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double rr = __fma_rn(-b, q0, a);
    return __fma_rn(rr, y, q0);
}

// bits j (j < W) of the pattern of row i at relative column tx: slot tx + W j
template <int W>
__device__ __forceinline__ unsigned colbits(const uint32_t *mrow, int tx) {
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < W; ++j) {
        const int s = tx + W * j;
        m |= ((__ldg(mrow + (s >> 5)) >> (s & 31)) & 1u) << j;
    }
    return m;
}

// One pivot application to the warp's two rows.  j0 (static): the pivot's
// line relative to the rows (j0 = oy + r); Lk: lane of the pivot's column;
// up[0] = u_kk, up[dx + W dy] = its upper entries; rc = RN(1/u_kk).
// FULL (both rows have every slot in the pattern): the updates run
// unpredicated; entries that must not change are multiplied by a zero
// multiplier or a zero pivot entry (x - 0 = x exactly), so they keep their bits.
template <int R, bool FULL>
__device__ __forceinline__ void apply2(double (&vA)[2 * R + 1], double (&vB)[2 * R + 1],
                                       unsigned cmA, unsigned cmB, bool useA, bool useB, int j0,
                                       int Lk, const double *up, double rc, const double *zeros,
                                       int lane, const Args &a, int64_t iA, int64_t k) {
    constexpr int W = 2 * R + 1;
    const int dx = lane - Lk;
    const bool inp = dx >= -R && dx <= R;
    // lanes outside the pivot's window read a zero block instead (no per-entry selects)
    const double *ub = inp ? up + dx : zeros;
    double u[R + 1];
    u[0] = dx > 0 ? ub[0] : 0.0;
#pragma unroll
    for (int dy = 1; dy <= R; ++dy) u[dy] = ub[W * dy];
    const double upiv = up[0];
    double aA = 0.0, aB = 0.0;
#pragma unroll
    for (int j = 0; j < W; ++j)
        if (j == j0) {
            aA = __shfl_sync(FULLM, vA[j], Lk & 31);
            aB = __shfl_sync(FULLM, vB[j], Lk & 31);
        }
    double lA = qdiv(aA, upiv, rc), lB = qdiv(aB, upiv, rc);
    if (lane == 0 && fabs(upiv) < a.tol) {
        if (useA) atomicMin(a.bad, (unsigned long long)(iA * a.n + k));
        if (useB) atomicMin(a.bad, (unsigned long long)((iA + 1) * a.n + k));
    }
    if (FULL) {
        const double mA = useA ? lA : 0.0, mB = useB ? lB : 0.0;
#pragma unroll
        for (int dy = 0; dy <= R; ++dy) {
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (j == j0 + dy) {
                    vA[j] = __dsub_rn(vA[j], __dmul_rn(mA, u[dy]));
                    vB[j] = __dsub_rn(vB[j], __dmul_rn(mB, u[dy]));
                }
        }
    } else {
#pragma unroll
        for (int dy = 0; dy <= R; ++dy) {
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (j == j0 + dy) {
                    const bool ok = inp && (dy > 0 || dx > 0);
                    if (useA && ok && ((cmA >> j) & 1u)) vA[j] = __dsub_rn(vA[j], __dmul_rn(lA, u[dy]));
                    if (useB && ok && ((cmB >> j) & 1u)) vB[j] = __dsub_rn(vB[j], __dmul_rn(lB, u[dy]));
                }
        }
    }
    if (lane == Lk) {
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (j == j0) {
                if (useA) vA[j] = lA;
                if (useB) vB[j] = lB;
            }
    }
}

struct Consumer {
    int task, y, x0, xlo, xhi, xa, lane, warp;
    bool liveA, liveB;
    int64_t iA;
    unsigned gbase, mbar0;
    const double *ring, *rdr, *lbuf, *rcl, *zeros;
    const int *lready;
    int *prog;
    int nk;
};

// E part (pivot lines y-R .. y-1 from the ring) and in-line part (rows
// xa-R .. xa-1 from the line buffer) of a warp's two rows.
template <int R, bool FULL>
__device__ __forceinline__ void consume(const Args &a, const Consumer &c, double (&vA)[2 * R + 1],
                                        double (&vB)[2 * R + 1], unsigned cmA, unsigned cmB) {
    constexpr int W = 2 * R + 1, S = W * W, C = (S - 1) / 2;
    constexpr int US = ((S - C + 1) + 1) & ~1;
    constexpr int LS = ((S - C + R) + 1) & ~1;
    const int lane = c.lane, xa = c.xa, y = c.y, K = a.K;
#ifdef LP_ILU2D_TRACE
    long long wait_cycles = 0;
#endif
    const int nx = c.xhi - c.xlo + 1;
    const int ylo = y > R ? y - R : 0;
    // Every warp waits on every ring entry in order, used or not: a slot's
    // mbarrier only tells the last two phases apart, so a warp may wait on
    // entry G only once entry G - NRING (same slot) has completed.
#pragma unroll
    for (int j0 = 0; j0 < R; ++j0) {
        const int yk = y - R + j0;
        if (yk < 0) continue;
        const unsigned Gl = c.gbase + (unsigned)((yk - ylo) * nx - c.xlo);
        const int64_t kl = (int64_t)yk * K;
        for (int xk = c.xlo; xk <= c.xhi; ++xk) {
            const unsigned G = Gl + (unsigned)xk, slot = G % NRING;
            const int Lk = xk - xa + R;
            bool useA = c.liveA && Lk >= 0 && Lk <= 2 * R;
            bool useB = c.liveB && Lk >= 1 && Lk <= 2 * R + 1;
            if (!FULL) {
                const unsigned cA = __shfl_sync(FULLM, cmA, Lk & 31);
                const unsigned cB = __shfl_sync(FULLM, cmB, Lk & 31);
                useA = useA && ((cA >> j0) & 1u);
                useB = useB && ((cB >> j0) & 1u);
            }
#ifdef LP_ILU2D_TRACE
            const long long tw = clock64();
            mbar_wait(c.mbar0 + 8 * slot, (G / NRING) & 1u);
            wait_cycles += clock64() - tw;
#else
            mbar_wait(c.mbar0 + 8 * slot, (G / NRING) & 1u);
#endif
            if (useA || useB) {
                const int64_t k = kl + xk;
                apply2<R, FULL>(vA, vB, cmA, cmB, useA, useB, j0, Lk,
                                c.ring + (size_t)slot * US + (int)((k ^ C) & 1), c.rdr[2 * slot],
                                c.zeros, lane, a, c.iA, k);
            }
            if (lane == 0) st_vol_cta(c.prog + c.warp, (int)(G + 1));   // entries <= G done
        }
    }
    if (lane == 0) st_vol_cta(c.prog + c.warp, (int)(c.gbase + c.nk));
    if (lane == 0) TSTAMP(c.task, 3);
#ifdef LP_ILU2D_TRACE
    if (lane == 0) atomicAdd(a.trace + (size_t)c.task * 8 + 6, (unsigned long long)wait_cycles);
#endif
#pragma unroll 1
    for (int m = R; m >= 1; --m) {
        const int xk = xa - m;
        if (xk < 0) continue;
        const int Lk = R - m;
        bool useA = c.liveA, useB = c.liveB && m < R;
        if (!FULL) {
            const unsigned cA = __shfl_sync(FULLM, cmA, Lk);
            const unsigned cB = __shfl_sync(FULLM, cmB, Lk);
            useA = useA && ((cA >> R) & 1u);
            useB = useB && ((cB >> R) & 1u);
        }
        if (!useA && !useB) continue;
        const int ls = xk % NLR;
        while (ld_acq_cta(c.lready + ls) != ltag(c.task, xk - c.x0)) {
        }
        apply2<R, FULL>(vA, vB, cmA, cmB, useA, useB, R, Lk, c.lbuf + (size_t)ls * LS + R, c.rcl[ls],
                        c.zeros, lane, a, c.iA, (int64_t)y * K + xk);
    }
}

template <int R>
__global__ void __launch_bounds__(NTHR, 1) ilu2d_kernel(const __grid_constant__ Args a) {
    constexpr int W = 2 * R + 1, S = W * W, C = (S - 1) / 2;
    constexpr int US = ((S - C + 1) + 1) & ~1;   // ring slot: diag + upper half (+ alignment)
    constexpr int LS = ((S - C + R) + 1) & ~1;   // line-buffer slot: from slot C - R
    constexpr int NL = NLR;                      // line-buffer slots (row x -> x mod NLR)
    extern __shared__ __align__(128) double sm[];
    double *ring = sm;                           // [NRING][US]
    double *rdr = ring + NRING * US;             // [NRING][2]
    double *lbuf = rdr + 2 * NRING;              // [NL][LS]
    double *rcl = lbuf + NL * LS;                // [NL]
    double *zeros = rcl + NL;                    // [W R + 1] zeros
    for (int i = threadIdx.x; i < W * R + 1; i += NTHR) zeros[i] = 0.0;
    __shared__ __align__(8) unsigned long long mbar[NRING];
    __shared__ int s_lready[NL];
    __shared__ int s_prog[NWC];
    __shared__ int s_task;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = a.K;
    const unsigned mbar0 = smem_addr(mbar);
    if (tid == 0) {
        for (int i = 0; i < NRING; ++i) mbar_init(mbar0 + 8 * i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < NL; i += NTHR) s_lready[i] = -1;   // never a tag
    if (tid < NWC) s_prog[tid] = 0;
    unsigned gbase = 0;   // ring sequence number of the task's first pivot
    for (;;) {
        __syncthreads();
        if (tid == 0) s_task = atomicAdd(a.ticket, 1);
        __syncthreads();
        const int task = s_task;
        if (task >= a.ntask) return;
        const int yb = a.tasks[task];
        const int y = yb / a.nb, b = yb - y * a.nb;
        const int x0 = b * RB;
        const int ylo = y > R ? y - R : 0;
        const int xlo = max(0, x0 - R), xhi = min(K - 1, x0 + RB - 1 + R);
        const int nx = xhi - xlo + 1;
        const int nk = (y - ylo) * nx;
        if (tid == 0) TSTAMP(task, 0);

        if (warp == NWC) {
            // ------------------------------------------------------------ loader
            // pivot blocks of lines ylo..y-1 (b-1..b+1): one parallel round of
            // acquire loads first, then lane 0 re-polls only the blocks not yet done
            const int bl = max(0, b - 1), bh = min(a.nb - 1, (xhi) / RB);
            const int nbk = bh - bl + 1;
            const int nchk = (y - ylo) * nbk;   // <= 3 R <= 45
            unsigned long long dmask = 0;
            for (int q0 = 0; q0 < nchk; q0 += 32) {
                const int q = q0 + lane;
                bool ok = false;
                if (q < nchk) ok = ld_acq_gpu(a.done + (ylo + q / nbk) * a.nb + bl + q % nbk) == a.epoch;
                dmask |= (unsigned long long)__ballot_sync(FULLM, ok) << q0;
            }
            // pivots go out in batches of LB, lane j issuing pivot q0 + j
            asm volatile("fence.proxy.async.global;" ::: "memory");
            int minprog = 0;
            for (int q0 = 0; q0 < nk; q0 += LB) {
                const int nq = min(LB, nk - q0);
                const unsigned Glast = gbase + (unsigned)(q0 + nq - 1);
                if (Glast >= NRING && minprog < (int)(Glast - NRING + 1)) {
                    // every consumer is past the pivot that last used the batch's slots
#ifdef LP_ILU2D_TRACE
                    const long long tw = clock64();
#endif
                    for (;;) {
                        int mp = lane < NWC ? ld_vol_cta(s_prog + lane) : 0x7fffffff;
#pragma unroll
                        for (int o = 4; o; o >>= 1) mp = min(mp, __shfl_xor_sync(FULLM, mp, o));
                        minprog = __shfl_sync(FULLM, mp, 0);
                        if (minprog >= (int)(Glast - NRING + 1)) break;
                        __nanosleep(20);
                    }
#ifdef LP_ILU2D_TRACE
                    if (lane == 0) atomicAdd(a.trace + (size_t)task * 8 + 7, (unsigned long long)(clock64() - tw));
#endif
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                const int q = q0 + lane;
                const bool act = lane < nq;
                const int lq = q / nx;
                const int yk = ylo + lq, xk = xlo + q - lq * nx;
                const int bq = lq * nbk + xk / RB - bl;
                bool polled = false;
                if (act && !((dmask >> bq) & 1ull)) {
                    while (ld_acq_gpu(a.done + yk * a.nb + xk / RB) != a.epoch) __nanosleep(64);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    polled = true;
                }
                const unsigned long long pb = polled ? 1ull << bq : 0ull;
                dmask |= (unsigned long long)__reduce_or_sync(FULLM, (unsigned)pb) |
                         ((unsigned long long)__reduce_or_sync(FULLM, (unsigned)(pb >> 32)) << 32);
                if (act) {
                    const unsigned G = gbase + (unsigned)q, slot = G % NRING;
                    const int64_t k = (int64_t)yk * K + xk;
                    const int sh = (int)((k ^ C) & 1);   // parity of k S + C (S odd)
                    const unsigned bytes = (unsigned)(((S - C + sh) + 1) & ~1) * 8u;
                    mbar_expect(mbar0 + 8 * slot, bytes + 16u);
                    bulk_g2s(smem_addr(ring + (size_t)slot * US), a.lu + (k * S + C - sh), bytes, mbar0 + 8 * slot);
                    bulk_g2s(smem_addr(rdr + 2 * slot), a.rd + 2 * k, 16u, mbar0 + 8 * slot);
                }
            }
            if (lane == 0) TSTAMP(task, 1);
            __syncwarp();
            // in-line rows x0-R .. x0-1 of the previous block into the line buffer
            if (x0 > 0) {
                if (lane == 0)
                    while (ld_acq_gpu(a.done + y * a.nb + b - 1) != a.epoch) __nanosleep(64);
                __syncwarp();
                for (int xk = max(0, x0 - R); xk < x0; ++xk) {
                    const int ls = xk % NLR;
                    const int64_t k = (int64_t)y * K + xk;
                    const double *g = a.lu + k * S + (C - R);
                    for (int q = lane; q < S - C + R; q += 32) lbuf[ls * LS + q] = __ldcg(g + q);
                    if (lane == 0) rcl[ls] = __ldcg(a.rd + 2 * k);
                    __syncwarp();
                    if (lane == 0) st_rel_cta(s_lready + ls, ltag(task, xk - x0));
                }
            }
            if (lane == 0) TSTAMP(task, 2);
        } else {
            // --------------------------------------------------------- consumers
            const int xa = x0 + 2 * warp;
            const bool liveA = xa < K, liveB = xa + 1 < K;
            const int64_t iA = (int64_t)y * K + xa;
            const bool colA = lane <= 2 * R, colB = lane >= 1 && lane <= 2 * R + 1;
            double vA[W], vB[W];
            unsigned cmA = 0, cmB = 0;
            {
                const double *pa = a.src + iA * S + lane, *pb = a.src + (iA + 1) * S + (lane - 1);
                const bool la = liveA && colA, lb = liveB && colB;
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    vA[j] = la ? ld_stream(pa + W * j) : 0.0;
                    vB[j] = lb ? ld_stream(pb + W * j) : 0.0;
                }
                if (la) cmA = a.full[iA] ? (1u << W) - 1u : colbits<W>(a.mask + iA * a.mw, lane);
                if (lb) cmB = a.full[iA + 1] ? (1u << W) - 1u : colbits<W>(a.mask + (iA + 1) * a.mw, lane - 1);
            }
            {
                Consumer cs;
                cs.task = task;
                cs.y = y;
                cs.x0 = x0;
                cs.xlo = xlo;
                cs.xhi = xhi;
                cs.xa = xa;
                cs.lane = lane;
                cs.warp = warp;
                cs.liveA = liveA;
                cs.liveB = liveB;
                cs.iA = iA;
                cs.gbase = gbase;
                cs.mbar0 = mbar0;
                cs.ring = ring;
                cs.rdr = rdr;
                cs.lbuf = lbuf;
                cs.rcl = rcl;
                cs.lready = s_lready;
                cs.prog = s_prog;
                cs.zeros = zeros;
                cs.nk = nk;
                const bool wfull = __all_sync(FULLM, (!liveA || a.full[iA]) && (!liveB || a.full[iA + 1]));
                if (wfull) consume<R, true>(a, cs, vA, vB, cmA, cmB);
                else consume<R, false>(a, cs, vA, vB, cmA, cmB);
                if (lane == 0) TSTAMP(task, 4);
            }
            double rcA = 0.0;
            if (liveA) {
                // row A is final: line buffer (for the sibling warps) first
                const int ls = xa % NLR;
                if (colA) {
#pragma unroll
                    for (int dy = 0; dy <= R; ++dy) lbuf[ls * LS + lane + W * dy] = vA[R + dy];
                }
                if (lane == R) {
                    rcA = __drcp_rn(vA[R]);
                    rcl[ls] = rcA;
                }
                __syncwarp();
                if (lane == 0) st_rel_cta(s_lready + ls, ltag(task, xa - x0));
            }
            double rcB = 0.0;
            if (liveB) {
                // row B applies row A from registers (same lane = same column)
                const unsigned cB = __shfl_sync(FULLM, cmB, R);
                if ((cB >> R) & 1u) {
                    const double upiv = __shfl_sync(FULLM, vA[R], R);
                    const double rc = __shfl_sync(FULLM, rcA, R);
                    const double lB = qdiv(__shfl_sync(FULLM, vB[R], R), upiv, rc);
                    if (lane == 0 && fabs(upiv) < a.tol)
                        atomicMin(a.bad, (unsigned long long)((iA + 1) * a.n + iA));
                    const int dx = lane - R;
                    const bool inp = lane <= 2 * R;
#pragma unroll
                    for (int dy = 0; dy <= R; ++dy) {
                        const bool ok = inp && (dy > 0 || dx > 0) && ((cmB >> (R + dy)) & 1u);
                        if (ok) vB[R + dy] = __dsub_rn(vB[R + dy], __dmul_rn(lB, vA[R + dy]));
                    }
                    if (lane == R) vB[R] = lB;
                }
                const int ls = (xa + 1) % NLR;
                if (colB) {
#pragma unroll
                    for (int dy = 0; dy <= R; ++dy) lbuf[ls * LS + (lane - 1) + W * dy] = vB[R + dy];
                }
                if (lane == R + 1) {
                    rcB = __drcp_rn(vB[R]);
                    rcl[ls] = rcB;
                }
                __syncwarp();
                if (lane == 0) st_rel_cta(s_lready + ls, ltag(task, xa + 1 - x0));
            }
            // global rows and reciprocals (published with the block below)
            if (liveA && colA) {
                double *pa = a.lu + iA * S + lane;
#pragma unroll
                for (int j = 0; j < W; ++j) pa[W * j] = vA[j];
                if (lane == R) {
                    a.rd[2 * iA] = rcA;
                    a.rd[2 * iA + 1] = 0.0;
                }
            }
            if (liveB && colB) {
                double *pb = a.lu + (iA + 1) * S + (lane - 1);
#pragma unroll
                for (int j = 0; j < W; ++j) pb[W * j] = vB[j];
                if (lane == R + 1) {
                    a.rd[2 * iA + 2] = rcB;
                    a.rd[2 * iA + 3] = 0.0;
                }
            }
        }
        gbase += (unsigned)nk;
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_rel_gpu(a.done + yb, a.epoch);
            TSTAMP(task, 5);
        }
    }
}

template <int R>
int launch(const Args &a, cudaStream_t st) {
    constexpr int W = 2 * R + 1, S = W * W, C = (S - 1) / 2;
    constexpr int US = ((S - C + 1) + 1) & ~1;
    constexpr int LS = ((S - C + R) + 1) & ~1;
    const size_t smem = ((size_t)NRING * US + 2 * NRING + (size_t)NLR * LS + NLR + W * R + 1) *
                        sizeof(double);
    if (smem > 220 * 1024) {
        set_error("2-D ILU: %zu bytes of shared memory", smem);
        return LP_ERR_ARG;
    }
    LP_CUDA(cudaFuncSetAttribute(ilu2d_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, nsm = 0, occ = 0;
    LP_CUDA(cudaGetDevice(&dev));
    LP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ilu2d_kernel<R>, NTHR, smem));
    if (occ < 1) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, ilu2d_kernel<R>);
        set_error("2-D ILU kernel does not fit an SM (%zu + %zu bytes of shared memory, %d registers, "
                  "%d threads max, %zu local)", smem, fa.sharedSizeBytes, fa.numRegs,
                  fa.maxThreadsPerBlock, fa.localSizeBytes);
        return LP_ERR_ARG;
    }
    int64_t blocks = (int64_t)occ * nsm;
    if (blocks > a.ntask) blocks = a.ntask;
    ilu2d_kernel<R><<<(unsigned)blocks, NTHR, smem, st>>>(a);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

// tasks (y, b) in key order key = b + 2y (ties by y)
int task_list(BoxLayout &b, int nb, cudaStream_t st) {
    const int nlines = (int)(b.n / b.K);
    const int ntask = nlines * nb;
    if (b.ilu_tasks && b.ilu_ntask == ntask && b.ilu_nb == nb) return LP_OK;
    std::vector<int> t;
    t.reserve(ntask);
    const int nkeys = nb + 2 * (nlines - 1);
    for (int key = 0; key < nkeys; ++key)
        for (int y = 0; y < nlines && 2 * y <= key; ++y) {
            const int bb = key - 2 * y;
            if (bb < nb) t.push_back(y * nb + bb);
        }
    if (b.ilu_tasks) dfree(b.ilu_tasks);
    b.ilu_tasks = nullptr;
    int rc;
    if ((rc = dalloc(&b.ilu_tasks, (size_t)ntask, "ILU task list"))) return rc;
    LP_CUDA(cudaMemcpyAsync(b.ilu_tasks, t.data(), (size_t)ntask * sizeof(int), cudaMemcpyHostToDevice, st));
    LP_CUDA(cudaStreamSynchronize(st));
    b.ilu_ntask = ntask;
    b.ilu_nb = nb;
    return LP_OK;
}

}  // namespace

// Launches the factorisation of a 2-D box (src -> b.lu); returns a negative
// code when the kernel does not apply (the caller falls back to the other
// kernels).  `done` holds nlines * ceil(K / 16) ints.
int box_ilu0_2d_tasks(lp_ilu *m, const double *src, double tol, unsigned long long *key, int *done,
                      cudaStream_t st) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    if (g.d != 2 || g.r < 1 || g.r > RB || !b.full) return LP_ERR_ARG;
    const int nb = (int)ceil_div(g.K, RB);
    int rc;
    if ((rc = task_list(b, nb, st))) return rc;
    if (!b.rdiag && (rc = dalloc(&b.rdiag, (size_t)b.n * 2, "ILU reciprocals"))) return rc;
    Args a;
    a.K = g.K;
    a.nlines = g.nlines;
    a.nb = nb;
    a.ntask = b.ilu_ntask;
    a.epoch = 1;
    a.mw = g.mw;
    a.n = g.n;
    a.src = src;
    a.lu = b.lu;
    a.rd = b.rdiag;
    a.mask = b.mask;
    a.full = b.full;
    a.tasks = b.ilu_tasks;
    a.done = done;
    a.ticket = m->ticket;
    a.tol = tol;
    a.bad = key;
    a.trace = nullptr;
#ifdef LP_ILU2D_TRACE
    if (g_ilu2d_trace_n < (size_t)a.ntask * 8) {
        if (g_ilu2d_trace) dfree(g_ilu2d_trace);
        g_ilu2d_trace_n = (size_t)a.ntask * 8;
        if ((rc = dalloc(&g_ilu2d_trace, g_ilu2d_trace_n, "ilu trace"))) return rc;
    }
    LP_CUDA(cudaMemsetAsync(g_ilu2d_trace, 0, g_ilu2d_trace_n * 8, st));
    a.trace = g_ilu2d_trace;
#endif
    switch (g.r) {
        case 1: return launch<1>(a, st);
        case 2: return launch<2>(a, st);
        case 3: return launch<3>(a, st);
        case 4: return launch<4>(a, st);
        case 5: return launch<5>(a, st);
        case 6: return launch<6>(a, st);
        case 7: return launch<7>(a, st);
        case 8: return launch<8>(a, st);
        case 9: return launch<9>(a, st);
        case 10: return launch<10>(a, st);
        case 11: return launch<11>(a, st);
        case 12: return launch<12>(a, st);
        case 13: return launch<13>(a, st);
        default: return launch<14>(a, st);
    }
}

}  // namespace lp

// LP_ILU2D_TRACE builds: per task [start, loader E issued, loader done, last
// warp E done, last warp done, published] (globaltimer ns); returns the count.
extern "C" int lp_debug_ilu2d_trace(unsigned long long *host, int64_t n) {
    if (!lp::g_ilu2d_trace) return -1;
    const size_t m = (size_t)n < lp::g_ilu2d_trace_n ? (size_t)n : lp::g_ilu2d_trace_n;
    cudaDeviceSynchronize();
    cudaMemcpy(host, lp::g_ilu2d_trace, m * 8, cudaMemcpyDeviceToHost);
    return (int)m;
}
