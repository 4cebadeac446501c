// ILU(0) of a 2-D box matrix as a task graph on a persistent grid.
//
// IKJ elimination (sparse.py:116-139) of row i = (y, x) visits its lower slots in
// column order: first the rows of lines y-r..y-1, then the in-line rows x-r..x-1.
// Every entry receives its updates in that order, each a separately rounded
// multiply and subtract, so any schedule that keeps the per-entry k order yields
// the reference's factors bit for bit.  The work splits into
//
//  * block tasks E(y, b): rows x in [16b, 16b+16) of line y eliminated against
//    lines y-r..y-1 -- about 95% of the arithmetic, one warp per row.  Most of
//    it uses lines that finished long ago, so these tasks run in parallel on
//    many SMs; the pivot rows' upper parts stream through a shared-memory ring
//    (TMA bulk copies), shared by the 16 rows of the task;
//  * line tasks L(y): one CTA walks line y and finishes every row with its r
//    in-line pivots, the sequential part; rows are taken round-robin by 16 warps
//    and the pivots are read from the sibling warps' shared-memory buffers.
//
// One pivot application ("apply") is a shifted axpy over slot ranges: the
// targets of pivot k = (ox, oy) are the offsets (tx, ty) with ty in
// [oy, oy + r], |tx - ox| <= r, past k itself, and the pivot entry of target t
// is slot t - s + c.  Interior rows have every slot in the pattern and skip the
// mask; out-of-pattern pivot entries are stored zeros.
//
// Tasks are handed out by one ticket in the order L(0), E(1, *), L(1), E(2, *),
// L(2), ...; a task only waits on tasks with smaller tickets, all held by
// resident CTAs, so the grid cannot deadlock.  Completion is published per row
// (values stored and fenced, then a flag) and per block task.
#include <math.h>

#include "box_geom.cuh"
#include "ilu.cuh"
#include "smem_tma.cuh"

namespace lp {

unsigned long long *g_ilu_trace = nullptr;   // LP_ILU_TRACE builds
size_t g_ilu_trace_n = 0;

namespace {

constexpr int NW = 16;   // warps per CTA; early-task rows; line-task rows in flight
constexpr int NR = 8;    // pivot-row ring slots of the early tasks

__device__ __forceinline__ int ld_flag(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long gtime_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Apply pivot row uk (uk[c] = pivot, uk[slot] its upper entries) at offset
// (ox, oy) to the target row buffer `row` (slot s = the pivot's slot in the
// row); returns l = row[s] / pivot (the caller stores it into row[s]).  Lane m
// owns target column tx = max(-r, ox - r) + m and walks the target lines
// oy .. oy + r; colmask[tx + r] has bit ty + r set when slot (tx, ty) is in
// the row's pattern (interior rows: FULL, no mask).  All loads are issued
// before any arithmetic (clamped indices, predicated stores): the warp is
// latency bound, so one shared-memory round trip per pivot instead of 16.
template <bool FULL, int R>
__device__ __forceinline__ double apply_pivot(double *row, const uint32_t *colmask, const double *uk,
                                              int s, int ox, int oy, int r, int W, int S, int c,
                                              int lane) {
    // R = r when specialised (every index below is in range, loads use immediate
    // offsets); R = 0 for the generic path (clamped indices, up to 16 lines)
    constexpr int MJ = R > 0 ? R + 1 : 16;
    const int txlo = max(-r, ox - r), txhi = min(r, ox + r);
    const int tx = txlo + lane;
    const bool act = tx <= txhi;
    const int nty = min(r, oy + r) - oy + 1;   // r + 1: pivots have oy <= 0
    unsigned jm = (nty >= 32 ? ~0u : (1u << nty) - 1u);
    if (tx <= ox) jm &= ~1u;
    if (!act) jm = 0;
    else if (!FULL) jm &= colmask[tx + r] >> (oy + r);
    const int t0 = act ? (tx + r) + W * (oy + r) : r;
    const int d = act ? c - s : 0;
    double u[MJ], v[MJ];
#pragma unroll
    for (int j = 0; j < MJ; ++j) {
        const int t = R > 0 ? t0 + W * j : min(t0 + W * j, S - 1);
        u[j] = uk[R > 0 ? t + d : min(t + d, S - 1)];
        v[j] = row[t];
    }
    const double l = __ddiv_rn(row[s], uk[c]);
#pragma unroll
    for (int j = 0; j < MJ; ++j)
        if ((jm >> j) & 1u) row[t0 + W * j] = __dsub_rn(v[j], __dmul_rn(l, u[j]));
    __syncwarp();
    return l;
}

// colmask[tx] (tx = 0..W-1): bit ty set when slot tx + W ty is in the pattern.
__device__ __forceinline__ void build_colmask(const uint32_t *bits, uint32_t *colmask, int W, int lane) {
    if (lane < W) {
        uint32_t m = 0;
        for (int ty = 0; ty < W; ++ty) {
            const int t = lane + W * ty;
            m |= ((bits[t >> 5] >> (t & 31)) & 1u) << ty;
        }
        colmask[lane] = m;
    }
}

struct TaskArgs {
    Geom g;
    double *lu;
    const uint32_t *mask;
    const unsigned char *full;
    int *rowf;     // [n]: row final (its values stored and fenced)
    int *edone;    // [nlines][nb]: early task finished
    int *ticket;
    double tol;
    unsigned long long *bad;
    int nb;        // early tasks per line
    int rs;        // ring row stride (doubles)
    int ntask;
    unsigned long long *trace;   // LP_ILU_TRACE builds: [task][4] timestamps
};

template <int R>
__global__ void __launch_bounds__(32 * NW, 1) box_ilu0_tasks(const __grid_constant__ TaskArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) unsigned long long s_full[NR];
    __shared__ unsigned s_cons[NR];
    __shared__ int s_rowdone[2 * NW];
    __shared__ int s_task;
    volatile unsigned *v_cons = s_cons;
    volatile int *v_done = s_rowdone;
    const Geom &g = a.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = g.K, r = g.r, W = g.W, S = g.S, c = g.c;
    const int mwS = (g.mw + 1) & ~1;          // mask words, padded to 8 bytes
    const int bufd = S + mwS / 2 + 16;        // doubles per row buffer: values, mask bits, column masks
    if (tid == 0) {
        for (int i = 0; i < NR; ++i) {
            mbar_init(smem_addr(s_full + i), 1);
            s_cons[i] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    unsigned kbase = 0;   // pivot rows this CTA has streamed (ring slot / phase)
    for (;;) {
        __syncthreads();
        if (tid == 0) s_task = atomicAdd(a.ticket, 1);
        for (int q = tid; q < 2 * NW; q += blockDim.x) s_rowdone[q] = -1;
        __syncthreads();
        const int task = s_task;
        if (task >= a.ntask) return;
        int y, b;   // b < 0: line task
        if (task == 0) {
            y = 0;
            b = -1;
        } else {
            const int u = task - 1;
            y = 1 + u / (a.nb + 1);
            b = u % (a.nb + 1);
            if (b == a.nb) b = -1;
        }
        const int64_t row0 = (int64_t)y * K;

        if (b >= 0) {
            // ------------------------------------------------ block task E(y, b)
#ifdef LP_ILU_TRACE
            if (tid == 0 && a.trace) a.trace[(size_t)task * 8] = gtime_ns();
#endif
            const int x0 = NW * b;
            const int x = x0 + warp;
            const bool live = x < K;
            const int64_t i = row0 + x;
            double *row = sm + (size_t)warp * bufd;
            uint32_t *bits = reinterpret_cast<uint32_t *>(row + S);
            bool full_row = false;
            uint32_t *colmask = bits + mwS;
            if (live) {
                for (int q = lane; q < S; q += 32) row[q] = a.lu[(size_t)i * S + q];
                for (int q = lane; q < g.mw; q += 32) bits[q] = a.mask[(size_t)i * g.mw + q];
                full_row = __ldg(a.full + i) != 0;
                __syncwarp();
                build_colmask(bits, colmask, W, lane);
            }
            __syncwarp();
            const unsigned ring0 = smem_addr(sm + (size_t)NW * bufd);
            const unsigned full0 = smem_addr(s_full);
            const int ylo = max(0, y - r), yhi = y - 1;   // pivot lines
            const int xlo = max(0, x0 - r), xhi = min(K - 1, x0 + NW - 1 + r);
            const int nx = xhi - xlo + 1;
            const int nk = (yhi - ylo + 1) * nx;
            const int ncopy = S - c;                     // diag + upper slots of a pivot row
            int qi = 0;                                  // next pivot to stream (warp 0)
            auto issue = [&](int q) {
                const int yk = ylo + q / nx, xk = xlo + q % nx;
                const unsigned G = kbase + (unsigned)q, slot = G % NR;
                if (lane == 0) {
                    while (v_cons[slot] < NW * (G / NR)) __nanosleep(32);
                    while (ld_flag(a.rowf + (int64_t)yk * K + xk) == 0) __nanosleep(64);
#ifdef LP_ILU_TRACE
                    if (a.trace && yk == y - 1 && xk == xlo) a.trace[(size_t)task * 8 + 1] = gtime_ns();
                    if (a.trace && yk == y - 1 && xk == xhi) a.trace[(size_t)task * 8 + 2] = gtime_ns();
#endif
                    const int64_t gi = ((int64_t)yk * K + xk) * S + c;
                    const int sh = (int)(gi & 1);
                    const unsigned bytes = (unsigned)((ncopy + sh + 1) & ~1) * 8;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect(full0 + 8 * slot, bytes);
                    bulk_g2s(ring0 + slot * (unsigned)a.rs * 8, a.lu + (gi - sh), bytes, full0 + 8 * slot);
                }
                __syncwarp();
            };
            for (int q = 0; q < nk; ++q) {
                if (warp == 0)
                    while (qi < nk && qi < q + NR) issue(qi++);
                const int yk = ylo + q / nx, xk = xlo + q % nx;
                const unsigned G = kbase + (unsigned)q, slot = G % NR;
                mbar_wait(full0 + 8 * slot, (G / NR) & 1);
                const int ox = xk - x, oy = yk - y;
                if (live && ox >= -r && ox <= r) {
                    const int s = (ox + r) + W * (oy + r);
                    if (full_row || ((bits[s >> 5] >> (s & 31)) & 1u)) {
                        const int64_t k = (int64_t)yk * K + xk;
                        const int sh = (int)((k * S + c) & 1);
                        const double *uk = sm + (size_t)NW * bufd + (size_t)slot * a.rs + sh - c;   // uk[c] = pivot
                        if (lane == 0 && fabs(uk[c]) < a.tol) atomicMin(a.bad, (unsigned long long)(i * g.n + k));
                        const double l = full_row ? apply_pivot<true, R>(row, colmask, uk, s, ox, oy, r, W, S, c, lane)
                                                  : apply_pivot<false, R>(row, colmask, uk, s, ox, oy, r, W, S, c, lane);
                        if (lane == 0) row[s] = l;
                    }
                }
                __syncwarp();
                if (lane == 0) atomicAdd(&s_cons[slot], 1u);
            }
            kbase += (unsigned)nk;
            if (live)
                for (int q = lane; q < S; q += 32) __stcg(a.lu + (size_t)i * S + q, row[q]);
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                *((volatile int *)(a.edone + (size_t)y * a.nb + b)) = 1;
#ifdef LP_ILU_TRACE
                if (a.trace) a.trace[(size_t)task * 8 + 3] = gtime_ns();
#endif
            }
            continue;
        }

        // -------------------------------------------------------- line task L(y)
        // Rows of the line are taken round-robin by the warps, each row double-
        // buffered in shared memory.  A row arrives from its block task with all
        // earlier lines applied and is finished with its in-line pivots x-r..x-1,
        // read from the sibling warps' buffers.  Requires NW >= r + 1.
#ifdef LP_ILU_TRACE
        if (tid == 0 && a.trace) a.trace[(size_t)task * 8] = gtime_ns();
#endif
        for (int ix = warp; ix < K; ix += NW) {
            const int buf = (ix / NW) & 1;
            double *row = sm + (size_t)(warp * 2 + buf) * bufd;
            uint32_t *bits = reinterpret_cast<uint32_t *>(row + S);
            const int64_t i = row0 + ix;
#ifdef LP_ILU_TRACE
            const bool trow = a.trace && ix == K / 2 && lane == 0;
            if (trow) a.trace[(size_t)task * 8 + 4] = gtime_ns();
#endif
            if (y >= 1 && lane == 0)
                while (ld_flag(a.edone + (size_t)y * a.nb + ix / NW) == 0) __nanosleep(64);
            __syncwarp();
#ifdef LP_ILU_TRACE
            if (trow) a.trace[(size_t)task * 8 + 5] = gtime_ns();
#endif
            uint32_t *colmask = bits + mwS;
            for (int q = lane; q < S; q += 32) row[q] = __ldcg(a.lu + (size_t)i * S + q);
            for (int q = lane; q < g.mw; q += 32) bits[q] = a.mask[(size_t)i * g.mw + q];
            const bool full_row = __ldg(a.full + i) != 0;
            __syncwarp();
            build_colmask(bits, colmask, W, lane);
            __syncwarp();
            for (int m = r; m >= 1; --m) {   // pivots x-m, ascending columns
                const int kix = ix - m;
                if (kix < 0) continue;
                const int s = (r - m) + W * r;
                if (!full_row && !((bits[s >> 5] >> (s & 31)) & 1u)) continue;
                // back off while polling: 15 spinning warps would otherwise flood the
                // shared-memory pipe the working warps need
                while (v_done[kix % (2 * NW)] != kix) __nanosleep(32);
#ifdef LP_ILU_TRACE
                unsigned long long tw0 = 0;
                if (trow && m == 1) tw0 = gtime_ns();
#endif
                const double *uk = sm + (size_t)((kix % NW) * 2 + ((kix / NW) & 1)) * bufd;
                if (lane == 0 && fabs(uk[c]) < a.tol) atomicMin(a.bad, (unsigned long long)(i * g.n + (i - m)));
                const double l = full_row ? apply_pivot<true, R>(row, colmask, uk, s, -m, 0, r, W, S, c, lane)
                                          : apply_pivot<false, R>(row, colmask, uk, s, -m, 0, r, W, S, c, lane);
                if (lane == 0) row[s] = l;
                __syncwarp();
#ifdef LP_ILU_TRACE
                if (trow && m == 1) {
                    a.trace[(size_t)task * 8 + 1] = tw0;               // overwrite row0 slot
                    a.trace[(size_t)task * 8 + 4] = gtime_ns() - tw0;  // last apply duration
                }
#endif
            }
            // siblings may use the row as soon as it is final in shared memory;
            // other CTAs once it is stored and fenced (per-row flag)
#ifdef LP_ILU_TRACE
            if (trow) a.trace[(size_t)task * 8 + 6] = gtime_ns();
#endif
            if (lane == 0) v_done[ix % (2 * NW)] = ix;
            for (int q = lane; q < S; q += 32) __stcg(a.lu + (size_t)i * S + q, row[q]);
            __threadfence();
            __syncwarp();
            if (lane == 0) {
                *((volatile int *)(a.rowf + i)) = 1;
#ifdef LP_ILU_TRACE
                if (trow) a.trace[(size_t)task * 8 + 7] = gtime_ns();
#endif
#ifdef LP_ILU_TRACE
                if (a.trace && (ix == 0 || ix == K / 2 || ix == K - 1))
                    a.trace[(size_t)task * 8 + (ix == 0 ? 1 : (ix == K - 1 ? 3 : 2))] = gtime_ns();
#endif
            }
            __syncwarp();
        }
    }
}

template <int R>
int launch_tasks(const TaskArgs &a, size_t smem, cudaStream_t st) {
    LP_CUDA(cudaFuncSetAttribute(box_ilu0_tasks<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, nsm = 148, occ = 1;
    LP_CUDA(cudaGetDevice(&dev));
    LP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, box_ilu0_tasks<R>, 32 * NW, smem));
    if (occ < 1) return LP_ERR_ARG;
    int64_t blocks = (int64_t)occ * nsm;
    if (blocks > a.ntask) blocks = a.ntask;
    box_ilu0_tasks<R><<<(unsigned)blocks, 32 * NW, smem, st>>>(a);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

}  // namespace

// Returns LP_OK after launching, or a negative code when the task kernel does
// not apply (the caller falls back to the other kernels).
int box_ilu0_2d_tasks(lp_ilu *m, double tol, unsigned long long *key, const unsigned char *full,
                      int *edone, cudaStream_t st) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    if (g.d != 2 || g.r + 1 > NW || g.r > 15) return LP_ERR_ARG;
    const int mwS = (g.mw + 1) & ~1;
    const size_t bufd = (size_t)g.S + mwS / 2 + 16;
    const int rs = (int)round_up(g.S - g.c + 1, 2);
    const size_t smem_l = 2 * NW * bufd * sizeof(double);
    const size_t smem_e = (NW * bufd + (size_t)NR * rs) * sizeof(double);
    const size_t smem = smem_l > smem_e ? smem_l : smem_e;
    if (smem > 220 * 1024) return LP_ERR_ARG;
    TaskArgs a;
    a.g = g;
    a.lu = b.lu;
    a.mask = b.mask;
    a.full = full;
    a.nb = (g.K + NW - 1) / NW;
    a.rowf = m->flags;
    a.edone = edone;
    a.ticket = m->ticket;
    a.tol = tol;
    a.bad = key;
    a.rs = rs;
    a.ntask = 1 + (g.nlines - 1) * (a.nb + 1);
    a.trace = nullptr;
#ifdef LP_ILU_TRACE
    {
        static unsigned long long *tr = nullptr;
        static size_t trn = 0;
        if (trn < (size_t)a.ntask * 8) {
            if (tr) dfree(tr);
            trn = (size_t)a.ntask * 8;
            dalloc(&tr, trn, "ilu trace");
        }
        cudaMemsetAsync(tr, 0, trn * 8, st);
        a.trace = tr;
        g_ilu_trace = tr;
        g_ilu_trace_n = trn;
    }
#endif
    switch (g.r) {
        case 10: return launch_tasks<10>(a, smem, st);
        case 12: return launch_tasks<12>(a, smem, st);
        case 14: return launch_tasks<14>(a, smem, st);
        default: return launch_tasks<0>(a, smem, st);
    }
}

}  // namespace lp

extern "C" int lp_debug_ilu_trace(unsigned long long *host, int64_t n) {
    if (!lp::g_ilu_trace) return -1;
    const size_t m = (size_t)n < lp::g_ilu_trace_n ? (size_t)n : lp::g_ilu_trace_n;
    cudaDeviceSynchronize();
    cudaMemcpy(host, lp::g_ilu_trace, m * 8, cudaMemcpyDeviceToHost);
    return (int)m;
}
