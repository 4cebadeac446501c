// ILU(0) forward / backward sweeps of a 3-D box matrix (forward_sub /
// backward_sub, sparse.py:175-216) as a bandwidth-first line wavefront.
//
// In 3-D a row carries (2r+1)^3 / 2 factor entries (4,630 at r = 10, 37 KB), so
// a sweep streams ~67 GB at cfg 4 while its dependency chain is short
// (16,759 levels, 0.6 us per level at the HBM roofline).  The
// kernel is therefore built around the factor stream:
//
//  * a CTA owns one x-line at a time (lines by atomic ticket in sweep order, so
//    it only waits on lines held by running CTAs);
//  * a loader lane streams the line's rows, each row's lower (forward) or
//    diagonal+upper (backward) half one contiguous TMA bulk copy, into a ring
//    of shared-memory row buffers (full / empty mbarriers);
//  * producer thread q owns source line q of the stencil (the r (2r+1) + r
//    off-line slot lines): it keeps the 2r+1 values y(src, x-r..x+r) it needs
//    in a register window that slides by one value per row (loads issued P rows
//    ahead, polled only if they came back as the sentinel), and contributes
//    sum_ox L(x; q, ox) y(src, x+ox); warp sums go to a shared ring;
//  * the serial warp adds the warp sums and runs the in-line recurrence
//    y_x = rhs_x - C_x - sum_d L(x, x-d) y_{x-d}  (backward: z_x = (...)/U_xx)
//    and publishes y_x.
//
// Synchronisation is fence-free as in box_sweep.cu: the output is pre-filled
// with a NaN sentinel and every value is its own flag (aligned 64-bit
// accesses are single-copy atomic; relaxed .gpu loads), computed NaNs are
// canonicalised.  The backward sweep is the mirror image (lines and rows in
// reverse, the upper half of each row, division by the diagonal).
#include <math.h>
#include <string.h>

#include <vector>

#include "box_geom.cuh"
#include "ilu.cuh"
#include "smem_tma.cuh"

namespace lp {

extern unsigned long long *g_trace;   // LP_SWEEP_TRACE builds (box_sweep.cu)
extern size_t g_trace_n;

namespace {

__device__ __forceinline__ unsigned long long gtime_s3() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr unsigned long long SENT3 = 0xFFF4C0FFEE5EED00ull;   // = SWEEP_SENTINEL (box_sweep.cu)
constexpr int RRED = 16;   // rows of warp sums in flight
constexpr int MAX_RANKS = 8;

template <int R>
struct S3 {
    static constexpr int W = 2 * R + 1;
    static constexpr int W2 = W * W;
    static constexpr int S = W2 * W;
    static constexpr int C = (S - 1) / 2;
    static constexpr int NQ = R * W + R;                  // off-line slot lines per side
    static constexpr int NPW = (NQ + 31) / 32;            // producer warps
    static constexpr int NT = 32 * (NPW + 2);             // + serial warp + loader warp
    static constexpr int ROWD = (C + 1 + 1 + 1) / 2 * 2;  // staged doubles per row (+ alignment shift)
#ifdef LP_S3_NR
    static constexpr int NR = LP_S3_NR;
#else
    static constexpr int NR = (190 * 1024) / (ROWD * 8) < 6 ? (190 * 1024) / (ROWD * 8) : 6;
#endif
    // rows of look-ahead of the window loads (P) and of their re-polls (PR); both
    // divide W (static register rotation)
#ifdef LP_S3_P
    static constexpr int P = LP_S3_P;
    static constexpr int PR = LP_S3_PR;
#else
    static constexpr int P = W % 7 == 0 ? 7 : W;
    static constexpr int PR = 1;   // measured (cfg-4 recipe, N=64): 1 row 17.9 ms, 3 rows 22.0 ms per pair
#endif
};

struct Sweep3Args {
    Geom g;
    const double *lu;            // factor rows, a.rows doubles apart
    int64_t rows;                // row stride of lu (S for the box layout)
    const double *rhs;
    double *out;
    int *ticket;
    const int *order;            // ticket -> forward line index (wavefront order)
    const int *gpos;             // small reach: group g = lines order[gpos[g] .. gpos[g+1])
    int ngroups;
    int nrun;                    // entries of `order` to process (plain kernel)
    // y-slab ranks: rank v owns the lines with y in [ys[v], ys[v+1]).
    // Every rank keeps a replica of the vector (rep[v]; rhs in rhsrep[v]); a line
    // is read from and written to its owner's replica and also written to every
    // rank whose stencil halo [ys[u] - r, ys[u+1] + r) contains it.  In the
    // one-launch emulation all replicas are slices of one device buffer and
    // `order` holds every line; in a multi-GPU run each process launches its own
    // lines only (`order` filtered to them) and the neighbours' replicas are
    // peer (CUDA IPC) mappings, written over NVLink with .sys-scope stores and
    // polled with .sys-scope loads (sys != 0).  nranks = 1 is the plain sweep.
    int nranks;
    int ys[MAX_RANKS + 1];
    double *rep[MAX_RANKS];
    const double *rhsrep[MAX_RANKS];
    int sys;
    unsigned long long *trace;   // LP_SWEEP_TRACE: [nlines][8] (ticket time, rows 0 / K/4 / K/2 / K-1 done)
};

__device__ __forceinline__ double ld_rel(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// Weak L2 load for the look-ahead reads: a strong (.relaxed.gpu) load holds
// back the warp's following shared-memory loads until it completes (measured:
// one L2 round trip per row), while a value read too early is only re-polled.
__device__ __forceinline__ double ld_l2(const double *p, unsigned long long pol) {
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// Published values stay in L2 (evict_last) while the factor stream passes
// through it (evict_first): a consumer's poll must not queue behind the
// stream's HBM traffic.
__device__ __forceinline__ void st_keep(double *p, double v, unsigned long long pol) {
    asm volatile("st.relaxed.gpu.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ bool is_sent(double v) {
    return (unsigned long long)__double_as_longlong(v) == SENT3;
}

__device__ __forceinline__ double canon3(double v) {
    return isnan(v) ? __longlong_as_double(0x7FF8000000000000ll) : v;
}

__device__ __forceinline__ double ld_rel_sys(const double *p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// halo copy into a (possibly peer) replica
__device__ __forceinline__ void st_halo(double *p, double v, bool sys, unsigned long long pol) {
    if (sys) asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ double wait_value(const double *p, double v, bool sys = false) {
    while (is_sent(v)) v = sys ? ld_rel_sys(p) : ld_rel(p);
    return v;
}

template <bool FWD, int R>
__global__ void __launch_bounds__(S3<R>::NT, 1) box_sweep3d_kernel(const __grid_constant__ Sweep3Args a) {
    using G = S3<R>;
    constexpr int W = G::W, S = G::S, C = G::C, NQ = G::NQ, NPW = G::NPW, ROWD = G::ROWD, NR = G::NR;
    constexpr int P3 = G::P, PR3 = G::PR;
    extern __shared__ __align__(16) double ring[];                         // [NR][ROWD], rhs [K]
    __shared__ __align__(8) unsigned long long mbar[NR];                    // full[NR]
    __shared__ double red[RRED][NPW];
    __shared__ int sh_line;
    __shared__ int rowready[NR];   // row (CTA step) whose TMA copy has landed in the slot
    __shared__ int slotdone[NR];   // consumers done with the slot, cumulative
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = a.g.K;
    const int nlines = a.g.nlines;
    const unsigned ring_s = smem_addr(ring);
    double *rhs_s = ring + NR * ROWD;
    const unsigned full_s = smem_addr(mbar);
    if (tid == 0) {
        for (int q = 0; q < NR; ++q) mbar_init(full_s + q * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int q = tid; q < NR; q += blockDim.x) {
        rowready[q] = -1;
        slotdone[q] = 0;
    }
    for (int q = tid; q < RRED * NPW; q += blockDim.x)
        (&red[0][0])[q] = __longlong_as_double((long long)SENT3);
    __syncthreads();
    const unsigned red_s = smem_addr(&red[0][0]);
    // Consumers never touch an mbarrier: an mbarrier wait or arrive in a warp
    // with outstanding global loads waits for those loads (measured: one L2
    // round trip per row).  A watcher lane turns each TMA completion into a
    // shared flag, and consumers count themselves off a slot with a shared atomic.
    auto wait_row = [&](int slot, long long gs) {
        const unsigned fa = smem_addr(&rowready[slot]);
        int f;
        do {
            asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(f) : "r"(fa) : "memory");
        } while (f != (int)gs);
    };

    // region of a row staged per step: forward slots [0, C), backward [C, S)
    constexpr int base = FWD ? 0 : C;
    constexpr int len = FWD ? C : C + 1;
    long long gstep = 0;   // rows processed by this CTA (mbarrier phases run across lines)
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    for (;;) {
        if (tid == 64) sh_line = atomicAdd(a.ticket, 1);
        __syncthreads();
        const int t = sh_line;
        __syncthreads();
        if (t >= a.nrun) return;
        const int L = FWD ? a.order[t] : nlines - 1 - a.order[t];
        const int ly = L % K, lz = L / K;
        const int64_t row0 = (int64_t)L * K;
        int owner = 0;
        while (owner + 1 < a.nranks && ly >= a.ys[owner + 1]) ++owner;
        double *const out = a.rep[owner];    // this line's replica
        const double *const rhs = a.rhsrep[owner];
#ifdef LP_SWEEP_TRACE
        if (tid == 0) a.trace[(size_t)t * 8] = gtime_s3();
#endif

        if (warp == 0) {
            // ---------------- loader lane
            if (lane == 0) {
                for (int u = 0; u < K; ++u) {
                    const long long gs = gstep + u;
                    const int slot = (int)(gs % NR);
                    if (gs >= NR) {
                        // all NPW + 1 consumers of the slot's previous row are done
                        const int need = (int)(gs / NR) * (NPW + 1);
                        const unsigned ca = smem_addr(&slotdone[slot]);
                        int f;
                        for (;;) {
                            asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(f) : "r"(ca) : "memory");
                            if (f >= need) break;
                            __nanosleep(32);
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
                    const int x = FWD ? u : K - 1 - u;
                    const int64_t e0 = (row0 + x) * S + base;
                    const int64_t ea = e0 & ~(int64_t)1;
                    const unsigned bytes = (unsigned)(((e0 - ea) + len + 1) / 2 * 2) * 8;
                    mbar_expect(full_s + slot * 8, bytes);
                    bulk_g2s_hint(ring_s + (unsigned)slot * ROWD * 8, a.lu + ea, bytes, full_s + slot * 8, pol_stream);
                }
            }
            else if (lane == 1) {
                // watcher: turns each row's TMA completion into a shared flag, so the
                // producer warps (which hold outstanding global loads) never execute
                // an mbarrier wait
                for (int u = 0; u < K; ++u) {
                    const long long gs = gstep + u;
                    const int slot = (int)(gs % NR);
                    mbar_wait(full_s + slot * 8, (unsigned)((gs / NR) & 1));
                    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(smem_addr(&rowready[slot])), "r"((int)gs) : "memory");
                }
            }
        } else if (warp == 1) {
            // ---------------- serial warp: in-line recurrence (lane 0)
            // the line's right-hand side, one coalesced pass into shared memory
            for (int x = lane; x < K; x += 32) rhs_s[x] = __ldcg(rhs + row0 + x);
            __syncwarp();
            if (lane == 0) {
                double h[R];   // h[d-1] = output of the row d steps back in processing order
#pragma unroll
                for (int d = 0; d < R; ++d) h[d] = 0.0;
                for (int u = 0; u < K; ++u) {
                    const long long gs = gstep + u;
                    const int slot = (int)(gs % NR);
                    const int x = FWD ? u : K - 1 - u;
                    const int64_t i = row0 + x;
                    const double rhs = rhs_s[x];
                    wait_row(slot, gs);
                    const int sh = (int)(((i * S + base) & 1));
                    const unsigned rowa = ring_s + (unsigned)(slot * ROWD + sh) * 8;
                    // in-line coefficients: forward L(x, x-d) at slot C-d; backward U(x, x+d) at C+d
                    double acc = rhs;
#pragma unroll
                    for (int d = R; d >= 2; --d) {
                        const bool ok = FWD ? x - d >= 0 : x + d < K;
                        const double cf = lds(rowa + (unsigned)(FWD ? C - d : d) * 8);
                        if (ok) acc = __fma_rn(-cf, h[d - 1], acc);
                    }
                    const double c1 = lds(rowa + (unsigned)(FWD ? C - 1 : 1) * 8);
                    const double diag = FWD ? 1.0 : lds(rowa);
                    atomicAdd(&slotdone[slot], 1);
                    // warp sums of the producers
                    const int rr = (int)(gs % RRED);
                    double csum = 0.0;
#pragma unroll
                    for (int w = NPW - 1; w >= 0; --w) {
                        const unsigned ra = red_s + (unsigned)(rr * NPW + w) * 8;
                        double v = lds_v(ra);
                        while (is_sent(v)) v = lds_v(ra);
                        sts_v(ra, __longlong_as_double((long long)SENT3));
                        csum += v;
                    }
                    acc -= csum;
                    if (FWD ? x >= 1 : x + 1 < K) acc = __fma_rn(-c1, h[0], acc);
                    const double y = canon3(FWD ? acc : __ddiv_rn(acc, diag));
                    st_keep(out + i, y, pol_keep);
#ifdef LP_SWEEP_TRACE
                    if (u == 0 || u == K / 4 || u == K / 2 || u == K - 1)
                        a.trace[(size_t)t * 8 + 1 + (u == 0 ? 0 : u == K / 4 ? 1 : u == K / 2 ? 2 : 3)] = gtime_s3();
#endif
                    for (int v = 0; v < a.nranks; ++v)   // halo copies (multi-rank only)
                        if (v != owner && ly >= a.ys[v] - R && ly < a.ys[v + 1] + R)
                            st_halo(a.rep[v] + i, y, a.sys != 0, pol_keep);
#pragma unroll
                    for (int d = R - 1; d >= 1; --d) h[d] = h[d - 1];
                    h[0] = y;
                }
            }
        } else {
            // ---------------- producers: thread q owns off-line slot line q
            const int pw = warp - 2;   // producer warp index
            const int q = tid - 64;
            const int ql = FWD ? q : NQ + 1 + q;           // slot-line index (oy, oz)
            const int oy = ql % W - R, oz = ql / W - R;
            const bool active = q < NQ && ly + oy >= 0 && ly + oy < K && lz + oz >= 0 && lz + oz < K;
            const double *src = out + (active ? (int64_t)(L + oy + (int64_t)K * oz) * K : 0);
            // processing coordinate p' -> x: forward x = p', backward x = K-1-p'
            auto srcp = [&](int pp) { return src + (FWD ? pp : K - 1 - pp); };
            auto fetch = [&](int pp) {
                return (active && pp >= 0 && pp < K) ? ld_l2(srcp(pp), pol_keep) : 0.0;
            };
            double win[W];   // win[(p' mod W)]
            double yq[P3];   // loads issued P3 rows ahead
            double yr[PR3];  // re-polls issued PR3 rows ahead (used when yq came back empty)
#pragma unroll
            for (int j = 0; j < W; ++j) win[j] = 0.0;
            // positions 0 .. R-1 (window of step 0 except its newest value)
#pragma unroll
            for (int pp = 0; pp < R; ++pp) win[pp % W] = fetch(pp);   // all loads in flight first
#pragma unroll
            for (int j = 0; j < P3; ++j) yq[j] = fetch(R + j);
#pragma unroll
            for (int j = 0; j < PR3; ++j) yr[j] = yq[j];
#pragma unroll
            for (int pp = 0; pp < R; ++pp)
                if (active && pp < K) win[pp % W] = wait_value(srcp(pp), win[pp % W], a.sys != 0);
            const int coff = ql * W;   // slot of (ox = -R) in this slot line, relative to `base`
            for (int u0 = 0; u0 < K; u0 += W) {
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const int u = u0 + k;
                    if (u < K) {
                        const long long gs = gstep + u;
                        const int slot = (int)(gs % NR);
                        const int x = FWD ? u : K - 1 - u;
                        const int64_t i = row0 + x;
                        // newest window value p' = u + R (consumed P3 steps after its load)
                        {
                            const int pp = u + R;
                            // A source line just ahead of this one leaves the deep load
                            // empty; the re-poll issued PR3 rows ahead (always, so
                            // nothing waits on the deep load's result to decide) usually
                            // has it, and only if both are empty does the thread spin.
                            double v = yq[k % P3];
                            if (is_sent(v)) v = yr[k % PR3];
                            if (active && pp < K) v = wait_value(srcp(pp), v, a.sys != 0);
                            win[(k + R) % W] = v;
                            yq[k % P3] = fetch(pp + P3);
                            yr[k % PR3] = fetch(pp + PR3);
                        }
                        wait_row(slot, gs);
                        const int sh = (int)(((i * S + base) & 1));
                        const unsigned rowa = ring_s + (unsigned)(slot * ROWD + sh + coff - base) * 8;
                        double s0 = 0.0, s1 = 0.0;
                        if (q < NQ) {
#pragma unroll
                            for (int j = 0; j < W; ++j) {
                                // slot ox = j - R pairs with x + ox, i.e. p' = u + (FWD ? ox : -ox)
                                const int d = FWD ? j - R : R - j;
                                const double lv = lds(rowa + (unsigned)j * 8);
                                if (j & 1) s1 = __fma_rn(lv, win[((k + d) % W + W) % W], s1);
                                else s0 = __fma_rn(lv, win[((k + d) % W + W) % W], s0);
                            }
                        }
                        double s = s0 + s1;
#pragma unroll
                        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                        if (lane == 0) {
                            atomicAdd(&slotdone[slot], 1);
                            sts_v(red_s + (unsigned)((int)(gs % RRED) * NPW + pw) * 8, s);
                        }
                    }
                }
            }
        }
        gstep += K;
        __syncthreads();
    }
}


// ---------------------------------------------------------------- small reach
// For r <= 4 a row is only (2r+1)^3 / 2 entries (62 at r = 2), so one line per CTA
// leaves most lanes idle and the per-row overhead dominates.  This variant takes a
// group of up to LPB lines with the SAME wavefront key (independent of each other)
// and advances them in lockstep: one TMA copy per line per step, producer lane
// (line j, source q) in segments of NQP lanes, serial lane j runs line j.
// ST = 2: the even-offset pattern of T = 0 (all in-pattern offsets even in every
// axis; 27 of the 125 slots at r = 2).  The factors are then compacted to the
// even slots (EvenBox, a reach-1 box of stride 2: 27 values per row) and the
// kernel runs with virtual reach R = 1: slot (a, b, c) is the real offset
// (2a, 2b, 2c), the in-line recurrence steps back 2 rows, and the producers'
// windows hold real x offsets -2R..2R.  Per row the sweeps stream 13 / 14
// values instead of 62 / 63.
template <int R, int ST = 1>
struct S3m {
    static constexpr int W = 2 * R + 1, W2 = W * W, S = W2 * W, C = (S - 1) / 2;
    static constexpr int NQ = R * W + R;
    static constexpr int NQP = NQ <= 16 ? 16 : NQ <= 32 ? 32 : 64;     // lanes per line
    static constexpr int LPB = NQP <= 16 ? 8 : 4;                      // lines per CTA
    static constexpr int NPW = LPB * NQP / 32;
    static constexpr int PPL = NQP > 32 ? NQP / 32 : 1;               // partial sums per line
    static constexpr int NT = 32 * (NPW + 3);   // + loader, serial, watcher warps
    static constexpr int ROWD = (C + 1 + 1 + 1) / 2 * 2;
    static constexpr int NR = 6;
    static constexpr int WR = 2 * R * ST + 1;   // producer window (real x offsets)
    static constexpr int P = WR;                // window look-ahead (divides WR)
    static constexpr int RR = R * ST;           // real reach
};

template <bool FWD, int R, int ST>
__global__ void __launch_bounds__(S3m<R, ST>::NT, 1) box_sweep3d_multi_kernel(const __grid_constant__ Sweep3Args a) {
    using G = S3m<R, ST>;
    constexpr int W = G::W, C = G::C, NQ = G::NQ, NQP = G::NQP, LPB = G::LPB;
    constexpr int NPW = G::NPW, PPL = G::PPL, ROWD = G::ROWD, NR = G::NR, P3 = G::P;
    constexpr int WR = G::WR, RR = G::RR;
    const int64_t S = a.rows;
    extern __shared__ __align__(16) double ring[];          // [NR][LPB][ROWD], then rhs [LPB][K]
    __shared__ __align__(8) unsigned long long mbar[NR];
    __shared__ double red[RRED][LPB][PPL];
    __shared__ int rowready[NR];
    __shared__ int slotdone[NR];
    __shared__ int sh_grp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = a.g.K;
    const int nlines = a.g.nlines;
    const unsigned ring_s = smem_addr(ring);
    double *rhs_s = ring + NR * LPB * ROWD;
    const unsigned full_s = smem_addr(mbar);
    if (tid == 0) {
        for (int q = 0; q < NR; ++q) mbar_init(full_s + q * 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int q = tid; q < NR; q += blockDim.x) {
        rowready[q] = -1;
        slotdone[q] = 0;
    }
    for (int q = tid; q < RRED * LPB * PPL; q += blockDim.x)
        (&red[0][0][0])[q] = __longlong_as_double((long long)SENT3);
    __syncthreads();
    const unsigned red_s = smem_addr(&red[0][0][0]);
    auto wait_row = [&](int slot, long long gs) {
        const unsigned fa = smem_addr(&rowready[slot]);
        int f;
        do {
            asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(f) : "r"(fa) : "memory");
        } while (f != (int)gs);
    };
    constexpr int base = FWD ? 0 : C;
    constexpr int len = FWD ? C : C + 1;
    long long gstep = 0;
    const unsigned long long pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    for (;;) {
        if (tid == 0) sh_grp = atomicAdd(a.ticket, 1);
        __syncthreads();
        const int t = sh_grp;
        __syncthreads();
        if (t >= a.ngroups) return;
        const int gp = a.gpos[t], cnt = a.gpos[t + 1] - gp;
        auto line_of = [&](int j) { return FWD ? a.order[gp + j] : nlines - 1 - a.order[gp + j]; };
        auto owner_of = [&](int ly) {
            int v = 0;
            while (v + 1 < a.nranks && ly >= a.ys[v + 1]) ++v;
            return v;
        };

        if (warp == 0) {
            // ---------------- loader warp: lane j issues line j's copy
            const int64_t lrow0 = lane < cnt ? (int64_t)line_of(lane) * K : 0;
            for (int u = 0; u < K; ++u) {
                const long long gs = gstep + u;
                const int slot = (int)(gs % NR);
                if (gs >= NR) {
                    const int need = (int)(gs / NR) * (NPW + 1);
                    const unsigned ca = smem_addr(&slotdone[slot]);
                    int f;
                    for (;;) {
                        asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(f) : "r"(ca) : "memory");
                        if (f >= need) break;
                        __nanosleep(32);
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                const int x = FWD ? u : K - 1 - u;
                const int64_t e0 = (lrow0 + x) * S + base;
                const int64_t ea = e0 & ~(int64_t)1;
                const unsigned bytes = lane < cnt ? (unsigned)(((e0 - ea) + len + 1) / 2 * 2) * 8 : 0u;
                unsigned total = bytes;
#pragma unroll
                for (int o = 16; o; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
                if (lane == 0) mbar_expect(full_s + slot * 8, total);
                __syncwarp();
                if (lane < cnt)
                    bulk_g2s_hint(ring_s + (unsigned)((slot * LPB + lane) * ROWD) * 8, a.lu + ea, bytes,
                                  full_s + slot * 8, pol_stream);
            }
        } else if (warp == 2) {
            // ---------------- watcher lane
            if (lane == 0) {
                for (int u = 0; u < K; ++u) {
                    const long long gs = gstep + u;
                    const int slot = (int)(gs % NR);
                    mbar_wait(full_s + slot * 8, (unsigned)((gs / NR) & 1));
                    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(smem_addr(&rowready[slot])), "r"((int)gs)
                                 : "memory");
                }
            }
        } else if (warp == 1) {
            // ---------------- serial warp: lane j runs line j
            for (int e = lane; e < cnt * K; e += 32) {
                const int j = e / K, x = e - j * K;
                const int L = line_of(j);
                const double *rh = a.rhsrep[owner_of(L % K)];
                rhs_s[j * K + x] = __ldcg(rh + (int64_t)L * K + x);
            }
            __syncwarp();
            const bool mine = lane < cnt;
            const int L = mine ? line_of(lane) : 0;
            const int ly = L % K;
            const int owner = owner_of(ly);
            double *const out = a.rep[owner];
            const int64_t row0 = (int64_t)L * K;
            double h[RR];   // h[d-1] = output of the row d (real) steps back in processing order
#pragma unroll
            for (int d = 0; d < RR; ++d) h[d] = 0.0;
            for (int u = 0; u < K; ++u) {
                const long long gs = gstep + u;
                const int slot = (int)(gs % NR);
                const int x = FWD ? u : K - 1 - u;
                const int64_t i = row0 + x;
                wait_row(slot, gs);
                double acc = 0.0, c1 = 0.0, diag = 1.0;
                if (mine) {
                    acc = rhs_s[lane * K + x];
                    const int sh = (int)((i * S + base) & 1);
                    const unsigned rowa = ring_s + (unsigned)((slot * LPB + lane) * ROWD + sh) * 8;
#pragma unroll
                    for (int d = R; d >= 2; --d) {   // virtual in-line slot d: real offset ST d
                        const bool ok = FWD ? x - ST * d >= 0 : x + ST * d < K;
                        const double cf = lds(rowa + (unsigned)(FWD ? C - d : d) * 8);
                        if (ok) acc = __fma_rn(-cf, h[ST * d - 1], acc);
                    }
                    c1 = lds(rowa + (unsigned)(FWD ? C - 1 : 1) * 8);
                    if (!FWD) diag = lds(rowa);
                }
                __syncwarp();
                if (lane == 0) atomicAdd(&slotdone[slot], 1);
                if (mine) {
                    const int rr = (int)(gs % RRED);
                    double csum = 0.0;
#pragma unroll
                    for (int w = 0; w < PPL; ++w) {
                        const unsigned ra = red_s + (unsigned)((rr * LPB + lane) * PPL + w) * 8;
                        double v = lds_v(ra);
                        while (is_sent(v)) v = lds_v(ra);
                        sts_v(ra, __longlong_as_double((long long)SENT3));
                        csum += v;
                    }
                    acc -= csum;
                    if (FWD ? x >= ST : x + ST < K) acc = __fma_rn(-c1, h[ST - 1], acc);
                    const double y = canon3(FWD ? acc : __ddiv_rn(acc, diag));
                    st_keep(out + i, y, pol_keep);
                    for (int v = 0; v < a.nranks; ++v)
                        if (v != owner && ly >= a.ys[v] - RR && ly < a.ys[v + 1] + RR)   // real reach
                            st_halo(a.rep[v] + i, y, a.sys != 0, pol_keep);
#pragma unroll
                    for (int d = RR - 1; d >= 1; --d) h[d] = h[d - 1];
                    h[0] = y;
                }
            }
        } else {
            // ---------------- producers: lane (j, q) = source q of line j
            const int p = tid - 96;
            const int j = p / NQP, q = p % NQP;
            const int ql = FWD ? q : NQ + 1 + q;
            const int oy = ST * (ql % W - R), oz = ST * (ql / W - R);   // real line offsets
            const int L = j < cnt ? line_of(j) : 0;
            const int ly = L % K, lz = L / K;
            const bool active = j < cnt && q < NQ && ly + oy >= 0 && ly + oy < K && lz + oz >= 0 && lz + oz < K;
            const double *out = a.rep[owner_of(ly)];
            const double *src = out + (active ? (int64_t)(L + oy + (int64_t)K * oz) * K : 0);
            auto srcp = [&](int pp) { return src + (FWD ? pp : K - 1 - pp); };
            auto fetch = [&](int pp) {
                return (active && pp >= 0 && pp < K) ? ld_l2(srcp(pp), pol_keep) : 0.0;
            };
            double win[WR], yq[P3];   // loads P3 rows ahead; a sentinel is polled again when needed
#pragma unroll
            for (int k = 0; k < WR; ++k) win[k] = 0.0;
#pragma unroll
            for (int pp = 0; pp < RR; ++pp) win[pp % WR] = fetch(pp);
#pragma unroll
            for (int k = 0; k < P3; ++k) yq[k] = fetch(RR + k);
#pragma unroll
            for (int pp = 0; pp < RR; ++pp)
                if (active && pp < K) win[pp % WR] = wait_value(srcp(pp), win[pp % WR], a.sys != 0);
            const int coff = ql * W;
            const int64_t row0 = (int64_t)L * K;
            for (int u0 = 0; u0 < K; u0 += WR) {
#pragma unroll
                for (int k = 0; k < WR; ++k) {
                    const int u = u0 + k;
                    if (u < K) {
                        const long long gs = gstep + u;
                        const int slot = (int)(gs % NR);
                        const int x = FWD ? u : K - 1 - u;
                        const int64_t i = row0 + x;
                        {
                            const int pp = u + RR;
                            double v = yq[k % P3];
                            if (active && pp < K) v = wait_value(srcp(pp), v, a.sys != 0);
                            win[(k + RR) % WR] = v;
                            yq[k % P3] = fetch(pp + P3);
                        }
                        wait_row(slot, gs);
                        double s0 = 0.0, s1 = 0.0;
                        if (active) {
                            const int sh = (int)((i * S + base) & 1);
                            const unsigned rowa = ring_s + (unsigned)((slot * LPB + j) * ROWD + sh + coff - base) * 8;
#pragma unroll
                            for (int jj = 0; jj < W; ++jj) {
                                const int d = ST * (FWD ? jj - R : R - jj);   // real x offset
                                const double lv = lds(rowa + (unsigned)jj * 8);
                                if (jj & 1) s1 = __fma_rn(lv, win[((k + d) % WR + WR) % WR], s1);
                                else s0 = __fma_rn(lv, win[((k + d) % WR + WR) % WR], s0);
                            }
                        }
                        double sum = s0 + s1;
#pragma unroll
                        for (int o = (NQP < 32 ? NQP : 32) / 2; o; o >>= 1)
                            sum += __shfl_xor_sync(0xffffffffu, sum, o);
                        if (lane == 0) atomicAdd(&slotdone[slot], 1);
                        if ((q & 31) == 0 && j < cnt)
                            sts_v(red_s + (unsigned)(((int)(gs % RRED) * LPB + j) * PPL + (q >> 5)) * 8, sum);
                    }
                }
            }
        }
        gstep += K;
        __syncthreads();
    }
}

template <bool FWD, int R, int ST = 1>
int launch3m(const Sweep3Args &a, cudaStream_t st) {
    using G = S3m<R, ST>;
    const size_t smem = ((size_t)G::NR * G::LPB * G::ROWD + (size_t)G::LPB * a.g.K) * sizeof(double);
    LP_ARG(smem <= 227 * 1024, "3-D sweep needs %zu bytes of shared memory (K = %d)", smem, a.g.K);
    auto kern = box_sweep3d_multi_kernel<FWD, R, ST>;
    const int nblocks = resident_blocks(reinterpret_cast<const void *>(kern), G::NT, smem);
    if (nblocks < 1) return LP_ERR_ARG;
    int blocks = nblocks < a.ngroups ? nblocks : a.ngroups;
    kern<<<blocks, G::NT, smem, st>>>(a);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

template <bool FWD, int R>
int launch3(const Sweep3Args &a, cudaStream_t st) {
    using G = S3<R>;
    const size_t smem = ((size_t)G::NR * G::ROWD + a.g.K) * sizeof(double);
    LP_ARG(smem <= 227 * 1024, "3-D sweep needs %zu bytes of shared memory (K = %d)", smem, a.g.K);
    auto kern = box_sweep3d_kernel<FWD, R>;
    const int nblocks = resident_blocks(reinterpret_cast<const void *>(kern), G::NT, smem);
    if (nblocks < 1) return LP_ERR_ARG;
    int blocks = nblocks < a.nrun ? nblocks : a.nrun;
    kern<<<blocks, G::NT, smem, st>>>(a);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

template <bool FWD>
int dispatch3(const Sweep3Args &a, int r, cudaStream_t st) {
    switch (r) {
        case 2: return launch3m<FWD, 2>(a, st);
        case 3: return launch3m<FWD, 3>(a, st);
        case 4: return launch3m<FWD, 4>(a, st);
        case 5: return launch3<FWD, 5>(a, st);
        case 6: return launch3<FWD, 6>(a, st);
        case 7: return launch3<FWD, 7>(a, st);
        case 8: return launch3<FWD, 8>(a, st);
        case 9: return launch3<FWD, 9>(a, st);
        case 10: return launch3<FWD, 10>(a, st);
        default: return LP_ERR_ARG;
    }
}

}  // namespace

namespace {
// any in-pattern slot with an odd offset coordinate?  oddm[w]: odd-offset slots of word w
__global__ void odd_slots_kernel(Geom g, const uint32_t *__restrict__ mask, const uint32_t *__restrict__ oddm,
                                 int *any) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.n * g.mw;
         q += (int64_t)gridDim.x * blockDim.x)
        if (mask[q] & oddm[q % g.mw]) {
            *any = 1;
            return;
        }
}

// even[i][e] = lu[i][slot of offset 2 (a, b, c)], (a, b, c) in {-1, 0, 1}^3, a fastest
__global__ void even_compact_kernel(Geom g, const double *__restrict__ lu, double *__restrict__ even) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.n * 27;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / 27;
        const int e = (int)(q - i * 27);
        const int ax = e % 3 - 1, ay = (e / 3) % 3 - 1, az = e / 9 - 1;
        const int s = (2 * ax + g.r) + g.W * ((2 * ay + g.r) + g.W * (2 * az + g.r));
        even[q] = lu[i * g.S + s];
    }
}
}  // namespace

// T = 0 patterns (reach 2, every in-pattern offset even): compact the factors to
// the 27 even slots for the sweeps (13 / 14 values per row instead of 62 / 63).
// Skipped when the pattern has odd offsets or the copy does not fit.
int box_build_even(lp_ilu *m, cudaStream_t st) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    if (g.d != 3 || g.r != 2 || !b.mask) return LP_OK;
    std::vector<uint32_t> oddm(g.mw, 0u);
    for (int s = 0; s < g.S; ++s) {
        const int ox = s % g.W - g.r, oy = (s / g.W) % g.W - g.r, oz = s / (g.W * g.W) - g.r;
        if ((ox & 1) || (oy & 1) || (oz & 1)) oddm[s >> 5] |= 1u << (s & 31);
    }
    uint32_t *d_odd = nullptr;
    int *d_any = nullptr;
    int rc;
    if ((rc = salloc(&d_odd, g.mw, "odd slots", st)) || (rc = salloc(&d_any, 1, "flag", st))) return rc;
    LP_CUDA(cudaMemcpyAsync(d_odd, oddm.data(), g.mw * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    LP_CUDA(cudaMemsetAsync(d_any, 0, sizeof(int), st));
    odd_slots_kernel<<<num_sms() * 8, 256, 0, st>>>(g, b.mask, d_odd, d_any);
    count_launch();
    int any = 1;
    LP_CUDA(cudaMemcpyAsync(&any, d_any, sizeof(int), cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaStreamSynchronize(st));
    sfree(d_odd, st);
    sfree(d_any, st);
    if (any) return LP_OK;
    if (!b.even && dalloc(&b.even, (size_t)g.n * 27 + 2, "even-slot factors") != LP_OK) {
        b.even = nullptr;   // no room: the sweeps stream the box rows
        return LP_OK;
    }
    even_compact_kernel<<<num_sms() * 16, 256, 0, st>>>(g, b.lu, b.even);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

bool box_sweep3d_applies(const Geom &g) {
    return g.d == 3 && g.r >= 2 && g.r <= 10 && g.K >= 1;
}

// Wavefront order of the x-lines.  With unit cost per row, row (x, y, z) can
// run at level x + (r+1) y + (r+1)^2 z, so line (y, z) starts at
// (r+1)(y + (r+1) z): lines with equal key y + (r+1) z are independent, and
// every line a line depends on -- (y', z) with y' < y, or (y', z') with z' < z
// and y' <= y + r -- has a smaller key.  Handing lines out in key order keeps
// the ~(r+2)K/(r+1)^2 planes of the wavefront in flight together (natural order
// would hold the running CTAs to one or two planes) while every line still only
// waits on lines with smaller tickets.  The backward sweep mirrors the order.
int ensure_line_order(BoxLayout &b, cudaStream_t st) {
    if (b.line_order) return LP_OK;
    const int K = b.K, r = b.r;
    std::vector<int> ord;
    ord.reserve((size_t)K * K);
    for (int key = 0; key <= (K - 1) + (r + 1) * (K - 1); ++key)
        for (int z = 0; z < K; ++z) {
            const int y = key - (r + 1) * z;
            if (y < 0) break;
            if (y < K) ord.push_back(y + K * z);
        }
    int rc = dalloc(&b.line_order, ord.size(), "sweep line order");
    if (rc) return rc;
    LP_CUDA(cudaMemcpyAsync(b.line_order, ord.data(), ord.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    LP_CUDA(cudaStreamSynchronize(st));
    return LP_OK;
}

// Groups of up to lpb consecutive lines of line_order with the same key (the
// small-reach kernel advances a group in lockstep; equal keys are independent).
static int ensure_line_groups(BoxLayout &b, int lpb, cudaStream_t st) {
    if (b.line_groups) return LP_OK;
    const int K = b.K, A = b.r + 1;
    std::vector<int> ord((size_t)K * K);
    LP_CUDA(cudaMemcpy(ord.data(), b.line_order, ord.size() * sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<int> gp;
    int prev_key = -1, run = 0;
    for (size_t p = 0; p < ord.size(); ++p) {
        const int key = ord[p] % K + A * (ord[p] / K);
        if (key != prev_key || run == lpb) {
            gp.push_back((int)p);
            run = 0;
            prev_key = key;
        }
        ++run;
    }
    gp.push_back((int)ord.size());
    int rc = dalloc(&b.line_groups, gp.size(), "sweep line groups");
    if (rc) return rc;
    LP_CUDA(cudaMemcpyAsync(b.line_groups, gp.data(), gp.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    LP_CUDA(cudaStreamSynchronize(st));
    b.n_line_groups = (int)gp.size() - 1;
    return LP_OK;
}

static int small_reach_lpb(int r) {
    switch (r) {
        case 2: return S3m<2>::LPB;
        case 3: return S3m<3>::LPB;
        case 4: return S3m<4>::LPB;
        default: return 0;
    }
}

// Forward / backward line order of one rank of a y-slab split (lines of the
// global wavefront order whose y -- mirrored for the backward sweep, which
// walks order[] from the other end -- lies in the rank's slab), cached.
static int rank_order(BoxLayout &b, const RankLayout &lay, bool fwd, int lpb, cudaStream_t st) {
    BoxLayout::RankOrder &ro = b.rank_order[fwd ? 0 : 1];
    int sig[11] = {lay.nranks, lay.own};
    for (int v = 0; v <= lay.nranks; ++v) sig[2 + v] = lay.ys[v];
    bool same = true;
    for (int i = 0; i < 2 + lay.nranks + 1; ++i) same = same && ro.sig[i] == sig[i];
    if (same && ro.order) return LP_OK;
    const int K = b.K, A = b.r + 1;
    std::vector<int> ord((size_t)K * K);
    LP_CUDA(cudaMemcpy(ord.data(), b.line_order, ord.size() * sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<int> mine, gp;
    const int y0 = lay.ys[lay.own], y1 = lay.ys[lay.own + 1];
    for (int o : ord) {
        const int y = fwd ? o % K : K - 1 - o % K;
        if (y >= y0 && y < y1) mine.push_back(o);
    }
    int prev_key = -1, run = 0;
    for (size_t p = 0; p < mine.size(); ++p) {
        const int key = mine[p] % K + A * (mine[p] / K);
        if (key != prev_key || run == lpb) {
            gp.push_back((int)p);
            run = 0;
            prev_key = key;
        }
        ++run;
    }
    gp.push_back((int)mine.size());
    dfree(ro.order);
    dfree(ro.groups);
    ro.order = ro.groups = nullptr;
    int rc;
    if ((rc = dalloc(&ro.order, mine.size(), "rank line order")) ||
        (rc = dalloc(&ro.groups, gp.size(), "rank line groups")))
        return rc;
    LP_CUDA(cudaMemcpy(ro.order, mine.data(), mine.size() * sizeof(int), cudaMemcpyHostToDevice));
    LP_CUDA(cudaMemcpy(ro.groups, gp.data(), gp.size() * sizeof(int), cudaMemcpyHostToDevice));
    ro.norder = (int)mine.size();
    ro.ngroups = (int)gp.size() - 1;
    for (int i = 0; i < 11; ++i) ro.sig[i] = i < 2 + lay.nranks + 1 ? sig[i] : -1;
    (void)st;
    return LP_OK;
}

// The caller has pre-filled `out` with the sentinel and reset the ticket.
int box_sweep3d(lp_ilu *m, bool fwd, const double *rhs, double *out, int *ticket, cudaStream_t st,
                const RankLayout *ranks) {
    Geom g = geom_of(m->box);
    if (!box_sweep3d_applies(g)) return LP_ERR_ARG;
    int rc = ensure_line_order(m->box, st);
    if (rc) return rc;
    const int lpb = small_reach_lpb(g.r);
    if (lpb && (rc = ensure_line_groups(m->box, lpb, st))) return rc;
    Sweep3Args a;
    a.g = g;
    a.lu = m->box.lu;
    a.rows = g.S;
    a.ticket = ticket;
    a.order = m->box.line_order;
    a.nrun = g.nlines;
    a.gpos = lpb ? m->box.line_groups : nullptr;
    a.ngroups = lpb ? m->box.n_line_groups : g.nlines;
    a.nranks = 1;
    a.ys[0] = 0;
    a.ys[1] = g.K;
    a.sys = 0;
    for (int v = 0; v < MAX_RANKS; ++v) {
        a.rep[v] = out;
        a.rhsrep[v] = rhs;
    }
    if (ranks && ranks->nranks > 1) {
        a.nranks = ranks->nranks;
        for (int v = 0; v <= a.nranks; ++v) a.ys[v] = ranks->ys[v];
        if (ranks->own < 0) {
            for (int v = 0; v < a.nranks; ++v) {
                a.rep[v] = out + (size_t)v * g.n;
                a.rhsrep[v] = rhs + (ranks->rhs_replicated ? (size_t)v * g.n : 0);
            }
        } else {
            for (int v = 0; v < a.nranks; ++v) a.rep[v] = v == ranks->own ? out : ranks->peers[v];
            a.sys = 1;
        }
    }
    if (ranks && ranks->own >= 0) {
        RankLayout lay = *ranks;
        if (lay.nranks == 1) {
            lay.ys[0] = 0;
            lay.ys[1] = g.K;
        }
        if ((rc = rank_order(m->box, lay, fwd, lpb ? lpb : 1, st))) return rc;
        const BoxLayout::RankOrder &ro = m->box.rank_order[fwd ? 0 : 1];
        a.order = ro.order;
        a.nrun = ro.norder;
        a.gpos = lpb ? ro.groups : nullptr;
        a.ngroups = lpb ? ro.ngroups : ro.norder;
    }
    a.trace = nullptr;
#ifdef LP_SWEEP_TRACE
    {
        static unsigned long long *tr = nullptr;
        static size_t trn = 0;
        if (trn < (size_t)g.nlines * 8) {
            if (tr) dfree(tr);
            trn = (size_t)g.nlines * 8;
            dalloc(&tr, trn, "sweep trace");
        }
        cudaMemsetAsync(tr, 0, trn * 8, st);
        a.trace = tr;
        g_trace = tr;
        g_trace_n = trn;
    }
#endif
    if (m->box.even && g.r == 2) {
        a.lu = m->box.even;
        a.rows = 27;
        return fwd ? launch3m<true, 1, 2>(a, st) : launch3m<false, 1, 2>(a, st);
    }
    return fwd ? dispatch3<true>(a, g.r, st) : dispatch3<false>(a, g.r, st);
}

namespace {
__global__ void fill_sent3(int64_t n, double *a) {
    const double v = __longlong_as_double((long long)SENT3);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}
}  // namespace

}  // namespace lp

using namespace lp;

// Sweeps with the vector distributed over y-slab ranks,
// emulated on one device in one launch: rank v owns the x-lines with y in
// [ys[v], ys[v+1]) and keeps a replica of the vector (replica v of `out` at
// out + v n); a line is computed from its owner's replica and published to the
// owner and to every rank whose stencil halo reaches it, exactly the stores a
// multi-GPU run makes into its neighbours' memory over NVLink.  rhs is one
// vector (forward) or nranks replicas (backward, rhs_replicated = 1).
extern "C" int lp_sweep_ranks(lp_ilu *f, int nranks, const int *ys, int dir, const double *rhs,
                              int rhs_replicated, double *out, void *stream) {
    LP_ARG(f->kind == MAT_BOX && f->factored, "lp_sweep_ranks needs a factored box matrix");
    Geom g = geom_of(f->box);
    LP_ARG(box_sweep3d_applies(g), "lp_sweep_ranks is for 3-D box factors (reach 2..10)");
    LP_ARG(nranks >= 1 && nranks <= MAX_RANKS, "nranks must be in 1..%d", MAX_RANKS);
    LP_ARG(ys[0] == 0 && ys[nranks] == g.K, "y slabs must cover [0, K)");
    for (int v = 0; v < nranks; ++v) LP_ARG(ys[v] < ys[v + 1], "empty y slab");
    cudaStream_t st = as_stream(stream);
    fill_sent3<<<num_sms() * 8, 256, 0, st>>>((int64_t)nranks * g.n, out);
    count_launch();
    RankLayout lay;
    lay.nranks = nranks;
    for (int v = 0; v <= nranks; ++v) lay.ys[v] = ys[v];
    lay.rhs_replicated = rhs_replicated != 0;
    int *tk = nullptr;
    int rc;
    if ((rc = salloc(&tk, 1, "sweep ticket", st))) return rc;
    LP_CUDA(cudaMemsetAsync(tk, 0, sizeof(int), st));
    rc = box_sweep3d(f, dir == 0, rhs, out, tk, st, &lay);
    sfree(tk, st);
    return rc;
}

// Sentinel pre-fill of a replica (lp_sweep_rank's `out`): every rank fills its
// replicas BEFORE the ranks synchronise (the neighbours' halo stores must not
// be overwritten).
extern "C" int lp_sweep_prefill(int64_t n, double *out, void *stream) {
    fill_sent3<<<num_sms() * 8, 256, 0, as_stream(stream)>>>(n, out);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

// One rank of a multi-GPU y-slab sweep: this process's lines
// only, in the global wavefront order; out = this rank's replica (pre-filled
// with lp_sweep_prefill before the ranks synchronise), peers[v] = the other ranks' replicas mapped through
// lp_ipc_open (NULL for rank `rank` itself and for ranks whose slab is not
// adjacent); rhs = this rank's replica of the right-hand side.  Every rank
// launches concurrently (one GPU each); the line values a neighbour needs are
// stored straight into its replica over NVLink.  Same arithmetic per line as
// lp_forward_sub / lp_backward_sub.
extern "C" int lp_sweep_rank(lp_ilu *f, int nranks, const int *ys, int rank, int dir,
                             const double *rhs, double *out, double *const *peers, void *stream) {
    LP_ARG(f->kind == MAT_BOX && f->factored, "lp_sweep_rank needs a factored box matrix");
    Geom g = geom_of(f->box);
    LP_ARG(box_sweep3d_applies(g), "lp_sweep_rank is for 3-D box factors (reach 2..10)");
    LP_ARG(nranks >= 1 && nranks <= MAX_RANKS, "nranks must be in 1..%d", MAX_RANKS);
    LP_ARG(rank >= 0 && rank < nranks, "rank %d outside [0, %d)", rank, nranks);
    LP_ARG(ys[0] == 0 && ys[nranks] == g.K, "y slabs must cover [0, K)");
    for (int v = 0; v < nranks; ++v) LP_ARG(ys[v] < ys[v + 1], "empty y slab");
    for (int v = 0; v < nranks; ++v)
        if (v != rank && (v == rank - 1 || v == rank + 1))
            LP_ARG(peers && peers[v], "missing replica of neighbour rank %d", v);
    cudaStream_t st = as_stream(stream);
    RankLayout lay;
    lay.nranks = nranks;
    for (int v = 0; v <= nranks; ++v) lay.ys[v] = ys[v];
    lay.own = rank;
    for (int v = 0; v < nranks; ++v) lay.peers[v] = (peers && v != rank) ? peers[v] : nullptr;
    int *tk = nullptr;
    int rc;
    if ((rc = salloc(&tk, 1, "sweep ticket", st))) return rc;
    LP_CUDA(cudaMemsetAsync(tk, 0, sizeof(int), st));
    rc = box_sweep3d(f, dir == 0, rhs, out, tk, st, &lay);
    sfree(tk, st);
    return rc;
}

// CUDA IPC plumbing for the replicas (one process per GPU).  lp_ipc_alloc:
// cudaMalloc'd device buffer plus its 64-byte IPC handle; lp_ipc_open maps a
// peer's handle (peer access over NVLink).
extern "C" int lp_ipc_alloc(int64_t bytes, void **ptr, unsigned char *handle64) {
    LP_CUDA(cudaMalloc(ptr, (size_t)bytes));
    cudaIpcMemHandle_t h;
    LP_CUDA(cudaIpcGetMemHandle(&h, *ptr));
    memcpy(handle64, &h, sizeof h);
    return LP_OK;
}

extern "C" int lp_ipc_free(void *ptr) {
    LP_CUDA(cudaFree(ptr));
    return LP_OK;
}

extern "C" int lp_ipc_open(const unsigned char *handle64, void **ptr) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof h);
    LP_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return LP_OK;
}

extern "C" int lp_ipc_close(void *ptr) {
    LP_CUDA(cudaIpcCloseMemHandle(ptr));
    return LP_OK;
}
