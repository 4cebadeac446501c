// ILU(0) forward / backward sweeps in the box layout (forward_sub / backward_sub,
// sparse.py:175-216), as a warp-specialised, fence-free line wavefront.
//
// A CTA owns one x-line at a time (lines handed out in sweep order by an
// atomic ticket, so a CTA only ever waits on lines owned by running CTAs).
// Row t of line L needs, besides its own line, the rows x <= t + r of the
// earlier lines of its stencil.  The work of a line is split so that the
// line-to-line critical path carries as little as possible:
//
//  * the serial warp owns everything that depends on the immediately
//    preceding line L-1 (the 2r+1 entries with offset oy = -1, oz = 0) and on
//    the line itself (the r in-line entries).  Lane k carries the running sum
//    of row t+k (k <= 2r).  Each step polls the one new value y(L-1, t+r) and
//    folds it into all 2r+1 running sums, adds y_{t-1} to the in-line sums,
//    and lane 0 finishes y_t = (c_t - A_t) - l1_t y_{t-1}: a line can trail
//    its predecessor by only ~r steps plus one L2 round trip;
//  * producer warps take rows round-robin and reduce the rest of the stencil
//    (lines L-2 and older, previous planes), which was produced long before:
//    c_t = rhs_t - sum L_ts y_col(s), into a shared ring, with the next row's
//    factor loads in flight (two register sets, ping-pong).
//
// Synchronisation carries no fences: every value is its own flag.  The output
// vector is pre-filled with a NaN sentinel; a consumer polls the 8-byte value
// it needs (aligned 64-bit accesses are single-copy atomic; relaxed .gpu
// loads, coherent at L2) until it is no longer the sentinel.  The shared ring
// uses per-step sentinels; computed NaNs are canonicalised so they can never
// alias a sentinel.  Band coefficients are staged by cp.async (register
// prefetch queues get their registers reused by the compiler, serialising
// every step on the load).  The backward sweep is the mirror image (rows and
// lines in reverse, scaling by 1/U_tt).
#include <math.h>

#include <type_traits>

#include "box_geom.cuh"
#include "ilu.cuh"
#include "smem_tma.cuh"
#include "vector_ops.cuh"

namespace lp {

unsigned long long *g_trace = nullptr;   // LP_SWEEP_TRACE builds only
__device__ long long g_chk[8];            // LP_SWEEP_CHECK builds: first failed check
size_t g_trace_n = 0;

constexpr unsigned long long SWEEP_SENTINEL = 0xFFF4C0FFEE5EED00ull;   // signalling NaN

namespace {

constexpr int RING = 64;    // rows in flight per line (power of two)
constexpr int BRING = 128;  // band rows staged for the serial warp (power of two)
constexpr int PR = 8;       // rows per producer stage (2-D)
constexpr int NSTAGE = 5;   // producer stages in flight (2-D)
constexpr unsigned long long RING_SENT = 0xFFF5000000000000ull;

#ifndef LP_SWEEP_SLEEP
#define LP_SWEEP_SLEEP 20
#endif

__device__ __forceinline__ unsigned long long bits(double v) {
    return (unsigned long long)__double_as_longlong(v);
}

__device__ __forceinline__ double canon(double v) {
    return isnan(v) ? __longlong_as_double(0x7FF8000000000000ll) : v;
}

// Relaxed gpu-scope load that the compiler may neither cache nor elide (a
// plain load in a side-effect-free spin loop can legally be removed).
__device__ __forceinline__ double ld_poll(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// Published values are stored with st.relaxed.gpu and polled with
// ld.relaxed.gpu: a morally strong pair (no data race under the PTX memory
// model), and an aligned 8-byte access is single-copy atomic, so a poller sees
// either the sentinel or the final value.
__device__ __forceinline__ void st_pub(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ double ring_sent(int t) {
    return __longlong_as_double((long long)(RING_SENT | (unsigned)t));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    return v;
}

__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

struct SweepArgs {
    Geom g;
    const double *lu;     // factors [n][S]
    const double *band;   // [n][NQ]: in-line coefficients (see band_kernel)
    const double *rhs;
    double *out;
    int *ticket;
    const double *band_g; // [n][gsz]: line L-/+1 coefficients (band + n * NQ)
    int gsz;              // their padded size (even)
    int lo, nslot;        // producers' slot range [lo, lo + nslot)
    int pr_rs, pr_ww;     // 2-D staged producers: factor row stride / y-window width (doubles)
    unsigned pr_ofs;      // byte offset of the producers' staging region in dynamic smem
    int nseg;             // 2-D: lines of the producers' stencil (r - 1)
    int csize;            // cluster size: lines of a batch (consecutive in sweep order)
    unsigned yr_ofs;      // byte offset of the line-handoff buffer [K] in dynamic smem
    unsigned long long *trace;   // LP_SWEEP_TRACE builds: per-line timestamps
    // fused dot product (pcg.py:151, r'z inside the backward sweep): the serial
    // warp of line L accumulates sum_x dotv[row] * out[row] and stores it to
    // dotpart[L]; null = no dot
    const double *dotv;
    double *dotpart;
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}


// One TMA bulk copy (two at the ring wrap) of the w-double rows of steps
// [32c, 32c + 32) of a line into a BRING-row shared ring (ring row = ix mod BRING),
// completing on mbarrier `mbar` (slot c mod 4).  Issued by one lane.
template <bool FWD>
__device__ __forceinline__ void stage_chunk(const double *src, int w, unsigned ring, int64_t row0,
                                            int K, int c, unsigned mbar) {
    const int u0 = 32 * c;
    if (u0 >= K) return;
    const int u1 = min(u0 + 32, K);
    const int ixlo = FWD ? u0 : K - u1, ixhi = FWD ? u1 : K - u0;
    const unsigned rb = (unsigned)w * 8;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect(mbar, (unsigned)(ixhi - ixlo) * rb);
    int p0 = ixlo;
    while (p0 < ixhi) {
        const int p1 = min(ixhi, (p0 / BRING + 1) * BRING);
        bulk_g2s(ring + (unsigned)(p0 & (BRING - 1)) * rb, src + (size_t)(row0 + p0) * w,
                 (unsigned)(p1 - p0) * rb, mbar);
        p0 = p1;
    }
}

// Warp roles: warps with id mod 4 in {0, 1} produce c_t = rhs_t - (stencil part
// in lines L-/+2 and older / other planes); warp NW-2 ("group") adds the 2r+1 entries of line
// L-/+1 as their values arrive and hands d_t = c_t - A_t to warp NW-1
// ("serial"), which runs the in-line recurrence y_t = d_t - sum_q l_q y_{t-q}
// entirely in registers (every lane redundantly; no shuffles on the chain).
template <bool FWD, int NW, int CH, int NQ>
__global__ void __launch_bounds__(32 * NW)
box_sweep_kernel(const __grid_constant__ SweepArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const Geom &g = a.g;
    double *s_in = reinterpret_cast<double *>(dsm);                     // [BRING][NQ]
    double *s_grp = s_in + (size_t)BRING * NQ;                          // [BRING][gsz]
    int *s_delta = reinterpret_cast<int *>(s_grp + (size_t)BRING * a.gsz);   // [nslot]
    signed char *s_ox = reinterpret_cast<signed char *>(s_delta + a.nslot);
    signed char *s_oy = s_ox + a.nslot;
    signed char *s_oz = s_oy + a.nslot;
    unsigned char *s_ok = reinterpret_cast<unsigned char *>(s_oz + a.nslot);
    __shared__ __align__(8) unsigned long long s_mbar[8];   // chunk barriers: serial 0-3, group 4-7
    __shared__ __align__(8) unsigned long long s_pfull[NSTAGE];
    // stages consumed per ring slot (a counter, not an mbarrier: a loader can be
    // two phases ahead of a slow consumer, where a parity wait would alias)
    __shared__ unsigned s_pcons[NSTAGE];
    __shared__ double s_c[RING];   // producers -> serial: c_t
    __shared__ double s_d[RING];   // group -> serial: A_t (line L-/+1 part)
    __shared__ int s_line;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = g.K, r = g.r;
    volatile double *v_c = s_c;
    volatile double *v_d = s_d;
    constexpr int SERIAL = NW - 1;   // highest warp ids: favoured by the SMSP arbiter
    constexpr int GROUP = NW - 2;

    if (tid == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(smem_addr(s_mbar + i), 1);
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(smem_addr(s_pfull + i), 1);
            s_pcons[i] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    unsigned chunk_base = 0;   // chunks this warp has staged on earlier lines (mbarrier phases)
    unsigned stage_base = 0;   // producer stages of earlier lines (2-D; mbarrier phases)
    int *s_yofs = reinterpret_cast<int *>(dsm + a.pr_ofs + (size_t)NSTAGE * (PR * a.pr_rs + a.nseg * a.pr_ww) * 8);
    if (g.d == 2)
        for (int j = tid; j < a.nslot; j += blockDim.x) s_yofs[j] = (j / g.W) * a.pr_ww + j % g.W;
    for (int j = tid; j < a.nslot; j += blockDim.x) {
        int sx, sy, sz;
        slot_axes(g, a.lo + j, sx, sy, sz);
        s_ox[j] = (signed char)(sx - r);
        s_oy[j] = (signed char)(sy - r);
        s_oz[j] = (signed char)(sz - r);
        s_delta[j] = (sx - r) + K * ((sy - r) + K * (sz - r));
    }

    // Lines are handed out in batches of csize consecutive lines, one per CTA of a
    // cluster; each CTA pushes its y values straight into the shared memory of
    // the CTA holding the next line (distributed shared memory), so the
    // line-to-line handoff inside a batch skips the L2 round trips.
    const unsigned crank = a.csize > 1 ? cluster_rank() : 0;
    double *s_yr = reinterpret_cast<double *>(dsm + a.yr_ofs);   // [K]: y of the previous line
    const unsigned yr0 = smem_addr(s_yr);
    const bool use_yr = a.csize > 1;
    const double sent = __longlong_as_double((long long)SWEEP_SENTINEL);
    for (;;) {
        __syncthreads();
        if (use_yr)
            for (int x = tid; x < K; x += blockDim.x) s_yr[x] = sent;
        if (crank == 0 && tid == 0) {
            const int tb = atomicAdd(a.ticket, 1);
            s_line = tb;
            for (int q = 1; q < a.csize; ++q) st_cluster_s32(map_rank(smem_addr(&s_line), q), tb);
        }
        for (int k = tid; k < RING; k += blockDim.x) {
            s_c[k] = ring_sent(k);
            s_d[k] = ring_sent(k);
        }
        if (use_yr) cluster_sync();
        else __syncthreads();
        const int tb = s_line;
        if (tb * a.csize >= g.nlines) return;
        const int tl = tb * a.csize + (int)crank;
        if (tl >= g.nlines) continue;   // idle rank of the last batch
        const int L = FWD ? tl : g.nlines - 1 - tl;
        const int iy = g.d > 1 ? L % K : 0, iz = g.d > 2 ? L / K : 0;
        for (int j = tid; j < a.nslot; j += blockDim.x) {
            const int y = iy + s_oy[j], z = iz + s_oz[j];
            s_ok[j] = (g.d < 2 || (y >= 0 && y < K)) && (g.d < 3 || (z >= 0 && z < K));
        }
        const int64_t row0 = (int64_t)L * K;
#ifdef LP_SWEEP_TRACE
        if (tid == 0 && a.trace) a.trace[(size_t)tl * 16] = gtime();
#endif
        __syncthreads();
        auto ix_of = [&](int t) { return FWD ? t : K - 1 - t; };

        if (warp == SERIAL) {
            // ------------------------------------------- serial recurrence
            // Lane k owns the rows t == k (mod 32): sp = its row's in-line sum over
            // the steps q >= 2, accumulated as those values are produced (one FMA
            // per lane per step).  Row t+1's finished sum is broadcast during step
            // t, off the chain; every lane then forms the same
            //   y_t = fma(-e_1(t-1), y_{t-1}, rd_t d_t - sp_t).
            // All addresses advance incrementally (the warp is latency bound: a
            // step is a few dozen dependent-issue instructions).
            constexpr unsigned RB = BRING * NQ * 8;        // ring bytes (power of two)
            const unsigned in0 = smem_addr(s_in), d0 = smem_addr(s_d), c0 = smem_addr(s_c);
            const unsigned mb = smem_addr(s_mbar);
            const bool has_prev = g.d > 1 && (FWD ? iy > 0 : iy < K - 1);
            const int nch = (K + 31) / 32;
            auto stage = [&](int c) {   // chunk c of this line (steps [32c, 32c+32))
                if (lane == 0 && c < nch)
                    stage_chunk<FWD>(a.band, NQ, in0, row0, K, c, mb + 8 * ((chunk_base + c) & 3));
            };
#ifdef LP_SWEEP_TRACE
            long long wcyc = 0;
#endif
            auto wait_chunk = [&](int c) {
#ifdef LP_SWEEP_TRACE
                const long long w0 = clock64();
#endif
                if (c < nch) mbar_wait(mb + 8 * ((chunk_base + c) & 3), ((chunk_base + c) >> 2) & 1);
#ifdef LP_SWEEP_TRACE
                wcyc += clock64() - w0;
#endif
            };
            // fused dot: lane k holds dotv of row 32c + k of the current chunk (the
            // next chunk's values are loaded a chunk ahead, off the chain)
            const bool dot = a.dotv != nullptr;
            double racc = 0.0, rv = 0.0, rvn = 0.0;
            if (dot && lane < K) rvn = __ldg(a.dotv + row0 + ix_of(lane));
            stage(0);
            stage(1);
            stage(2);
            wait_chunk(0);
            unsigned roff = FWD ? 0u : (unsigned)(((K - 1) & (BRING - 1)) * NQ * 8);
            const unsigned rstep = FWD ? NQ * 8u : (unsigned)(RB - NQ * 8);
            unsigned doff = 0;
            unsigned jl = (unsigned)lane;                   // (lane - t) & 31
            double sp = 0.0, yprev = 0.0, e1 = 0.0;
            double e1n, rdn;
            lds2(in0 + roff, e1n, rdn);
            double qn = (jl >= 2 && jl < NQ) ? lds(in0 + roff + 8 * jl) : 0.0;
            double spn = 0.0;
            double dn = has_prev ? lds_v(d0) : 0.0, cn = lds_v(c0);
            double *outp = a.out + row0 + (FWD ? 0 : K - 1);
            const ptrdiff_t ostep = FWD ? 1 : -1;
            // loop bounds in registers (a "memory" clobber would otherwise make the
            // compiler re-read them from the parameter bank every step)
            int Kr;
            asm volatile("mov.b32 %0, %1;" : "=r"(Kr) : "r"(K));
            unsigned qoff = 8u * (unsigned)lane;   // 8 * ((lane - t) & 31)
            // next line of the batch in the same plane: it reads this line's values
            const bool push = use_yr && crank + 1 < (unsigned)a.csize && tl + 1 < g.nlines &&
                              (g.d < 2 || (FWD ? iy < K - 1 : iy > 0));
            const unsigned push_base = push ? map_rank(yr0, crank + 1) : 0u;
#ifdef LP_SWEEP_TRACE
            long long nspin_c = 0, nspin_a = 0;
#endif
            // HP: the line has a previous line (A_t from the group); a compile-time
            // flag so the step carries no branch on it
            auto step = [&](const int t, auto HP, auto DT) {
                constexpr bool hp = decltype(HP)::value;
                const double q = qn, e1c = e1n, rd = rdn, spt = spn;
                double c = cn, av = dn;
                const unsigned long long sb = bits(ring_sent(t));
#ifdef LP_SWEEP_TRACE
                while (bits(c) == sb) { c = lds_v(c0 + doff); ++nspin_c; }
                if (hp)
                    while (bits(av) == sb) { av = lds_v(d0 + doff); ++nspin_a; }
#else
                while (bits(c) == sb) c = lds_v(c0 + doff);
                if (hp)
                    while (bits(av) == sb) av = lds_v(d0 + doff);
#endif
                const double y = fma(-e1, yprev, fma(rd, hp ? c - av : c, -spt));
                // every lane stores the same values (no divergent branch)
                sts_v(c0 + doff, ring_sent(t + RING));
                if (hp) sts_v(d0 + doff, ring_sent(t + RING));
                st_pub(outp, canon(y));
                if (push) st_cluster_f64(push_base + 8u * (unsigned)(FWD ? t : Kr - 1 - t), canon(y));
                outp += ostep;
                doff = (doff + 8) & (RING * 8 - 1);
                cn = lds_v(c0 + doff);
                if (hp) dn = lds_v(d0 + doff);
                roff = (roff + rstep) & (RB - 1);
                qoff = (qoff - 8) & 255;
                const unsigned rowa = in0 + roff;
                lds2(rowa, e1n, rdn);
                qn = (qoff - 16 < (NQ - 2) * 8) ? lds(rowa + qoff) : 0.0;
                // row t+1's finished sum: lane t+1 takes no update this step, so it is
                // broadcast before the update, off the y_t -> y_{t+1} chain
                spn = __shfl_sync(0xffffffff, sp, (t + 1) & 31);
                sp = ((unsigned)lane == ((unsigned)t & 31)) ? 0.0 : fma(q, y, sp);
                if (decltype(DT)::value) racc = ((unsigned)lane == ((unsigned)t & 31)) ? fma(rv, y, racc) : racc;
                e1 = e1c;
                yprev = y;
            };
#ifdef LP_SWEEP_TRACE
            auto mark = [&](int k) {
                if (lane == 0 && a.trace) {
                    a.trace[(size_t)tl * 16 + k] = gtime();
                    a.trace[(size_t)tl * 16 + 4 + k] = clock64();
                }
            };
            mark(1);
#endif
            for (int c = 0; c < nch; ++c) {
                // chunk c+1 must be resident before step 32c+31 prefetches its first row
                stage(c + 3);
                wait_chunk(c + 1);
                const int t1 = min(32 * c + 32, Kr);
#ifdef LP_SWEEP_TRACE
                const int th = Kr / 2, th2 = Kr / 2 + r + 1;
                if ((32 * c <= th && th < t1) || (32 * c <= th2 && th2 < t1)) {
                    for (int t = 32 * c; t < t1; ++t) {
                        if (t == th) mark(2);
                        if (t == th2 && lane == 0 && a.trace) a.trace[(size_t)tl * 16 + 15] = gtime();
                        if (has_prev) step(t, std::true_type{}, std::false_type{});
                        else step(t, std::false_type{}, std::false_type{});
                    }
                    continue;
                }
#endif
                if (dot) {
                    rv = rvn;
                    const int tn = 32 * c + 32 + lane;
                    rvn = tn < Kr ? __ldg(a.dotv + row0 + ix_of(tn)) : 0.0;
                    if (has_prev)
                        for (int t = 32 * c; t < t1; ++t) step(t, std::true_type{}, std::true_type{});
                    else
                        for (int t = 32 * c; t < t1; ++t) step(t, std::false_type{}, std::true_type{});
                } else if (has_prev) {
                    for (int t = 32 * c; t < t1; ++t) step(t, std::true_type{}, std::false_type{});
                } else {
                    for (int t = 32 * c; t < t1; ++t) step(t, std::false_type{}, std::false_type{});
                }
            }
            if (dot) {
                // the line's sum in a fixed order (xor butterfly over the lanes)
#pragma unroll
                for (int o = 16; o; o >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, o);
                if (lane == 0) a.dotpart[L] = racc;
            }
#ifdef LP_SWEEP_TRACE
            mark(3);
#endif
#ifdef LP_SWEEP_TRACE
            if (lane == 0 && a.trace) {
                a.trace[(size_t)tl * 16 + 4] = wcyc;
                a.trace[(size_t)tl * 16 + 13] = nspin_c;
                a.trace[(size_t)tl * 16 + 14] = nspin_a;
            }
#endif
            chunk_base += nch;
        } else if (warp == GROUP) {
            // ------------------- line L-/+1 group: A_t (the serial forms c_t - A_t)
            // Lane k owns the rows t == k (mod 32) and accumulates their 2r+1
            // products with line L-/+1 as its values arrive (no shuffles on the
            // sums).  The value y(L-/+1, x) arriving at step t = x -/+ r enters rows
            // t..t+2r with the coefficients of band row x's group section.  Values
            // are polled 32 at a time (one per lane) and the window is re-polled
            // while the value needed next is not yet produced.
            const bool has_prev = g.d > 1 && (FWD ? iy > 0 : iy < K - 1);
            if (!has_prev) continue;
            const double *prev = a.out + (FWD ? row0 - K : row0 + K);   // line L-/+1
            // line L-/+2 of the same plane (produced a line earlier: always complete
            // in the block polls, its coefficients follow the 2r+1 of line L-/+1)
            const bool has_prev2 = FWD ? iy > 1 : iy < K - 2;
            const double *prev2 = a.out + (FWD ? row0 - 2 * K : row0 + 2 * K);
            const int R = r;
            const unsigned gstride = (unsigned)a.gsz * 8;
            const unsigned grp0 = smem_addr(s_grp), c0 = smem_addr(s_c), d0 = smem_addr(s_d);
            const unsigned mb = smem_addr(s_mbar + 4);
            const int nch = has_prev ? (K + 31) / 32 : 0;
            // chunk c = arrival indices [32c, 32c+32): x = 32c.. (fwd) / K-1-32c.. (bwd)
            auto stage = [&](int c) {
                if (lane == 0 && c < nch)
                    stage_chunk<FWD>(a.band_g, a.gsz, grp0, row0, K, c, mb + 8 * ((chunk_base + c) & 3));
            };
            auto wait_chunk = [&](int c) {
                if (c < nch) mbar_wait(mb + 8 * ((chunk_base + c) & 3), ((chunk_base + c) >> 2) & 1);
            };
            stage(0);
            stage(1);
            stage(2);
            wait_chunk(0);
            // loop constants in registers (opaque: no per-step parameter-bank reloads)
            const int Kr = opaque(K), tw = opaque(2 * R);
            const unsigned gstr = opaque(gstride);
            double acc = 0.0;
            double yb = 0.0;   // lane l: y(L-/+1, arrival index 32 b + l)
            // previous line held by the CTA before us in the cluster: its values land
            // in our shared memory; otherwise poll them in L2
            const bool local = use_yr && crank > 0;
            auto pollv = [&](int x) -> double { return local ? lds_v(yr0 + 8u * (unsigned)x) : ld_poll(prev + x); };
            auto poll_block = [&](int u0) -> double {
                const int ua = u0 + lane;
                return ua < Kr ? pollv(FWD ? ua : Kr - 1 - ua) : 0.0;
            };
            double ybn = poll_block(0);   // the next block's values, polled half a block early
            auto poll_block2 = [&](int u0) -> double {
                const int ua = u0 + lane;
                return (has_prev2 && ua < Kr) ? ld_poll(prev2 + (FWD ? ua : Kr - 1 - ua)) : 0.0;
            };
            double yb2 = 0.0, ybn2 = poll_block2(0);
            const unsigned g2 = 8u * (unsigned)(2 * R + 1);   // byte offset of the line-2 coefficients
            const unsigned jl0 = (unsigned)(lane + R) & 31;   // j = (jl0 - i) & 31 at step i of a block
#ifdef LP_SWEEP_TRACE
            const long long gc0 = clock64();
            long long nrepoll = 0;
#endif
            const int nblk = (Kr + R + 31) / 32;
            for (int blk = 0; blk < nblk; ++blk) {
                const int u0 = 32 * blk;
                stage(blk + 3);
                wait_chunk(blk + 1);
                yb = ybn;
                yb2 = ybn2;
                // the serial has consumed every slot this block will write
                {
                    const int tl31 = u0 + 31 - R;
                    if (tl31 >= 0) {
                        const unsigned long long fb = bits(ring_sent(tl31));
                        while (bits(lds_v(d0 + (tl31 & (RING - 1)) * 8)) != fb) {
                        }
                    }
                }
                __syncwarp();
                if (has_prev2) {
                    // line -/+2 was produced a line earlier: check the whole block once
                    while (__any_sync(0xffffffff, bits(yb2) == SWEEP_SENTINEL)) {
                        const int ua = u0 + lane;
                        if (bits(yb2) == SWEEP_SENTINEL) yb2 = ld_poll(prev2 + (FWD ? ua : Kr - 1 - ua));
                    }
                }
                if (u0 >= R && u0 + 32 <= Kr) {
                    // interior block: every arrival valid and every step publishes; no
                    // bounds tests, addresses advance incrementally
                    const unsigned RBg = BRING * gstr;
                    unsigned rofs = (unsigned)((FWD ? u0 : Kr - 1 - u0) & (BRING - 1)) * gstr;
                    unsigned jq = jl0;
                    double ynx = __shfl_sync(0xffffffff, yb, 0);
                    double y2n = __shfl_sync(0xffffffff, yb2, 0);
                    double qn = (int)jq <= tw ? lds(grp0 + rofs + 8 * jq) : 0.0;
                    double q2n = (has_prev2 && (int)jq <= tw) ? lds(grp0 + rofs + g2 + 8 * jq) : 0.0;
                    const unsigned tb = (unsigned)(u0 - R);
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        if (i == 16) {
                            ybn = poll_block(u0 + 32);
                            ybn2 = poll_block2(u0 + 32);
                        }
                        const double acc2 = fma(q2n, y2n, acc);
                        const double q = qn;
                        double yn = ynx;
                        if (i < 31) {
                            ynx = __shfl_sync(0xffffffff, yb, i + 1);
                            y2n = __shfl_sync(0xffffffff, yb2, i + 1);
                            rofs = FWD ? (rofs + gstr == RBg ? 0u : rofs + gstr) : (rofs == 0u ? RBg - gstr : rofs - gstr);
                            jq = (jq - 1u) & 31u;
                            const bool ok = (int)jq <= tw;
                            qn = ok ? lds(grp0 + rofs + 8 * jq) : 0.0;
                            q2n = (has_prev2 && ok) ? lds(grp0 + rofs + g2 + 8 * jq) : 0.0;
                        }
                        while (bits(yn) == SWEEP_SENTINEL) {
                            const int ua = u0 + lane;
                            if (lane >= i) yb = pollv(FWD ? ua : Kr - 1 - ua);
                            yn = __shfl_sync(0xffffffff, yb, i);
                            if (i < 31) ynx = __shfl_sync(0xffffffff, yb, i + 1);
#ifdef LP_SWEEP_TRACE
                            ++nrepoll;
#endif
                        }
                        acc = fma(q, yn, acc2);
                        if (lane == ((i - R) & 31)) {
                            sts_v(d0 + ((tb + (unsigned)i) & (RING - 1)) * 8, acc);
                            acc = 0.0;
                        }
                    }
                    continue;
                }
                // operands of step i are fetched during step i-1, off the arrival path
                auto qaddr = [&](int i) -> unsigned {
                    const int uarr = u0 + i;
                    const int x = FWD ? uarr : Kr - 1 - uarr;
                    const unsigned j = (jl0 - (unsigned)i) & 31;
                    return grp0 + (unsigned)(x & (BRING - 1)) * gstr + 8 * j;
                };
                auto jok = [&](int i) { return (int)((jl0 - (unsigned)i) & 31) <= tw; };
                double ynx = __shfl_sync(0xffffffff, yb, 0);
                double y2n = __shfl_sync(0xffffffff, yb2, 0);
                double qn = (u0 < Kr && jok(0)) ? lds(qaddr(0)) : 0.0;
                double q2n = (has_prev2 && u0 < Kr && jok(0)) ? lds(qaddr(0) + g2) : 0.0;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int uarr = u0 + i, t = uarr - R;
                    if (i == 16) {
                        ybn = poll_block(u0 + 32);
                        ybn2 = poll_block2(u0 + 32);
                    }
                    if (uarr < Kr) {
                        const double acc2 = fma(q2n, y2n, acc);
                        const double q = qn;
                        double yn = ynx;
                        if (i < 31) {
                            const bool nok = uarr + 1 < Kr && jok(i + 1);
                            ynx = __shfl_sync(0xffffffff, yb, i + 1);
                            y2n = __shfl_sync(0xffffffff, yb2, i + 1);
                            qn = nok ? lds(qaddr(i + 1)) : 0.0;
                            q2n = (has_prev2 && nok) ? lds(qaddr(i + 1) + g2) : 0.0;
                        }
                        while (bits(yn) == SWEEP_SENTINEL) {
                            // re-poll the rest of the window: one round trip brings in
                            // every value produced since the last poll
                            const int ua = u0 + lane;
                            if (lane >= i && ua < Kr) yb = pollv(FWD ? ua : Kr - 1 - ua);
                            yn = __shfl_sync(0xffffffff, yb, i);
                            if (i < 31) ynx = __shfl_sync(0xffffffff, yb, i + 1);
#ifdef LP_SWEEP_TRACE
                            ++nrepoll;
#endif
                        }
#ifdef LP_SWEEP_TRACE
                        if (lane == 0 && a.trace && t == K / 2) a.trace[(size_t)tl * 16 + 10] = gtime();
                        if (lane == 0 && a.trace && t == K / 2 - 64) a.trace[(size_t)tl * 16 + 11] = clock64();
                        if (lane == 0 && a.trace && t == K / 2) a.trace[(size_t)tl * 16 + 11] = clock64() - a.trace[(size_t)tl * 16 + 11];
                        if (lane == 0 && a.trace && t == K / 2 - 64) a.trace[(size_t)tl * 16 + 12] = nrepoll;
                        if (lane == 0 && a.trace && t == K / 2) a.trace[(size_t)tl * 16 + 12] = nrepoll - a.trace[(size_t)tl * 16 + 12];
#endif
                        acc = fma(q, yn, acc2);
                    }
                    if (lane == ((i - R) & 31) && t >= 0 && t < Kr) {
                        sts_v(d0 + (unsigned)(t & (RING - 1)) * 8, acc);
                        acc = 0.0;
                    }
                }
            }
#ifdef LP_SWEEP_TRACE
            (void)gc0;
#endif
            chunk_base += nch;
        } else if ((warp & 3) >= 2) {
            // keeps SMSPs 2 and 3 (warp id mod 4) to the group and serial warps:
            // both are latency bound, and any co-scheduled busy warp steals their
            // issue slots
            continue;
        } else {
            constexpr int NP = NW / 2;   // warps 0, 1, 4, 5, ... (SMSPs 0 and 1)
            const int pw = (warp >> 2) * 2 + (warp & 1);
            if (g.d == 2) {
                // ---- staged producers (2-D).  Stage s = PR consecutive rows (steps
                // [PR s, PR s + PR)), taken by warp s mod NP.  Their factor rows arrive
                // by TMA bulk copies into a NSTAGE-slot ring (full/empty mbarriers);
                // the y values of lines L-/+2 .. L-/+r over the stage's x window are
                // loaded once per stage into shared memory (sentinel-checked), and each
                // row's dot product is then formed from shared memory only.
                const int ns = (K + PR - 1) / PR;
                const unsigned fb0 = smem_addr(dsm + a.pr_ofs);
                const unsigned fslot = (unsigned)(PR * a.pr_rs) * 8;
                const unsigned yb0 = fb0 + NSTAGE * fslot;
                const unsigned yslot = (unsigned)(a.nseg * a.pr_ww) * 8;
                const unsigned full0 = smem_addr(s_pfull);
                volatile unsigned *v_cons = s_pcons;
                const int W = g.W, nslot = a.nslot, ww = a.pr_ww;
                const int oy0 = FWD ? -r : 3;   // line offset of segment 0
                const int depL = FWD ? (iy >= 3 ? L - 3 : -1) : (iy <= K - 4 ? L + 3 : -1);
                for (int st = pw; st < ns; st += NP) {
                    const unsigned gs = stage_base + st;
                    const unsigned slot = gs % NSTAGE;
                    const int t0 = PR * st, t1 = min(t0 + PR, K), nr = t1 - t0;
                    const int ixlo = FWD ? t0 : K - t1, ixhi = FWD ? t1 : K - t0;
                    const unsigned fb = fb0 + slot * fslot, yb = yb0 + slot * yslot;
                    // slot free: stage gs - NSTAGE (the previous user) consumed
                    while (v_cons[slot] < gs / NSTAGE) {
                    }
                    // factor rows: one 16-byte aligned bulk copy per row
                    if (lane == 0) {
                        unsigned bytes = 0;
                        for (int q = 0; q < nr; ++q) {
                            const int64_t gi = (row0 + (FWD ? t0 + q : K - 1 - t0 - q)) * (int64_t)g.S + a.lo;
                            bytes += (unsigned)((nslot + (int)(gi & 1) + 1) & ~1) * 8;
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        mbar_expect(full0 + 8 * slot, bytes);
                    }
                    __syncwarp();
                    double rhs_t = 0.0;
                    int sh = 0;
                    if (lane < nr) {
                        const int ix = FWD ? t0 + lane : K - 1 - t0 - lane;
                        const int64_t gi = (row0 + ix) * (int64_t)g.S + a.lo;
                        sh = (int)(gi & 1);
#ifdef LP_SWEEP_CHECK
                        if (gi - sh < 0 || gi - sh + ((nslot + sh + 1) & ~1) > g.n * (int64_t)g.S + 2 || ix < 0 ||
                            ix >= K || (fb - fb0) >= NSTAGE * fslot || ((fb + (unsigned)(lane * a.pr_rs) * 8) & 15)) {
                            if (atomicCAS((unsigned long long *)g_chk, 0ull, 1ull) == 0ull) {
                                g_chk[1] = L; g_chk[2] = st; g_chk[3] = lane; g_chk[4] = ix; g_chk[5] = gi;
                                g_chk[6] = sh; g_chk[7] = fb - fb0;
                            }
                            asm volatile("exit;");
                        }
#endif
                        bulk_g2s(fb + (unsigned)(lane * a.pr_rs) * 8, a.lu + (gi - sh),
                                 (unsigned)((nslot + sh + 1) & ~1) * 8, full0 + 8 * slot);
                        rhs_t = a.rhs[row0 + ix];
                    }
                    // y window of each stencil line: x in [ixlo - r, ixlo - r + ww)
                    if (depL >= 0) {
                        const int fx = FWD ? min(ixhi - 1 + r, K - 1) : max(ixlo - r, 0);
                        const double *fp = a.out + (int64_t)depL * K + fx;
                        while (bits(ld_poll(fp)) == SWEEP_SENTINEL) __nanosleep(LP_SWEEP_SLEEP);
                    }
                    for (int e = lane; e < a.nseg * ww; e += 32) {
                        const int k = e / ww, w = e - k * ww;
                        const int ly = iy + oy0 + k, x = ixlo - r + w;
                        double v = 0.0;
                        if (ly >= 0 && ly < K && x >= 0 && x < K) {
                            const double *yp = a.out + (int64_t)ly * K + x;
#ifdef LP_SWEEP_CHECK
                            if (yp < a.out || yp >= a.out + g.n || 8 * e >= yslot) {
                                if (atomicCAS((unsigned long long *)g_chk, 0ull, 2ull) == 0ull) {
                                    g_chk[1] = L; g_chk[2] = st; g_chk[3] = e; g_chk[4] = ly; g_chk[5] = x;
                                }
                                asm volatile("exit;");
                            }
#endif
                            v = __ldcg(yp);
                            while (bits(v) == SWEEP_SENTINEL) {
                                __nanosleep(LP_SWEEP_SLEEP);
                                v = ld_poll(yp);
                            }
                        }
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(yb + 8 * e), "d"(v) : "memory");
                    }
                    __syncwarp();
                    mbar_wait(full0 + 8 * slot, (gs / NSTAGE) & 1);
                    // lane = (row q, part p): row q = lane & 7, slots p, p+4, ...
                    const int q = lane & 7, part = lane >> 3;
                    const int shq = __shfl_sync(0xffffffff, sh, q);
                    double acc = 0.0;
                    if (q < nr) {
                        const int ixq = FWD ? t0 + q : K - 1 - t0 - q;
                        const unsigned frow = fb + (unsigned)(q * a.pr_rs + shq) * 8;
                        const unsigned yrow = yb + (unsigned)(ixq - ixlo) * 8;
                        for (int j = part; j < nslot; j += 4) {
#ifdef LP_SWEEP_CHECK
                            if (frow + 8 * j >= fb0 + NSTAGE * fslot || yrow + 8 * s_yofs[j] >= yb + yslot ||
                                yrow < yb) {
                                if (atomicCAS((unsigned long long *)g_chk, 0ull, 3ull) == 0ull) {
                                    g_chk[1] = L; g_chk[2] = st; g_chk[3] = q; g_chk[4] = j; g_chk[5] = s_yofs[j];
                                    g_chk[6] = ixq; g_chk[7] = ixlo;
                                }
                                asm volatile("exit;");
                            }
#endif
                            acc = fma(lds(frow + 8 * j), lds(yrow + 8 * s_yofs[j]), acc);
                        }
                    }
                    acc += __shfl_xor_sync(0xffffffff, acc, 8);
                    acc += __shfl_xor_sync(0xffffffff, acc, 16);
                    __syncwarp();
                    if (lane == 0) v_cons[slot] = gs / NSTAGE + 1;
                    // hand c_t to the group (slots are freed in order: check the last)
                    const int tl1 = t1 - 1;
                    const unsigned long long free_tag = bits(ring_sent(tl1));
                    if (lane == 0)
                        while (bits(v_c[tl1 & (RING - 1)]) != free_tag) __nanosleep(LP_SWEEP_SLEEP);
                    __syncwarp();
                    const double rq = __shfl_sync(0xffffffff, rhs_t, q);
                    if (lane < nr) {
                        v_c[(t0 + lane) & (RING - 1)] = canon(rq - acc);
#ifdef LP_SWEEP_TRACE
                        if (a.trace && t0 + lane == K / 2) a.trace[(size_t)tl * 16 + 8] = gtime();
#endif
                    }
                }
                stage_base += ns;
                continue;
            }
            // The lex-latest line of the producers' stencil in each earlier row of
            // lines: once its value at the frontier x is visible, everything the
            // row needs has almost certainly been produced (per-value sentinel
            // checks remain the guard).
            int dep1, dep2;
            if (FWD) {
                dep1 = (g.d > 1 && iy > 2) ? L - 3 : -1;
                dep2 = (g.d > 2 && iz > 0) ? min(iy + r, K - 1) + K * (iz - 1) : -1;
            } else {
                dep1 = (g.d > 1 && iy < K - 3) ? L + 3 : -1;
                dep2 = (g.d > 2 && iz < K - 1) ? max(iy - r, 0) + K * (iz + 1) : -1;
            }
            double va[CH], vb[CH];
            double ra = 0.0, rb = 0.0;   // rhs of the row, loaded with its factors
            auto load_v = [&](int t, double (&dst)[CH], double &rd, int b0) {
                const int ix = FWD ? t : K - 1 - t;
                const double *row = a.lu + (size_t)(row0 + ix) * g.S + a.lo;
                if (b0 == 0 && t < K) rd = a.rhs[row0 + ix];
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    const int jj = b0 + lane + 32 * j;
                    dst[j] = (t < K && jj < a.nslot) ? __ldcs(row + jj) : 0.0;
                }
            };
            auto process = [&](int t, double (&v)[CH], double rhs_i) {
                const int ix = FWD ? t : K - 1 - t;
                const int64_t i = row0 + ix;
                if (lane < 2) {
                    const int dl = lane == 0 ? dep1 : dep2;
                    if (dl >= 0) {
                        const int fx = FWD ? min(ix + r, K - 1) : max(ix - r, 0);
                        const double *fp = a.out + (int64_t)dl * K + fx;
                        while (bits(ld_poll(fp)) == SWEEP_SENTINEL) __nanosleep(LP_SWEEP_SLEEP);
                    }
                }
                __syncwarp();
                double acc = 0.0;
                for (int b0 = 0; b0 < a.nslot; b0 += 32 * CH) {
                    if (b0 > 0) {
                        double dummy;
                        load_v(t, v, dummy, b0);
                    }
                    double yv[CH];
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        const int jj = b0 + lane + 32 * j;
                        const bool ok = jj < a.nslot && s_ok[jj] &&
                                        (unsigned)(ix + s_ox[jj]) < (unsigned)K;
                        yv[j] = ok ? __ldcg(a.out + i + s_delta[jj]) : 0.0;
                    }
#pragma unroll
                    for (int j = 0; j < CH; ++j) {
                        if (bits(yv[j]) == SWEEP_SENTINEL) {
                            const int jj = b0 + lane + 32 * j;
                            yv[j] = ld_poll(a.out + i + s_delta[jj]);
                            while (bits(yv[j]) == SWEEP_SENTINEL) {
                                __nanosleep(LP_SWEEP_SLEEP);
                                yv[j] = ld_poll(a.out + i + s_delta[jj]);
                            }
                        }
                        acc = fma(v[j], yv[j], acc);
                    }
                }
                __syncwarp();
                acc = warp_sum(acc);
                if (lane == 0) {
                    const int slot = t & (RING - 1);
                    const unsigned long long free_tag = bits(ring_sent(t));
                    while (bits(v_c[slot]) != free_tag) __nanosleep(LP_SWEEP_SLEEP);
                    v_c[slot] = canon(rhs_i - acc);
#ifdef LP_SWEEP_TRACE
                    if (a.trace && t == K / 2) a.trace[(size_t)tl * 16 + 8] = gtime();
#endif
                }
            };
            int t = pw;
            load_v(t, va, ra, 0);
            while (t < K) {
                load_v(t + NP, vb, rb, 0);
                process(t, va, ra);
                t += NP;
                if (t >= K) break;
                load_v(t + NP, va, ra, 0);
                process(t, vb, rb);
                t += NP;
            }
        }
    }
}

// Band arrays, section-major: [n][nq] in-line sections, then [n][gsz] group sections
// (each staged by contiguous TMA bulk copies), in the sweep's step order:
//   [0, nq):   e_1, rd, e_2, .., e_{nq-1}: e_j is the coefficient by which y(row) enters
//              the row j steps later on the same line (fwd: L(ix+j, ix); bwd:
//              U(ix-j, ix) / U(ix-j, ix-j)), 0 beyond r or the line end; rd = fwd 1,
//              bwd 1/U(ix, ix);
//   group section [2 (2r+1)], for line offsets m = 1, 2: the coefficients by which
//              y(line L-/+m, x = ix) enters the rows of line L that are j = 0..2r steps
//              after its arrival step (fwd: rows x-r+j, slot (r-j, -m); bwd: rows
//              x+r-j, slot (j-r, +m)).
__global__ void band_kernel(Geom g, const double *__restrict__ lu, int nq, int gsz,
                            double *__restrict__ blo, double *__restrict__ bup,
                            double *__restrict__ rdg) {
    const int bs = nq + gsz;
    const int64_t total = g.n * bs;
    const int K = g.K, r = g.r;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / bs;
        const int l = (int)(q % bs);
        const int ix = (int)(i % K);
        const int64_t row0 = i - ix;
        const double *row = lu + (size_t)i * g.S;
        double lo = 0.0, up = 0.0;
        size_t o;
        if (l < nq) {
            o = (size_t)i * nq + l;
            if (l == 1) {
                lo = 1.0;
                up = 1.0 / row[g.c];
            } else {
                const int j = l == 0 ? 1 : l;
                if (j <= r && ix + j < K) lo = lu[(size_t)(i + j) * g.S + g.c - j];
                if (j <= r && ix - j >= 0) {
                    const double *rj = lu + (size_t)(i - j) * g.S;
                    up = rj[g.c + j] * (1.0 / rj[g.c]);
                }
            }
        } else {
            const int jj = l - nq;
            o = (size_t)g.n * nq + (size_t)i * gsz + jj;
            const int line = jj / (2 * r + 1) + 1, j = jj % (2 * r + 1);   // line -/+1 or -/+2
            if (g.d > 1 && line <= 2) {
                const int ixf = ix - r + j, ixb = ix + r - j;
                if (ixf >= 0 && ixf < K) lo = lu[(size_t)(row0 + ixf) * g.S + g.c - line * g.W + r - j];
                if (ixb >= 0 && ixb < K) up = lu[(size_t)(row0 + ixb) * g.S + g.c + line * g.W + j - r];
            }
        }
        blo[o] = lo;
        bup[o] = up;
        if (l == 0) rdg[i] = 1.0 / row[g.c];
    }
}

__global__ void fill_sentinel(int64_t n, double *a, double *b) {
    const double s = __longlong_as_double((long long)SWEEP_SENTINEL);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        a[i] = s;
        if (b) b[i] = s;
    }
}

int prefill(int64_t n, double *a, double *b, cudaStream_t st) {
    int64_t blocks = ceil_div(n, 256);
    if (blocks > num_sms() * 16) blocks = num_sms() * 16;
    fill_sentinel<<<(unsigned)blocks, 256, 0, st>>>(n, a, b);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int band_nq(const Geom &g) { return g.r <= 7 ? 8 : 16; }
int band_gsz(const Geom &g) { return g.d > 1 ? (int)round_up(2 * (2 * g.r + 1), 2) : 0; }
int band_stride(const Geom &g) { return band_nq(g) + band_gsz(g); }

#ifndef LP_SWEEP_CLUSTER
#define LP_SWEEP_CLUSTER 8   // measured (cfg 2 sweep pair): 2 -> 2.30, 4 -> 2.22, 8 -> 2.17 ms
#endif

template <bool FWD, int CH, int NQ>
int run_sweep(SweepArgs a, const Geom &g, size_t smem, cudaStream_t st) {
    constexpr int NW = 16;
    auto kern = box_sweep_kernel<FWD, NW, CH, NQ>;
    const void *fn = reinterpret_cast<const void *>(kern);
    // clusters of LP_SWEEP_CLUSTER CTAs (line hand-off through distributed shared
    // memory) when the hand-off buffer exists (K <= 2048) and every CTA can be resident
    int csize = 1, blocks = 0;
    if (LP_SWEEP_CLUSTER > 1 && g.K <= 2048) {
        blocks = resident_cluster_blocks(fn, 32 * NW, smem, LP_SWEEP_CLUSTER);
        if (blocks > 0) csize = LP_SWEEP_CLUSTER;
    }
    if (csize == 1) blocks = resident_blocks(fn, 32 * NW, smem);
    LP_ARG(blocks > 0, "sweep kernel does not fit an SM (%zu bytes of shared memory)", smem);
    a.csize = csize;
    if (csize == 1 && blocks > g.nlines) blocks = g.nlines;
    if (csize > 1) {
        const int need = (g.nlines + csize - 1) / csize * csize;
        if (blocks > need) blocks = need;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csize;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(blocks, 1, 1);
        cfg.blockDim = dim3(32 * NW, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        LP_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    } else {
        kern<<<blocks, 32 * NW, smem, st>>>(a);
    }
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

template <bool FWD, int NQ>
int launch_nq(const SweepArgs &a, const Geom &g, size_t smem, cudaStream_t st) {
    if (a.nslot <= 32 * 8) return run_sweep<FWD, 8, NQ>(a, g, smem, st);
    if (a.nslot <= 32 * 13) return run_sweep<FWD, 13, NQ>(a, g, smem, st);
    return run_sweep<FWD, 16, NQ>(a, g, smem, st);
}

template <bool FWD>
int launch_sweep(lp_ilu *m, const double *rhs, double *out, int *ticket, cudaStream_t st,
                 const double *dotv = nullptr, double *dotpart = nullptr) {
    Geom g = geom_of(m->box);
    if (box_sweep3d_applies(g)) {
        LP_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
        return box_sweep3d(m, FWD, rhs, out, ticket, st);
    }
    LP_ARG(g.r <= 15, "stencil reach %d > 15 is not supported by the sweep kernel", g.r);
    SweepArgs a;
    a.g = g;
    a.lu = m->box.lu;
    a.band = FWD ? m->box.band_lo : m->box.band_up;
    a.rhs = rhs;
    a.out = out;
    a.ticket = ticket;
    const int nq = band_nq(g);
    a.gsz = band_gsz(g);
    a.band_g = a.band + (size_t)g.n * nq;
    // producers: everything except the in-line entries and (d >= 2) lines -/+1, -/+2
    const int excl = g.d > 1 ? 2 * g.W + g.r : g.r;
    a.lo = FWD ? 0 : g.c + excl + 1;
    a.nslot = FWD ? g.c - excl : g.S - (g.c + excl + 1);
    a.trace = nullptr;
    a.dotv = dotv;
    a.dotpart = dotpart;
#ifdef LP_SWEEP_TRACE
    {
        static unsigned long long *tr = nullptr;
        static size_t trn = 0;
        if (trn < (size_t)g.nlines * 16) {
            if (tr) dfree(tr);
            trn = (size_t)g.nlines * 16;
            dalloc(&tr, trn, "sweep trace");
        }
        cudaMemsetAsync(tr, 0, trn * 8, st);
        a.trace = tr;
        g_trace = tr;
        g_trace_n = trn;
    }
#endif
    size_t smem = (size_t)BRING * (nq + a.gsz) * sizeof(double) + (size_t)a.nslot * (sizeof(int) + 4);
    smem = (size_t)round_up((int64_t)smem, 16);
    a.pr_ofs = (unsigned)smem;
    a.nseg = g.d == 2 ? g.r - 2 : 0;
    a.pr_rs = (int)round_up(a.nslot + 1, 2);
    a.pr_ww = (int)round_up(PR + 2 * g.r, 2);
    if (g.d == 2)
        smem += (size_t)NSTAGE * (PR * a.pr_rs + a.nseg * a.pr_ww) * sizeof(double) +
                (size_t)a.nslot * sizeof(int);
    smem = (size_t)round_up((int64_t)smem, 16);
    a.yr_ofs = (unsigned)smem;
    a.csize = 1;
    if (g.K <= 2048) smem += (size_t)g.K * sizeof(double);   // line handoff buffer (clusters)
    smem += 16;
    LP_ARG(smem <= 227 * 1024, "sweep needs %zu bytes of shared memory (reach %d)", smem, g.r);
    LP_CUDA(cudaMemsetAsync(a.ticket, 0, sizeof(int), st));
    return nq == 8 ? launch_nq<FWD, 8>(a, g, smem, st) : launch_nq<FWD, 16>(a, g, smem, st);
}

}  // namespace

int box_build_bands(lp_ilu *m, cudaStream_t st) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    if (box_sweep3d_applies(g)) return box_build_even(m, st);   // the 3-D sweeps read the factors directly
    const int bs = band_stride(g);
    int rc;
    if (!b.band_lo && ((rc = dalloc(&b.band_lo, (size_t)b.n * bs, "band")) ||
                       (rc = dalloc(&b.band_up, (size_t)b.n * bs, "band")) ||
                       (rc = dalloc(&b.diag, (size_t)b.n, "diag"))))
        return rc;
    band_kernel<<<num_sms() * 8, 256, 0, st>>>(g, b.lu, band_nq(g), band_gsz(g), b.band_lo, b.band_up, b.diag);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int box_forward(lp_ilu *m, const double *r, double *y, int *ticket, cudaStream_t st) {
    int rc = prefill(m->n, y, nullptr, st);
    return rc ? rc : launch_sweep<true>(m, r, y, ticket, st);
}

int box_backward(lp_ilu *m, const double *y, double *z, int *ticket, cudaStream_t st) {
    int rc = prefill(m->n, z, nullptr, st);
    return rc ? rc : launch_sweep<false>(m, y, z, ticket, st);
}

// precond_apply: one prefill of both outputs, then the two sweeps.
int box_apply(lp_ilu *m, const double *r, double *z, const SweepScratch &s, cudaStream_t st) {
    int rc = prefill(m->n, s.ytmp, z, st);
    if (!rc) rc = launch_sweep<true>(m, r, s.ytmp, s.tickets, st);
    if (!rc) rc = launch_sweep<false>(m, s.ytmp, z, s.tickets + 1, st);
    return rc;
}

// The line-wavefront kernel can carry r'z in its backward sweep (1-D, 2-D and
// the 3-D boxes it serves); the bandwidth-first 3-D sweeps cannot.
bool box_apply_dot_fused(const lp_ilu *m) { return !box_sweep3d_applies(geom_of(m->box)); }

// precond_apply with rz = r'z fused into the backward sweep: every line's
// serial warp accumulates its part, the parts are summed in double-double in a
// fixed order (sum_lines_dd).  rz: device dd pair.
int box_apply_dot(lp_ilu *m, const double *r, double *z, const SweepScratch &s, double *rz, cudaStream_t st) {
    int rc = prefill(m->n, s.ytmp, z, st);
    if (!rc) rc = launch_sweep<true>(m, r, s.ytmp, s.tickets, st);
    if (!rc) rc = launch_sweep<false>(m, s.ytmp, z, s.tickets + 1, st, r, s.dotpart);
    if (!rc) rc = sum_lines_dd(s.dotpart, geom_of(m->box).nlines, rz, st);
    return rc;
}

}  // namespace lp

extern "C" int lp_debug_sweep_check(long long *host) {
    cudaDeviceSynchronize();
    return cudaMemcpyFromSymbol(host, lp::g_chk, 8 * sizeof(long long)) == cudaSuccess ? 0 : -1;
}

extern "C" int lp_debug_sweep_trace(unsigned long long *host, int64_t n) {
    if (!lp::g_trace) return -1;
    const size_t m = (size_t)n < lp::g_trace_n ? (size_t)n : lp::g_trace_n;
    cudaDeviceSynchronize();
    cudaMemcpy(host, lp::g_trace, m * 8, cudaMemcpyDeviceToHost);
    return (int)m;
}
