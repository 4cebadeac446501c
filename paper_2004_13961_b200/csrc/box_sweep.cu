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

#include "box_geom.cuh"
#include "ilu.cuh"

namespace lp {

unsigned long long *g_trace = nullptr;   // LP_SWEEP_TRACE builds only
size_t g_trace_n = 0;

constexpr unsigned long long SWEEP_SENTINEL = 0xFFF4C0FFEE5EED00ull;   // signalling NaN

namespace {

constexpr int RING = 64;    // rows in flight per line (power of two)
constexpr int BRING = 128;  // band rows staged for the serial warp (power of two)
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
    const double *band;   // [n][bs]: r in-line coefficients, then the 2r+1 of line L-/+1
    const double *rdiag;  // 1/U_tt
    const double *rhs;
    double *out;
    int *ticket;
    int bs;               // band row stride (even)
    int lo, nslot;        // producers' slot range [lo, lo + nslot)
    unsigned long long *trace;   // LP_SWEEP_TRACE builds: per-line timestamps
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <bool FWD, int NW, int CH>
__global__ void __launch_bounds__(32 * NW)
box_sweep_kernel(const __grid_constant__ SweepArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const Geom &g = a.g;
    double *s_band = reinterpret_cast<double *>(dsm);                  // [BRING][bs]
    double *s_rd = s_band + (size_t)BRING * a.bs;                       // [BRING]
    int *s_delta = reinterpret_cast<int *>(s_rd + BRING);               // [nslot]
    signed char *s_ox = reinterpret_cast<signed char *>(s_delta + a.nslot);
    signed char *s_oy = s_ox + a.nslot;
    signed char *s_oz = s_oy + a.nslot;
    unsigned char *s_ok = reinterpret_cast<unsigned char *>(s_oz + a.nslot);
    __shared__ double s_c[RING];
    __shared__ int s_line;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = g.K, r = g.r;
    volatile double *v_c = s_c;
    constexpr int SERIAL = NW - 1;   // highest warp id: favoured by the SMSP arbiter

    for (int j = tid; j < a.nslot; j += blockDim.x) {
        int sx, sy, sz;
        slot_axes(g, a.lo + j, sx, sy, sz);
        s_ox[j] = (signed char)(sx - r);
        s_oy[j] = (signed char)(sy - r);
        s_oz[j] = (signed char)(sz - r);
        s_delta[j] = (sx - r) + K * ((sy - r) + K * (sz - r));
    }

    for (;;) {
        __syncthreads();
        if (tid == 0) s_line = atomicAdd(a.ticket, 1);
        for (int k = tid; k < RING; k += blockDim.x) s_c[k] = ring_sent(k);
        __syncthreads();
        const int tl = s_line;
        if (tl >= g.nlines) return;
        const int L = FWD ? tl : g.nlines - 1 - tl;
        const int iy = g.d > 1 ? L % K : 0, iz = g.d > 2 ? L / K : 0;
        for (int j = tid; j < a.nslot; j += blockDim.x) {
            const int y = iy + s_oy[j], z = iz + s_oz[j];
            s_ok[j] = (g.d < 2 || (y >= 0 && y < K)) && (g.d < 3 || (z >= 0 && z < K));
        }
        const int64_t row0 = (int64_t)L * K;
#ifdef LP_SWEEP_TRACE
        if (tid == 0 && a.trace) a.trace[(size_t)tl * 4] = gtime();
#endif
        __syncthreads();

        if (warp == SERIAL) {
            // ------------------------------------------- serial recurrence
            const bool has_prev = g.d > 1 && (FWD ? iy > 0 : iy < K - 1);
            const double *prev = a.out + (FWD ? row0 - K : row0 + K);   // line L-/+1
            const int LW = g.d > 1 ? 2 * r : r - 1;   // lanes >= LW hold no pending sum
            auto ix_of = [&](int t) { return FWD ? t : K - 1 - t; };
            // band rows of steps [u0, u0+32), contiguous in memory, by ix mod BRING
            auto stage_chunk = [&](int u0) {
                if (u0 < K) {
                    const int u1 = min(u0 + 32, K);
                    const int ixlo = FWD ? u0 : K - u1, ixhi = FWD ? u1 : K - u0;
                    for (int p0 = ixlo; p0 < ixhi;) {
                        const int p1 = min(ixhi, (p0 / BRING + 1) * BRING);
                        const double *src = a.band + (size_t)(row0 + p0) * a.bs;
                        double *dst = s_band + (size_t)(p0 & (BRING - 1)) * a.bs;
                        const int n = (p1 - p0) * a.bs;
                        for (int e = 2 * lane; e < n; e += 64) cp_async16(dst + e, src + e);
                        if (!FWD)
                            for (int e = lane; e < p1 - p0; e += 32)
                                cp_async8(s_rd + ((p0 + e) & (BRING - 1)), a.rdiag + row0 + p0 + e);
                        p0 = p1;
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            // lane k's two coefficients for step t (row t+k):
            //   qi: in-line, multiplies y_{t-1} (lane 0: l1_t)
            //   qg: line L-/+1, multiplies the step's new value y(L-/+1, t -/+ r)
            auto coefs = [&](int t, double &qi, double &qg) {
                const int tk = t + lane;
                qi = 0.0;
                qg = 0.0;
                if (tk < 0 || tk >= K) return;
                const double *b = s_band + (size_t)(ix_of(tk) & (BRING - 1)) * a.bs;
                if (lane < r) qi = b[lane];
                if (g.d > 1 && lane <= 2 * r) qg = b[r + (FWD ? 2 * r - lane : lane)];
            };
            auto xnew_of = [&](int t) { return FWD ? t + r : K - 1 - t - r; };
            auto fetch_new = [&](int t) -> double {
                const int x = xnew_of(t);
                return (has_prev && x >= 0 && x < K) ? ld_poll(prev + x) : 0.0;
            };
            auto ready_new = [&](int t, double v) -> double {
                const int x = xnew_of(t);
                if (!has_prev || x < 0 || x >= K) return 0.0;
                while (bits(v) == SWEEP_SENTINEL) v = ld_poll(prev + x);
                return v;
            };

            stage_chunk(0);
            stage_chunk(32);
            stage_chunk(64);
            asm volatile("cp.async.wait_group 2;" ::: "memory");
            __syncwarp();
            double acc = 0.0, yprev = 0.0;
            double ynext = fetch_new(g.d > 1 ? -r : 0);
            // virtual steps t = -r..-1: values of line L-/+1 at x < r (x > K-1-r)
            if (g.d > 1)
                for (int t = -r; t < 0; ++t) {
                    double qi, qg;
                    coefs(t, qi, qg);
                    const double yn = ready_new(t, ynext);
                    ynext = fetch_new(t + 1);
                    acc = fma(qg, yn, acc);
                    acc = __shfl_down_sync(0xffffffff, acc, 1);
                    if (lane >= LW) acc = 0.0;
                }
            double cn = v_c[0];
            for (int t0 = 0; t0 < K; t0 += 32) {
                stage_chunk(t0 + 96);
                asm volatile("cp.async.wait_group 2;" ::: "memory");
                __syncwarp();
                const int tend = min(t0 + 32, K);
                for (int t = t0; t < tend; ++t) {
                    const int slot = t & (RING - 1);
                    double qi, qg;
                    coefs(t, qi, qg);
                    const double yn = ready_new(t, ynext);
                    ynext = fetch_new(t + 1);
                    const double yb = __shfl_sync(0xffffffff, yprev, 0);
                    acc = fma(qg, yn, acc);
                    if (lane != 0) acc = fma(qi, yb, acc);
                    // c_t from the producers, read one step ahead by all lanes
                    double cc = cn;
                    const unsigned long long sb = bits(ring_sent(t));
#ifdef LP_EXP_NOWAIT
                    if (false) {
#else
                    if (bits(cc) == sb) {
#endif
                        do {
                            cc = v_c[slot];
                        } while (bits(cc) == sb);
                    }
                    double y = fma(-qi, yprev, cc - acc);
                    if (!FWD) y *= s_rd[ix_of(t) & (BRING - 1)];
                    y = canon(y);
                    if (lane == 0) {
                        v_c[slot] = ring_sent(t + RING);
                        __stcg(a.out + row0 + ix_of(t), y);
                    }
#ifdef LP_SWEEP_TRACE
                    if (lane == 0 && a.trace && (t == 0 || t == K / 2 || t == K - 1))
                        a.trace[(size_t)tl * 4 + (t == 0 ? 1 : (t == K - 1 ? 3 : 2))] = gtime();
#endif
                    cn = v_c[(t + 1) & (RING - 1)];
                    yprev = y;
                    acc = __shfl_down_sync(0xffffffff, acc, 1);
                    if (lane >= LW) acc = 0.0;
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        } else {
            // ------------------------------------------------- producers
            constexpr int NP = NW - 1;
            // The lex-latest line of the producers' stencil in each earlier row of
            // lines: once its value at the frontier x is visible, everything the
            // row needs has almost certainly been produced (per-value sentinel
            // checks remain the guard).
            int dep1, dep2;
            if (FWD) {
                dep1 = (g.d > 1 && iy > 1) ? L - 2 : -1;
                dep2 = (g.d > 2 && iz > 0) ? min(iy + r, K - 1) + K * (iz - 1) : -1;
            } else {
                dep1 = (g.d > 1 && iy < K - 2) ? L + 2 : -1;
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
#ifdef LP_EXP_NOPROD
                    dst[j] = 0.0 * jj;
#else
                    dst[j] = (t < K && jj < a.nslot) ? __ldcs(row + jj) : 0.0;
#endif
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
#ifdef LP_EXP_NOPROD
                for (int b0 = 0; b0 < 0; b0 += 32 * CH) {
#else
                for (int b0 = 0; b0 < a.nslot; b0 += 32 * CH) {
#endif
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
                }
            };
            int t = warp;
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

// band[row] = [ in-line: M(row, row-1-q) or M(row, row+1+q), q < r |
//               line -/+1: M(row, slot(ox, -/+1)), ox = -r..r | pad ],  rdiag = 1/U_tt
__global__ void band_kernel(Geom g, const double *__restrict__ lu, int bs, double *__restrict__ blo,
                            double *__restrict__ bup, double *__restrict__ rdg) {
    const int64_t total = g.n * bs;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / bs;
        const int l = (int)(q % bs);
        const double *row = lu + (size_t)i * g.S;
        double lo = 0.0, up = 0.0;
        if (l < g.r) {
            lo = row[g.c - 1 - l];
            up = row[g.c + 1 + l];
        } else if (g.d > 1 && l < 3 * g.r + 1) {
            const int j = l - g.r;   // ox = j - r
            lo = row[g.c - g.W - g.r + j];
            up = row[g.c + g.W - g.r + j];
        }
        blo[q] = lo;
        bup[q] = up;
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
    if (blocks > 148 * 16) blocks = 148 * 16;
    fill_sentinel<<<(unsigned)blocks, 256, 0, st>>>(n, a, b);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int band_stride(const Geom &g) { return (int)round_up(3 * g.r + 1, 2); }

template <bool FWD, int CH>
int run_sweep(const SweepArgs &a, const Geom &g, size_t smem, cudaStream_t st) {
    constexpr int NW = 16;
    static int nblocks = 0;
    static size_t smem_set = 0;
    if (smem_set < smem) {
        LP_CUDA(cudaFuncSetAttribute(box_sweep_kernel<FWD, NW, CH>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 1, dev = 0, nsm = 148;
        LP_CUDA(cudaGetDevice(&dev));
        LP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, box_sweep_kernel<FWD, NW, CH>,
                                                              32 * NW, smem));
        nblocks = occ * nsm;
        smem_set = smem;
    }
    const int blocks = g.nlines < nblocks ? g.nlines : nblocks;
    box_sweep_kernel<FWD, NW, CH><<<blocks, 32 * NW, smem, st>>>(a);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

template <bool FWD>
int launch_sweep(lp_ilu *m, const double *rhs, double *out, cudaStream_t st) {
    Geom g = geom_of(m->box);
    LP_ARG(g.r <= 15, "stencil reach %d > 15 is not supported by the sweep kernel", g.r);
    SweepArgs a;
    a.g = g;
    a.lu = m->box.lu;
    a.band = FWD ? m->box.band_lo : m->box.band_up;
    a.rdiag = m->box.diag;
    a.rhs = rhs;
    a.out = out;
    a.ticket = m->ticket + (FWD ? 0 : 1);
    a.bs = band_stride(g);
    // producers: everything except the in-line entries and (d >= 2) line -/+1
    const int excl = g.d > 1 ? g.W + g.r : g.r;
    a.lo = FWD ? 0 : g.c + excl + 1;
    a.nslot = FWD ? g.c - excl : g.S - (g.c + excl + 1);
    a.trace = nullptr;
#ifdef LP_SWEEP_TRACE
    {
        static unsigned long long *tr = nullptr;
        static size_t trn = 0;
        if (trn < (size_t)g.nlines * 4) {
            if (tr) dfree(tr);
            trn = (size_t)g.nlines * 4;
            dalloc(&tr, trn, "sweep trace");
        }
        cudaMemsetAsync(tr, 0, trn * 8, st);
        a.trace = tr;
        g_trace = tr;
        g_trace_n = trn;
    }
#endif
    const size_t smem = (size_t)BRING * a.bs * sizeof(double) + BRING * sizeof(double) +
                        (size_t)a.nslot * (sizeof(int) + 4) + 16;
    LP_CUDA(cudaMemsetAsync(a.ticket, 0, sizeof(int), st));
    if (a.nslot <= 32 * 8) return run_sweep<FWD, 8>(a, g, smem, st);
    if (a.nslot <= 32 * 13) return run_sweep<FWD, 13>(a, g, smem, st);
    return run_sweep<FWD, 16>(a, g, smem, st);
}

}  // namespace

int box_build_bands(lp_ilu *m, cudaStream_t st) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    const int bs = band_stride(g);
    int rc;
    if (!b.band_lo && ((rc = dalloc(&b.band_lo, (size_t)b.n * bs, "band")) ||
                       (rc = dalloc(&b.band_up, (size_t)b.n * bs, "band")) ||
                       (rc = dalloc(&b.diag, (size_t)b.n, "diag"))))
        return rc;
    band_kernel<<<148 * 8, 256, 0, st>>>(g, b.lu, bs, b.band_lo, b.band_up, b.diag);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int box_forward(lp_ilu *m, const double *r, double *y, cudaStream_t st) {
    int rc = prefill(m->n, y, nullptr, st);
    return rc ? rc : launch_sweep<true>(m, r, y, st);
}

int box_backward(lp_ilu *m, const double *y, double *z, cudaStream_t st) {
    int rc = prefill(m->n, z, nullptr, st);
    return rc ? rc : launch_sweep<false>(m, y, z, st);
}

// precond_apply: one prefill of both outputs, then the two sweeps.
int box_apply(lp_ilu *m, const double *r, double *z, cudaStream_t st) {
    int rc = prefill(m->n, m->ytmp, z, st);
    if (!rc) rc = launch_sweep<true>(m, r, m->ytmp, st);
    if (!rc) rc = launch_sweep<false>(m, m->ytmp, z, st);
    return rc;
}

}  // namespace lp

extern "C" int lp_debug_sweep_trace(unsigned long long *host, int64_t n) {
    if (!lp::g_trace) return -1;
    const size_t m = (size_t)n < lp::g_trace_n ? (size_t)n : lp::g_trace_n;
    cudaDeviceSynchronize();
    cudaMemcpy(host, lp::g_trace, m * 8, cudaMemcpyDeviceToHost);
    return (int)m;
}
