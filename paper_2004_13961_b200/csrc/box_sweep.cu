// ILU(0) forward / backward sweeps in the box layout (forward_sub / backward_sub,
// sparse.py:175-216), as a warp-specialised, fence-free line wavefront.
//
// A CTA owns one x-line at a time (lines handed out in sweep order by an
// atomic ticket, so a CTA only ever waits on lines owned by running CTAs).
// Per line:
//  * producer warps (all but the serial warp) take rows round-robin.  Each keeps the next
//    row's off-line factor entries in flight (register double buffer), gathers
//    the solution values those entries multiply and reduces
//    c_i = rhs_i - sum L_is y_col(s) into a shared ring;
//  * the serial warp runs the in-line recurrence
//        y_i = c_i - sum_{q=1..r} L_{i,i-q} y_{i-q}
//    "right-looking": lane q carries the partial sum of row i+q, so a row
//    costs one broadcast, one lane shift and one FMA per lane.  The in-line
//    band values are staged from a compact band array into a shared ring by
//    cp.async (register prefetch queues get their registers reused as
//    temporaries by the compiler, which serialises every step on the load).
//
// Synchronisation carries no fences at all: every value is its own flag.
// The output vector is pre-filled with a NaN sentinel; a consumer spins on the
// 8-byte value it needs (aligned 64-bit accesses are single-copy atomic, and
// the loads/stores are .cg, i.e. coherent at L2) until it is no longer the
// sentinel.  The same trick, with per-step sentinels, carries the shared ring.
// Computed NaNs are canonicalised so they can never alias a sentinel.  The
// backward sweep is the mirror image (rows and lines in reverse, division by
// the diagonal).
#include <math.h>

#include "box_geom.cuh"
#include "ilu.cuh"

namespace lp {

unsigned long long *g_trace = nullptr;   // LP_SWEEP_TRACE builds only
size_t g_trace_n = 0;

constexpr unsigned long long SWEEP_SENTINEL = 0xFFF4C0FFEE5EED00ull;   // signalling NaN

namespace {

constexpr int RING = 64;   // rows in flight per line (power of two)
constexpr int BRING = 128;  // band rows staged for the serial warp (power of two)
constexpr unsigned long long RING_SENT = 0xFFF5000000000000ull;

#ifndef LP_SWEEP_SLEEP
#define LP_SWEEP_SLEEP 20
#endif
#if LP_SWEEP_SLEEP > 0
#define LP_BACKOFF() __nanosleep(LP_SWEEP_SLEEP)
#else
#define LP_BACKOFF() do {} while (0)
#endif

__device__ __forceinline__ unsigned long long bits(double v) {
    return (unsigned long long)__double_as_longlong(v);
}

__device__ __forceinline__ double canon(double v) {
    return isnan(v) ? __longlong_as_double(0x7FF8000000000000ll) : v;
}

// Relaxed gpu-scope load that the compiler may neither cache nor elide
// (a plain .cg load in a side-effect-free spin loop can legally be removed).
__device__ __forceinline__ double ld_poll(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

#ifndef LP_SWEEP_PUBMODE
#define LP_SWEEP_PUBMODE 2
#endif
// Publish a solution value to other SMs.  A plain .cg store can linger in the
// SM's write path for microseconds; an L2-performed reduction is visible as
// soon as it reaches L2.  The slot holds the sentinel, so xor-ing in
// (sentinel ^ value) leaves exactly the value.
__device__ __forceinline__ void publish(double *p, double y) {
#if LP_SWEEP_PUBMODE == 0
    __stcg(p, y);
#elif LP_SWEEP_PUBMODE == 1
    atomicExch(reinterpret_cast<unsigned long long *>(p), bits(y));
#elif LP_SWEEP_PUBMODE == 2
    const unsigned long long x = bits(y) ^ SWEEP_SENTINEL;
    asm volatile("red.relaxed.gpu.global.xor.b64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
#else
    asm volatile("st.release.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(y) : "memory");
#endif
}

__device__ __forceinline__ double ring_sent(int t) {
    return __longlong_as_double((long long)(RING_SENT | (unsigned)t));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    return v;
}

struct SweepArgs {
    Geom g;
    const double *lu, *band, *diag, *rhs;
    double *out;
    int *ticket;
    int lo, nslot;   // off-line slot range [lo, lo + nslot)
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
    int *s_delta = reinterpret_cast<int *>(dsm);
    signed char *s_ox = reinterpret_cast<signed char *>(s_delta + a.nslot);
    signed char *s_oy = s_ox + a.nslot;
    signed char *s_oz = s_oy + a.nslot;
    unsigned char *s_ok = reinterpret_cast<unsigned char *>(s_oz + a.nslot);
    __shared__ double s_c[RING];
    __shared__ __align__(16) double s_band[BRING * 30];   // serial warp's band ring
    __shared__ double s_rd[BRING];                         // 1/U_tt ring (backward)
    __shared__ int s_line;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = g.K, r = g.r;
    volatile double *v_c = s_c;

    for (int j = tid; j < a.nslot; j += blockDim.x) {
        int sx, sy, sz;
        slot_axes(g, a.lo + j, sx, sy, sz);
        s_ox[j] = (signed char)(sx - g.r);
        s_oy[j] = (signed char)(sy - g.r);
        s_oz[j] = (signed char)(sz - g.r);
        s_delta[j] = (sx - g.r) + K * ((sy - g.r) + K * (sz - g.r));
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
        // The lex-latest line of the stencil in each earlier plane-row: once its
        // value at the frontier x is visible, the row's whole stencil has almost
        // certainly been produced (per-value sentinel checks remain the guard).
        int dep1, dep2;
        if (FWD) {
            dep1 = (g.d > 1 && iy > 0) ? L - 1 : -1;
            dep2 = (g.d > 2 && iz > 0) ? min(iy + r, K - 1) + K * (iz - 1) : -1;
        } else {
            dep1 = (g.d > 1 && iy < K - 1) ? L + 1 : -1;
            dep2 = (g.d > 2 && iz < K - 1) ? max(iy - r, 0) + K * (iz + 1) : -1;
        }
#ifdef LP_SWEEP_TRACE
        if (tid == 0 && a.trace) a.trace[(size_t)tl * 4] = gtime();
#endif
        __syncthreads();

        // The serial warp is the highest-numbered one: the SMSP arbiter issues
        // highest-warp-id first, so it wins every slot it is eligible for.
#ifndef LP_SWEEP_SERIAL_WARP
#define LP_SWEEP_SERIAL_WARP (NW - 1)
#endif
        if (warp == LP_SWEEP_SERIAL_WARP) {
            // ------------------------------------------- serial recurrence
            // Lane 0 carries the scalar chain y_t = (c_t - A_t) - l1_t y_{t-1}
            // (one FMA per row on the critical path; backward also scales by
            // 1/U_tt).  Lane k >= 1 holds A_{t+k} = sum_{q>=2} L_{t+k,t+k-q} y_{t+k-q}
            // and adds y_{t-1} one step after it is produced; a lane shift then
            // hands A_{t+1} to lane 0.  Lane k's coefficient for step t is
            // band[row(t+k)][k] (lane 0: l1_t).  The band rows are staged into a
            // shared ring by cp.async, two 32-row chunks ahead.
            // Band rows live in the ring by memory row (ix mod BRING), r doubles
            // each; 1/U_tt in a separate ring.  A chunk = 32 steps = 32 rows,
            // contiguous in memory, copied with 16-byte cp.async when 16-byte
            // aligned (r even), else 8-byte.
            const bool vec16 = (r % 2) == 0;
            auto stage_chunk = [&](int u0) {
                if (u0 < K) {
                    const int u1 = min(u0 + 32, K);
                    const int ixlo = FWD ? u0 : K - u1, ixhi = FWD ? u1 : K - u0;   // [ixlo, ixhi)
                    // split at the ring wrap so each piece is contiguous in smem
                    for (int p0 = ixlo; p0 < ixhi;) {
                        const int p1 = min(ixhi, (p0 / BRING + 1) * BRING);
                        const double *src = a.band + (size_t)(row0 + p0) * r;
                        double *dst = s_band + (size_t)(p0 & (BRING - 1)) * r;
                        const int n = (p1 - p0) * r;
                        if (vec16) {
                            for (int e = 2 * lane; e < n; e += 64) {
                                const unsigned d = (unsigned)__cvta_generic_to_shared(dst + e);
                                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                                             "l"(src + e) : "memory");
                            }
                        } else {
                            for (int e = lane; e < n; e += 32) {
                                const unsigned d = (unsigned)__cvta_generic_to_shared(dst + e);
                                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d),
                                             "l"(src + e) : "memory");
                            }
                        }
                        if (!FWD)
                            for (int e = lane; e < p1 - p0; e += 32) {
                                const unsigned d = (unsigned)__cvta_generic_to_shared(
                                    s_rd + ((p0 + e) & (BRING - 1)));
                                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d),
                                             "l"(a.diag + row0 + p0 + e) : "memory");
                            }
                        p0 = p1;
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            stage_chunk(0);
            stage_chunk(32);
            double acc = 0.0, yprev = 0.0;
            // The next step's c is read one step ahead by all lanes (a uniform,
            // non-divergent poll); a divergent single-lane spin costs ~280 cycles.
            double cn = v_c[0];
            for (int t0 = 0; t0 < K; t0 += 32) {
                stage_chunk(t0 + 64);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                __syncwarp();
                const int tend = min(t0 + 32, K);
                for (int t = t0; t < tend; ++t) {
                    const int slot = t & (RING - 1);
                    const int ixq = FWD ? t + lane : K - 1 - t - lane;
                    const double qv = (lane < r && t + lane < K)
                                          ? s_band[(ixq & (BRING - 1)) * r + lane] : 0.0;
                    const double yb = __shfl_sync(0xffffffff, yprev, 0);
                    if (lane != 0) acc = fma(qv, yb, acc);
                    double cc = cn;
                    const unsigned long long sb = bits(ring_sent(t));
                    if (bits(cc) == sb) {
                        do {
#ifdef LP_SWEEP_SERIAL_SLEEP
                            __nanosleep(LP_SWEEP_SERIAL_SLEEP);
#endif
                            cc = v_c[slot];
                        } while (bits(cc) == sb);
                    }
                    double y = fma(-qv, yprev, cc - acc);
                    if (!FWD) y *= s_rd[(K - 1 - t) & (BRING - 1)];
                    y = canon(y);
                    if (lane == 0) {
                        v_c[slot] = ring_sent(t + RING);
                        publish(a.out + row0 + (FWD ? t : K - 1 - t), y);
                    }
#ifdef LP_SWEEP_TRACE
                    if (lane == 0 && a.trace && (t == 0 || t == K / 2 || t == K - 1))
                        a.trace[(size_t)tl * 4 + (t == 0 ? 1 : (t == K - 1 ? 3 : 2))] = gtime();
#endif
#ifdef LP_SWEEP_TRACE
                    if (lane == 0 && a.trace && (tl == g.nlines / 2 - 1 || tl == g.nlines / 2))
                        a.trace[(size_t)g.nlines * 4 + (size_t)(tl == g.nlines / 2 - 1 ? 0 : 1) * K * 6 +
                                (size_t)t * 6 + 3] = gtime();
#endif
                    cn = v_c[(t + 1) & (RING - 1)];
                    yprev = y;
                    acc = __shfl_down_sync(0xffffffff, acc, 1);
                    if (lane >= r - 1) acc = 0.0;
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        } else {
            // ------------------------------------------------- producers
            // Two register buffers alternate so the next row's factor loads are
            // always in flight while the current row gathers and reduces.
            constexpr int NP = NW - 1;
            double va[CH], vb[CH];
            double ra = 0.0, rb = 0.0;   // rhs of the row, loaded with its factors
            auto load_v = [&](int t, double (&dst)[CH], int b0) {
                const int ix = FWD ? t : K - 1 - t;
                const double *row = a.lu + (size_t)(row0 + ix) * g.S + a.lo;
                if (b0 == 0 && t < K) (&dst == &va ? ra : rb) = a.rhs[row0 + ix];
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    const int jj = b0 + lane + 32 * j;
                    dst[j] = (t < K && jj < a.nslot) ? __ldcs(row + jj) : 0.0;
                }
            };
            auto process = [&](int t, double (&v)[CH], double rhs_i) {
                const int ix = FWD ? t : K - 1 - t;
                const int64_t i = row0 + ix;
                double acc = 0.0;
#ifdef LP_SWEEP_TRACE
                int npoll = 0, lastjj = -1;
                unsigned long long *rt = nullptr;
                if (a.trace && (tl == g.nlines / 2 - 1 || tl == g.nlines / 2))
                    rt = a.trace + (size_t)g.nlines * 4 + (size_t)(tl == g.nlines / 2 - 1 ? 0 : 1) * K * 6 + (size_t)t * 6;
                if (rt && lane == 0) rt[0] = gtime();
#endif
                if (lane < 2) {
                    const int dl = lane == 0 ? dep1 : dep2;
                    if (dl >= 0) {
                        const int fx = FWD ? min(ix + r, K - 1) : max(ix - r, 0);
                        const double *fp = a.out + (int64_t)dl * K + fx;
                        while (bits(ld_poll(fp)) == SWEEP_SENTINEL) LP_BACKOFF();
                    }
                }
                __syncwarp();
#ifdef LP_SWEEP_TRACE
                if (rt && lane == 0) rt[4] = gtime();
#endif
#ifdef LP_SWEEP_SERIAL_ONLY
                for (int b0 = 0; b0 < 0; b0 += 32 * CH) {
#else
                for (int b0 = 0; b0 < a.nslot; b0 += 32 * CH) {
#endif
                    if (b0 > 0) load_v(t, v, b0);
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
                        // values not yet produced by their (earlier) lines: re-poll
                        if (bits(yv[j]) == SWEEP_SENTINEL) {
                            const int jj = b0 + lane + 32 * j;
                            yv[j] = ld_poll(a.out + i + s_delta[jj]);
                            while (bits(yv[j]) == SWEEP_SENTINEL) {
                                LP_BACKOFF();
                                yv[j] = ld_poll(a.out + i + s_delta[jj]);
#ifdef LP_SWEEP_TRACE
                                ++npoll;
                                lastjj = jj;
#endif
                            }
                        }
                        acc = fma(v[j], yv[j], acc);
                    }
                }
#ifdef LP_SWEEP_TRACE
                {
                    unsigned long long tg = gtime();
                    for (int o = 16; o; o >>= 1) {
                        tg = max(tg, (unsigned long long)__shfl_xor_sync(0xffffffff, (long long)tg, o));
                        npoll += __shfl_xor_sync(0xffffffff, npoll, o);
                        lastjj = max(lastjj, __shfl_xor_sync(0xffffffff, lastjj, o));
                    }
                    if (rt && lane == 0) {
                        rt[1] = tg;

                    }
                }
#endif
                acc = warp_sum(acc);
                if (lane == 0) {
                    const int slot = t & (RING - 1);
                    const unsigned long long free_tag = bits(ring_sent(t));
#ifdef LP_SWEEP_TRACE
                    int ringspins = 0;
#endif
                    while (bits(v_c[slot]) != free_tag) {
#ifdef LP_SWEEP_TRACE
                        ++ringspins;
#endif
#ifndef LP_SWEEP_RINGSPIN
                        LP_BACKOFF();
#endif
                    }
#ifdef LP_SWEEP_TRACE
                    if (rt) rt[5] = (unsigned long long)ringspins;
#endif
#ifdef LP_SWEEP_NORHS
                    v_c[slot] = canon(-acc);
#else
                    v_c[slot] = canon(rhs_i - acc);
#endif
#ifdef LP_SWEEP_TRACE
                    if (rt) rt[2] = gtime();
#endif
                }
            };
            int t = warp < LP_SWEEP_SERIAL_WARP ? warp : warp - 1;
            load_v(t, va, 0);
            while (t < K) {
#ifndef LP_SWEEP_NOPREFETCH
                load_v(t + NP, vb, 0);
#endif
                process(t, va, ra);
                t += NP;
                if (t >= K) break;
#ifndef LP_SWEEP_NOPREFETCH
                load_v(t + NP, va, 0);
#endif
                process(t, vb, rb);
                t += NP;
            }
        }
    }
}

__global__ void band_kernel(Geom g, const double *__restrict__ lu, double *__restrict__ blo,
                            double *__restrict__ bup, double *__restrict__ dg) {
    const int64_t total = g.n * g.r;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / g.r;
        const int l = (int)(q % g.r);
        const double *row = lu + (size_t)i * g.S;
        blo[q] = row[g.c - 1 - l];
        bup[q] = row[g.c + 1 + l];
        if (l == 0) dg[i] = 1.0 / row[g.c];
    }
    if (g.r == 0)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
             i += (int64_t)gridDim.x * blockDim.x)
            dg[i] = 1.0 / lu[(size_t)i * g.S + g.c];
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

template <bool FWD, int CH>
int run_sweep(const SweepArgs &a, const Geom &g, size_t smem, cudaStream_t st);

template <bool FWD>
int launch_sweep(lp_ilu *m, const double *rhs, double *out, cudaStream_t st) {
    Geom g = geom_of(m->box);
    LP_ARG(g.r <= 30, "stencil reach %d > 30 is not supported by the sweep kernel", g.r);
    SweepArgs a;
    a.g = g;
    a.lu = m->box.lu;
    a.band = FWD ? m->box.band_lo : m->box.band_up;
    a.diag = m->box.diag;
    a.rhs = rhs;
    a.out = out;
    a.ticket = m->ticket + (FWD ? 0 : 1);
    a.lo = FWD ? 0 : g.c + g.r + 1;
    a.nslot = FWD ? g.c - g.r : g.S - (g.c + g.r + 1);
    a.trace = nullptr;
#ifdef LP_SWEEP_TRACE
    {
        static unsigned long long *tr = nullptr;
        static size_t trn = 0;
        if (trn < (size_t)g.nlines * 4 + (size_t)12 * g.K) {
            if (tr) dfree(tr);
            trn = (size_t)g.nlines * 4 + (size_t)12 * g.K;
            dalloc(&tr, trn, "sweep trace");
        }
        cudaMemsetAsync(tr, 0, trn * 8, st);
        a.trace = tr;
        g_trace = tr;
        g_trace_n = trn;
    }
#endif
    const size_t smem = (size_t)a.nslot * (sizeof(int) + 4) + 16;
    LP_CUDA(cudaMemsetAsync(a.ticket, 0, sizeof(int), st));
    if (a.nslot <= 32 * 8) return run_sweep<FWD, 8>(a, g, smem, st);
    if (a.nslot <= 32 * 13) return run_sweep<FWD, 13>(a, g, smem, st);
    return run_sweep<FWD, 16>(a, g, smem, st);
}

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

}  // namespace

int box_build_bands(lp_ilu *m, cudaStream_t st) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    int rc;
    if (!b.band_lo && ((rc = dalloc(&b.band_lo, (size_t)b.n * g.r, "band")) ||
                       (rc = dalloc(&b.band_up, (size_t)b.n * g.r, "band")) ||
                       (rc = dalloc(&b.diag, (size_t)b.n, "diag"))))
        return rc;
    band_kernel<<<148 * 8, 256, 0, st>>>(g, b.lu, b.band_lo, b.band_up, b.diag);
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
