// Parity-split fp64 line transforms on DMMA.  See line_transform.cuh.
#include "line_transform.cuh"

namespace lp {

namespace {

constexpr int BM = LT_BM, BN = LT_BN, BK = LT_BK;
constexpr int LDS = BK + 4;          // smem row stride (doubles): conflict-free fragment loads
constexpr int THREADS = 256;         // 8 warps: 2 along M (32 rows) x 4 along N (16 cols)
constexpr int TILE_A = BM * LDS;     // doubles per A part
constexpr int TILE_B = BN * LDS;
constexpr int STAGE = 2 * TILE_A + 2 * TILE_B;
constexpr size_t SMEM_BYTES = 2 * STAGE * sizeof(double);

__device__ __forceinline__ void dmma_16x8x8(double (&c)[4], const double (&a)[4],
                                            const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

struct Prefetch {
    double2 a[2][2];     // [part][i]
    double b[8];         // UNFOLD: 8 raw values; FOLD: 4 (s, d) pairs
};

__device__ __forceinline__ void load_tile(Prefetch &pf, const LtArgs &a, const LtTerm &t,
                                          int m0, int n0, int k0, int tid) {
    // A: 2 parts x 64 rows x 16 cols -> 2 double2 per part per thread
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int idx = tid + i * THREADS;
        const int r = idx >> 3, c2 = idx & 7;
        const size_t off = (size_t)(m0 + r) * a.lda + k0 + 2 * c2;
        pf.a[0][i] = __ldg(reinterpret_cast<const double2 *>(t.A0 + off));
        pf.a[1][i] = __ldg(reinterpret_cast<const double2 *>(t.A1 + off));
    }
    if (a.mode == 0) {
        // UNFOLD: In[b][2k0 .. 2k0+32) raw, split by parity when stored
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int idx = tid + i * THREADS;
            const int r = idx >> 5, c = idx & 31;
            const int b = n0 + r, k = 2 * k0 + c;
            pf.b[i] = (b < a.B && k < a.nk) ? __ldg(t.in + (size_t)b * a.nk + k) : 0.0;
        }
    } else {
        // FOLD: s/d of the node pairs (jh, P-1-jh), jh in [k0, k0+16)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * THREADS;
            const int r = idx >> 4, c = idx & 15;
            const int b = n0 + r, jh = k0 + c;
            double lo = 0.0, hi = 0.0;
            if (b < a.B && jh < a.Hm) {
                const double *row = t.in + (size_t)b * a.P;
                lo = __ldg(row + jh);
                hi = __ldg(row + (a.P - 1 - jh));
            }
            pf.b[2 * i] = lo + hi;
            pf.b[2 * i + 1] = lo - hi;
        }
    }
}

__device__ __forceinline__ void store_tile(const Prefetch &pf, double *stage, int mode, int tid) {
    double *As = stage, *Bs = stage + 2 * TILE_A;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int idx = tid + i * THREADS;
        const int r = idx >> 3, c2 = idx & 7;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            double *dst = As + p * TILE_A + r * LDS + 2 * c2;
            dst[0] = pf.a[p][i].x;
            dst[1] = pf.a[p][i].y;
        }
    }
    if (mode == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int idx = tid + i * THREADS;
            const int r = idx >> 5, c = idx & 31;
            Bs[(c & 1) * TILE_B + r * LDS + (c >> 1)] = pf.b[i];
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * THREADS;
            const int r = idx >> 4, c = idx & 15;
            Bs[r * LDS + c] = pf.b[2 * i];
            Bs[TILE_B + r * LDS + c] = pf.b[2 * i + 1];
        }
    }
}

// MINB = 2 caps registers at 128 (a few spilled) so two CTAs share an SM:
// measured on B200, cfg 5 matvec 69.1 -> 52.7 ms (50 -> 66 % of DGEMM peak), cfg 3
// 4.57 -> 3.61 ms; grids smaller than two waves keep the 1-CTA form (cfg 2: 0.118 vs
// 0.139 ms).
template <int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
line_transform_kernel(const __grid_constant__ LtArgs a) {
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tq = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
    const LtOut &o = a.outs[blockIdx.z];

    const int nkt = (a.mode == 0 ? (a.lda) : (a.lda)) / BK;   // k-tiles per term
    const int ntiles = nkt * o.nterms;

    double acc[2][2][2][4];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[p][i][j][v] = 0.0;
    double midacc = 0.0;   // UNFOLD middle node (x = 0), lines n0 + tid, tid < BN
    const bool do_mid = (a.mode == 0) && (a.mid >= 0) && (blockIdx.y == 0) && (tid < BN);

    Prefetch pf;
    load_tile(pf, a, o.term[0], m0, n0, 0, tid);
    store_tile(pf, smem, a.mode, tid);
    __syncthreads();

    for (int t = 0; t < ntiles; ++t) {
        const int term = t / nkt, kt = t - term * nkt;
        double *cur = smem + (t & 1) * STAGE;
        if (t + 1 < ntiles) {
            const int nterm = (t + 1) / nkt, nkt1 = (t + 1) - nterm * nkt;
            load_tile(pf, a, o.term[nterm], m0, n0, nkt1 * BK, tid);
        }
        const int ps = o.term[term].ps;
        const double *As0 = cur, *As1 = cur + TILE_A;
        const double *Bsym = cur + 2 * TILE_A + ps * TILE_B;
        const double *Banti = cur + 2 * TILE_A + (1 - ps) * TILE_B;
#pragma unroll
        for (int ks = 0; ks < BK; ks += 8) {
            double af[2][2][4], bf[2][2][2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int r = wm * 32 + mt * 16 + g;
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const double *A = p ? As1 : As0;
                    af[p][mt][0] = A[r * LDS + ks + tq];
                    af[p][mt][1] = A[(r + 8) * LDS + ks + tq];
                    af[p][mt][2] = A[r * LDS + ks + tq + 4];
                    af[p][mt][3] = A[(r + 8) * LDS + ks + tq + 4];
                }
            }
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int c = wn * 16 + nt * 8 + g;
                bf[0][nt][0] = Bsym[c * LDS + ks + tq];
                bf[0][nt][1] = Bsym[c * LDS + ks + tq + 4];
                bf[1][nt][0] = Banti[c * LDS + ks + tq];
                bf[1][nt][1] = Banti[c * LDS + ks + tq + 4];
            }
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) dmma_16x8x8(acc[p][mt][nt], af[p][mt], bf[p][nt]);
        }
        if (do_mid) {
            const double *um = o.term[term].mid0 + kt * BK;
            const double *brow = Bsym + tid * LDS;
#pragma unroll
            for (int c = 0; c < BK; ++c) midacc = fma(__ldg(um + c), brow[c], midacc);
        }
        if (t + 1 < ntiles) {
            store_tile(pf, smem + ((t + 1) & 1) * STAGE, a.mode, tid);
        }
        __syncthreads();
    }

    // ---------------------------------------------------------------- epilogue
    if (a.mode == 1 && a.mid >= 0) {
        // middle node rank-1 update: acc_p[kk][b] += Tmid_p[kk] * In[b][mid]
        for (int term = 0; term < o.nterms; ++term) {
            const LtTerm &tr = o.term[term];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int v1 = 0; v1 < 2; ++v1) {
                    const int b = n0 + wn * 16 + nt * 8 + 2 * tq + v1;
                    const double xm = (b < a.B) ? __ldg(tr.in + (size_t)b * a.P + a.mid) : 0.0;
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int v0 = 0; v0 < 2; ++v0) {
                            const int kk = m0 + wm * 32 + mt * 16 + g + 8 * v0;
                            acc[0][mt][nt][2 * v0 + v1] =
                                fma(__ldg(tr.mid0 + kk), xm, acc[0][mt][nt][2 * v0 + v1]);
                            acc[1][mt][nt][2 * v0 + v1] =
                                fma(__ldg(tr.mid1 + kk), xm, acc[1][mt][nt][2 * v0 + v1]);
                        }
                }
        }
    }
    double pw = 0.0;   // this thread's part of the fused dot (FOLD, a.dotv)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int v0 = 0; v0 < 2; ++v0) {
            const int row = m0 + wm * 32 + mt * 16 + g + 8 * v0;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int v1 = 0; v1 < 2; ++v1) {
                    const int b = n0 + wn * 16 + nt * 8 + 2 * tq + v1;
                    if (b >= a.B) continue;
                    const double x0 = acc[0][mt][nt][2 * v0 + v1];
                    const double x1 = acc[1][mt][nt][2 * v0 + v1];
                    if (a.mode == 0) {
                        if (row >= a.Hm) continue;
                        const size_t lo = (size_t)row * a.B + b;
                        const size_t hi = (size_t)(a.P - 1 - row) * a.B + b;
                        double vlo = x0 + x1, vhi = x0 - x1;
                        if (o.grid) {
                            vlo *= __ldg(o.grid + lo);
                            vhi *= __ldg(o.grid + hi);
                        }
                        o.out[lo] = vlo;
                        o.out[hi] = vhi;
                    } else {
                        const int k0 = 2 * row;
                        if (k0 < a.nk) o.out[(size_t)k0 * a.B + b] = x0;
                        if (k0 + 1 < a.nk) o.out[(size_t)(k0 + 1) * a.B + b] = x1;
                        if (a.dotv) {
                            if (k0 < a.nk) pw = fma(x0, __ldg(a.dotv + (size_t)k0 * a.B + b), pw);
                            if (k0 + 1 < a.nk) pw = fma(x1, __ldg(a.dotv + (size_t)(k0 + 1) * a.B + b), pw);
                        }
                    }
                }
        }
    if (do_mid) {
        const int b = n0 + tid;
        if (b < a.B) {
            const size_t idx = (size_t)a.mid * a.B + b;
            o.out[idx] = o.grid ? midacc * __ldg(o.grid + idx) : midacc;
        }
    }
    if (a.dotv) {
        // the CTA's sum in a fixed order: xor butterfly per warp, the warps in order
#pragma unroll
        for (int s = 16; s; s >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, s);
        __syncthreads();   // the tile buffers are free
        if (lane == 0) smem[warp] = pw;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
#pragma unroll
            for (int w8 = 0; w8 < THREADS / 32; ++w8) t += smem[w8];
            a.dotpart[blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z)] = t;
        }
    }
}

// Fill the parity-split forms of a P x nk table T (row-major, device).
__global__ void fill_table_forms(LineTable t, const double *__restrict__ T) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nu = (int64_t)t.u_rows * t.u_ld;
    const int64_t nf = (int64_t)t.f_rows * t.f_ld;
    if (i < nu) {
        const int jh = (int)(i / t.u_ld), kk = (int)(i % t.u_ld);
        const int ks = 2 * kk + t.ps, ka = 2 * kk + 1 - t.ps;
        const bool rowok = jh < t.Hm;
        t.u_sym[i] = (rowok && ks < t.nk) ? T[(size_t)jh * t.nk + ks] : 0.0;
        t.u_anti[i] = (rowok && ka < t.nk) ? T[(size_t)jh * t.nk + ka] : 0.0;
    }
    if (i < nf) {
        const int kk = (int)(i / t.f_ld), jh = (int)(i % t.f_ld);
        const int ke = 2 * kk, ko = 2 * kk + 1;
        const bool colok = jh < t.Hm;
        t.f_even[i] = (colok && ke < t.nk) ? T[(size_t)jh * t.nk + ke] : 0.0;
        t.f_odd[i] = (colok && ko < t.nk) ? T[(size_t)jh * t.nk + ko] : 0.0;
    }
    const int mid = (t.P & 1) ? t.P / 2 : -1;
    if (i < t.u_ld) {
        const int ks = 2 * (int)i + t.ps;
        t.u_mid[i] = (mid >= 0 && ks < t.nk) ? T[(size_t)mid * t.nk + ks] : 0.0;
    }
    if (i < t.f_rows) {
        const int ke = 2 * (int)i, ko = ke + 1;
        t.f_mid_e[i] = (mid >= 0 && ke < t.nk) ? T[(size_t)mid * t.nk + ke] : 0.0;
        t.f_mid_o[i] = (mid >= 0 && ko < t.nk) ? T[(size_t)mid * t.nk + ko] : 0.0;
    }
}

}  // namespace

int line_table_build(LineTable &t, const double *Tdev, int P, int nk, int ps,
                     cudaStream_t st) {
    t.P = P;
    t.nk = nk;
    t.ps = ps;
    t.Hm = P / 2;
    t.KE = (nk + 1) / 2;
    t.KO = nk / 2;
    const int kh = t.KE > t.KO ? t.KE : t.KO;
    t.u_rows = (int)round_up(t.Hm > 0 ? t.Hm : 1, BM);
    t.u_ld = (int)round_up(kh, BK);
    t.f_rows = (int)round_up(kh, BM);
    t.f_ld = (int)round_up(t.Hm > 0 ? t.Hm : 1, BK);
    const size_t nu = (size_t)t.u_rows * t.u_ld, nf = (size_t)t.f_rows * t.f_ld;
    int rc;
    if ((rc = dalloc(&t.u_sym, nu, "table")) || (rc = dalloc(&t.u_anti, nu, "table")) ||
        (rc = dalloc(&t.f_even, nf, "table")) || (rc = dalloc(&t.f_odd, nf, "table")) ||
        (rc = dalloc(&t.u_mid, t.u_ld, "table")) || (rc = dalloc(&t.f_mid_e, t.f_rows, "table")) ||
        (rc = dalloc(&t.f_mid_o, t.f_rows, "table")))
        return rc;
    const size_t n = nu > nf ? nu : nf;
    fill_table_forms<<<(unsigned)ceil_div((int64_t)n, 256), 256, 0, st>>>(t, Tdev);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

void line_table_free(LineTable &t) {
    double **ps[] = {&t.u_sym, &t.u_anti, &t.u_mid, &t.f_even, &t.f_odd, &t.f_mid_e, &t.f_mid_o};
    for (double **p : ps) {
        if (*p) dfree(*p);
        *p = nullptr;
    }
}

LtArgs lt_unfold(const LineTable &s, int B) {
    LtArgs a{};
    a.mode = 0;
    a.P = s.P;
    a.nk = s.nk;
    a.B = B;
    a.Hm = s.Hm;
    a.mid = (s.P & 1) ? s.P / 2 : -1;
    a.lda = s.u_ld;
    a.Mdim = s.u_rows;
    a.Kdim = s.u_ld;
    return a;
}

LtArgs lt_fold(const LineTable &s, int B) {
    LtArgs a{};
    a.mode = 1;
    a.P = s.P;
    a.nk = s.nk;
    a.B = B;
    a.Hm = s.Hm;
    a.mid = (s.P & 1) ? s.P / 2 : -1;
    a.lda = s.f_ld;
    a.Mdim = s.f_rows;
    a.Kdim = s.f_ld;
    return a;
}

void lt_add_term(LtArgs &a, int oi, const LineTable &t, const double *in) {
    LtOut &o = a.outs[oi];
    LtTerm &tr = o.term[o.nterms++];
    if (a.mode == 0) {
        tr.A0 = t.u_sym;
        tr.A1 = t.u_anti;
        tr.mid0 = t.u_mid;
        tr.mid1 = nullptr;
    } else {
        tr.A0 = t.f_even;
        tr.A1 = t.f_odd;
        tr.mid0 = t.f_mid_e;
        tr.mid1 = t.f_mid_o;
    }
    tr.in = in;
    tr.ps = t.ps;
    if (oi + 1 > a.nouts) a.nouts = oi + 1;
}

void lt_set_out(LtArgs &a, int oi, double *out, const double *grid) {
    a.outs[oi].out = out;
    a.outs[oi].grid = grid;
    if (oi + 1 > a.nouts) a.nouts = oi + 1;
}

int64_t line_transform_ctas(const LtArgs &a) {
    return ceil_div(a.B, BN) * (int64_t)(a.Mdim / BM) * a.nouts;
}

int line_transform(const LtArgs &a, cudaStream_t st) {
    // per device (cached): sets the kernels' dynamic shared-memory limit
    if (resident_blocks(reinterpret_cast<const void *>(line_transform_kernel<1>), THREADS, SMEM_BYTES) < 1 ||
        resident_blocks(reinterpret_cast<const void *>(line_transform_kernel<2>), THREADS, SMEM_BYTES) < 1) {
        set_error("line transform kernel does not fit an SM");
        return LP_ERR_CUDA;
    }
    if (a.B <= 0 || a.nouts <= 0) return LP_OK;
    dim3 grid((unsigned)ceil_div(a.B, BN), (unsigned)(a.Mdim / BM), (unsigned)a.nouts);
    const int64_t ctas = (int64_t)grid.x * grid.y * grid.z;
    if (ctas > 2 * num_sms())
        line_transform_kernel<2><<<grid, THREADS, SMEM_BYTES, st>>>(a);
    else
        line_transform_kernel<1><<<grid, THREADS, SMEM_BYTES, st>>>(a);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

}  // namespace lp
