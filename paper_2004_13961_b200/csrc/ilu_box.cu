// Kronecker-banded preconditioner M in the implicit-offset "box" layout:
// assembly, ILU(0) factorisation, forward/backward sweeps, SpMV, export.
//
// Reference: precond.py:207-297 (assemble_M, _symmetrize, _compress),
// sparse.py:116-221 (ilu0, forward_sub, backward_sub, precond_apply).
//
// Layout: values[row][slot], row = ix + K (iy + K iz) (x fastest, the CSR row
// order of precond.py:275-285), slot s <-> offset (ox, oy, oz) in [-r, r]^d,
// s = (ox+r) + W ((oy+r) + W (oz+r)).  No column indices are stored.  For the
// valid slots of a row, slot order is column order, so the reference's
// "k < i in increasing column order" is "s < c in increasing slot order",
// c = (S-1)/2 the diagonal.  An in-pattern bit per (row, slot) reproduces the
// reference's stored pattern (valid column and |m| >= 1e-300); out-of-pattern
// values are exactly zero.
#include <math.h>

#include <vector>

#include "box_geom.cuh"
#include "ilu.cuh"

namespace lp {
namespace {

// ----------------------------------------------------------------- assembly

struct GroupDesc {
    int lens[3];
    int kind[3];       // 0 = stiff block, 1 = mass block, per axis
    int64_t hat_off;   // offset into the concatenated hat array
};

struct AsmArgs {
    Geom g;
    int ngroups, tmax, R;
    GroupDesc grp[4];
    const double *hats;
    const double *blocks;   // [2][tmax+1][2R+1][K]
};

__device__ __forceinline__ double blk(const AsmArgs &a, int kind, int t, int o, int i) {
    return __ldg(a.blocks + (((size_t)kind * (a.tmax + 1) + t) * (2 * a.R + 1) + (o + a.R)) * a.g.K + i);
}

// One CTA per (line, slot-line): H_g[a] = sum_{b,c} hat_g[a,b,c] Y_b[oy](iy) Z_c[oz](iz)
// over parity-matched degrees, then raw(ix, ox) = sum_g sum_a H_g[a] X_a[ox](ix).
__global__ void box_raw_kernel(const __grid_constant__ AsmArgs a, double *__restrict__ vals) {
    const Geom &g = a.g;
    __shared__ double H[4][64];
    const int line = blockIdx.x, sl = blockIdx.y;
    const int iy = g.d > 1 ? line % g.K : 0, iz = g.d > 2 ? line / g.K : 0;
    const int oy = g.d > 1 ? sl % g.W - g.r : 0, oz = g.d > 2 ? sl / g.W - g.r : 0;
    for (int q = threadIdx.x; q < a.ngroups * 64; q += blockDim.x) {
        const int gi = q / 64, ax = q % 64;
        const GroupDesc &G = a.grp[gi];
        if (ax >= G.lens[0]) continue;
        double h = 0.0;
        const int ly = G.lens[1], lz = G.lens[2];
        for (int b = (oy & 1); b < ly; b += 2) {
            const double yb = g.d > 1 ? blk(a, G.kind[1], b, oy, iy) : 1.0;
            for (int c = (oz & 1); c < lz; c += 2) {
                const double zc = g.d > 2 ? blk(a, G.kind[2], c, oz, iz) : 1.0;
                h += a.hats[G.hat_off + ((size_t)ax * ly + b) * lz + c] * yb * zc;
            }
        }
        H[gi][ax] = h;
    }
    __syncthreads();
    const int64_t rowbase = (int64_t)line * g.K;
    const int sbase = g.W * sl;
    for (int q = threadIdx.x; q < g.K * g.W; q += blockDim.x) {
        const int ix = q / g.W, sx = q % g.W, ox = sx - g.r;
        double v = 0.0;
        for (int gi = 0; gi < a.ngroups; ++gi) {
            const GroupDesc &G = a.grp[gi];
            for (int t = (ox & 1); t < G.lens[0]; t += 2) v += H[gi][t] * blk(a, G.kind[0], t, ox, ix);
        }
        vals[(rowbase + ix) * g.S + sbase + sx] = v;
    }
}

// Average every lower entry with its transpose (precond.py:255-269).
__global__ void box_sym_kernel(Geom g, double *vals) {
    const int64_t total = g.n * g.c;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / g.c;
        const int s = (int)(q % g.c);
        int ix, iy, iz;
        row_pos(g, i, ix, iy, iz);
        const int64_t j = slot_col(g, i, ix, iy, iz, s);
        if (j < 0) continue;
        const size_t a = (size_t)i * g.S + s, b = (size_t)j * g.S + (g.S - 1 - s);
        const double avg = 0.5 * (vals[a] + vals[b]);
        vals[a] = avg;
        vals[b] = avg;
    }
}

// Pattern bits (valid column and |v| >= 1e-300, precond.py:281), zero the rest,
// count nnz, flag rows whose diagonal is not stored.
__global__ void box_mask_kernel(Geom g, double *vals, uint32_t *mask,
                                unsigned long long *nnz, unsigned long long *missing) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned long long cnt = 0;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < g.n * g.mw;
         w += nwarps) {
        const int64_t i = w / g.mw;
        const int word = (int)(w % g.mw);
        const int s = word * 32 + lane;
        bool in = false;
        if (s < g.S) {
            int ix, iy, iz;
            row_pos(g, i, ix, iy, iz);
            double *p = vals + (size_t)i * g.S + s;
            in = slot_col(g, i, ix, iy, iz, s) >= 0 && fabs(*p) >= 1e-300;
            if (!in) *p = 0.0;
            if (s == g.c && !in) atomicMin(missing, (unsigned long long)i);
        }
        const unsigned bits = __ballot_sync(0xffffffff, in);
        if (lane == 0) {
            mask[(size_t)i * g.mw + word] = bits;
            cnt += __popc(bits);
        }
    }
    if (lane == 0 && cnt) atomicAdd(nnz, cnt);
}

// Fused assembly (raw products, pattern, nnz and the full-row flags in one
// pass over M).  The raw entry of (row, slot) is
//   sum_g sum_t H_g[t](line, slot-line) X_t[ox](ix),  H_g[t] = sum_{b,c} hat_g[t,b,c] Y_b[oy](iy) Z_c[oz](iz),
// and the 1-D block diagonals are stored mirrored exactly (building_blocks_1d),
// so entry (j, i) is evaluated from bitwise the same operands in the same order
// as entry (i, j): the raw M is exactly symmetric and the averaging of
// precond.py:255-269 returns every value unchanged (0.5 (v + v) = v).  The
// separate symmetrisation pass is therefore not needed.
// CTA = (x-line, chunk of ASM_RB rows); H of every slot-line of the line in
// shared memory; warp = row, lane = x offset, looping over the slot-lines, so
// each store is a run of W contiguous doubles and the row's pattern bits are
// built by ballots in warp-private shared memory.
constexpr int ASM_RB = 32;
constexpr int ASM_MAXJ = 8;   // parity-matched degrees per group in registers (tmax <= 15)

// NG groups, J parity-matched degrees per group (t = (ox & 1) + 2j, j < J):
// H is stored [slot-line][group][2J] with zeros past the group's degree and
// each lane's X values past its degree are zero, so every entry is the same
// unpredicated chain of NG * J FMAs (an x 0 term leaves the sum unchanged;
// the mirror entry runs the same chain, so M stays exactly symmetric).
template <int NG, int J>
__global__ void __launch_bounds__(256, 2)
box_assemble_kernel(const __grid_constant__ AsmArgs a, double *__restrict__ vals,
                    uint32_t *__restrict__ mask, unsigned char *__restrict__ full,
                    unsigned long long *nnz, unsigned long long *missing) {
    extern __shared__ __align__(16) double sm[];
    constexpr int HT = 2 * J;
    const Geom &g = a.g;
    const int W = g.W, r = g.r;
    const int nsl = g.d == 1 ? 1 : (g.d == 2 ? W : W * W);
    double *H = sm;   // [nsl][NG][HT]
    uint32_t *mk = reinterpret_cast<uint32_t *>(H + (size_t)nsl * NG * HT);   // [ASM_RB][mw]
    const int line = blockIdx.x;
    const int iy = g.d > 1 ? line % g.K : 0, iz = g.d > 2 ? line / g.K : 0;
    const int x0 = blockIdx.y * ASM_RB;
    const int nrows = min(ASM_RB, g.K - x0);
    for (int q = threadIdx.x; q < nsl * NG * HT; q += blockDim.x) {
        const int t = q % HT, gi = (q / HT) % NG, sl = q / (HT * NG);
        const int oy = g.d > 1 ? sl % W - r : 0, oz = g.d > 2 ? sl / W - r : 0;
        const GroupDesc &G = a.grp[gi];
        double h = 0.0;
        if (t < G.lens[0]) {
            const int ly = G.lens[1], lz = G.lens[2];
            for (int b = (oy & 1); b < ly; b += 2) {
                const double yb = g.d > 1 ? blk(a, G.kind[1], b, oy, iy) : 1.0;
                for (int c = (oz & 1); c < lz; c += 2) {
                    const double zc = g.d > 2 ? blk(a, G.kind[2], c, oz, iz) : 1.0;
                    h += a.hats[G.hat_off + ((size_t)t * ly + b) * lz + c] * yb * zc;
                }
            }
        }
        H[q] = h;
    }
    for (int q = threadIdx.x; q < nrows * g.mw; q += blockDim.x) mk[q] = 0u;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ox = lane - r;
    const bool xlane = lane < W;
    const int par = ox & 1;
    unsigned long long cnt = 0;
    for (int rl = warp; rl < nrows; rl += blockDim.x >> 5) {
        const int ix = x0 + rl;
        const int64_t i = (int64_t)line * g.K + ix;
        double xr[NG][J];
#pragma unroll
        for (int gi = 0; gi < NG; ++gi)
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int t = par + 2 * j;
                xr[gi][j] = (xlane && t < a.grp[gi].lens[0]) ? blk(a, a.grp[gi].kind[0], t, ox, ix) : 0.0;
            }
        const bool xok = xlane && ix + ox >= 0 && ix + ox < g.K;
        uint32_t *mrow = mk + rl * g.mw;
        double *vrow = vals + (size_t)i * g.S + lane;
        const double *Hs = H + par;
        int sl = 0;
        const int nz = g.d > 2 ? W : 1, ny = g.d > 1 ? W : 1;
        for (int sz = 0; sz < nz; ++sz) {
            const bool zok = g.d < 3 || (iz + sz - r >= 0 && iz + sz - r < g.K);
            for (int sy = 0; sy < ny; ++sy, ++sl, Hs += NG * HT) {
                const bool ok = xok && zok && (g.d < 2 || (iy + sy - r >= 0 && iy + sy - r < g.K));
                double v = 0.0;
#pragma unroll
                for (int gi = 0; gi < NG; ++gi)
#pragma unroll
                    for (int j = 0; j < J; ++j) v += Hs[gi * HT + 2 * j] * xr[gi][j];
                const bool in = ok && fabs(v) >= 1e-300;
                if (xlane) vrow[sl * W] = in ? v : 0.0;
                const unsigned bits = __ballot_sync(0xffffffffu, in);
                if (lane == 0 && bits) {
                    const int s0 = sl * W, w0 = s0 >> 5, sh = s0 & 31;
                    mrow[w0] |= bits << sh;
                    if (sh && (bits >> (32 - sh))) mrow[w0 + 1] |= bits >> (32 - sh);
                }
            }
        }
        __syncwarp();
        int pc = 0;
        for (int w = lane; w < g.mw; w += 32) pc += __popc(mrow[w]);
#pragma unroll
        for (int o = 16; o; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
        if (lane == 0) {
            full[i] = pc == g.S;
            cnt += (unsigned long long)pc;
            if (!((mrow[g.c >> 5] >> (g.c & 31)) & 1u)) atomicMin(missing, (unsigned long long)i);
        }
    }
    if (lane == 0 && cnt) atomicAdd(nnz, cnt);
    __syncthreads();
    uint32_t *mdst = mask + ((size_t)line * g.K + x0) * g.mw;
    for (int q = threadIdx.x; q < nrows * g.mw; q += blockDim.x) mdst[q] = mk[q];
}

template <int NG>
const void *assemble_kernel_j(int J) {
    switch (J) {
        case 1: return reinterpret_cast<const void *>(box_assemble_kernel<NG, 1>);
        case 2: return reinterpret_cast<const void *>(box_assemble_kernel<NG, 2>);
        case 3: return reinterpret_cast<const void *>(box_assemble_kernel<NG, 3>);
        case 4: return reinterpret_cast<const void *>(box_assemble_kernel<NG, 4>);
        case 5: return reinterpret_cast<const void *>(box_assemble_kernel<NG, 5>);
        case 6: return reinterpret_cast<const void *>(box_assemble_kernel<NG, 6>);
        case 7: return reinterpret_cast<const void *>(box_assemble_kernel<NG, 7>);
        default: return reinterpret_cast<const void *>(box_assemble_kernel<NG, 8>);
    }
}

const void *assemble_kernel(int NG, int J) {
    switch (NG) {
        case 1: return assemble_kernel_j<1>(J);
        case 2: return assemble_kernel_j<2>(J);
        case 3: return assemble_kernel_j<3>(J);
        default: return assemble_kernel_j<4>(J);
    }
}

// full[i] = 1 when every slot of row i is in the pattern (interior rows of a
// full box): the factorisation then needs no boundary or pattern checks.
__global__ void box_full_kernel(Geom g, const uint32_t *__restrict__ mask,
                                unsigned char *__restrict__ full) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int cnt = 0;
        for (int w = 0; w < g.mw; ++w) cnt += __popc(mask[(size_t)i * g.mw + w]);
        full[i] = cnt == g.S;
    }
}

// ----------------------------------------------------------- factorisation
//
// IKJ ILU(0) (sparse.py:116-139) with one CTA per row, rows handed out in
// natural order by a ticket.  Row i lives in shared memory; for every lower
// in-pattern slot s (ascending = column order) the CTA waits for row
// k = i + off(s) to be final, forms l = a_is / u_kk, and applies
// a_it -= l u_ks' for every upper slot s' of row k whose target offset
// off(s) + off(s') is an in-pattern slot t of row i.  Updates of one step hit
// distinct targets; steps are separated by a barrier, so each entry receives
// its updates in the reference's k order, each as a separately rounded
// multiply and subtract: the factors are bit-identical to the reference's for
// the same M.

__device__ __forceinline__ int ld_flag(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int TPR>
__device__ __forceinline__ void row_sync() {
    if (TPR == 32) __syncwarp();
    else __syncthreads();
}

template <int TPR>
__global__ void __launch_bounds__(TPR)
box_ilu0_kernel(Geom g, double *lu, const uint32_t *__restrict__ mask, int *flags, int epoch,
                int *ticket, double tol, unsigned long long *bad) {
    extern __shared__ __align__(16) double sm[];
    double *row = sm;                     // [S]
    double *lval = sm + g.S;              // [c]
    uint32_t *bits = reinterpret_cast<uint32_t *>(lval + g.c);   // [mw]
    __shared__ int64_t sh_row;
    const int tid = threadIdx.x;
    for (;;) {
        if (tid == 0) sh_row = atomicAdd(ticket, 1);
        row_sync<TPR>();
        const int64_t i = sh_row;
        if (i >= g.n) return;
        int ix, iy, iz;
        row_pos(g, i, ix, iy, iz);
        for (int s = tid; s < g.S; s += TPR) {
            const double v = lu[(size_t)i * g.S + s];
            row[s] = v;
            if (s < g.c) lval[s] = v;
        }
        for (int w = tid; w < g.mw; w += TPR) bits[w] = mask[(size_t)i * g.mw + w];
        row_sync<TPR>();
        for (int s = 0; s < g.c; ++s) {
            if (!((bits[s >> 5] >> (s & 31)) & 1u)) continue;
            int sx, sy, sz;
            slot_axes(g, s, sx, sy, sz);
            const int64_t k = i + (sx - g.r) + (int64_t)g.K * ((sy - g.r) + (int64_t)g.K * (sz - g.r));
            // all threads poll the same flag (uniform, no divergent spin); the
            // writer fences before publishing, and row k is read through L2
            while (ld_flag(flags + k) != epoch) {
            }
            const double *uk = lu + (size_t)k * g.S;
            const double piv = __ldcg(uk + g.c);
            const double l = __ddiv_rn(row[s], piv);
            if (tid == 0) {
                lval[s] = l;
                if (fabs(piv) < tol) atomicMin(bad, (unsigned long long)(i * g.n + k));
            }
            // row k position and the sub-box of upper slots s' whose target stays in the box
            const int kx = ix + sx - g.r, ky = iy + sy - g.r, kz = iz + sz - g.r;
            const int xlo = max(g.r - sx, 0), xhi = min(g.W + g.r - sx, g.W);
            // the most significant axis of an upper slot is >= r; the others span their range
            const int ylo = g.d > 1 ? max(g.r - sy, g.d == 2 ? g.r : 0) : 0;
            const int yhi = g.d > 1 ? min(g.W + g.r - sy, g.W) : 1;
            const int zlo = g.d > 2 ? max(g.r - sz, g.r) : 0, zhi = g.d > 2 ? min(g.W + g.r - sz, g.W) : 1;
            // threads: lane along x, the rest along (y, z) pairs; the loads of one
            // batch are all issued before any update uses them
            constexpr int B = 16;
            const int nx = xhi - xlo;
            const int tx = tid & 31, tyz = tid >> 5, nyz_threads = TPR / 32;
            const int ny = yhi - ylo, nz = zhi - zlo;
            const int sxp = xlo + tx;
            const int colx = kx + sxp - g.r;
            const bool xok = tx < nx && colx >= 0 && colx < g.K;
            for (int q0 = tyz; q0 < ny * nz; q0 += nyz_threads * B) {
                double u[B];
                int tt[B];
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int q = q0 + j * nyz_threads;
                    const int syp = g.d > 1 ? ylo + q % ny : g.r;
                    const int szp = g.d > 2 ? zlo + q / ny : g.r;
                    const int sp = sxp + (g.d > 1 ? g.W * syp : 0) + (g.d > 2 ? g.W * g.W * szp : 0);
                    bool ok = xok && q < ny * nz && sp > g.c;
                    if (g.d > 1) {
                        const int cy = ky + syp - g.r;
                        ok = ok && cy >= 0 && cy < g.K;
                    }
                    if (g.d > 2) {
                        const int cz = kz + szp - g.r;
                        ok = ok && cz >= 0 && cz < g.K;
                    }
                    const int t = (sx + sxp - g.r) + (g.d > 1 ? g.W * (sy + syp - g.r) : 0) +
                                  (g.d > 2 ? g.W * g.W * (sz + szp - g.r) : 0);
                    ok = ok && ((bits[t >> 5] >> (t & 31)) & 1u);
                    u[j] = ok ? __ldcg(uk + sp) : 0.0;
                    tt[j] = ok ? t : -1;
                }
#pragma unroll
                for (int j = 0; j < B; ++j)
                    if (tt[j] >= 0) row[tt[j]] = __dsub_rn(row[tt[j]], __dmul_rn(l, u[j]));
            }
            row_sync<TPR>();
        }
        for (int s = tid; s < g.S; s += TPR) __stcg(lu + (size_t)i * g.S + s, s < g.c ? lval[s] : row[s]);
        __threadfence();
        row_sync<TPR>();
        if (tid == 0) {
            __threadfence();
            *((volatile int *)(flags + i)) = epoch;
        }
    }
}

// Line-pipelined ILU(0) for 1-D/2-D boxes.  A CTA owns one x-line at a time
// (lines in natural order by ticket); its NW warps take the line's rows
// round-robin, one row per warp in flight, each row double-buffered in shared
// memory.  The row's last r elimination steps (the in-line slots, k = i-1..i-r)
// are the critical path of the whole factorisation; they read the sibling rows'
// finished U parts straight from shared memory.  Off-line steps read rows of
// earlier lines through L2 once that line's published contiguous-prefix row
// count covers them (flags[line], one relaxed poll per offset group).  Arithmetic and per-entry update order are exactly those of
// box_ilu0_kernel (and of the reference), so the factors are identical.
// Requires NW >= r + 1 (a row buffer is recycled only after every row that
// reads it has finished) and 2 * NW * S doubles of shared memory.
template <int NW>
__global__ void __launch_bounds__(32 * NW)
box_ilu0_line_kernel(Geom g, double *lu, const uint32_t *__restrict__ mask,
                     const unsigned char *__restrict__ full, int *flags, int epoch, int *ticket,
                     double tol, unsigned long long *bad) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int s_rowdone[2 * NW];
    __shared__ int s_prefix;
    __shared__ int s_line;
    volatile int *v_prefix = &s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = g.K, r = g.r;
    const int S = g.S, c = g.c;
    const int mwS = (g.mw + 1) & ~1;                     // mask words, padded to 8 bytes
    const int bufd = S + mwS / 2;                        // doubles per row buffer
    volatile int *v_done = s_rowdone;
    for (;;) {
        __syncthreads();
        if (tid == 0) s_line = atomicAdd(ticket, 1);
        for (int q = tid; q < 2 * NW; q += blockDim.x) s_rowdone[q] = -1;
        if (tid == 0) s_prefix = 0;
        __syncthreads();
        const int L = s_line;
        if (L >= g.nlines) return;
        const int iy = g.d > 1 ? L : 0;
        const int64_t row0 = (int64_t)L * K;
        for (int ix = warp, it = 0; ix < K; ix += NW, ++it) {
            const int buf = (ix / NW) & 1;
            double *row = sm + (size_t)(warp * 2 + buf) * bufd;
            uint32_t *bits = reinterpret_cast<uint32_t *>(row + S);
            const int64_t i = row0 + ix;
            for (int q = lane; q < S; q += 32) row[q] = lu[(size_t)i * S + q];
            for (int q = lane; q < g.mw; q += 32) bits[q] = mask[(size_t)i * g.mw + q];
            __syncwarp();
            // Elimination steps over the in-pattern lower slots, software
            // pipelined: while step s updates the row, the flag check and the U
            // loads of the next off-line step are already in flight (two
            // register sets, ping-pong).  In-line steps read shared memory.
            constexpr int B = 16;   // >= r + 1 rows of upper slots in 2-D
            struct Step {
                int s, sx, sy;
                bool inl;
                int64_t k;
                double piv;
                double u[B];
                int tt[B];
            };
            auto next_slot = [&](int s0) {
                for (int s1 = s0; s1 < c; ++s1)
                    if ((bits[s1 >> 5] >> (s1 & 31)) & 1u) return s1;
                return c;
            };
            // gather row k's upper entries that land in row i's pattern
            const bool full_i = full[i] != 0;
            auto gather = [&](Step &st, const double *uk, bool shared) {
                if (full_i && full[st.k]) {
                    // every slot of rows i and k is in the pattern: the targets are
                    // t = s' + s - c, no boundary or pattern tests needed
                    const int xlo = max(r - st.sx, 0), xhi = min(g.W + r - st.sx, g.W);
                    const int ylo = g.d > 1 ? max(r - st.sy, r) : 0;
                    const int yhi = g.d > 1 ? min(g.W + r - st.sy, g.W) : 1;
                    const int sxp = xlo + lane;
                    const bool xok = lane < xhi - xlo;
                    const int shift = st.s - c;
                    st.piv = shared ? uk[c] : __ldcg(uk + c);
#pragma unroll
                    for (int j = 0; j < B; ++j) {
                        const int sp = sxp + g.W * (ylo + j);
                        const bool ok = xok && ylo + j < yhi && sp > c;
                        st.u[j] = ok ? (shared ? uk[sp] : __ldcg(uk + sp)) : 0.0;
                        st.tt[j] = ok ? sp + shift : -1;
                    }
                    return;
                }
                const int kx = ix + st.sx - r, ky = iy + st.sy - r;
                const int xlo = max(r - st.sx, 0), xhi = min(g.W + r - st.sx, g.W);
                const int ylo = g.d > 1 ? max(r - st.sy, r) : 0;
                const int yhi = g.d > 1 ? min(g.W + r - st.sy, g.W) : 1;
                const int nx = xhi - xlo, ny = yhi - ylo;
                const int sxp = xlo + lane;
                const int colx = kx + sxp - r;
                const bool xok = lane < nx && colx >= 0 && colx < K;
                st.piv = shared ? uk[c] : __ldcg(uk + c);
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int syp = g.d > 1 ? ylo + j : r;
                    const int sp = sxp + (g.d > 1 ? g.W * syp : 0);
                    bool ok = xok && j < ny && sp > c;
                    if (g.d > 1) {
                        const int cy = ky + syp - r;
                        ok = ok && cy >= 0 && cy < K;
                    }
                    const int t = (st.sx + sxp - r) + (g.d > 1 ? g.W * (st.sy + syp - r) : 0);
                    ok = ok && ((bits[t >> 5] >> (t & 31)) & 1u);
                    st.u[j] = ok ? (shared ? uk[sp] : __ldcg(uk + sp)) : 0.0;
                    st.tt[j] = ok ? t : -1;
                }
            };
            // decode slot s; for an off-line step wait for row k and issue its loads
            // Earlier lines publish a contiguous-prefix row count; the rows of
            // line L + oy this row needs are those with x <= ix + r, checked once
            // per offset group oy.
            int oy_ready = -1 << 20;
            auto prepare = [&](Step &st, int s) {
                st.s = s;
                if (s >= c) return;
                st.sx = s % g.W;
                st.sy = g.d > 1 ? s / g.W : r;
                st.inl = st.sy == r;
                st.k = i + (st.sx - r) + (int64_t)K * (st.sy - r);
                if (!st.inl) {
                    if (st.sy != oy_ready) {
                        const int need = min(K, ix + r + 1);
                        while (ld_flag(flags + (L + st.sy - r)) < need) {
                        }
                        oy_ready = st.sy;
                    }
                    gather(st, lu + (size_t)st.k * S, false);
                }
            };
            auto execute = [&](Step &st) {
                if (st.inl) {
                    const int kix = ix - (r - st.sx);
                    while (v_done[kix % (2 * NW)] != kix) {
                    }
                    gather(st, sm + (size_t)((kix % NW) * 2 + ((kix / NW) & 1)) * bufd, true);
                }
                const double l = __ddiv_rn(row[st.s], st.piv);
                if (lane == 0 && fabs(st.piv) < tol)
                    atomicMin(bad, (unsigned long long)(i * g.n + st.k));
#pragma unroll
                for (int j = 0; j < B; ++j)
                    if (st.tt[j] >= 0) row[st.tt[j]] = __dsub_rn(row[st.tt[j]], __dmul_rn(l, st.u[j]));
                __syncwarp();
                if (lane == 0) row[st.s] = l;     // no later step touches slot s
                __syncwarp();
            };
            Step A, Bq;
            prepare(A, next_slot(0));
            while (A.s < c) {
                prepare(Bq, next_slot(A.s + 1));
                execute(A);
                if (Bq.s >= c) break;
                prepare(A, next_slot(Bq.s + 1));
                execute(Bq);
            }
            for (int q = lane; q < S; q += 32) __stcg(lu + (size_t)i * S + q, row[q]);
            __threadfence();
            __syncwarp();
            if (lane == 0) {
                v_done[ix % (2 * NW)] = ix;
                // publish the line's contiguous prefix in row order
                while (*v_prefix != ix) {
                }
                __threadfence();
                *((volatile int *)(flags + L)) = ix + 1;
                *v_prefix = ix + 1;
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    return v;
}

__global__ void box_spmv_kernel(Geom g, const double *__restrict__ vals, const double *__restrict__ x,
                                double *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= g.n) return;
    int ix, iy, iz;
    row_pos(g, i, ix, iy, iz);
    double acc = 0.0;
    for (int s = lane; s < g.S; s += 32) {
        const double v = vals[(size_t)i * g.S + s];
        if (v != 0.0) acc = fma(v, x[slot_col(g, i, ix, iy, iz, s)], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) y[i] = acc;
}

}  // namespace

int box_spmv(lp_ilu *m, const double *x, double *y, cudaStream_t st) {
    Geom g = geom_of(m->box);
    LP_ARG(m->box.values != nullptr, "original matrix was released (factored in place)");
    box_spmv_kernel<<<(unsigned)ceil_div(g.n * 32, 256), 256, 0, st>>>(g, m->box.values, x, y);
    count_launch();
    LP_CHECK_LAUNCH();
    return LP_OK;
}

int box_ilu0(lp_ilu *m, double tol, int64_t *bad_row, cudaStream_t st) {
    BoxLayout &b = m->box;
    Geom g = geom_of(b);
    if (m->missing_diag >= 0) {
        *bad_row = m->missing_diag;
        set_error("zero pivot at elimination step %lld", (long long)*bad_row);
        return LP_ERR_ZERO_PIVOT;
    }
    const size_t bytes = (size_t)b.n * b.S * sizeof(double);
    if (!b.lu) {
        // +2 doubles: the sweeps stage factor rows with 16-byte aligned bulk copies
        if (dalloc(&b.lu, (size_t)b.n * b.S + 2, "ILU factors") != LP_OK) {
            // not enough memory for a separate copy: factor in place, drop M
            b.lu = b.values;
            b.values = nullptr;
        }
    }
    if (!b.values && m->factored) {
        set_error("matrix was factored in place; re-assemble before refactoring");
        return LP_ERR_ARG;
    }
    // the 2-D block-wavefront kernel reads M and writes the factors itself; the
    // other kernels factor a copy in place
    const bool wave2d = g.d == 2 && g.r >= 1 && g.r <= 14 && b.full;
    if (b.values && !wave2d) LP_CUDA(cudaMemcpyAsync(b.lu, b.values, bytes, cudaMemcpyDeviceToDevice, st));
    unsigned long long *key = reinterpret_cast<unsigned long long *>(m->bad);
    const unsigned long long none = ~0ull;
    LP_CUDA(cudaMemcpyAsync(key, &none, sizeof none, cudaMemcpyHostToDevice, st));
    // row flags: reuse `flags` as int per row (progress counters are re-based per sweep call)
    LP_CUDA(cudaMemsetAsync(m->flags, 0, b.n * sizeof(int), st));
    LP_CUDA(cudaMemsetAsync(m->ticket, 0, sizeof(int), st));
    const int epoch = 1;
    const size_t smem = (size_t)g.S * sizeof(double) + (size_t)g.c * sizeof(double) +
                        (size_t)g.mw * sizeof(uint32_t) + 16;
    int dev;
    LP_CUDA(cudaGetDevice(&dev));
    int nsm = 0;
    LP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    constexpr int LNW = 16;
    const size_t line_smem = (size_t)2 * LNW * (g.S + ((g.mw + 1) & ~1) / 2) * sizeof(double);
    // The row-ticket kernel keeps ~(resident CTAs) rows in flight in natural
    // order; that window must span the wavefront, about K (r + 1) rows.  When
    // it does not (long lines), the line-pipelined kernel is used instead.
    // (Measured on B200: cfg 2, K (r+1) = 3315 -> row kernel 57 ms vs line kernel
    // 198 ms; cfg 3, K (r+1) = 30705 -> row kernel 9.5 s vs line kernel 3.1 s.)
    const bool window_ok = (int64_t)g.K * (g.r + 1) <= 8192;
    bool done = false;
    if (wave2d) {
        // block-wavefront factorisation (ilu_box2d.cu)
        int *bdone = nullptr;
        const int nb = (g.K + 13) / 14;
        int rcf;
        if ((rcf = dalloc(&bdone, (size_t)g.nlines * nb, "block flags"))) return rcf;
        LP_CUDA(cudaMemsetAsync(bdone, 0, (size_t)g.nlines * nb * sizeof(int), st));
        const int rt = box_ilu0_2d_tasks(m, b.values ? b.values : b.lu, tol, key, bdone, st);
        dfree(bdone);
        if (rt != LP_OK) return rt;
        LP_CUDA(cudaStreamSynchronize(st));
        done = true;
    }
    if (g.d == 3 && b.mask) {
        // row-per-CTA kernel (ilu_box3d.cu)
        const int rt = box_ilu0_3d_rows(m, tol, key, st);
        if (rt == LP_OK) done = true;
    }
    if (done) {
    } else if (g.d <= 2 && !window_ok && g.r + 1 <= LNW && line_smem <= 220 * 1024) {
        LP_CUDA(cudaFuncSetAttribute(box_ilu0_line_kernel<LNW>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)line_smem));
        int occ = 1;
        LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, box_ilu0_line_kernel<LNW>,
                                                              32 * LNW, line_smem));
        int64_t blocks = (int64_t)occ * nsm;
        if (blocks > g.nlines) blocks = g.nlines;
        box_ilu0_line_kernel<LNW><<<(unsigned)blocks, 32 * LNW, line_smem, st>>>(
            g, b.lu, b.mask, b.full, m->flags, epoch, m->ticket, tol, key);
        count_launch();
        LP_CUDA(cudaStreamSynchronize(st));
    } else if (g.S <= 1200) {
        LP_CUDA(cudaFuncSetAttribute(box_ilu0_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        int occ = 1;
        LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, box_ilu0_kernel<32>, 32, smem));
        int64_t blocks = (int64_t)occ * nsm;
        if (blocks > g.n) blocks = g.n;
        box_ilu0_kernel<32><<<(unsigned)blocks, 32, smem, st>>>(g, b.lu, b.mask, m->flags, epoch,
                                                               m->ticket, tol, key);
    } else {
        LP_CUDA(cudaFuncSetAttribute(box_ilu0_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        int occ = 1;
        LP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, box_ilu0_kernel<256>, 256, smem));
        int64_t blocks = (int64_t)occ * nsm;
        if (blocks > g.n) blocks = g.n;
        box_ilu0_kernel<256><<<(unsigned)blocks, 256, smem, st>>>(g, b.lu, b.mask, m->flags, epoch,
                                                                 m->ticket, tol, key);
    }
    if (!done) count_launch();
    LP_CHECK_LAUNCH();
    unsigned long long hk;
    double plast;
    LP_CUDA(cudaMemcpyAsync(&hk, key, sizeof hk, cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaMemcpyAsync(&plast, b.lu + (size_t)(b.n - 1) * b.S + g.c, sizeof plast,
                            cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaStreamSynchronize(st));
    // progress counters for the sweeps start from a clean slate
    LP_CUDA(cudaMemset(m->flags, 0, b.n * sizeof(int)));
    m->epoch = 0;
    if (hk != none) *bad_row = (int64_t)(hk % (unsigned long long)b.n);
    else if (fabs(plast) < tol) *bad_row = b.n - 1;
    if (*bad_row >= 0) {
        set_error("zero pivot at elimination step %lld (row %lld)", (long long)*bad_row,
                  hk != none ? (long long)(hk / (unsigned long long)b.n) : (long long)(b.n - 1));
        return LP_ERR_ZERO_PIVOT;
    }
    m->factored = true;
    return box_build_bands(m, st);
}

// Factor storage of one rank ready for lp_ilu0_rank(s): M copied into the
// factor array, line flags cleared (synchronises the stream).
int box_ilu0_prepare(lp_ilu *m, int64_t *bad_row, cudaStream_t st) {
    BoxLayout &b = m->box;
    if (m->missing_diag >= 0) {
        *bad_row = m->missing_diag;
        set_error("zero pivot at elimination step %lld", (long long)*bad_row);
        return LP_ERR_ZERO_PIVOT;
    }
    const size_t bytes = (size_t)b.n * b.S * sizeof(double);
    if (!b.lu) {
        if (dalloc(&b.lu, (size_t)b.n * b.S + 2, "ILU factors") != LP_OK) {
            b.lu = b.values;
            b.values = nullptr;
        }
    }
    if (!b.values && m->factored) {
        set_error("matrix was factored in place; re-assemble before refactoring");
        return LP_ERR_ARG;
    }
    if (b.values) LP_CUDA(cudaMemcpyAsync(b.lu, b.values, bytes, cudaMemcpyDeviceToDevice, st));
    LP_CUDA(cudaMemsetAsync(m->flags, 0, b.n * sizeof(int), st));
    LP_CUDA(cudaStreamSynchronize(st));
    return LP_OK;
}

// ILU(0) of a 3-D box matrix distributed over y-slab ranks (the
// factorisation uses the sweeps' wavefront and needs the neighbours' U rows of
// the r halo lines).  own = -1: ms[0..nranks) are the ranks' matrices (each
// assembled from the same problem), factored in ONE launch on this device --
// the emulation of the multi-GPU run, every rank reading only its own array
// (its rows plus the halo rows its neighbours stored there).  own >= 0: ms[0]
// is this rank's matrix; peer_lu / peer_flags hold the neighbours' factor and
// flag arrays mapped over CUDA IPC (entries of non-neighbours may be null).
// Every row's arithmetic is the single-GPU kernel's: the owners' rows equal the
// single-GPU factors bit for bit.
int box_ilu0_ranks(lp_ilu *const *ms, int nranks, const int *ys, int own, double *const *peer_lu,
                   int *const *peer_flags, double tol, int64_t *bad_row, cudaStream_t st) {
    LP_ARG(nranks >= 1 && nranks <= 8, "1 to 8 ranks");
    const int nh = own >= 0 ? 1 : nranks;
    lp_ilu *m0 = ms[0];
    Geom g = geom_of(m0->box);
    LP_ARG(g.d == 3 && g.r >= 1 && g.r <= 10 && m0->box.mask, "the distributed ILU(0) serves 3-D boxes of reach 1..10");
    LP_ARG(ys[0] == 0 && ys[nranks] == g.K, "ys must split [0, K)");
    for (int v = 0; v < nranks; ++v) LP_ARG(ys[v + 1] > ys[v], "empty y-slab");
    IluRanks rk;
    rk.nranks = nranks;
    rk.own = own;
    for (int v = 0; v <= nranks; ++v) rk.ys[v] = ys[v];
    *bad_row = -1;
    for (int h = 0; h < nh; ++h) {
        lp_ilu *m = ms[h];
        BoxLayout &b = m->box;
        LP_ARG(m->kind == MAT_BOX && b.n == m0->box.n && b.r == g.r, "rank matrices differ");
        // one rank of a multi-GPU run is prepared (and the ranks synchronised) by the
        // caller: a neighbour may already be storing halo rows and flags here
        if (own < 0) {
            const int rp = box_ilu0_prepare(m, bad_row, st);
            if (rp) return rp;
        } else {
            LP_ARG(b.lu != nullptr, "call lp_ilu0_rank_prepare (and synchronise the ranks) first");
        }
        const int v = own >= 0 ? own : h;
        rk.lu[v] = b.lu;
        rk.flags[v] = m->flags;
    }
    if (own >= 0)
        for (int v = 0; v < nranks; ++v)
            if (v != own) {
                rk.lu[v] = peer_lu ? peer_lu[v] : nullptr;
                rk.flags[v] = peer_flags ? peer_flags[v] : nullptr;
                const bool neighbour = v == own - 1 || v == own + 1;
                LP_ARG(!neighbour || (rk.lu[v] && rk.flags[v]), "the slab neighbours' arrays are required");
            }
    unsigned long long *key = reinterpret_cast<unsigned long long *>(m0->bad);
    const unsigned long long none = ~0ull;
    LP_CUDA(cudaMemcpyAsync(key, &none, sizeof none, cudaMemcpyHostToDevice, st));
    LP_CUDA(cudaMemsetAsync(m0->ticket, 0, sizeof(int), st));
    int rc = box_ilu0_3d_rows(m0, tol, key, st, &rk);
    if (rc != LP_OK) return rc;
    unsigned long long hk;
    LP_CUDA(cudaMemcpyAsync(&hk, key, sizeof hk, cudaMemcpyDeviceToHost, st));
    LP_CUDA(cudaStreamSynchronize(st));
    if (hk != none) {
        *bad_row = (int64_t)(hk % (unsigned long long)g.n);
        set_error("zero pivot at elimination step %lld (row %lld)", (long long)*bad_row,
                  (long long)(hk / (unsigned long long)g.n));
        return LP_ERR_ZERO_PIVOT;
    }
    for (int h = 0; h < nh; ++h) {
        lp_ilu *m = ms[h];
        LP_CUDA(cudaMemsetAsync(m->flags, 0, m->box.n * sizeof(int), st));
        m->epoch = 0;
        m->factored = true;
        if ((rc = box_build_bands(m, st))) return rc;
    }
    LP_CUDA(cudaStreamSynchronize(st));
    return LP_OK;
}

int box_export(const lp_ilu *m, int which, int64_t *indptr, int32_t *indices, double *values) {
    const BoxLayout &b = m->box;
    const double *src = which == 0 ? b.values : b.lu;
    LP_ARG(src != nullptr, "original matrix was released (factored in place)");
    Geom g = geom_of(b);
    std::vector<uint32_t> mk((size_t)b.n * b.mask_words);
    LP_CUDA(cudaMemcpy(mk.data(), b.mask, mk.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    const int64_t chunk = 1 << 14;
    std::vector<double> buf;
    int64_t out = 0;
    indptr[0] = 0;
    const int slo = which == 2 ? g.c : 0, shi = which == 1 ? g.c : g.S;
    for (int64_t i0 = 0; i0 < b.n; i0 += chunk) {
        const int64_t rows = (b.n - i0) < chunk ? (b.n - i0) : chunk;
        if (values) {
            buf.resize((size_t)rows * b.S);
            LP_CUDA(cudaMemcpy(buf.data(), src + (size_t)i0 * b.S, buf.size() * sizeof(double),
                               cudaMemcpyDeviceToHost));
        }
        for (int64_t i = i0; i < i0 + rows; ++i) {
            for (int s = slo; s < shi; ++s) {
                if (!((mk[(size_t)i * b.mask_words + (s >> 5)] >> (s & 31)) & 1u)) continue;
                const int sx = s % g.W, qq = s / g.W;
                const int sy = g.d > 1 ? qq % g.W : g.r, sz = g.d > 2 ? qq / g.W : g.r;
                const int64_t col = i + (sx - g.r) + (int64_t)g.K * ((sy - g.r) + (int64_t)g.K * (sz - g.r));
                if (indices) indices[out] = (int32_t)col;
                if (values) values[out] = buf[(size_t)(i - i0) * b.S + s];
                ++out;
            }
            indptr[i + 1] = out;
        }
    }
    return LP_OK;
}

}  // namespace lp

using namespace lp;

extern "C" int lp_box_assemble(int d, int K, int n_groups, const int *lens, const int *stiff_axis,
                               const double *const *hats, int tmax, const double *blocks,
                               lp_ilu **out) {
    *out = nullptr;
    LP_ARG(d >= 1 && d <= 3, "dim must be 1, 2 or 3");
    LP_ARG(K >= 1, "empty preconditioner: K = 0");
    LP_ARG(n_groups >= 1 && n_groups <= 4, "1..4 coefficient groups supported");
    LP_ARG(tmax >= 0 && tmax < 64, "truncation degree out of range");
    AsmArgs a{};
    a.ngroups = n_groups;
    a.tmax = tmax;
    a.R = tmax + 2;
    int r = 0;
    int64_t hat_total = 0;
    for (int gi = 0; gi < n_groups; ++gi) {
        GroupDesc &G = a.grp[gi];
        int64_t cnt = 1;
        for (int ax = 0; ax < 3; ++ax) {
            G.lens[ax] = ax < d ? lens[gi * d + ax] : 1;
            G.kind[ax] = (stiff_axis[gi] == ax) ? 0 : 1;
            LP_ARG(G.lens[ax] >= 1 && G.lens[ax] <= tmax + 1, "hat extent out of range");
            cnt *= G.lens[ax];
            if (ax < d) {
                const int reach = G.lens[ax] - 1 + (G.kind[ax] == 0 ? 0 : 2);
                if (reach > r) r = reach;
            }
        }
        G.hat_off = hat_total;
        hat_total += cnt;
    }
    lp_ilu *m = new lp_ilu();
    m->kind = MAT_BOX;
    BoxLayout &b = m->box;
    b.d = d;
    b.K = K;
    b.r = r;
    b.W = 2 * r + 1;
    b.S = b.W;
    for (int ax = 1; ax < d; ++ax) b.S *= b.W;
    b.n = K;
    for (int ax = 1; ax < d; ++ax) b.n *= K;
    b.mask_words = (b.S + 31) / 32;
    m->n = b.n;
    int rc;
    double *dhats = nullptr, *dblocks = nullptr;
    unsigned long long *cnt = nullptr;
    const size_t nblk = (size_t)2 * (tmax + 1) * (2 * a.R + 1) * K;
    auto fail = [&](int code) {
        if (dhats) dfree(dhats);
        if (dblocks) dfree(dblocks);
        if (cnt) dfree(cnt);
        lp_ilu_destroy(m);
        return code;
    };
    if ((rc = dalloc(&b.values, (size_t)b.n * b.S + 2, "preconditioner values")) ||
        (rc = dalloc(&b.mask, (size_t)b.n * b.mask_words, "pattern bits")) ||
        (rc = dalloc(&dhats, hat_total, "hats")) || (rc = dalloc(&dblocks, nblk, "1-D blocks")) ||
        (rc = dalloc(&cnt, 2, "counters")) ||
        (rc = dalloc(&m->flags, b.n > 2 * (b.n / K) + 2 ? b.n : 2 * (b.n / K) + 2, "flags")) ||
        (rc = dalloc(&m->ticket, 4, "tickets")) || (rc = dalloc(&m->bad, 1, "pivot key")))
        return fail(rc);
    for (int gi = 0; gi < n_groups; ++gi) {
        const GroupDesc &G = a.grp[gi];
        const int64_t c = (int64_t)G.lens[0] * G.lens[1] * G.lens[2];
        cudaError_t e = cudaMemcpy(dhats + G.hat_off, hats[gi], c * sizeof(double), cudaMemcpyDefault);
        if (e != cudaSuccess) return fail(cuda_fail(e, "hat upload", __FILE__, __LINE__));
    }
    cudaError_t e = cudaMemcpy(dblocks, blocks, nblk * sizeof(double), cudaMemcpyDefault);
    if (e != cudaSuccess) return fail(cuda_fail(e, "block upload", __FILE__, __LINE__));
    a.hats = dhats;
    a.blocks = dblocks;
    a.g = geom_of(b);
    const unsigned long long init[2] = {0ull, ~0ull};
    e = cudaMemcpy(cnt, init, sizeof init, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(cuda_fail(e, "counter init", __FILE__, __LINE__));
    const int wd = d > 1 ? b.W : 1;
    const unsigned slot_lines = (unsigned)(d > 2 ? wd * wd : wd);
    unsigned long long *cnt1 = cnt + 1;
    const int asm_j = (tmax + 2) / 2;   // parity-matched degrees per group
    const size_t asm_smem = (size_t)slot_lines * n_groups * 2 * asm_j * sizeof(double) +
                            (size_t)ASM_RB * b.mask_words * sizeof(uint32_t);
    if ((rc = dalloc(&b.full, (size_t)b.n, "full-row flags"))) return fail(rc);
    const void *akern = assemble_kernel(n_groups, asm_j);
    if (b.W <= 32 && asm_j <= ASM_MAXJ && asm_smem <= 200 * 1024 &&
        resident_blocks(akern, 256, asm_smem) > 0) {
        void *args[] = {(void *)&a, (void *)&b.values, (void *)&b.mask, (void *)&b.full,
                        (void *)&cnt, (void *)&cnt1};
        e = cudaLaunchKernel(akern, dim3((unsigned)a.g.nlines, (unsigned)ceil_div(K, ASM_RB)), dim3(256),
                             args, asm_smem, 0);
        if (e != cudaSuccess) return fail(cuda_fail(e, "assembly launch", __FILE__, __LINE__));
        count_launch(1);
    } else {
        // general reach / degree: raw products, symmetrisation, pattern (three passes)
        box_raw_kernel<<<dim3((unsigned)a.g.nlines, slot_lines), 128>>>(a, b.values);
        box_sym_kernel<<<num_sms() * 8, 256>>>(a.g, b.values);
        box_mask_kernel<<<num_sms() * 8, 256>>>(a.g, b.values, b.mask, cnt, cnt + 1);
        box_full_kernel<<<num_sms() * 8, 256>>>(a.g, b.mask, b.full);
        count_launch(4);
    }
    unsigned long long host[2];
    e = cudaMemcpy(host, cnt, sizeof host, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(cuda_fail(e, "assembly", __FILE__, __LINE__));
    LP_CUDA(cudaMemset(m->flags, 0, b.n * sizeof(int)));
    dfree(dhats);
    dfree(dblocks);
    dfree(cnt);
    b.nnz = (int64_t)host[0];
    m->nnz = b.nnz;
    if (b.nnz == 0) {
        lp_ilu_destroy(m);
        set_error("assembled preconditioner has no nonzero entries");
        return LP_ERR_ARG;
    }
    // a row without a stored diagonal is reported by lp_ilu0 (IluZeroPivotError(i))
    m->missing_diag = host[1] != ~0ull ? (int64_t)host[1] : -1;
    *out = m;
    return LP_OK;
}
