"""Slab-sharded 3-D matvec over G ranks.

Vectors (K^3, x fastest) are split into z-slabs, rank g holding planes
[z0_g, z0_g + nz_g).  ``apply_system`` (operator.py:204-210) then runs as three
compute stages between three all-to-alls (csrc/slab.cu has the layouts):

  S1 S2 on the z-slab            -> 3 fields [y'][x'][z_g]      E1: y'-slabs
  S3 (+ grids) B1 on a y'-slab   -> 3 fields [kx][z'][y'_g]     E2: kx-slabs
  B2 B3 on a kx-slab             -> [kz][ky][kx_g]              E3: z-slabs

Each rank's chunk for rank h is contiguous (the distributed axis is the
slowest), so the exchanges are plain ``all_to_all_single`` calls over NCCL
(NVLink/NVSwitch); ``lp_copy2d`` drops each received chunk into place.  Every
line is computed by the same kernel as on one GPU, so the sharded matvec is
bit-identical to ``apply_system``.

``SlabMatvec`` holds the per-rank schedule; ``apply_local`` runs all G ranks
in one process on one device with the exchanges done as device copies (the
single-GPU emulation used by the GPU tests), ``apply_rank`` is one rank of a
torch.distributed job.  PCG dot products across ranks use
``distributed.ordered_dd_allreduce``.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib


def slab_bounds(n, G):
    """Balanced contiguous split of range(n) into G parts: list of (start, count)."""
    base, extra = divmod(n, G)
    out, s = [], 0
    for g in range(G):
        c = base + (1 if g < extra else 0)
        out.append((s, c))
        s += c
    return out


@dataclass
class Schedule:
    K: int
    P: int
    G: int

    def __post_init__(self):
        if self.G < 1 or self.G > self.K:
            raise ValueError(f"cannot split {self.K} planes over {self.G} ranks")
        self.z = slab_bounds(self.K, self.G)    # vectors and E3
        self.y = slab_bounds(self.P, self.G)    # middle stage (y' nodes)
        self.kx = slab_bounds(self.K, self.G)   # backward stage (kx modes)

    # element counts of the chunks rank g sends to rank h in each exchange
    def e1(self, g, h):
        return self.y[h][1] * self.P * self.z[g][1]

    def e2(self, g, h):
        return self.kx[h][1] * self.P * self.y[g][1]

    def e3(self, g, h):
        return self.z[h][1] * self.K * self.kx[g][1]


class SlabMatvec:
    """(A+B) u for z-slab sharded u, on the device of the calling process."""

    device = "cuda"

    def __init__(self, spec, plan, G, which=3):
        if spec.dim != 3:
            raise ValueError("slab sharding is for the 3-D operator")
        import torch
        self.torch = torch
        self.which = which
        self.s = Schedule(spec.n_modes, plan.order, G)
        self._setup(spec, plan)

    def _setup(self, spec, plan):
        self.lib = _lib.load()
        self.op = spec.device_operator(plan)

    # ---------------------------------------------------------------- stages
    def _empty(self, n):
        return self.torch.empty(max(n, 1), dtype=self.torch.float64, device=self.device)

    def stage1(self, g, u_slab):
        s = self.s
        nz = s.z[g][1]
        f = [self._empty(s.P * s.P * nz) for _ in range(3)]
        _lib.check(self.lib.lp_slab_forward(self.op, self.which, nz, u_slab.data_ptr(),
                                            f[0].data_ptr(), f[1].data_ptr(), f[2].data_ptr(),
                                            _lib.stream_ptr()), "slab forward")
        return f

    def stage2(self, h, f_in):
        s = self.s
        y0, ny = s.y[h]
        w = [self._empty(s.K * s.P * ny) for _ in range(3)]
        _lib.check(self.lib.lp_slab_middle(self.op, self.which, y0, ny, f_in[0].data_ptr(),
                                           f_in[1].data_ptr(), f_in[2].data_ptr(),
                                           w[0].data_ptr(), w[1].data_ptr(), w[2].data_ptr(),
                                           _lib.stream_ptr()), "slab middle")
        return w

    def stage3(self, h, w_in):
        s = self.s
        nkx = s.kx[h][1]
        out = self._empty(s.K * s.K * nkx)
        _lib.check(self.lib.lp_slab_backward(self.op, self.which, nkx, w_in[0].data_ptr(),
                                             w_in[1].data_ptr(), w_in[2].data_ptr(),
                                             out.data_ptr(), _lib.stream_ptr()), "slab backward")
        return out

    # ------------------------------------------------------------- placement
    def _copy2d(self, rows, cols, src, dst, col, ld):
        _lib.check(self.lib.lp_copy2d(rows, cols, src.data_ptr(), cols, dst.data_ptr() + 8 * col,
                                      ld, _lib.stream_ptr()), "copy2d")

    def _place(self, chunks, rows_of, cols_of, ld, n_out):
        """Received chunks (one per source rank, [rows][cols_g]) -> [rows][ld] at col offsets."""
        out = self._empty(n_out)
        col = 0
        for g, c in enumerate(chunks):
            cols = cols_of(g)
            if cols and rows_of:
                self._copy2d(rows_of, cols, c, out, col, ld)
            col += cols
        return out

    def place_e1(self, h, chunks):
        s = self.s
        ny = s.y[h][1]
        return self._place(chunks, ny * s.P, lambda g: s.z[g][1], s.K, ny * s.P * s.K)

    def place_e2(self, h, chunks):
        s = self.s
        nkx = s.kx[h][1]
        return self._place(chunks, nkx * s.P, lambda g: s.y[g][1], s.P, nkx * s.P * s.P)

    def place_e3(self, h, chunks):
        s = self.s
        nz = s.z[h][1]
        return self._place(chunks, nz * s.K, lambda g: s.kx[g][1], s.K, nz * s.K * s.K)

    @staticmethod
    def split(t, sizes):
        out, o = [], 0
        for n in sizes:
            out.append(t[o:o + n])
            o += n
        return out

    # ----------------------------------------------------------- schedules
    def apply_local(self, u_slabs):
        """All G ranks in this process (single-device emulation of the exchanges)."""
        s, G = self.s, self.s.G
        f = [self.stage1(g, u_slabs[g]) for g in range(G)]
        sent = [[self.split(f[g][k], [s.e1(g, h) for h in range(G)]) for k in range(3)]
                for g in range(G)]
        mid = [[self.place_e1(h, [sent[g][k][h] for g in range(G)]) for k in range(3)]
               for h in range(G)]
        w = [self.stage2(h, mid[h]) for h in range(G)]
        sent = [[self.split(w[g][k], [s.e2(g, h) for h in range(G)]) for k in range(3)]
                for g in range(G)]
        back = [[self.place_e2(h, [sent[g][k][h] for g in range(G)]) for k in range(3)]
                for h in range(G)]
        o = [self.stage3(h, back[h]) for h in range(G)]
        sent = [self.split(o[g], [s.e3(g, h) for h in range(G)]) for g in range(G)]
        return [self.place_e3(h, [sent[g][h] for g in range(G)]) for h in range(G)]

    def apply_rank(self, rank, u_slab, group=None):
        """One rank of a torch.distributed job: three NCCL all-to-alls."""
        import torch.distributed as dist
        s, G = self.s, self.s.G

        def exchange(t, send_sizes, recv_sizes):
            recv = self._empty(sum(recv_sizes))
            dist.all_to_all_single(recv[:sum(recv_sizes)], t[:sum(send_sizes)],
                                   output_split_sizes=recv_sizes,
                                   input_split_sizes=send_sizes, group=group)
            return self.split(recv, recv_sizes)

        f = self.stage1(rank, u_slab)
        mid = [self.place_e1(rank, exchange(f[k], [s.e1(rank, h) for h in range(G)],
                                            [s.e1(g, rank) for g in range(G)])) for k in range(3)]
        w = self.stage2(rank, mid)
        back = [self.place_e2(rank, exchange(w[k], [s.e2(rank, h) for h in range(G)],
                                             [s.e2(g, rank) for g in range(G)])) for k in range(3)]
        o = self.stage3(rank, back)
        return self.place_e3(rank, exchange(o, [s.e3(rank, h) for h in range(G)],
                                            [s.e3(g, rank) for g in range(G)]))


def split_vector(u_flat, K, G):
    """z-slabs (views) of an x-fastest K^3 vector."""
    return [u_flat[z0 * K * K:(z0 + nz) * K * K] for z0, nz in slab_bounds(K, G)]


# ------------------------------------------------------------------ PCG

def _dd_add(x, y):
    from .distributed import dd_add
    return dd_add(x, y)


class SlabSweeps:
    """The ILU(0) sweeps with the vector over G y-slab ranks (lp_sweep_ranks):
    rank v owns the x-lines with y in its slab of [0, K) and a replica of the
    vector; every line is published to its owner and to the ranks whose
    stencil halo (+-r lines) reaches it.  Emulated on one device."""

    def __init__(self, factors, K, G):
        import torch
        self.torch = torch
        self.lib = _lib.load()
        self.f = factors
        self.K, self.G = K, G
        self.ys = [z0 for z0, _ in slab_bounds(K, G)] + [K]
        import ctypes
        self._ys = (ctypes.c_int * (G + 1))(*self.ys)
        n = K ** 3
        self.yrep = torch.empty(G * n, dtype=torch.float64, device="cuda")
        self.zrep = torch.empty(G * n, dtype=torch.float64, device="cuda")

    def apply(self, r_full):
        """z = M^-1 r; r_full is the assembled residual (what the y-slab owners
        hold after the z-slab -> y-slab exchange); returns the assembled z."""
        lib, K, G = self.lib, self.K, self.G
        _lib.check(lib.lp_sweep_ranks(self.f._handle, G, self._ys, 0, r_full.data_ptr(), 0,
                                      self.yrep.data_ptr(), _lib.stream_ptr()), "forward sweep")
        _lib.check(lib.lp_sweep_ranks(self.f._handle, G, self._ys, 1, self.yrep.data_ptr(), 1,
                                      self.zrep.data_ptr(), _lib.stream_ptr()), "backward sweep")
        return self.gather(self.zrep)

    def gather(self, reps):
        """Each rank's own lines from its replica -> one x-fastest vector."""
        K, G = self.K, self.G
        n = K ** 3
        out = self.torch.empty(n, dtype=self.torch.float64, device="cuda")
        for v in range(G):
            y0, ny = self.ys[v], self.ys[v + 1] - self.ys[v]
            _lib.check(self.lib.lp_copy2d(K, ny * K, reps.data_ptr() + 8 * (v * n + y0 * K), K * K,
                                          out.data_ptr() + 8 * y0 * K, K * K, _lib.stream_ptr()),
                       "gather")
        return out


def ilu0_sharded_local(matrices, pivot_tol=1e-300):
    """ILU(0) over G y-slab ranks, emulated on one device (``lp_ilu0_ranks``):
    ``matrices[v]`` is rank v's assembled M (``assemble_M`` of the same problem,
    one per rank, as each GPU of a multi-GPU run assembles its own).  Every
    rank factors the x-lines with y in its slab in its own factor array,
    reading its neighbours' rows of the r halo lines from the copies they
    stored there (sparse.py:116-139 per row).  Returns one
    ``IluFactors`` per rank: the rows of the rank's slab equal the single-GPU
    factors bit for bit; rows outside its slab are not factors."""
    import ctypes
    from .sparse import IluFactors, IluZeroPivotError
    G = len(matrices)
    K = round(matrices[0].n ** (1.0 / 3.0))
    ys = [y0 for y0, _ in slab_bounds(K, G)] + [K]
    cys = (ctypes.c_int * (G + 1))(*ys)
    hs = (ctypes.c_void_p * G)(*[m._handle for m in matrices])
    bad = ctypes.c_int64(-1)
    rc = _lib.load().lp_ilu0_ranks(hs, G, cys, pivot_tol, ctypes.byref(bad), _lib.stream_ptr())
    if rc == _lib.LP_ERR_ZERO_PIVOT:
        raise IluZeroPivotError(int(bad.value))
    _lib.check(rc, "ilu0 (y-slab ranks)")
    return [IluFactors(m, m._handle) for m in matrices], ys


def ilu0_rank(matrix, rank, G, group=None, pivot_tol=1e-300):
    """This process's part of the ILU(0) over G y-slab ranks (one process per
    GPU, ``lp_ilu0_rank``): ``matrix`` is this rank's assembled M.  The ranks
    exchange the CUDA IPC handles of their factor and flag arrays, map their
    slab neighbours', synchronise and factor concurrently; a finished halo row
    is stored into the neighbour's array over NVLink, followed by its flag.
    Returns this rank's ``IluFactors`` (its slab's rows are the single-GPU
    factors bit for bit)."""
    import ctypes

    import torch.distributed as dist
    from .sparse import IluFactors, IluZeroPivotError
    lib = _lib.load()
    K = round(matrix.n ** (1.0 / 3.0))
    ys = [y0 for y0, _ in slab_bounds(K, G)] + [K]
    cys = (ctypes.c_int * (G + 1))(*ys)
    lu, fl = ctypes.c_void_p(), ctypes.c_void_p()
    h_lu, h_fl = (ctypes.c_ubyte * 64)(), (ctypes.c_ubyte * 64)()
    _lib.check(lib.lp_ilu_rank_arrays(matrix._handle, ctypes.byref(lu), ctypes.byref(fl), h_lu, h_fl),
               "rank arrays")
    allh = [None] * G
    dist.all_gather_object(allh, (bytes(h_lu), bytes(h_fl)), group=group)
    peer_lu, peer_fl, opened = (ctypes.c_void_p * G)(), (ctypes.c_void_p * G)(), []
    for v in range(G):
        if abs(v - rank) == 1:
            for which, dst in ((0, peer_lu), (1, peer_fl)):
                p = ctypes.c_void_p()
                hb = (ctypes.c_ubyte * 64).from_buffer_copy(allh[v][which])
                _lib.check(lib.lp_ipc_open(hb, ctypes.byref(p)), "ipc open")
                dst[v] = p.value
                opened.append(p.value)
    bad = ctypes.c_int64(-1)
    rc = lib.lp_ilu0_rank_prepare(matrix._handle, ctypes.byref(bad), _lib.stream_ptr())
    dist.barrier(group=group)   # every rank's arrays are ready before any halo store
    if rc == _lib.LP_OK:
        rc = lib.lp_ilu0_rank(matrix._handle, G, cys, rank, peer_lu, peer_fl, pivot_tol,
                              ctypes.byref(bad), _lib.stream_ptr())
    dist.barrier(group=group)   # the neighbours are done storing into this rank's arrays
    for p in opened:
        lib.lp_ipc_close(p)
    if rc == _lib.LP_ERR_ZERO_PIVOT:
        raise IluZeroPivotError(int(bad.value))
    _lib.check(rc, "ilu0 (rank)")
    return IluFactors(matrix, matrix._handle)


# ------------------------------------------------------------ PCG driver
#
# One PCG loop (pcg.py:145-164) written against per-slab operations, run either
# by one process for all G ranks (LocalOps: the one-device emulation) or by
# each process of a torch.distributed job for its own rank (RankOps).  Vectors
# are lists of this process's z-slabs; dots are per-slab double-double partials
# combined in rank order (a plain loop locally, ordered_dd_allreduce across
# processes), so both paths produce the same bits.


def pcg_loop(ops, config, f):
    """Algorithm 1 over ops (this process's slabs).  Returns (x slabs, report)."""
    import math
    x = ops.zeros()
    r = ops.copy(f)
    p = ops.empty()
    fnorm = math.sqrt(ops.dot(f, f))
    rr = ops.dot(r, r)
    hist = [math.sqrt(rr)]
    tol = config.epsilon * fnorm
    it, rho_old = 0, None
    while math.sqrt(rr) > tol and it < config.k_max:
        z = ops.precond(r)
        it += 1
        rho = ops.dot(r, z)
        beta = 0.0 if it == 1 else rho / rho_old
        ops.update_p(z, p, beta, it == 1)
        w = ops.matvec(p)
        curv = ops.dot(p, w)
        if curv <= 0.0:
            from .pcg import IndefiniteOperatorError
            raise IndefiniteOperatorError(it, curv)
        rr = ops.update_xr(x, r, p, w, rho / curv)
        rho_old = rho
        hist.append(math.sqrt(rr))
    return x, {"iterations": it, "converged": math.sqrt(rr) <= tol,
               "final_relative_residual": math.sqrt(rr) / fnorm if fnorm else 0.0,
               "residual_history": hist, "ranks": ops.G}


class _GpuSlabOps:
    """Per-slab vector kernels (lp_dot, lp_update_p, lp_update_xr) on CUDA slabs."""

    def __init__(self, K, G, sizes):
        import torch
        self.torch = torch
        self.lib = _lib.load()
        self.K, self.G = K, G
        self.sizes = sizes                          # this process's slab lengths
        self._two = torch.empty(2, dtype=torch.float64, device="cuda")

    def _new(self):
        return [self.torch.empty(max(c, 1), dtype=self.torch.float64, device="cuda")[:c]
                for c in self.sizes]

    def zeros(self):
        return [t.zero_() for t in self._new()]

    def empty(self):
        return self._new()

    def copy(self, v):
        return [t.clone() for t in v]

    def _partial(self, a, b):
        _lib.check(self.lib.lp_dot(a.numel(), a.data_ptr(), b.data_ptr(), self._two.data_ptr(),
                                   _lib.stream_ptr()), "dot")
        h = self._two.cpu().numpy()
        return float(h[0]), float(h[1])

    def dot(self, a, b):
        return self.combine([self._partial(u, v) for u, v in zip(a, b)])[0]

    def update_p(self, z, p, beta, first):
        for zs, ps in zip(z, p):
            _lib.check(self.lib.lp_update_p(zs.numel(), zs.data_ptr(), ps.data_ptr(), beta,
                                            int(first), _lib.stream_ptr()), "update p")

    def update_xr(self, x, r, p, w, alpha):
        parts = []
        for xs, rs, ps, ws in zip(x, r, p, w):
            _lib.check(self.lib.lp_update_xr(xs.numel(), xs.data_ptr(), rs.data_ptr(), ps.data_ptr(),
                                             ws.data_ptr(), alpha, self._two.data_ptr(),
                                             _lib.stream_ptr()), "update x r")
            h = self._two.cpu().numpy()
            parts.append((float(h[0]), float(h[1])))
        return self.combine(parts)[0]


class LocalOps(_GpuSlabOps):
    """All G ranks in this process on one device (exchanges as device copies,
    the sweeps' halo publication in one launch, lp_sweep_ranks)."""

    def __init__(self, spec, plan, G, factors):
        K = spec.n_modes
        super().__init__(K, G, [nz * K * K for _, nz in slab_bounds(K, G)])
        self.sm = SlabMatvec(spec, plan, G)
        self.sw = SlabSweeps(factors, K, G) if factors is not None else None

    def combine(self, parts):
        acc = (0.0, 0.0)
        for pr in parts:
            acc = _dd_add(acc, pr)
        return acc

    def matvec(self, p):
        return [o[:c] for o, c in zip(self.sm.apply_local(p), self.sizes)]

    def precond(self, r):
        if self.sw is None:
            return r
        z = self.sw.apply(self.torch.cat(r))
        return SlabMatvec.split(z, self.sizes)


class RankSweeps:
    """The ILU(0) sweeps of one rank of a multi-GPU run: the residual's
    z-slab -> y-slab redistribution (one all-to-all), the forward and backward
    sweeps over this rank's y-slab lines with halo lines stored straight into
    the neighbours' replicas (lp_sweep_rank, CUDA IPC peer mappings), and the
    y-slab -> z-slab redistribution of z (one all-to-all).

    Replicas are full-length vectors (n values) addressed by global row; only
    the rank's own lines and its +-r halo lines are meaningful.  Per iteration
    a rank sends and receives (G-1)/G of its z-slab twice (r and z) and, during
    each sweep, r K values per plane to each neighbour (the halo lines)."""

    def __init__(self, factors, K, G, rank, group=None):
        import ctypes

        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.ctypes = torch, dist, ctypes
        self.f, self.K, self.G, self.rank, self.group = factors, K, G, rank, group
        self.z = slab_bounds(K, G)
        self.y = slab_bounds(K, G)
        self.ys = [y0 for y0, _ in self.y] + [K]
        self.n = K ** 3
        self._setup()

    # ------------------------------------------------------ device hooks
    def _setup(self):
        ctypes = self.ctypes
        self.lib = _lib.load()
        self._ys = (ctypes.c_int * (self.G + 1))(*self.ys)
        # replicas: rhs (r, own lines), forward output y, backward output z
        self.bufs, handles = [], []
        for _ in range(3):
            ptr = ctypes.c_void_p()
            h = (ctypes.c_ubyte * 64)()
            _lib.check(self.lib.lp_ipc_alloc(8 * self.n, ctypes.byref(ptr), h), "ipc alloc")
            self.bufs.append(ptr.value)
            handles.append(bytes(h))
        allh = [None] * self.G
        self.dist.all_gather_object(allh, handles, group=self.group)
        self.peers = []   # [buffer][rank] -> mapped pointer (own: local buffer)
        self._opened = []
        for b in range(3):
            row = (ctypes.c_void_p * self.G)()
            for v in range(self.G):
                if v == self.rank:
                    row[v] = self.bufs[b]
                elif abs(v - self.rank) == 1:
                    p = ctypes.c_void_p()
                    hb = (ctypes.c_ubyte * 64).from_buffer_copy(allh[v][b])
                    _lib.check(self.lib.lp_ipc_open(hb, ctypes.byref(p)), "ipc open")
                    row[v] = p.value
                    self._opened.append(p.value)
            self.peers.append(row)

    def close(self):
        for p in self._opened:
            self.lib.lp_ipc_close(p)
        for p in self.bufs:
            self.lib.lp_ipc_free(p)
        self._opened, self.bufs = [], []

    def _empty(self, n):
        return self.torch.empty(max(n, 1), dtype=self.torch.float64, device="cuda")

    @staticmethod
    def _addr(buf, off):
        return (buf if isinstance(buf, int) else buf.data_ptr()) + 8 * off

    def _copy2d(self, rows, cols, src, soff, lds, dst, doff, ldd):
        _lib.check(self.lib.lp_copy2d(rows, cols, self._addr(src, soff), lds, self._addr(dst, doff),
                                      ldd, _lib.stream_ptr()), "copy2d")

    def _prefill(self):
        # both output replicas hold the sentinel before any rank starts sweeping
        st = _lib.stream_ptr()
        for b in self.bufs[1:]:
            _lib.check(self.lib.lp_sweep_prefill(self.n, b, st), "prefill")

    def _sweeps(self):
        lib, h, st = self.lib, self.f._handle, _lib.stream_ptr()
        rrep, yrep, zrep = self.bufs
        _lib.check(lib.lp_sweep_rank(h, self.G, self._ys, self.rank, 0, rrep, yrep, self.peers[1],
                                     st), "forward sweep")
        _lib.check(lib.lp_sweep_rank(h, self.G, self._ys, self.rank, 1, yrep, zrep, self.peers[2],
                                     st), "backward sweep")

    # ------------------------------------------------------------ schedule
    def _exchange(self, send, send_sizes, recv_sizes):
        recv = self._empty(sum(recv_sizes))
        self.dist.all_to_all_single(recv[:sum(recv_sizes)], send[:sum(send_sizes)],
                                    output_split_sizes=recv_sizes, input_split_sizes=send_sizes,
                                    group=self.group)
        return recv

    def apply(self, r_slab):
        """z = M^-1 r on this rank's z-slab of r (x fastest); returns its z-slab of z."""
        K, me = self.K, self.rank
        nz = self.z[me][1]
        y0, ny = self.y[me]
        rrep, zrep = self.bufs[0], self.bufs[2]
        self._prefill()
        # z -> y: to rank h the rows (my planes, h's lines): [nz][ny_h][K]
        send_sizes = [nz * nyh * K for _, nyh in self.y]
        recv_sizes = [nzg * ny * K for _, nzg in self.z]
        send = self._empty(sum(send_sizes))
        o = 0
        for (yh, nyh), c in zip(self.y, send_sizes):
            if c:
                self._copy2d(nz, nyh * K, r_slab, yh * K, K * K, send, o, nyh * K)
            o += c
        recv = self._exchange(send, send_sizes, recv_sizes)
        o = 0
        for (zg, nzg), c in zip(self.z, recv_sizes):
            if c:
                self._copy2d(nzg, ny * K, recv, o, ny * K, rrep, (zg * K + y0) * K, K * K)
            o += c
        self._sweeps()
        # y -> z: to rank g my lines of its planes: [nz_g][ny][K]
        send_sizes, recv_sizes = recv_sizes, send_sizes
        send = self._empty(sum(send_sizes))
        o = 0
        for (zg, nzg), c in zip(self.z, send_sizes):
            if c:
                self._copy2d(nzg, ny * K, zrep, (zg * K + y0) * K, K * K, send, o, ny * K)
            o += c
        recv = self._exchange(send, send_sizes, recv_sizes)
        z = self._empty(nz * K * K)[:nz * K * K]
        o = 0
        for (yh, nyh), c in zip(self.y, recv_sizes):
            if c:
                self._copy2d(nz, nyh * K, recv, o, nyh * K, z, yh * K, K * K)
            o += c
        return z


class RankOps(_GpuSlabOps):
    """This process's rank of a torch.distributed job (one GPU per rank):
    z-slab matvec with three NCCL all-to-alls, y-slab sweeps with peer halo
    stores, dots combined with ordered_dd_allreduce."""

    def __init__(self, spec, plan, factors, rank, G, group=None):
        K = spec.n_modes
        super().__init__(K, G, [slab_bounds(K, G)[rank][1] * K * K])
        self.rank, self.group = rank, group
        self.sm = SlabMatvec(spec, plan, G)
        self.sw = RankSweeps(factors, K, G, rank, group) if factors is not None else None

    def combine(self, parts):
        from .distributed import ordered_dd_allreduce
        acc = (0.0, 0.0)
        for pr in parts:
            acc = _dd_add(acc, pr)
        return ordered_dd_allreduce(acc[0], acc[1], device="cuda")

    def matvec(self, p):
        return [self.sm.apply_rank(self.rank, p[0], self.group)[:self.sizes[0]]]

    def precond(self, r):
        return [self.sw.apply(r[0])] if self.sw is not None else r

    def close(self):
        if self.sw is not None:
            self.sw.close()


def pcg_solve_sharded_local(spec, config, plan, f_flat, G, factors=None):
    """PCG (pcg.py:111-179) with every stage distributed over G ranks, emulated
    on one device: the matvec z-slab sharded (SlabMatvec, three all-to-alls),
    the sweeps over y-slab ranks with halo publication (SlabSweeps), vector
    updates per z-slab (lp_update_p / lp_update_xr) and the three dots per
    iteration as per-slab double-double partials combined in rank order (what
    ordered_dd_allreduce does across processes).  Returns (x_full, report)."""
    import torch
    from .pcg import setup_preconditioner
    if factors is None:
        factors = setup_preconditioner(spec, config, plan)
    ops = LocalOps(spec, plan, G, factors)
    x, rep = pcg_loop(ops, config, SlabMatvec.split(f_flat, ops.sizes))
    return torch.cat(x), rep


def pcg_solve_sharded_rank(spec, config, plan, f_slab, factors=None, group=None):
    """One rank of the distributed PCG under torch.distributed (torchrun, one
    GPU per rank, NCCL): f_slab is this rank's z-slab of F (x fastest);
    returns (this rank's z-slab of x, report).  Every rank factors M itself
    (the factors are replicated; each rank's sweeps read only its own lines)."""
    import torch.distributed as dist
    from .pcg import setup_preconditioner
    G = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if factors is None:
        factors = setup_preconditioner(spec, config, plan)
    ops = RankOps(spec, plan, factors, rank, G, group)
    try:
        x, rep = pcg_loop(ops, config, [f_slab])
    finally:
        ops.close()
    return x[0], rep
