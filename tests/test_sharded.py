"""Slab-sharded 3-D matvec (paper_2004_13961_b200/sharded.py, csrc/slab.cu).

CPU (gloo, world_size 2): the exchange schedule -- chunk sizes, all-to-all
splits, placement of received chunks -- run with numpy stand-ins for the three
compute stages (the same sum-factorised passes, test-only), checked against the
CPU oracle's apply_system.  GPU: the CUDA stages, with the exchanges emulated
on one device, are bit-identical to the single-GPU apply_system."""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import legpcg_port as orc
from paper_2004_13961_b200 import ProblemSpec, workloads as wl
from paper_2004_13961_b200.sharded import Schedule, SlabMatvec, slab_bounds


def spec_of(w, N):
    return ProblemSpec(dim=w.dim, N=N, beta=w.beta, alpha=w.alpha)


class NumpySlab(SlabMatvec):
    """The stages of csrc/slab.cu restated with numpy einsum on CPU tensors."""

    device = "cpu"

    def _setup(self, spec, plan):
        s = self.s
        K, P = s.K, s.P
        op = orc.Plan(P)
        V = op.table
        self.F = V[:, :K] - V[:, 2:K + 2]                                   # phi_k(x_i)
        self.D = V[:, 1:K + 1] * (-(2.0 * np.arange(K) + 3.0))              # phi_k'(x_i)
        w3 = np.einsum("i,j,l->ijl", op.weights, op.weights, op.weights)
        b = orc.grid(spec, op, "beta") * w3                                 # [x][y][z]
        self.bw = np.ascontiguousarray(b.transpose(2, 1, 0))               # [z][y][x]
        self.aw = None
        if spec.alpha is not None and not spec.alpha.is_zero:
            a = np.broadcast_to(orc.grid(spec, op, "alpha"), (P, P, P)) * w3
            self.aw = np.ascontiguousarray(a.transpose(2, 1, 0))

    def _t(self, a):
        return torch.from_numpy(np.ascontiguousarray(a).reshape(-1).copy())

    def stage1(self, g, u_slab):
        s, F, D = self.s, self.F, self.D
        u = u_slab.numpy().reshape(s.z[g][1], s.K, s.K)                     # [z][y][x]
        g0 = np.einsum("ax,zyx->azy", F, u)
        g1 = np.einsum("ax,zyx->azy", D, u)
        return [self._t(np.einsum("by,azy->baz", F, g1)), self._t(np.einsum("by,azy->baz", D, g0)),
                self._t(np.einsum("by,azy->baz", F, g0))]

    def stage2(self, h, f_in):
        s, F, D = self.s, self.F, self.D
        y0, ny = s.y[h]
        f = [t.numpy().reshape(ny, s.P, s.K) for t in f_in]                 # [y'][x'][z]
        bw = self.bw[:, y0:y0 + ny, :]
        q0 = np.einsum("cz,yxz->cyx", F, f[0]) * bw
        q1 = np.einsum("cz,yxz->cyx", F, f[1]) * bw
        q2 = np.einsum("cz,yxz->cyx", D, f[2]) * bw
        w0 = np.einsum("xk,cyx->kcy", D, q0)
        if self.aw is not None:
            w0 = w0 + np.einsum("xk,cyx->kcy", F, np.einsum("cz,yxz->cyx", F, f[2])
                                * self.aw[:, y0:y0 + ny, :])
        return [self._t(w0), self._t(np.einsum("xk,cyx->kcy", F, q1)),
                self._t(np.einsum("xk,cyx->kcy", F, q2))]

    def stage3(self, h, w_in):
        s, F, D = self.s, self.F, self.D
        nkx = s.kx[h][1]
        w = [t.numpy().reshape(nkx, s.P, s.P) for t in w_in]               # [kx][z'][y']
        v0 = np.einsum("yk,xcy->kxc", F, w[0]) + np.einsum("yk,xcy->kxc", D, w[1])
        v1 = np.einsum("yk,xcy->kxc", F, w[2])
        return self._t(np.einsum("ck,yxc->kyx", F, v0) + np.einsum("ck,yxc->kyx", D, v1))

    def _copy2d(self, rows, cols, src, dst, col, ld):
        dst[:rows * ld].view(rows, ld)[:, col:col + cols] = src[:rows * cols].view(rows, cols)


def _problem(name="cfg5", N=14, seed=3):
    w = wl.CONFIGS[name]()
    spec = spec_of(w, N)
    K = N - 1
    u = np.random.default_rng(seed).standard_normal((K, K, K))             # oracle: [x][y][z]
    ref = orc.apply_system(spec, orc.Plan(N + 1), u)
    flat = np.ascontiguousarray(u.transpose(2, 1, 0)).reshape(-1)           # x fastest
    ref_flat = np.ascontiguousarray(ref.transpose(2, 1, 0)).reshape(-1)
    return w, spec, flat, ref_flat


def _slabs(flat, K, G):
    return [torch.from_numpy(flat[z0 * K * K:(z0 + nz) * K * K].copy()) for z0, nz in slab_bounds(K, G)]


def relerr(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_schedule_chunk_sizes():
    for K, G in [(13, 1), (13, 2), (13, 3), (127, 8), (511, 8), (9, 9)]:
        s = Schedule(K, K + 2, G)
        for g in range(G):
            assert sum(s.e1(g, h) for h in range(G)) == s.P * s.P * s.z[g][1]
            assert sum(s.e2(g, h) for h in range(G)) == s.K * s.P * s.y[g][1]
            assert sum(s.e3(g, h) for h in range(G)) == s.K * s.K * s.kx[g][1]
        for h in range(G):
            assert sum(s.e1(g, h) for g in range(G)) == s.y[h][1] * s.P * s.K
    with pytest.raises(ValueError):
        Schedule(4, 6, 5)


@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_sharded_schedule_numpy_local(name, G):
    w, spec, flat, ref = _problem(name, N=12)
    K = spec.n_modes
    sm = _numpy_slab(spec, G)
    out = torch.cat(sm.apply_local(_slabs(flat, K, G))).numpy()
    assert relerr(out, ref) < 1e-12


def _numpy_slab(spec, G):
    sm = NumpySlab.__new__(NumpySlab)
    sm.torch = torch
    sm.which = 3
    sm.s = Schedule(spec.n_modes, spec.N + 1, G)
    sm._setup(spec, None)
    return sm


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    from paper_2004_13961_b200 import distributed as Dm
    dist = Dm.init("gloo")
    try:
        w, spec, flat, ref = _problem("cfg5", N=14)
        K = spec.n_modes
        sm = _numpy_slab(spec, ws)
        mine = sm.apply_rank(rank, _slabs(flat, K, ws)[rank])
        out[rank] = mine[:K * K * slab_bounds(K, ws)[rank][1]].numpy().tobytes()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(240)
def test_gloo_two_ranks_sharded_matvec():
    ws = 2
    port = _free_port()
    import torch.multiprocessing as mp
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
        res = dict(out)
    got = np.concatenate([np.frombuffer(res[r], dtype=np.float64) for r in range(ws)])
    w, spec, flat, ref = _problem("cfg5", N=14)
    assert relerr(got, ref) < 1e-12
    # the exchanges over gloo give exactly the single-process schedule's bits
    local = torch.cat(_numpy_slab(spec, ws).apply_local(_slabs(flat, spec.n_modes, ws))).numpy()
    assert np.array_equal(got, local)


# ------------------------------------------------ distributed PCG (numpy stand-ins)

from paper_2004_13961_b200.distributed import dd_add, dd_of  # noqa: E402
from paper_2004_13961_b200.sharded import RankSweeps, SlabMatvec, pcg_loop  # noqa: E402


class _NumpyVecOps:
    """Per-slab vector operations on CPU tensors with sequential double-double
    dots (a stand-in for lp_dot / lp_update_p / lp_update_xr)."""

    def zeros(self):
        return [torch.zeros(c, dtype=torch.float64) for c in self.sizes]

    def empty(self):
        return [torch.empty(c, dtype=torch.float64) for c in self.sizes]

    def copy(self, v):
        return [t.clone() for t in v]

    def dot(self, a, b):
        return self.combine([dd_of((u * v).numpy()) for u, v in zip(a, b)])[0]

    def update_p(self, z, p, beta, first):
        for zs, ps in zip(z, p):
            ps.copy_(zs if first else zs + beta * ps)

    def update_xr(self, x, r, p, w, alpha):
        for xs, rs, ps, ws in zip(x, r, p, w):
            xs.add_(alpha * ps)
            rs.sub_(alpha * ws)
        return self.combine([dd_of((rs * rs).numpy()) for rs in r])[0]


def _oracle_precond(spec, T):
    fac = orc.ilu0(orc.assemble_M(spec, T, T))
    return lambda r: torch.from_numpy(np.asarray(orc.precond_apply(fac, r.numpy()), dtype=np.float64))


class NumpyLocalOps(_NumpyVecOps):
    def __init__(self, spec, T, G):
        K = spec.n_modes
        self.G = G
        self.sizes = [nz * K * K for _, nz in slab_bounds(K, G)]
        self.sm = _numpy_slab(spec, G)
        self.pre = _oracle_precond(spec, T)

    def combine(self, parts):
        acc = (0.0, 0.0)
        for pr in parts:
            acc = dd_add(acc, pr)
        return acc

    def matvec(self, p):
        return [o[:c] for o, c in zip(self.sm.apply_local(p), self.sizes)]

    def precond(self, r):
        return SlabMatvec.split(self.pre(torch.cat(r)), self.sizes)


class NumpyRankSweeps(RankSweeps):
    """RankSweeps' redistribution schedule on CPU tensors; the sweeps themselves
    by the oracle on the rank-summed residual (each rank contributes its lines)."""

    def _setup(self):
        self.bufs = [torch.zeros(self.n, dtype=torch.float64) for _ in range(3)]

    def close(self):
        pass

    def _empty(self, n):
        return torch.empty(max(n, 1), dtype=torch.float64)

    def _copy2d(self, rows, cols, src, soff, lds, dst, doff, ldd):
        s = src[soff:soff + (rows - 1) * lds + cols].as_strided((rows, cols), (lds, 1))
        d = dst[doff:doff + (rows - 1) * ldd + cols].as_strided((rows, cols), (ldd, 1))
        d.copy_(s)

    def _prefill(self):
        for b in self.bufs:
            b.zero_()

    def _sweeps(self):
        r = self.bufs[0].clone()
        self.dist.all_reduce(r)            # each rank placed only its own lines
        self.bufs[2].copy_(self.pre(r))


class NumpyRankOps(_NumpyVecOps):
    def __init__(self, spec, T, rank, G):
        K = spec.n_modes
        self.G, self.rank = G, rank
        self.sizes = [slab_bounds(K, G)[rank][1] * K * K]
        self.sm = _numpy_slab(spec, G)
        self.sw = NumpyRankSweeps(None, K, G, rank)
        self.sw.pre = _oracle_precond(spec, T)

    def combine(self, parts):
        from paper_2004_13961_b200.distributed import ordered_dd_allreduce
        acc = (0.0, 0.0)
        for pr in parts:
            acc = dd_add(acc, pr)
        return ordered_dd_allreduce(*acc)

    def matvec(self, p):
        return [self.sm.apply_rank(self.rank, p[0])[:self.sizes[0]]]

    def precond(self, r):
        return [self.sw.apply(r[0])]


def _pcg_problem(N=9, T=1):
    from types import SimpleNamespace
    from paper_2004_13961_b200 import SolverConfig
    w = wl.cfg5()
    spec = spec_of(w, N)
    K = N - 1
    F = wl.mass_contract_series(wl.seeded_fhat(3, N + 1))
    f = np.ascontiguousarray(F.transpose(2, 1, 0)).reshape(-1)           # x fastest
    return spec, f, SolverConfig(epsilon=1e-10, preconditioner=(T, T)), K


def _pcg_worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    from paper_2004_13961_b200 import distributed as Dm
    dist = Dm.init("gloo")
    try:
        spec, f, cfg, K = _pcg_problem()
        ops = NumpyRankOps(spec, 1, rank, ws)
        mine = _slabs(f, K, ws)[rank]
        x, rep = pcg_loop(ops, cfg, [mine])
        out[rank] = (x[0].numpy().tobytes(), rep["iterations"], rep["residual_history"])
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_two_ranks_distributed_pcg():
    """The per-rank PCG driver (pcg_loop over RankOps' schedule: z->y and y->z
    redistributions around the sweeps, three all-to-alls per matvec, rank-ordered
    dots) on two gloo processes with numpy stand-ins for the kernels is bit
    for bit the single-process emulation over the same two slabs, and solves
    the system like the CPU oracle."""
    ws = 2
    port = _free_port()
    import torch.multiprocessing as mp
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_pcg_worker, args=(ws, port, out), nprocs=ws, join=True)
        res = dict(out)
    got = np.concatenate([np.frombuffer(res[r][0], dtype=np.float64) for r in range(ws)])
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]
    spec, f, cfg, K = _pcg_problem()
    xl, rl = pcg_loop(NumpyLocalOps(spec, 1, ws), cfg, _slabs(f, K, ws))
    assert np.array_equal(got, torch.cat(xl).numpy())
    assert res[0][1] == rl["iterations"] and res[0][2] == rl["residual_history"]
    # and the oracle's own PCG (x-fastest flat -> [x][y][z])
    F = f.reshape(K, K, K).transpose(2, 1, 0)
    xo, ro = orc.pcg_solve(spec, F, epsilon=cfg.epsilon, preconditioner=cfg.preconditioner)
    xo_flat = np.ascontiguousarray(np.asarray(xo).transpose(2, 1, 0)).reshape(-1)
    assert abs(ro["iterations"] - rl["iterations"]) <= 1
    assert relerr(got, xo_flat) < 1e-10


# ----------------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("name,N", [("cfg4", 24), ("cfg5", 20)])
@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_cuda_stages_bit_identical(name, N, G):
    from paper_2004_13961_b200 import TransformPlan
    from paper_2004_13961_b200.operator import apply_flat
    w = wl.CONFIGS[name]()
    spec = spec_of(w, N)
    plan = TransformPlan(N + 1)
    K = N - 1
    u = torch.randn(K ** 3, dtype=torch.float64, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(7))
    full = apply_flat(spec, plan, 3, u)
    sm = SlabMatvec(spec, plan, G)
    slabs = [u[z0 * K * K:(z0 + nz) * K * K].contiguous() for z0, nz in slab_bounds(K, G)]
    out = torch.cat([o[:K * K * nz] for o, (_, nz) in zip(sm.apply_local(slabs), slab_bounds(K, G))])
    assert torch.equal(out, full)


@pytest.mark.gpu
def test_cuda_stages_match_oracle():
    from paper_2004_13961_b200 import TransformPlan
    w, spec, flat, ref = _problem("cfg5", N=14)
    plan = TransformPlan(15)
    K = 13
    u = torch.from_numpy(flat).cuda()
    sm = SlabMatvec(spec, plan, 3)
    slabs = [u[z0 * K * K:(z0 + nz) * K * K].contiguous() for z0, nz in slab_bounds(K, 3)]
    out = torch.cat([o[:K * K * nz] for o, (_, nz) in zip(sm.apply_local(slabs), slab_bounds(K, 3))])
    assert relerr(out.cpu().numpy(), ref) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,T,G", [("cfg4", 24, 8, 2), ("cfg4", 24, 8, 3), ("cfg5", 20, 3, 4),
                                        ("cfg5", 26, 0, 3), ("cfg5", 21, 0, 2),
                                        ("cfg4", 40, 8, 4), ("cfg5", 24, 0, 3), ("cfg5", 20, 2, 2)])
def test_rank_sweeps_bit_identical(name, N, T, G):
    """Sweeps over G y-slab ranks with halo publication == the one-rank sweeps."""
    from paper_2004_13961_b200 import TransformPlan, _lib
    from paper_2004_13961_b200.precond import assemble_M
    from paper_2004_13961_b200.sharded import SlabSweeps
    from paper_2004_13961_b200.sparse import ilu0
    w = wl.CONFIGS[name]()
    spec = spec_of(w, N)
    f = ilu0(assemble_M(spec, T, T, TransformPlan(N + 1)))
    K = N - 1
    n = K ** 3
    r = torch.randn(n, dtype=torch.float64, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(5))
    lib = _lib.load()
    y1 = torch.empty_like(r)
    z1 = torch.empty_like(r)
    _lib.check(lib.lp_forward_sub(f._handle, r.data_ptr(), y1.data_ptr(), _lib.stream_ptr()))
    _lib.check(lib.lp_backward_sub(f._handle, y1.data_ptr(), z1.data_ptr(), _lib.stream_ptr()))
    sw = SlabSweeps(f, K, G)
    z = sw.apply(r)
    assert torch.equal(sw.gather(sw.yrep), y1)
    assert torch.equal(z, z1)


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,T,G", [("cfg4", 24, 8, 2), ("cfg5", 20, 8, 3), ("cfg4", 32, 8, 4)])
def test_sharded_pcg_matches_single_gpu(name, N, T, G):
    """The fully distributed PCG (emulated on one GPU) against the one-GPU solve
    and the CPU oracle: same iteration count (+-1), solution within 1e-10."""
    from paper_2004_13961_b200 import SolverConfig, TransformPlan, device
    from paper_2004_13961_b200.pcg import pcg_solve_device, setup_preconditioner
    from paper_2004_13961_b200.sharded import pcg_solve_sharded_local
    w = wl.CONFIGS[name]()
    spec = spec_of(w, N)
    plan = TransformPlan(N + 1)
    cfg = SolverConfig(epsilon=w.rtol, preconditioner=(T, T))
    F = wl.mass_contract_series(wl.seeded_fhat(3, N + 1))
    fd = device.to_device(F.flatten(order="F"))
    fac = setup_preconditioner(spec, cfg, plan)
    x1, r1 = pcg_solve_device(spec, cfg, plan, fd, factors=fac)
    xg, rg = pcg_solve_sharded_local(spec, cfg, plan, fd, G, factors=fac)
    assert abs(rg["iterations"] - r1["iterations"]) <= 1
    assert rg["converged"]
    assert relerr(xg.cpu().numpy(), x1.cpu().numpy()) < 1e-10
    if N <= 24:
        xo, ro = orc.pcg_solve(spec, F, epsilon=w.rtol, preconditioner=(T, T))
        assert abs(rg["iterations"] - ro["iterations"]) <= 1
        assert relerr(xg.cpu().numpy(), np.asarray(xo).flatten(order="F")) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,T", [("cfg5", 20, 1), ("cfg4", 14, 8)])
def test_rank_pcg_one_rank_nccl_bit_identical(name, N, T):
    """pcg_solve_sharded_rank -- the per-process driver of a multi-GPU run (NCCL
    all-to-alls, IPC replicas, lp_sweep_rank, ordered allreduce) -- as a
    one-rank NCCL job on this GPU is bit for bit the single-process emulation."""
    import torch.distributed as dist
    from paper_2004_13961_b200 import SolverConfig, TransformPlan, device
    from paper_2004_13961_b200.pcg import setup_preconditioner
    from paper_2004_13961_b200.sharded import pcg_solve_sharded_local, pcg_solve_sharded_rank
    w = wl.CONFIGS[name]()
    spec = spec_of(w, N)
    plan = TransformPlan(N + 1)
    cfg = SolverConfig(epsilon=w.rtol, preconditioner=(T, T))
    F = wl.mass_contract_series(wl.seeded_fhat(3, N + 1))
    fd = device.to_device(F.flatten(order="F"))
    fac = setup_preconditioner(spec, cfg, plan)
    xl, rl = pcg_solve_sharded_local(spec, cfg, plan, fd, 1, factors=fac)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1)
    try:
        xr, rr = pcg_solve_sharded_rank(spec, cfg, plan, fd, factors=fac)
    finally:
        dist.destroy_process_group()
    assert rr["iterations"] == rl["iterations"]
    assert rr["residual_history"] == rl["residual_history"]
    assert torch.equal(xr, xl)


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,T", [("cfg5", 24, 0), ("cfg5", 37, 0), ("cfg4", 22, 0),
                                      ("cfg5", 20, 1), ("cfg4", 18, 2), ("cfg5", 16, 3),
                                      ("cfg4", 14, 8)])
def test_box_sweeps_match_csr_sweeps(name, N, T):
    """The 3-D box sweeps (small-reach multi-line kernel for r <= 4, the line kernel
    above) against the general CSR sweeps on the same factors."""
    from paper_2004_13961_b200 import TransformPlan
    from paper_2004_13961_b200.precond import assemble_M
    from paper_2004_13961_b200.sparse import SparseMatrix, ilu0, precond_apply
    w = wl.CONFIGS[name]()
    m = assemble_M(spec_of(w, N), T, T, TransformPlan(N + 1))
    csr = SparseMatrix(m.n, m.indptr, m.indices, m.values)
    fb, fc = ilu0(m), ilu0(csr)
    r = np.random.default_rng(9).standard_normal(m.n)
    zb, zc = precond_apply(fb, r), precond_apply(fc, r)
    assert relerr(zb, zc) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,T,G", [("cfg5", 16, 2, 2), ("cfg5", 16, 2, 3), ("cfg4", 14, 8, 2),
                                        ("cfg5", 20, 0, 4), ("cfg4", 24, 6, 3), ("cfg5", 26, 8, 2)])
def test_distributed_ilu0_bitwise(name, N, T, G):
    """ILU(0) over G y-slab ranks (lp_ilu0_ranks, one-device emulation of the
    multi-GPU factorisation: every rank reads only its own factor array, its
    neighbours' halo rows arrive as stores): the rows of every rank's slab equal
    the single-GPU factors bit for bit (sparse.py:116-139 per row)."""
    from paper_2004_13961_b200 import ProblemSpec, TransformPlan, assemble_M, ilu0, workloads as wl
    from paper_2004_13961_b200.sharded import ilu0_sharded_local
    w = wl.CONFIGS[name]()
    spec = ProblemSpec(dim=3, N=N, beta=w.beta, alpha=w.alpha)
    plan = TransformPlan(N + 1)
    K = N - 1
    ref = ilu0(assemble_M(spec, T, T, plan))
    facs, ys = ilu0_sharded_local([assemble_M(spec, T, T, plan) for _ in range(G)])
    for part in ("L", "U"):
        rp = getattr(ref, part)
        for v, f in enumerate(facs):
            fp = getattr(f, part)
            np.testing.assert_array_equal(fp.indptr, rp.indptr)
            rows = np.arange(K ** 3)
            own = ((rows // K) % K >= ys[v]) & ((rows // K) % K < ys[v + 1])
            sel = np.repeat(own, np.diff(rp.indptr))
            np.testing.assert_array_equal(fp.values[sel], rp.values[sel])
            assert sel.any()


@pytest.mark.gpu
def test_comm_abi_one_rank_nccl():
    """lp_comm_* (the C-ABI collectives on a caller-owned ncclComm_t) with a
    one-rank communicator created straight from libnccl: the rank-ordered
    double-double allreduce is the identity, lp_comm_dot equals lp_dot bit for
    bit, and the all-to-all moves the own chunk."""
    import ctypes
    from paper_2004_13961_b200 import _lib
    lib = _lib.load()
    torch.zeros(1, device="cuda")
    nccl = None
    for name in ("libnccl.so.2", "libnccl.so"):
        try:
            nccl = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if nccl is None:
        import glob
        import os
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "nccl", "lib",
                                       "libnccl.so.2"))
        assert cands, "no libnccl.so.2"
        nccl = ctypes.CDLL(cands[0], mode=ctypes.RTLD_GLOBAL)
    uid = (ctypes.c_byte * 128)()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()

    class Uid(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_byte * 128)]
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, Uid, ctypes.c_int]
    u = Uid()
    ctypes.memmove(ctypes.byref(u), uid, 128)
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, u, 0) == 0
    h = ctypes.c_void_p()
    try:
        _lib.check(lib.lp_comm_init(comm, 0, 1, 2, ctypes.byref(h)), "comm init")
        st = _lib.stream_ptr()
        n = 100003
        a = torch.randn(n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, dtype=torch.float64, device="cuda")
        d1 = torch.empty(2, dtype=torch.float64, device="cuda")
        d2 = torch.empty(2, dtype=torch.float64, device="cuda")
        _lib.check(lib.lp_dot(n, a.data_ptr(), b.data_ptr(), d1.data_ptr(), st))
        _lib.check(lib.lp_comm_dot(h, n, a.data_ptr(), b.data_ptr(), d2.data_ptr(), st))
        assert torch.equal(d1, d2)
        cnt = (ctypes.c_int64 * 1)(n)
        out = torch.zeros_like(a)
        _lib.check(lib.lp_comm_alltoall(h, a.data_ptr(), cnt, out.data_ptr(), cnt, st))
        torch.cuda.synchronize()
        assert torch.equal(out, a)
    finally:
        if h.value:
            lib.lp_comm_destroy(h)
        nccl.ncclCommDestroy.argtypes = [ctypes.c_void_p]
        nccl.ncclCommDestroy(comm)


@pytest.mark.gpu
@pytest.mark.parametrize("name,N,T", [("cfg5", 18, 2), ("cfg4", 14, 8)])
def test_rank_ilu0_one_rank_nccl_bitwise(name, N, T):
    """ilu0_rank -- the per-process entry of the multi-GPU factorisation (factor
    and flag arrays in CUDA-IPC memory, handle exchange, lp_ilu0_rank_prepare,
    barrier, lp_ilu0_rank) -- as a one-rank NCCL job reproduces the single-GPU
    factors bit for bit, and the solve with them is the single-GPU solve."""
    import torch.distributed as dist
    from paper_2004_13961_b200 import ProblemSpec, TransformPlan, assemble_M, ilu0, precond_apply
    from paper_2004_13961_b200.sharded import ilu0_rank
    w = wl.CONFIGS[name]()
    spec = ProblemSpec(dim=3, N=N, beta=w.beta, alpha=w.alpha)
    plan = TransformPlan(N + 1)
    ref = ilu0(assemble_M(spec, T, T, plan))
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1)
    try:
        fac = ilu0_rank(assemble_M(spec, T, T, plan), 0, 1)
    finally:
        dist.destroy_process_group()
    np.testing.assert_array_equal(fac.L.values, ref.L.values)
    np.testing.assert_array_equal(fac.U.values, ref.U.values)
    r = np.random.default_rng(2).standard_normal(ref.n)
    np.testing.assert_array_equal(precond_apply(fac, r), precond_apply(ref, r))
