"""3-D measurements beside the CPU reference, one JSON
line per workload:

  * cfg 4 (3-D N=128, T=8): setup (GPU assembly + ILU(0)) once, then PCG loops with
    the factors reused, sweep pair and matvec timed with CUDA events; roofline of the
    sweep pair (B_sw = 8 nnz + 32 n bytes vs the measured HBM peak) and of the matvec
    (F_alg vs a cuBLAS DGEMM measured here); CPU reference: the oracle port's
    apply_system on all host cores (its ILU(0) needs 134 GB of RAM and days of one
    core, so only the matvec is timed);
  * cfg 5 (3-D N=512) at T=0 (the largest truncation whose ILU(0) fits one GPU):
    one full solve and the matvec; CPU reference: one oracle apply_system call
    (~70 s; --no-cpu5 skips it).

  python scripts/bench_3d.py [--no-cpu5] [--loops 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import dgemm_tflops, matvec_flops, measured_peaks, time_events  # noqa: E402
from oracle import legpcg_port as orc  # noqa: E402
from paper_2004_13961_b200 import ProblemSpec, SolverConfig, TransformPlan, _lib, device  # noqa: E402
from paper_2004_13961_b200 import workloads as wl  # noqa: E402
from paper_2004_13961_b200.operator import apply_flat  # noqa: E402
from paper_2004_13961_b200.pcg import pcg_solve_device  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--no-cpu5", action="store_true")
ap.add_argument("--loops", type=int, default=3)
args = ap.parse_args()
peaks, _ = measured_peaks()
fp64 = dgemm_tflops(torch)
lib = _lib.load()


def cpu_matvec(w, reps):
    spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
    plan = orc.Plan(w.N + 1)
    u = np.random.default_rng(1).standard_normal((w.K,) * w.dim)
    cache = {}
    orc.apply_system(spec, plan, u, cache)       # warm-up: fills the grid cache
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        orc.apply_system(spec, plan, u, cache)
        best = min(best, time.perf_counter() - t0)
    return best


def run(w, loops, cpu_reps):
    spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
    plan = TransformPlan(w.N + 1)
    cfg = SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T))
    fd = wl.rhs_on_device(w.fhat)   # GPU mass contraction of the seeded series
    spec.device_operator(plan)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    m = assemble_M(spec, w.T, w.T, plan)
    ev[1].record()
    f = ilu0(m)
    ev[2].record()
    ev[2].synchronize()
    t_asm, t_ilu = ev[0].elapsed_time(ev[1]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3
    pcg_solve_device(spec, cfg, plan, fd, factors=f)     # warm-up (module loading)
    loop = []
    it = None
    for _ in range(loops):
        ev[0].record()
        x, rep = pcg_solve_device(spec, cfg, plan, fd, factors=f)
        ev[1].record()
        ev[1].synchronize()
        loop.append(ev[0].elapsed_time(ev[1]) / 1e3)
        it = rep["iterations"]
    n = w.dofs
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    t_sw = time_events(torch, lambda: lib.lp_precond_apply(f._handle, r.data_ptr(), z.data_ptr(),
                                                           _lib.stream_ptr()), 3)
    t_mv = time_events(torch, lambda: apply_flat(spec, plan, 3, r), 5)
    nnz = m.nnz
    B_sw = 8.0 * nnz + 32.0 * n
    F_alg = matvec_flops(3, w.P, w.K)
    t_loop = float(np.median(loop))
    solve = t_asm + t_ilu + t_loop
    cpu = cpu_matvec(w, cpu_reps) if cpu_reps else None
    res = {"workload": f"{w.name}: 3-D N={w.N} T={w.T} rtol={w.rtol} ILU(0)-PCG", "dofs": n,
           "nnz_M": nnz, "iterations": it, "assemble_s": t_asm, "ilu0_s": t_ilu,
           "pcg_loop_s": t_loop, "solve_s": solve, "solve_dof_per_s": n / solve,
           "precond_apply_s": t_sw, "matvec_s": t_mv, "matvec_dof_per_s": n / t_mv,
           "roofline": {
               "sweeps": {"kernel": "box_sweep3d_kernel fwd+bwd", "bound": "hbm",
                          "achieved": B_sw / t_sw / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                          "frac": B_sw / t_sw / 1e9 / peaks["hbm_gbs"], "algorithmic_bytes": B_sw},
               "matvec": {"kernel": "line_transform_kernel x6", "bound": "fp64",
                          "achieved": F_alg / t_mv / 1e12, "peak": fp64, "unit": "TFLOP/s",
                          "frac": F_alg / t_mv / 1e12 / fp64, "algorithmic_flops": F_alg}},
           "cpu_baseline": None if cpu is None else {
               "what": "oracle apply_system (numpy/OpenBLAS, the reference's dense transform "
                       "mode), best of %d after warm-up" % cpu_reps,
               "matvec_s": cpu, "matvec_dof_per_s": n / cpu, "cores": os.cpu_count(),
               "gpu_speedup_matvec": cpu / t_mv}}
    del m, f
    torch.cuda.empty_cache()
    return res


print(json.dumps(run(wl.cfg4(), args.loops, 3)), flush=True)
print(json.dumps(run(wl.cfg5(T=0), 1, 0 if args.no_cpu5 else 1)), flush=True)
