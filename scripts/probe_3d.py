"""3-D scaling probe (dev tool): assemble / ILU(0) / sweep / matvec / PCG times
for the cfg-4 (or cfg-5) coefficient recipe at growing N.

  python scripts/probe_3d.py cfg4 24 32 48 64 [--T 8] [--nopcg]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import matvec_flops, time_events  # noqa: E402
from paper_2004_13961_b200 import ProblemSpec, SolverConfig, TransformPlan, _lib, device  # noqa: E402
from paper_2004_13961_b200 import workloads as wl  # noqa: E402
from paper_2004_13961_b200.operator import apply_flat  # noqa: E402
from paper_2004_13961_b200.pcg import pcg_solve_device  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

args = sys.argv[1:]
T = None
nopcg = "--nopcg" in args
if "--T" in args:
    T = int(args[args.index("--T") + 1])
    del args[args.index("--T"):args.index("--T") + 2]
args = [a for a in args if not a.startswith("--")]
name = args[0]
lib = _lib.load()
for N in map(int, args[1:]):
    kw = {"N": N}
    if T is not None:
        kw["T"] = T
    w = wl.CONFIGS[name](**kw)
    spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
    plan = TransformPlan(w.N + 1)
    spec.device_operator(plan)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = assemble_M(spec, w.T, w.T, plan)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    f = ilu0(m)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    n = w.dofs
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    h = f._handle
    tsw = time_events(torch, lambda: lib.lp_precond_apply(h, r.data_ptr(), z.data_ptr(),
                                                          _lib.stream_ptr()), 3)
    tmv = time_events(torch, lambda: apply_flat(spec, plan, 3, r), 5)
    nnz = m.nnz
    out = {"cfg": name, "N": N, "T": w.T, "n": n, "nnz": nnz, "assemble_s": t1 - t0,
           "ilu0_s": t2 - t1, "sweep_pair_s": tsw,
           "sweep_gbs": (8.0 * nnz + 32.0 * n) / tsw / 1e9, "matvec_s": tmv,
           "matvec_tflops": matvec_flops(3, w.P, w.K) / tmv / 1e12,
           "mem_alloc_gb": torch.cuda.max_memory_allocated() / 1e9}
    if not nopcg:
        F = wl.mass_contract_series(w.fhat)
        fd = device.to_device(F.flatten(order="F"))
        cfg = SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T))
        t3 = time.perf_counter()
        x, rep = pcg_solve_device(spec, cfg, plan, fd, factors=f)
        torch.cuda.synchronize()
        out.update({"pcg_loop_s": time.perf_counter() - t3, "iterations": rep["iterations"],
                    "relres": rep["final_relative_residual"]})
    print(json.dumps(out), flush=True)
    del m, f
    torch.cuda.empty_cache()
