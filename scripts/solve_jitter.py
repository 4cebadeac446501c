"""Where do slow solves spend their time? (dev tool)"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, SolverConfig, device, workloads as wl  # noqa: E402
from paper_2004_13961_b200.pcg import pcg_solve_device, setup_preconditioner  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402


def ev_time(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    s.record()
    out = fn()
    e.record()
    e.synchronize()
    return round(s.elapsed_time(e), 1), round(1e3 * (time.perf_counter() - h0), 1), out


name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = wl.CONFIGS[name]()
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field)
plan = TransformPlan(w.N + 1)
cfg = SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T))
F = wl.mass_contract_series(w.fhat)
f_dev = device.to_device(np.asarray(F).flatten(order="F"))
spec.device_operator(plan)
m = assemble_M(spec, w.T, w.T, plan)
print("assemble", [ev_time(lambda: assemble_M(spec, w.T, w.T, plan))[:2] for _ in range(8)])
print("ilu0", [ev_time(lambda: ilu0(m))[:2] for _ in range(12)])
fac = setup_preconditioner(spec, cfg, plan)
print("loop", [ev_time(lambda: pcg_solve_device(spec, cfg, plan, f_dev, factors=fac))[:2] for _ in range(12)])
print("solve", [ev_time(lambda: pcg_solve_device(spec, cfg, plan, f_dev))[:2] for _ in range(12)])
