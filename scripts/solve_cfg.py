"""Full-size ILU(0)-PCG solve of a BASELINE config on one GPU with a residual
certificate (dev tool; where the CPU oracle cannot run, the
true residual ||F - (A+B) x|| / ||F|| is recomputed with the matvec that the
parity tests verify against the oracle at full size).

  python scripts/solve_cfg.py cfg3 [--N 2048] [--T 12]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, SolverConfig, TransformPlan, device  # noqa: E402
from paper_2004_13961_b200 import workloads as wl  # noqa: E402
from paper_2004_13961_b200.operator import apply_flat  # noqa: E402
from paper_2004_13961_b200.pcg import pcg_solve_device, setup_preconditioner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--N", type=int)
ap.add_argument("--T", type=int)
args = ap.parse_args()
kw = {}
if args.N:
    kw["N"] = args.N
if args.T is not None:
    kw["T"] = args.T
w = wl.CONFIGS[args.cfg](**kw)
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
plan = TransformPlan(w.N + 1)
cfg = SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T))
t0 = time.perf_counter()
fd = wl.rhs_on_device(w.fhat)   # GPU mass contraction of the seeded series
spec.device_operator(plan)
torch.cuda.synchronize()
t1 = time.perf_counter()
fac = setup_preconditioner(spec, cfg, plan)
torch.cuda.synchronize()
t2 = time.perf_counter()
x, rep = pcg_solve_device(spec, cfg, plan, fd, factors=fac)
torch.cuda.synchronize()
t3 = time.perf_counter()
r = fd - apply_flat(spec, plan, 3, x)
cert = float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(fd))
print(json.dumps({"cfg": args.cfg, "dim": w.dim, "N": w.N, "T": w.T, "dofs": w.dofs, "rtol": w.rtol,
                  "host_inputs_and_grids_s": t1 - t0, "setup_s": t2 - t1, "loop_s": t3 - t2,
                  "solve_s": t3 - t1, "iterations": rep["iterations"],
                  "reported_relres": rep["final_relative_residual"],
                  "certified_relres": cert, "converged": rep["converged"]}))
