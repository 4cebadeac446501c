"""Matvec-only timing at the BASELINE sizes (dev tool): DOF/s and FP64 roofline."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import dgemm_tflops, matvec_flops, time_events  # noqa: E402
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, device, workloads as wl  # noqa: E402
from paper_2004_13961_b200.operator import apply_flat  # noqa: E402

fp64 = dgemm_tflops(torch)
print(json.dumps({"dgemm_tflops": fp64}), flush=True)
for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]:
    w = wl.CONFIGS[name]()
    spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
    plan = TransformPlan(w.N + 1)
    spec.device_operator(plan)
    u = torch.randn(w.dofs, dtype=torch.float64, device="cuda")
    t = time_events(torch, lambda: apply_flat(spec, plan, 3, u), 5 if w.dim == 3 and w.N > 256 else 20)
    F = matvec_flops(w.dim, w.P, w.K)
    print(json.dumps({"cfg": name, "matvec_s": t, "dof_per_s": w.dofs / t,
                      "tflops": F / t / 1e12, "frac_fp64": F / t / 1e12 / fp64}), flush=True)
