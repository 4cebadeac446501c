"""Per-call timing distribution of precond_apply and of whole solves (dev tool)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, SolverConfig, _lib, device, workloads as wl  # noqa: E402
from paper_2004_13961_b200.pcg import pcg_solve_device, setup_preconditioner  # noqa: E402
from paper_2004_13961_b200.operator import assemble_rhs  # noqa: E402


def ev_time(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e)


name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = wl.CONFIGS[name]()
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field)
plan = TransformPlan(w.N + 1)
cfg = SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T))
fac = setup_preconditioner(spec, cfg, plan)
lib = _lib.load()
n = w.dofs
r = torch.randn(n, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
ts = [ev_time(lambda: lib.lp_precond_apply(fac._handle, r.data_ptr(), z.data_ptr(), _lib.stream_ptr()))
      for _ in range(200)]
q = np.percentile(ts, [0, 10, 50, 90, 99, 100])
print(json.dumps({"precond_apply_ms_pcts_0_10_50_90_99_100": [round(v, 3) for v in q]}))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
F = assemble_rhs(spec, plan).data if w.rhs_field is not None else None
from bench import build_workload  # noqa: E402
import argparse
_, F = build_workload(argparse.Namespace(workload=name, N=None, T=None))
if F is None:
    F = assemble_rhs(spec, plan).data
f_dev = device.to_device(np.asarray(F).flatten(order="F"))
for flush_on in (False, True, False, True):
    out = []
    for _ in range(5):
        if flush_on:
            flush.zero_()
            torch.cuda.synchronize()
        out.append(ev_time(lambda: pcg_solve_device(spec, cfg, plan, f_dev)))
    print(json.dumps({"flush": flush_on, "solve_ms": [round(v, 1) for v in out]}))
