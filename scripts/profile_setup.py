"""Setup-time breakdown of pcg_solve (dev tool)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, workloads as wl  # noqa: E402
from paper_2004_13961_b200 import precond  # noqa: E402
from paper_2004_13961_b200.quadrature import gauss_rule  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = wl.CONFIGS[name]()
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
plan = TransformPlan(w.N + 1)
for rep in range(2):
    t = {}
    t0 = time.perf_counter()
    g = precond._groups(spec, w.T, w.T)
    t["groups(expand_coefficient)"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rule = gauss_rule(w.K + w.T // 2 + 2)
    t["gauss_rule"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    precond.building_blocks_1d(w.T, w.K, rule)
    t["building_blocks_1d"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    m = precond.assemble_M(spec, w.T, w.T, plan)
    torch.cuda.synchronize()
    t["assemble_M total"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    f = ilu0(m)
    torch.cuda.synchronize()
    t["ilu0"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    spec._op_cache.clear()
    spec.device_operator(plan)
    torch.cuda.synchronize()
    t["device_operator"] = time.perf_counter() - t0
    print(name, {k: round(v * 1e3, 2) for k, v in t.items()}, "ms")
