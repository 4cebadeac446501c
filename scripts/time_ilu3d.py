"""Time the 3-D ILU(0) alone (dev tool; tolerates a zero-pivot error from experiment builds).

  python scripts/time_ilu3d.py cfg4 64 [T]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, workloads as wl  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

name, N = sys.argv[1], int(sys.argv[2])
kw = {"N": N}
if len(sys.argv) > 3:
    kw["T"] = int(sys.argv[3])
w = wl.CONFIGS[name](**kw)
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
m = assemble_M(spec, w.T, w.T, TransformPlan(w.N + 1))
torch.cuda.synchronize()
t0 = time.perf_counter()
try:
    ilu0(m)
except Exception as ex:  # noqa: BLE001
    print("error:", str(ex)[:80])
torch.cuda.synchronize()
print(f"{name} N={N} T={w.T}: ilu0 {time.perf_counter() - t0:.3f} s")
