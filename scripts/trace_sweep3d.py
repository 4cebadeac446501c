"""Line timeline of the 3-D sweep kernel (dev tool; LP_SWEEP_TRACE build).

  LP_LIB_PATH=build/variants/trace.so python scripts/trace_sweep3d.py cfg4 64 [T]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, _lib, workloads as wl  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

name, N = sys.argv[1], int(sys.argv[2])
kw = {"N": N}
if len(sys.argv) > 3:
    kw["T"] = int(sys.argv[3])
w = wl.CONFIGS[name](**kw)
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
f = ilu0(assemble_M(spec, w.T, w.T, TransformPlan(w.N + 1)))
lib = _lib.load()
n, K = w.dofs, w.K
r = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(r)
for _ in range(2):
    lib.lp_forward_sub(f._handle, r.data_ptr(), y.data_ptr(), _lib.stream_ptr())
torch.cuda.synchronize()
nl = K * K
buf = np.zeros(nl * 8, dtype=np.uint64)
lib.lp_debug_sweep_trace.restype = ctypes.c_int
lib.lp_debug_sweep_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size))
tr = buf[:nl * 8].reshape(nl, 8).astype(np.int64)[:, :5]
t0 = tr[:, 0].min()
tr = (tr - t0) / 1e3
print(f"K={K} lines={nl} sweep {tr[:, 4].max():.1f} us")
start, r0, rq, rh, rl = tr.T
print("median: ticket->row0 %.1f  row0->rowK/4 %.1f  ->K/2 %.1f  ->K-1 %.1f us" % (
    np.median(r0 - start), np.median(rq - r0), np.median(rh - rq), np.median(rl - rh)))
d = np.diff(r0)
print("row-0 lead between consecutive lines (us): median %.2f q10 %.2f q90 %.2f" % (
    np.median(d), np.quantile(d, .1), np.quantile(d, .9)))
pl = r0.reshape(K, K)[:, 0]
print("plane lead (row0 of line y=0), median %.1f us" % np.median(np.diff(pl)))
print("per-row slope in line (us/row): median %.3f" % np.median((rl - r0) / (K - 1)))
for L in [0, 1, 2, K // 2, K, K + 1, K * K // 2, K * K // 2 + 1, nl - 1]:
    print(L, (tr[L] ).round(1))
