"""Per-line timeline of the box sweep (dev tool; needs the LP_SWEEP_TRACE build)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, _lib, workloads as wl  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

name = sys.argv[1]
w = wl.CONFIGS[name]()
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
f = ilu0(assemble_M(spec, w.T, w.T, TransformPlan(w.N + 1)))
lib = _lib.load()
n = w.dofs
r = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(r)
for _ in range(3):
    lib.lp_forward_sub(f._handle, r.data_ptr(), y.data_ptr(), _lib.stream_ptr())
torch.cuda.synchronize()
nl = n // w.K
buf = np.zeros(nl * 16, dtype=np.uint64)
lib.lp_debug_sweep_trace.restype = ctypes.c_int
lib.lp_debug_sweep_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size))
tc = buf.reshape(nl, 16).astype(np.int64)
t = tc[:, :4]
cy = tc[:, 4:]
t0 = t[:, 0].min()
t = (t - t0) / 1e3
print(name, "line  start  row0  rowmid  rowlast   (us)")
for L in list(range(0, 12)) + list(range(nl // 2, nl // 2 + 4)) + list(range(nl - 4, nl)):
    print(L, *[f"{v:9.2f}" for v in t[L]])
d0 = np.diff(t[:, 1])
print("lead (row0 to row0) median us", np.median(d0), "line duration median",
      np.median(t[:, 3] - t[:, 1]), "start->row0 median", np.median(t[:, 1] - t[:, 0]))
half = w.K - 1 - w.K // 2
cps = (cy[:, 3] - cy[:, 2]) / half
nsps = (t[:, 3] - t[:, 2]) / half
print("second-half-of-line cycles/step: line0", cps[0], "median", np.median(cps),
      "| ns/step line0", nsps[0] * 1e3, "median", np.median(nsps) * 1e3,
      "| implied MHz", np.median(cps / (nsps * 1e3)) * 1e3)
print("serial cycles waiting for band chunks per line: line0", cy[0, 0], "median", np.median(cy[:, 0]))
ev = (tc[:, 8:11] - t0) / 1e3   # producer c_mid, group d_mid, group arrival at mid (us)
print("mid-row events (us): line  c_mid(prod)  arrival(grp)  d_mid(grp)  y_mid(serial)")
for L in list(range(0, 6)) + [nl // 2]:
    print(L, *[f"{v:9.2f}" for v in (ev[L, 0], ev[L, 2], ev[L, 1], t[L, 2])])
print("group loop cycles/step (median over lines)", np.median(tc[1:, 11] / (w.K + w.T + 2)),
      "| group re-polls per line: median", np.median(tc[1:, 12]), "max", tc[1:, 12].max(),
      "| serial spins on c per line", np.median(tc[:, 13]), "on A", np.median(tc[1:, 14]))
# y(L-1, K/2 + r) is produced just before line L-1's step K/2 + r + 1 is marked
prod = (tc[:, 15] - t0) / 1e3
arr = ev[:, 2]
lam = arr[1:] - prod[:-1]
print("detect latency y(L-1, mid+r) produced -> seen by line L's group (us): median", np.median(lam),
      "p10", np.percentile(lam, 10), "p90", np.percentile(lam, 90))
print("arrival -> y_mid of line L (us): median", np.median(t[1:, 2] - arr[1:]))
print("line-L-1 r steps (y_mid -> y_mid+r) (us): median", np.median(prod - t[:, 2]))
slope = (t[:, 3] - t[:, 2]) / half * 1e3
print("per-line slope ns/step (lines 0..15):", " ".join(f"{v:.0f}" for v in slope[:16]))
print("per-line detect latency us (lines 1..15):", " ".join(f"{v:.2f}" for v in lam[:15]))
print("slope ns/step at lines 50,100,150,200,250:", " ".join(f"{slope[i]:.0f}" for i in (50, 100, 150, 200, 250) if i < nl))
print("group: cycles per step over the 64 steps before mid (median over lines 1..)", np.median(tc[1:, 11] / 64.0),
      "| re-polls in that window: median", np.median(tc[1:, 12]))
