"""Task timeline of the 2-D ILU(0) task kernel (dev tool; LP_ILU_TRACE build)."""
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
m = assemble_M(spec, w.T, w.T, TransformPlan(w.N + 1))
ilu0(m)
torch.cuda.synchronize()
lib = _lib.load()
K = w.K
nl = K
nb = (K + 15) // 16
nt = 1 + (nl - 1) * (nb + 1)
buf = np.zeros(nt * 8, dtype=np.uint64)
lib.lp_debug_ilu_trace.restype = ctypes.c_int
lib.lp_debug_ilu_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size))
tr8 = buf.reshape(nt, 8).astype(np.int64)
tr = tr8[:, :4]
t0 = tr[tr > 0].min()
tr = np.where(tr > 0, tr - t0, -1) / 1e3
def task_of(y, b):
    if y == 0:
        return 0
    return 1 + (y - 1) * (nb + 1) + (nb if b < 0 else b)
print("line: L start, row0, rowmid, rowlast | E(y,0): start, last-kline first, last-kline end, done | E(y,nb-1) done (us)")
for y in list(range(0, 8)) + [nl // 2, nl // 2 + 1, nl - 1]:
    L = tr[task_of(y, -1)]
    s = f"{y:4d} " + " ".join(f"{v:9.1f}" for v in L)
    if y >= 1:
        E0 = tr[task_of(y, 0)]
        El = tr[task_of(y, nb - 1)]
        s += " | " + " ".join(f"{v:9.1f}" for v in E0) + " | " + f"{El[3]:9.1f}"
    print(s)
Ls = np.array([tr[task_of(y, -1)] for y in range(nl)])
print("median line row0->rowlast us", np.median(Ls[:, 3] - Ls[:, 1]), " median lead (rowmid) us", np.median(np.diff(Ls[:, 2])))
E = np.array([tr[task_of(y, b)] for y in range(1, nl) for b in range(nb)])
print("E task: median start->done us", np.median(E[:, 3] - E[:, 0]), " median lastkline-ready->done us", np.median(E[:, 3] - E[:, 1]))
tq = np.where(tr8 > 0, tr8 - t0, -1) / 1e3
print("row K/2 of line tasks: row-start, after E wait, after in-line, after fence (us), lines 0..5, mid")
for y in list(range(0, 6)) + [nl // 2]:
    v = tq[task_of(y, -1), 4:8]
    print(y, " ".join(f"{x:9.2f}" for x in v), " | wait E", f"{v[1]-v[0]:.2f}", "inline", f"{v[2]-v[1]:.2f}", "store+fence", f"{v[3]-v[2]:.2f}")
print("last in-line apply of row K/2 (ns), lines 0..5:", [int(tr8[task_of(y, -1), 4]) for y in range(6)])
