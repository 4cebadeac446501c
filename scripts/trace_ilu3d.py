"""Row timeline of the 3-D ILU(0) row kernel (dev tool; LP_ILU_TRACE build).

  LP_LIB_PATH=build/variants/trace.so python scripts/trace_ilu3d.py cfg4 48
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
w = wl.CONFIGS[name](N=N)
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
m = assemble_M(spec, w.T, w.T, TransformPlan(w.N + 1))
ilu0(m)
torch.cuda.synchronize()
lib = _lib.load()
n = w.dofs
K = w.K
buf = np.zeros(n * 8, dtype=np.uint64)
lib.lp_debug_ilu_trace.restype = ctypes.c_int
lib.lp_debug_ilu_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(buf.size))
tr8 = buf.reshape(n, 8).astype(np.int64)
tr = tr8[:, :4]
spin_line, spin_in, npiv = tr8[:, 4], tr8[:, 5], tr8[:, 6]
t0 = tr[:, 0].min()
tr = (tr - t0) / 1e3   # us
start, plane0, elim, pub = tr.T
print(f"n={n} K={K} total {pub.max()/1e3:.1f} ms")
print(f"per row (us): bulk (start->pz=0) median {np.median(plane0-start):.1f}, "
      f"same-plane (pz=0 -> elim) median {np.median(elim-plane0):.1f}, "
      f"store+publish median {np.median(pub-elim):.1f}, total median {np.median(pub-start):.1f}")
for q in [0.1, 0.5, 0.9, 0.99]:
    print(f"  q{q}: bulk {np.quantile(plane0-start,q):.1f} plane0 {np.quantile(elim-plane0,q):.1f} "
          f"pub {np.quantile(pub-elim,q):.1f}")
# finishing rate per line / plane
lines = pub.reshape(-1, K)
print("line finish times (ms) for lines 0..5 of plane K/2:", (lines[(K//2)*K:(K//2)*K+6, -1]/1e3).round(3))
planes = pub.reshape(K, K * K)
print("plane finish (ms):", (planes[:, -1][::max(1, K//10)]/1e3).round(2))
st = np.sort(start)
print("start spacing median (us):", np.median(np.diff(st)))
print("spins per row: line median %d q90 %d, inline median %d q90 %d; pivots median %d" % (
    np.median(spin_line), np.quantile(spin_line, .9), np.median(spin_in), np.quantile(spin_in, .9), np.median(npiv)))
print("bulk us per pivot (median):", np.median((plane0 - start) / np.maximum(npiv, 1)))
