"""Per-task timeline of the 2-D ILU(0) block wavefront (dev tool; needs the
LP_ILU2D_TRACE build:  make -C paper_2004_13961_b200/csrc VAR=trace DEFS=-DLP_ILU2D_TRACE).

  LP_LIB_PATH=paper_2004_13961_b200/_lib/trace/liblegpcg_b200.so python scripts/trace_ilu2d.py cfg3 [--N 512]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, _lib, workloads as wl  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--N", type=int)
ap.add_argument("--T", type=int)
args = ap.parse_args()
kw = {k: v for k, v in (("N", args.N), ("T", args.T)) if v is not None}
w = wl.CONFIGS[args.cfg](**kw)
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
lib = _lib.load()
lib.lp_debug_ilu2d_trace.restype = ctypes.c_int
lib.lp_debug_ilu2d_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
m = assemble_M(spec, w.T, w.T)
ilu0(m)
torch.cuda.synchronize()
ilu0(m)
torch.cuda.synchronize()
K, RB = w.K, 14
nb = -(-K // RB)
ntask = K * nb
buf = np.zeros(ntask * 8, dtype=np.uint64)
got = lib.lp_debug_ilu2d_trace(buf.ctypes.data, buf.size)
assert got > 0, "not a trace build"
t = buf.reshape(ntask, 8).astype(np.int64)
tasks = []
for key in range(nb + 2 * (K - 1)):
    for y in range(K):
        b = key - 2 * y
        if 0 <= b < nb:
            tasks.append((y, b, key))
tasks = np.array(tasks)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3   # us
tot = rel[:, 5] - rel[:, 0]
print(f"N={w.N} K={K} tasks={ntask} span {rel[:, 5].max() / 1e3:.1f} ms")
names = ["loader E issued", "loader done", "warps E done", "warps done", "published"]
for i, nm in zip([1, 2, 3, 4, 5], names):
    d = rel[:, i] - rel[:, 0]
    print(f"  start -> {nm:16s}: mean {d.mean():8.1f} us  p50 {np.median(d):8.1f}  p90 {np.percentile(d, 90):8.1f}")
d = rel[:, 5] - rel[:, 3]
print(f"  warps E done -> published: mean {d.mean():.1f} us p50 {np.median(d):.1f}")
d = rel[:, 4] - rel[:, 3]
print(f"  in-line part (E done -> warps done): mean {d.mean():.1f} us")
print(f"  consumer mbarrier wait per task (sum over 7 warps): {t[:, 6].mean() / 1.965e3 / 7:.1f} us per warp")
print(f"  loader slot-free wait per task: {t[:, 7].mean() / 1.965e3:.1f} us")
# key steps: time each key's last task published
keys = tasks[:, 2]
kpub = np.zeros(keys.max() + 1)
for i in range(ntask):
    kpub[keys[i]] = max(kpub[keys[i]], rel[i, 5])
dk = np.diff(kpub)
print(f"  key step: mean {dk.mean():.2f} us p50 {np.median(dk):.2f} p90 {np.percentile(dk, 90):.2f}")
# concurrency
ev = np.concatenate([np.stack([rel[:, 0], np.ones(ntask)], 1), np.stack([rel[:, 5], -np.ones(ntask)], 1)])
ev = ev[np.argsort(ev[:, 0])]
c = np.cumsum(ev[:, 1])
dt = np.diff(ev[:, 0])
print(f"  mean resident tasks {np.sum(c[:-1] * dt) / (ev[-1, 0] - ev[0, 0]):.1f}")
