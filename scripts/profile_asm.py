"""Breakdown of assemble_M (host prep vs the lp_box_assemble call) and ilu0 (dev tool).

  python scripts/profile_asm.py cfg3 [--N 2048] [--T 12]
"""
import argparse
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, _lib, workloads as wl  # noqa: E402
from paper_2004_13961_b200 import precond  # noqa: E402
from paper_2004_13961_b200.quadrature import gauss_rule  # noqa: E402
from paper_2004_13961_b200.sparse import SparseMatrix, ilu0  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--N", type=int)
ap.add_argument("--T", type=int)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
kw = {k: v for k, v in (("N", args.N), ("T", args.T)) if v is not None}
w = wl.CONFIGS[args.cfg](**kw)
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
plan = TransformPlan(w.N + 1)
lib = _lib.load()
for rep in range(args.reps):
    t = {}
    t0 = time.perf_counter()
    groups = precond._groups(spec, w.T, w.T)
    t["groups"] = time.perf_counter() - t0
    d, K = spec.dim, spec.n_modes
    tmax = max(h.shape[a] for h, _ in groups for a in range(d)) - 1
    t0 = time.perf_counter()
    rule = gauss_rule(K + tmax // 2 + 2)
    t["gauss_rule"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    s_blocks, m_blocks = precond.building_blocks_1d(tmax, K, rule)
    t["blocks_1d"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    R = tmax + 2
    blocks = np.zeros((2, tmax + 1, 2 * R + 1, K))
    for kind, bl in enumerate((s_blocks, m_blocks)):
        for tt, b in enumerate(bl):
            for o, dg in b.diags.items():
                blocks[kind, tt, o + R] = dg
    lens = np.array([h.shape for h, _ in groups], dtype=np.int32).reshape(-1)
    stiff = np.array([-1 if s is None else s for _, s in groups], dtype=np.int32)
    hats = [np.ascontiguousarray(h, dtype=float) for h, _ in groups]
    hat_ptrs = (ctypes.c_void_p * len(hats))(*[h.ctypes.data for h in hats])
    t["pack"] = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = ctypes.c_void_p()
    _lib.check(lib.lp_box_assemble(d, K, len(groups), lens.ctypes.data, stiff.ctypes.data,
                                   hat_ptrs, tmax, blocks.ctypes.data, ctypes.byref(h)))
    torch.cuda.synchronize()
    t["lp_box_assemble"] = time.perf_counter() - t0
    m = SparseMatrix(K ** d, _handle=h.value)
    t0 = time.perf_counter()
    f = ilu0(m)
    torch.cuda.synchronize()
    t["ilu0"] = time.perf_counter() - t0
    print(args.cfg, {k: round(v * 1e3, 2) for k, v in t.items()}, "ms", flush=True)
    del f, m
