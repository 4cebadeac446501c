"""Sweep/factorisation timing at BASELINE sizes (dev tool).  LP_LIB_PATH selects a variant."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import time_events  # noqa: E402
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, _lib, workloads as wl  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

for name in sys.argv[1:]:
    w = wl.CONFIGS[name]()
    spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
    t0 = time.perf_counter()
    m = assemble_M(spec, w.T, w.T, TransformPlan(w.N + 1))
    torch.cuda.synchronize()
    f = ilu0(m)           # first call: includes lazy module loading
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    f = ilu0(m)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    n = w.dofs
    r = torch.randn(n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    y = torch.empty_like(r)
    lib = _lib.load()
    h = f._handle
    tf = time_events(torch, lambda: lib.lp_forward_sub(h, r.data_ptr(), y.data_ptr(), _lib.stream_ptr()), 5)
    tb = time_events(torch, lambda: lib.lp_backward_sub(h, y.data_ptr(), z.data_ptr(), _lib.stream_ptr()), 5)
    nnz = m.nnz
    B = 8.0 * nnz + 32.0 * n
    print(json.dumps({"cfg": name, "lib": os.path.basename(_lib.LIB_PATH), "assemble_s": t1 - t0,
                      "ilu0_s": t2 - t1, "fwd_s": tf, "bwd_s": tb,
                      "pair_gbs": B / (tf + tb) / 1e9, "nnz": nnz}), flush=True)
    rz = torch.empty(2, dtype=torch.float64, device="cuda")
    ta = time_events(torch, lambda: lib.lp_precond_apply(h, r.data_ptr(), z.data_ptr(), _lib.stream_ptr()), 5)
    tz = time_events(torch, lambda: lib.lp_precond_apply_rz(h, r.data_ptr(), z.data_ptr(), rz.data_ptr(),
                                                            _lib.stream_ptr()), 5)
    print(json.dumps({"cfg": name, "precond_apply_s": ta, "precond_apply_rz_s": tz}), flush=True)
