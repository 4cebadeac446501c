"""One forward + backward sweep of a 2-D problem (dev tool: run under compute-sanitizer)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, TransformPlan, _lib, workloads as wl  # noqa: E402
from paper_2004_13961_b200.precond import assemble_M  # noqa: E402
from paper_2004_13961_b200.sparse import ilu0  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = wl.CONFIGS["cfg2"](N=N, T=T)
spec = ProblemSpec(dim=w.dim, N=w.N, beta=w.beta, alpha=w.alpha)
f = ilu0(assemble_M(spec, w.T, w.T, TransformPlan(w.N + 1)))
lib = _lib.load()
r = torch.randn(w.dofs, dtype=torch.float64, device="cuda")
y = torch.empty_like(r)
z = torch.empty_like(r)
print("fwd", lib.lp_forward_sub(f._handle, r.data_ptr(), y.data_ptr(), _lib.stream_ptr()))
if hasattr(lib, "lp_debug_sweep_check"):
    import ctypes
    import numpy as np
    chk = np.zeros(8, dtype=np.int64)
    lib.lp_debug_sweep_check(chk.ctypes.data_as(ctypes.c_void_p))
    print("check", chk.tolist())
torch.cuda.synchronize()
print("bwd", lib.lp_backward_sub(f._handle, y.data_ptr(), z.data_ptr(), _lib.stream_ptr()))
torch.cuda.synchronize()
print("ok", float(z.norm()))
