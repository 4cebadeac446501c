"""Distributed 3-D ILU(0)-PCG, one process per GPU (torchrun).

  python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \\
      scripts/distributed_pcg.py --workload cfg4 [--N 128] [--T 8]

Each rank holds a z-slab of F and x; the matvec runs z-slab sharded (three NCCL
all-to-alls), the sweeps over y-slabs with halo lines stored into the
neighbours' replicas over NVLink (lp_sweep_rank), the dots as rank-ordered
double-double allreduces.  Prints one JSON line (rank 0): iterations, setup and
loop seconds as the max over ranks, and the solution's relative difference to a
one-GPU solve when --check is given (needs the factors to fit one GPU).
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_13961_b200 import ProblemSpec, SolverConfig, TransformPlan, device  # noqa: E402
from paper_2004_13961_b200 import workloads as wl  # noqa: E402
from paper_2004_13961_b200.distributed import max_over_ranks  # noqa: E402
from paper_2004_13961_b200.pcg import setup_preconditioner  # noqa: E402
from paper_2004_13961_b200.sharded import pcg_solve_sharded_rank, slab_bounds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg4")
ap.add_argument("--N", type=int)
ap.add_argument("--T", type=int)
ap.add_argument("--check", action="store_true")
ap.add_argument("--rank-ilu", action="store_true",
                help="factor with the distributed ILU(0) (ilu0_rank: each rank its y-slab, halo rows over CUDA IPC)")
args = ap.parse_args()
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl")
rank, G = dist.get_rank(), dist.get_world_size()
kw = {k: v for k, v in (("N", args.N), ("T", args.T)) if v is not None}
w = wl.CONFIGS[args.workload](**kw)
spec = ProblemSpec(dim=3, N=w.N, beta=w.beta, alpha=w.alpha)
plan = TransformPlan(w.N + 1)
cfg = SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T))
K = w.K
F = wl.mass_contract_series(w.fhat).flatten(order="F")
z0, nz = slab_bounds(K, G)[rank]
f_slab = device.to_device(F[z0 * K * K:(z0 + nz) * K * K])
torch.cuda.synchronize()
dist.barrier()
t0 = time.perf_counter()
if args.rank_ilu:
    from paper_2004_13961_b200 import assemble_M
    from paper_2004_13961_b200.sharded import ilu0_rank
    fac = ilu0_rank(assemble_M(spec, w.T, w.T, plan), rank, G)
else:
    fac = setup_preconditioner(spec, cfg, plan)
torch.cuda.synchronize()
t1 = time.perf_counter()
x, rep = pcg_solve_sharded_rank(spec, cfg, plan, f_slab, factors=fac)
torch.cuda.synchronize()
t2 = time.perf_counter()
out = {"workload": args.workload, "N": w.N, "T": w.T, "ranks": G, "rank_ilu": bool(args.rank_ilu), "iterations": rep["iterations"],
       "converged": rep["converged"], "relres": rep["final_relative_residual"],
       "setup_s": max_over_ranks(t1 - t0, "cuda"), "loop_s": max_over_ranks(t2 - t1, "cuda")}
if args.check:
    from paper_2004_13961_b200.pcg import pcg_solve_device
    fac1 = setup_preconditioner(spec, cfg, plan) if args.rank_ilu else fac
    x1, _ = pcg_solve_device(spec, cfg, plan, device.to_device(F), factors=fac1)
    mine = x1[z0 * K * K:(z0 + nz) * K * K]
    num = torch.linalg.vector_norm(x - mine) ** 2
    den = torch.linalg.vector_norm(mine) ** 2
    dist.all_reduce(num)
    dist.all_reduce(den)
    out["rel_diff_vs_1gpu"] = float((num / den).sqrt())
if rank == 0:
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
