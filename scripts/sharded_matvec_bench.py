"""Slab-sharded 3-D matvec across the GPUs of one node, one process per GPU:

  python -m torch.distributed.run --nnodes=1 --nproc-per-node G --master-addr 127.0.0.1 \
      --master-port 29511 scripts/sharded_matvec_bench.py [--cfg cfg5] [--N 512] [--reps 5]

Each rank holds its z-slab of u, runs the three compute stages of csrc/slab.cu and
the three NCCL all-to-alls (SlabMatvec.apply_rank).  Rank 0 checks the gathered
result bit for bit against the one-GPU apply_system (when it fits) and prints one
JSON line: DOF/s of the whole job, the time as the max over ranks (CUDA events),
and the FP64 rate per GPU.  With G = 1 the same code path runs with a 1-rank NCCL
communicator (how it is exercised on a one-GPU pool).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import matvec_flops  # noqa: E402
from paper_2004_13961_b200 import ProblemSpec, TransformPlan  # noqa: E402
from paper_2004_13961_b200 import workloads as wl  # noqa: E402
from paper_2004_13961_b200.operator import apply_flat  # noqa: E402
from paper_2004_13961_b200.sharded import SlabMatvec, slab_bounds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--N", type=int, default=None)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
rank, ws = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
dist.init_process_group("nccl")
w = wl.CONFIGS[args.cfg](**({"N": args.N} if args.N else {}))
spec = ProblemSpec(dim=3, N=w.N, beta=w.beta, alpha=w.alpha)
plan = TransformPlan(w.N + 1)
K = w.K
sm = SlabMatvec(spec, plan, ws)
z0, nz = slab_bounds(K, ws)[rank]
g = torch.Generator(device="cuda").manual_seed(11)
u_full = torch.randn(K ** 3, dtype=torch.float64, device="cuda", generator=g)   # same on every rank
u = u_full[z0 * K * K:(z0 + nz) * K * K].contiguous()
out = sm.apply_rank(rank, u)                                                       # warm-up
torch.cuda.synchronize()
dist.barrier()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(args.reps):
    out = sm.apply_rank(rank, u)
e.record()
e.synchronize()
t = torch.tensor([s.elapsed_time(e) / 1e3 / args.reps], dtype=torch.float64, device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX)
mine = out[:nz * K * K].contiguous()
parts = [torch.empty(cnt * K * K, dtype=torch.float64, device="cuda") for _, cnt in slab_bounds(K, ws)]
dist.all_gather(parts, mine)
if rank == 0:
    got = torch.cat(parts)
    ref = apply_flat(spec, plan, 3, u_full)
    F = matvec_flops(3, w.P, K)
    print(json.dumps({"metric": "sharded fast-matvec DOF/s (fp64)", "cfg": w.name, "N": w.N, "ranks": ws,
                      "seconds": float(t.item()), "dof_per_s": K ** 3 / float(t.item()),
                      "tflops_per_gpu": F / float(t.item()) / ws / 1e12,
                      "bit_identical_to_one_gpu": bool(torch.equal(got, ref))}), flush=True)
dist.barrier()
dist.destroy_process_group()
