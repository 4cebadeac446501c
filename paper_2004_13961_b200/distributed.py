"""Multi-process plumbing (torch.distributed): one process per GPU.

The 2-D configurations do not shard (BASELINE runs them on one GPU), so
multi-GPU runs of them are independent replicas timed as the max over ranks.
``ordered_dd_allreduce`` is the deterministic cross-rank combination the
slab-sharded 3-D PCG uses for its three dots per iteration: every
rank gathers all ranks' double-double partials and sums them in rank order,
so every rank gets the same bits and a G-rank run rounds like a fixed-order
single-rank reduction of the same partials.
"""

from __future__ import annotations

import os

import numpy as np


def env_world():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend=None):
    """Initialise the default process group (nccl on GPUs, gloo otherwise)."""
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        return dist
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend)
    return dist


def max_over_ranks(value, device=None):
    """Max of a scalar over all ranks (timings are reported as the max)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def dd_add(x, y):
    """Double-double addition of (hi, lo) pairs (same algorithm as vector_ops.cuh)."""
    s, e = _two_sum(x[0], y[0])
    t, f = _two_sum(x[1], y[1])
    e += t
    s, e = s + e, e - ((s + e) - s)
    e += f
    hi = s + e
    return hi, e - (hi - s)


def ordered_dd_allreduce(hi, lo, device=None):
    """Sum a double-double partial over ranks in rank order; identical on every rank."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(hi), float(lo)
    ws = dist.get_world_size()
    mine = torch.tensor([hi, lo], dtype=torch.float64, device=device or "cpu")
    parts = [torch.empty_like(mine) for _ in range(ws)]
    dist.all_gather(parts, mine)
    acc = (0.0, 0.0)
    for p in parts:
        v = p.cpu().numpy()
        acc = dd_add(acc, (float(v[0]), float(v[1])))
    return acc


def dd_of(values):
    """Double-double sum of a float64 array in index order (reference helper)."""
    acc = (0.0, 0.0)
    for v in np.asarray(values, dtype=np.float64):
        acc = dd_add(acc, (float(v), 0.0))
    return acc
