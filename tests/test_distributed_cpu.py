"""Multi-process host logic on CPU (gloo, world_size 2): max-over-ranks timing
and the rank-ordered double-double reduction used for sharded PCG dots."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(ws),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    from paper_2004_13961_b200 import distributed as D
    dist = D.init("gloo")
    try:
        t = D.max_over_ranks(1.0 + rank)
        rng = np.random.default_rng(100 + rank)
        x = rng.standard_normal(1000) * 10.0 ** rng.integers(-8, 8, 1000)
        hi, lo = D.dd_of(x)
        tot = D.ordered_dd_allreduce(hi, lo)
        out[rank] = (t, tot[0], tot[1])
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gloo_two_ranks_max_and_ordered_reduction():
    ws = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 2.0
    # identical bits on every rank
    assert res[0][1:] == res[1][1:]
    # equal to the single-process rank-ordered reduction of the same partials
    from paper_2004_13961_b200 import distributed as D
    acc = (0.0, 0.0)
    for rank in range(ws):
        rng = np.random.default_rng(100 + rank)
        x = rng.standard_normal(1000) * 10.0 ** rng.integers(-8, 8, 1000)
        acc = D.dd_add(acc, D.dd_of(x))
    assert res[0][1:] == acc
    # and accurate to the double-double level against an exact sum
    import math
    xs = []
    for r in range(ws):
        rng = np.random.default_rng(100 + r)
        xs.append(rng.standard_normal(1000) * 10.0 ** rng.integers(-8, 8, 1000))
    exact = math.fsum(np.concatenate(xs))
    assert abs(res[0][1] - exact) <= 1e-15 * abs(exact)
