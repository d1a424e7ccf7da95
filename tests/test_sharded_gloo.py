"""CPU (gloo, world size 2): the model-parallel exchange of pooled rows and
gradients (paper_2201_10095_b200/sharded.py) reassembles exactly what a single
device would compute."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2201_10095_b200.sharded import Exchange, column_index, local_tables, rank_dims
from paper_2201_10095_b200.types import PlanEntry, ShardingPlan


def _plan():
    gpus = [1, 0, 0, 1, 1, 0, 1]
    return ShardingPlan("t", 1, [PlanEntry(j, g, 0, 0) for j, g in enumerate(gpus)])


DIMS = [8, 4, 16, 4, 12, 8, 4]


def _full(B):
    # deterministic "single device" pooled output [B, sum D]: value = sample*1000 + column
    return torch.arange(B, dtype=torch.float32)[:, None] * 1000 + torch.arange(sum(DIMS))[None, :]


def _worker(rank, world, port, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = _plan()
        ex = Exchange(plan, DIMS, world, rank, B, torch.device("cpu"))
        full = _full(B)
        cols = np.concatenate([[0], np.cumsum(DIMS)[:-1]])
        mine = local_tables(plan, rank)
        local = torch.cat([full[:, cols[j]:cols[j] + DIMS[j]] for j in mine], dim=1)
        got = ex.to_owners(local)
        bl = B // world
        ok_fwd = torch.equal(got, full[rank * bl:(rank + 1) * bl])
        grad_owned = -got * 2  # any function of the owned rows
        back = ex.to_tables(grad_owned)
        want = torch.cat([(-2 * full)[:, cols[j]:cols[j] + DIMS[j]] for j in mine], dim=1)
        ok_bwd = torch.equal(back.view(B, -1), want)
        q.put((rank, ok_fwd, ok_bwd))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_rank_dims_and_columns():
    plan = _plan()
    assert rank_dims(plan, DIMS, 2) == [4 + 16 + 8, 8 + 4 + 12 + 4]
    idx = column_index(plan, DIMS, 2)
    assert sorted(np.concatenate(idx).tolist()) == list(range(sum(DIMS)))
    assert local_tables(plan, 0) == [1, 2, 5]


@pytest.mark.parametrize("B", [8, 64])
def test_exchange_world2_gloo(B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res), "pooled rows did not reach their sample owners intact"
    assert all(r[2] for r in res), "gradients did not return to the table owners intact"
