"""CPU (gloo, world size 2): the K6 exchange contract (tests/k6_reference.py,
the layout csrc/exchange.cu implements: pooled rows to sample owners in global
table order, gradients back as [B, D_local]) reassembles exactly what a single
device would compute; the table split of the sharded profile reassembles the
whole-trace profile.  The CUDA exchange itself is exercised with two
processes on one GPU in tests/test_exchange_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from k6_reference import RefExchange
from paper_2201_10095_b200.sharded import column_index, local_tables, rank_dims
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
        ex = RefExchange(plan, DIMS, world, rank, B, torch.device("cpu"))
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


# ---------------------------------------------------------------- HP1 by table
def _small_trace(seed=3):
    from paper_2201_10095_b200.types import TableSpec, Trace

    rng = np.random.default_rng(seed)
    tables = [TableSpec(j * 5 + 2, 1000, int(h), 8, 4) for j, h in enumerate([300, 2000, 50, 999, 4096])]
    S, J = 400, len(tables)
    lens = rng.integers(0, 6, S * J).astype(np.uint32)
    keep = lens > 0
    rec_sample = np.repeat(np.arange(S, dtype=np.uint64), J)[keep]
    rec_table = np.tile(np.array([t.table_id for t in tables], np.uint32), S)[keep]
    lens = lens[keep]
    rec_offset = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    hs = {t.table_id: t.hash_size for t in tables}
    ids = np.concatenate([rng.integers(0, hs[int(t)], int(n)) for t, n in zip(rec_table, lens)]).astype(np.uint32)
    return Trace(tables, S, rec_sample, rec_table, rec_offset, lens, ids=ids)


def _cpu_profile(tr, rate, seed):
    """The C oracle's profile() as FeatureStats (what profile_sharded gathers)."""
    import oracle
    from paper_2201_10095_b200.types import FeatureStats

    return [FeatureStats(**d) for d in oracle.C().profile(tr.tables, tr.num_samples, tr.rec_sample, tr.rec_table,
                                                          tr.rec_offset, tr.rec_len, tr.ids, rate, seed)]


def _profile_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_10095_b200.sharded import profile_sharded

        tr = _small_trace()
        got = profile_sharded(tr, 0.6, 11, profile_fn=_cpu_profile)
        want = _cpu_profile(tr, 0.6, 11)
        ok = len(got) == len(want) and all(
            g.table_id == w.table_id and g.total_accesses == w.total_accesses
            and g.distinct_rows_accessed == w.distinct_rows_accessed
            and float(g.coverage) == float(w.coverage) and float(g.avg_pooling) == float(w.avg_pooling)
            and np.array_equal(np.asarray(g.rows_by_rank), np.asarray(w.rows_by_rank))
            and np.array_equal(np.asarray(g.icdf_steps), np.asarray(w.icdf_steps))
            and np.array_equal(np.asarray(g.access_cdf).view(np.uint64), np.asarray(w.access_cdf).view(np.uint64))
            for g, w in zip(got, want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_profile_split_balances_counters():
    from paper_2201_10095_b200.sharded import profile_split

    tabs = _small_trace().tables
    for world in (1, 2, 3, 7):
        parts = profile_split(tabs, world)
        assert sorted(sum(parts, [])) == list(range(len(tabs)))
    assert profile_split(tabs, 2) == [[4], [0, 1, 2, 3]]  # LPT on hash sizes: 4096 vs 2000+999+300+50


def test_subtrace_keeps_each_tables_profile():
    """A table's statistics on the sub-trace of its shard equal those on the
    whole trace (selection is per sample)."""
    from paper_2201_10095_b200.sharded import profile_split, subtrace

    tr = _small_trace()
    want = _cpu_profile(tr, 0.6, 11)
    for pos in profile_split(tr.tables, 3):
        got = _cpu_profile(subtrace(tr, pos), 0.6, 11)
        for j, g in zip(pos, got):
            w = want[j]
            assert g.table_id == w.table_id
            assert np.array_equal(np.asarray(g.rows_by_rank), np.asarray(w.rows_by_rank))
            assert float(g.coverage) == float(w.coverage) and float(g.avg_pooling) == float(w.avg_pooling)


def test_profile_sharded_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_profile_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res), "sharded profile differs from the whole-trace profile"
