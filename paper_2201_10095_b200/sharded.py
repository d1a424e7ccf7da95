"""Table-wise model-parallel EmbeddingBag over ranks.

Each rank owns the tables its plan entries name (``PlanEntry.gpu``; both tiers
of a table on its owner), pools them for the whole global
batch, and an all-to-all hands every sample owner (rank r owns samples
[r*B/N, (r+1)*B/N)) its pooled row block; gradients travel back the same way.
The exchange is expressed with ``torch.distributed.all_to_all_single`` so it
runs over NCCL (NVLink) on GPUs and over gloo in the CPU tests.
"""
from __future__ import annotations

import numpy as np


def local_tables(plan, rank):
    """Indices (in plan/spec order) of the tables ``rank`` owns."""
    return [j for j, e in enumerate(plan.entries) if e.gpu == rank]


def rank_dims(plan, dims, world):
    """Sum of embedding dims each rank owns."""
    out = [0] * world
    for e, d in zip(plan.entries, dims):
        out[e.gpu] += d
    return out


def column_index(plan, dims, world):
    """For the sample owner's assembled row [sum D] in GLOBAL table order:
    position of every received element (received layout: src-major blocks
    [src][B/N][D_src], tables in plan order inside a block)."""
    cols = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int64)
    per_src = [[] for _ in range(world)]
    for j, e in enumerate(plan.entries):
        per_src[e.gpu].extend(range(cols[j], cols[j] + dims[j]))
    return [np.array(p, np.int64) for p in per_src]


class Exchange:
    """All-to-all of pooled rows to sample owners and of gradients back."""

    def __init__(self, plan, dims, world, rank, batch, device, group=None):
        import torch

        if batch % world:
            raise ValueError("global batch must divide by the world size")
        self.world, self.rank, self.B, self.bl = world, rank, batch, batch // world
        self.group = group
        self.dims_all = rank_dims(plan, dims, world)
        self.D_local = self.dims_all[rank]
        self.D_total = int(sum(dims))
        self.send_splits = [self.bl * self.D_local] * world
        self.recv_splits = [self.bl * d for d in self.dims_all]
        idx = column_index(plan, dims, world)
        self._cols = [torch.as_tensor(c, device=device) for c in idx]
        self.recv = torch.empty(sum(self.recv_splits), dtype=torch.float32, device=device)
        self.back = torch.empty(batch * max(1, self.D_local), dtype=torch.float32, device=device)

    def to_owners(self, pooled_local):
        """[B, D_local] -> this rank's samples [B/N, sum D] in global column order."""
        import torch
        import torch.distributed as dist

        src = pooled_local.reshape(-1)[:self.B * self.D_local].contiguous()
        dist.all_to_all_single(self.recv, src, self.recv_splits, self.send_splits, group=self.group)
        out = torch.empty(self.bl, self.D_total, dtype=torch.float32, device=self.recv.device)
        off = 0
        for s in range(self.world):
            n = self.recv_splits[s]
            if n:
                out[:, self._cols[s]] = self.recv[off:off + n].view(self.bl, self.dims_all[s])
            off += n
        return out

    def to_tables(self, grad_owned):
        """[B/N, sum D] gradients of this rank's samples -> [B, D_local] for its tables."""
        import torch
        import torch.distributed as dist

        parts = []
        for s in range(self.world):
            if self.dims_all[s]:
                parts.append(grad_owned[:, self._cols[s]].reshape(-1))
        send = torch.cat(parts) if parts else self.recv[:0]
        out = self.back[:self.B * self.D_local]
        dist.all_to_all_single(out, send.contiguous(), self.send_splits, self.recv_splits,
                               group=self.group)
        return out.view(self.B, max(1, self.D_local)) if self.D_local else out


class ShardedEmbeddingBag:
    """The rank-local TieredEmbeddingBag plus the exchange."""

    def __init__(self, plan, specs, remaps_local, world, rank, batch, max_lookups,
                 optimizer="rowwise_adagrad", ctx=None, group=None):
        import torch

        from .embedding import TieredEmbeddingBag

        self.local = local_tables(plan, rank)
        dims = [s.dim for s in specs]
        self.ex = Exchange(plan, dims, world, rank, batch,
                           torch.device("cuda", torch.cuda.current_device()), group)
        self.op = (TieredEmbeddingBag([specs[j] for j in self.local], remaps_local, batch,
                                      max_lookups, optimizer, ctx=ctx) if self.local else None)
        self.B = batch

    def forward(self, offsets, indices, hits=None):
        import torch

        pooled = (self.op.forward(offsets, indices, self.B, hits=hits) if self.op else
                  torch.empty(self.B, 0, device=self.ex.recv.device))
        self._pooled = pooled
        return self.ex.to_owners(pooled)

    def backward(self, offsets, indices, grad_owned, lr):
        g = self.ex.to_tables(grad_owned)
        if self.op:
            self.op.backward(offsets, indices, g.contiguous(), self.B, lr)


# ---------------------------------------------------------------- HP1 across GPUs
def profile_split(tables, world: int):
    """Tables -> ranks for a sharded profile: longest-processing-
    time on hash sizes (the per-table counter footprint), ties by table order.
    Returns one list of table positions per rank."""
    load = [0] * world
    out = [[] for _ in range(world)]
    for j in sorted(range(len(tables)), key=lambda j: (-int(tables[j].hash_size), j)):
        r = min(range(world), key=lambda m: (load[m], m))
        out[r].append(j)
        load[r] += int(tables[j].hash_size)
    return [sorted(x) for x in out]


def subtrace(trace, positions):
    """The records (and their ids, re-packed contiguously) of the tables at
    `positions`; num_samples unchanged.  Profile statistics of a table depend
    only on its own records and the sample ids (selection is per sample,
    core/src/profiler.cpp:68-76), so they are identical on the sub-trace."""
    from .types import Trace

    tabs = [trace.tables[j] for j in positions]
    ids = trace.ids if trace.ids is not None else trace.raw_ids
    if hasattr(trace.rec_table, "is_cuda"):
        import torch

        want = torch.tensor([int(t.table_id) for t in tabs], dtype=torch.int64, device=trace.rec_table.device)
        keep = torch.isin(trace.rec_table.long() & 0xFFFFFFFF, want)
        rl = trace.rec_len[keep]
        lens = rl.long()
        offs = torch.cumsum(lens, 0) - lens
        n = int(lens.sum().item()) if lens.numel() else 0
        src = trace.rec_offset[keep].long()
        gather = (src.repeat_interleave(lens) + torch.arange(n, device=lens.device)
                  - offs.repeat_interleave(lens))
        new_ids = ids[gather].contiguous()
        rs, rt, ro = trace.rec_sample[keep].contiguous(), trace.rec_table[keep].contiguous(), offs.contiguous()
        rl = rl.contiguous()
    else:
        want = np.array([int(t.table_id) for t in tabs], np.uint32)
        keep = np.isin(np.asarray(trace.rec_table, np.uint32), want)
        rl = np.asarray(trace.rec_len, np.uint32)[keep]
        lens = rl.astype(np.int64)
        offs = (np.cumsum(lens) - lens).astype(np.uint64)
        src = np.asarray(trace.rec_offset, np.uint64)[keep].astype(np.int64)
        gather = np.repeat(src - offs.astype(np.int64), lens) + np.arange(int(lens.sum()), dtype=np.int64)
        new_ids = np.asarray(ids)[gather]
        rs, rt, ro = np.asarray(trace.rec_sample, np.uint64)[keep], np.asarray(trace.rec_table, np.uint32)[keep], offs
    if trace.ids is not None:
        return Trace(tabs, trace.num_samples, rs, rt, ro, rl, ids=new_ids)
    return Trace(tabs, trace.num_samples, rs, rt, ro, rl, raw_ids=new_ids)


def profile_sharded(trace, sample_rate: float, seed: int, group=None, profile_fn=None):
    """profile() with the tables split over the ranks of `group` (no exchange
    of ids: each rank profiles its tables' records; the FeatureStats are then
    all-gathered).  Every rank returns the full list, in trace table order —
    equal to profile() of the whole trace.  `profile_fn(trace, rate, seed)`
    defaults to the GPU profile()."""
    import torch.distributed as dist

    if profile_fn is None:
        from .profiler import profile as profile_fn
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    split = profile_split(trace.tables, world)
    mine = split[rank]
    got = profile_fn(subtrace(trace, mine), sample_rate, seed) if mine else []
    parts = [None] * world
    dist.all_gather_object(parts, (mine, list(got)), group=group)
    out = [None] * len(trace.tables)
    for pos, stats in parts:
        for j, st in zip(pos, stats):
            out[j] = st
    return out
