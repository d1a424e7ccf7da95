"""Table-wise model-parallel EmbeddingBag over ranks.

Each rank owns the tables its plan entries name (``PlanEntry.gpu``; both tiers
of a table on its owner), pools them for the whole global
batch, and every sample owner (rank r owns samples [r*B/N, (r+1)*B/N))
receives its pooled rows of ALL tables, [B/N, sum D] in global table order;
gradients travel back the same way.  The exchange is K6 in the C-ABI
(csrc/exchange.cu, ``rs_exchange_*`` / ``rs_emb_*_owners``):

* ``transport="peer"`` — NVLink peer memory between the ranks' processes
  (CUDA IPC): K4 stores every pooled row straight into its owner's block and
  a flag barrier publishes it; the backward pulls the gradient rows on a side
  stream while K5 sorts.
* ``transport="nccl"`` — grouped ncclSend/ncclRecv, K4's [B, D_local] output
  is the send layout; received blocks are scattered into column order by
  one kernel.

``torch.distributed`` (gloo or NCCL) only bootstraps: it all-gathers the
exchange blobs (IPC handles / the NCCL unique id).  ``column_index`` and
``rank_dims`` restate the layout in Python for tests.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .runtime import default_context, ptr

TRANSPORTS = {"peer": _lib.RS_EX_PEER, "nccl": _lib.RS_EX_NCCL}


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
    """For the sample owner's row [sum D] in GLOBAL table order: the global
    column of every element of source rank s's block [B/N, D_s] (its tables in
    plan order) — the layout K6 assembles (csrc/exchange.cu gsrc/gcol)."""
    cols = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int64)
    per_src = [[] for _ in range(world)]
    for j, e in enumerate(plan.entries):
        per_src[e.gpu].extend(range(cols[j], cols[j] + dims[j]))
    return [np.array(p, np.int64) for p in per_src]


class Exchange:
    """K6: one rank's end of the pooled-row / gradient exchange."""

    def __init__(self, plan, dims, world, rank, batch, transport="peer", ctx=None, group=None):
        import torch.distributed as dist

        if batch % world:
            raise ValueError("global batch must divide by the world size")
        self.ctx = ctx or default_context()
        self.world, self.rank, self.B, self.bl = world, rank, batch, batch // world
        self.dims = [int(d) for d in dims]
        self.owner = [int(e.gpu) for e in plan.entries]
        self.D_total = int(sum(dims))
        self.D_local = int(sum(d for d, o in zip(self.dims, self.owner) if o == rank))
        d = np.array(self.dims, np.uint32)
        o = np.array(self.owner, np.uint32)
        h = C.c_void_p()
        _lib.check(_lib.lib().rs_exchange_create(self.ctx.h, TRANSPORTS[transport], world, rank,
                                                 C.c_uint64(batch), len(dims), ptr(d), ptr(o), C.byref(h)))
        self.h = h
        blob = (C.c_char * _lib.RS_EX_BLOB_BYTES)()
        _lib.check(_lib.lib().rs_exchange_blob(self.h, blob))
        blobs = [None] * world
        if world > 1:
            dist.all_gather_object(blobs, bytes(blob), group=group)
        else:
            blobs = [bytes(blob)]
        allb = np.frombuffer(b"".join(blobs), np.uint8).copy()
        _lib.check(_lib.lib().rs_exchange_connect(self.h, ptr(allb)))

    def owned(self):
        """This step's owner block [B/N, sum D] (a torch view of device memory)."""
        import torch

        f = C.c_void_p()
        _lib.check(_lib.lib().rs_exchange_info(self.h, None, None, None, C.byref(f)))
        return _device_view(f.value, self.bl * self.D_total, self.ctx.device).view(self.bl, self.D_total)

    def to_owners(self, pooled_local, out=None):
        """K6 forward primitive: [B, D_local] -> [B/N, sum D]."""
        import torch

        if out is None:
            out = torch.empty(self.bl, self.D_total, dtype=torch.float32, device=pooled_local.device)
        _lib.check(_lib.lib().rs_emb_alltoall_fwd(self.h, ptr(pooled_local), ptr(out)))
        return out

    def to_tables(self, grad_owned, out=None):
        """K6 backward primitive: [B/N, sum D] -> [B, D_local]."""
        import torch

        if out is None:
            out = torch.empty(self.B, max(1, self.D_local), dtype=torch.float32, device=grad_owned.device)
        _lib.check(_lib.lib().rs_emb_alltoall_bwd(self.h, ptr(grad_owned.contiguous()), ptr(out)))
        return out

    def close(self):
        if self.h:
            _lib.lib().rs_exchange_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _device_view(addr, n, device):
    """A float32 torch tensor over n floats of library-owned device memory."""
    import torch

    class _Holder:
        pass

    h = _Holder()
    h.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4", "data": (int(addr), False),
                                  "version": 3, "strides": None}
    return torch.as_tensor(h, device=torch.device("cuda", device))


class ShardedEmbeddingBag:
    """This rank's TieredEmbeddingBag (its tables of the plan) plus K6."""

    def __init__(self, plan, specs, remaps_local, world, rank, batch, max_lookups,
                 optimizer="rowwise_adagrad", transport="peer", ctx=None, group=None):
        from .embedding import TieredEmbeddingBag

        self.ctx = ctx or default_context()
        self.local = local_tables(plan, rank)
        dims = [s.dim for s in specs]
        self.op = (TieredEmbeddingBag([specs[j] for j in self.local], remaps_local, batch,
                                      max_lookups, optimizer, ctx=self.ctx) if self.local else None)
        self.ex = Exchange(plan, dims, world, rank, batch, transport, ctx=self.ctx, group=group)
        self.B = batch

    def forward(self, offsets, indices, hits=None):
        """offsets/indices: this rank's tables for all B samples (table-major
        CSR).  Returns this rank's samples [B/N, sum D] (global table order);
        write the gradient into it in place (or pass one to backward)."""
        if self.op is None:
            raise ValueError("ShardedEmbeddingBag: this rank owns no tables")
        self.op._check_dev(offsets, indices, hits)
        f = C.c_void_p()
        _lib.check(_lib.lib().rs_emb_forward_to_owners(self.op.h, self.ex.h, ptr(offsets), ptr(indices),
                                                       ptr(hits), C.byref(f)))
        return self.ex.owned()

    def backward(self, offsets, indices, lr, grad_owned=None):
        _lib.check(_lib.lib().rs_emb_backward_from_owners(self.op.h, self.ex.h, ptr(offsets), ptr(indices),
                                                          ptr(grad_owned), C.c_float(lr)))

    def close(self):
        if self.op:
            self.op.close()
        self.ex.close()


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
    import torch

    from .types import FeatureStats

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    split = profile_split(trace.tables, world)
    mine = split[rank]
    got = profile_fn(subtrace(trace, mine), sample_rate, seed) if mine else []
    # the small fields (scalars, 101-step ICDFs, array lengths) as objects;
    # rows_by_rank (u32) and access_cdf (f64 bits) of all of a rank's tables
    # as ONE flat int64 tensor per rank — not pickled — all-gathered padded to
    # the longest rank (device tensors over NCCL, host tensors over gloo)
    meta = [(int(st.table_id), float(st.coverage), float(st.avg_pooling), int(st.distinct_rows_accessed),
             int(st.total_accesses), np.asarray(st.icdf_steps, np.uint64)) for st in got]
    parts = [None] * world
    dist.all_gather_object(parts, (mine, meta), group=group)
    flat = np.concatenate([np.concatenate([np.asarray(st.rows_by_rank, np.uint32).astype(np.int64),
                                           np.asarray(st.access_cdf, np.float64).view(np.int64)])
                           for st in got]) if got else np.zeros(0, np.int64)
    sizes = [sum(2 * m[3] for m in meta_r) for _, meta_r in parts]
    n = max(1, max(sizes))
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    buf = torch.zeros(n, dtype=torch.int64, device=dev)
    buf[:flat.size] = torch.from_numpy(flat).to(dev)
    bufs = [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    out = [None] * len(trace.tables)
    for (pos, meta_r), b in zip(parts, bufs):
        arr = b.cpu().numpy()
        at = 0
        for j, (tid, cov, pool, d, tot, icdf) in zip(pos, meta_r):
            rows = arr[at:at + d].astype(np.uint32)
            cdf = arr[at + d:at + 2 * d].view(np.float64).copy()
            at += 2 * d
            out[j] = FeatureStats(tid, cov, pool, d, tot, icdf, cdf, rows)
    return out
