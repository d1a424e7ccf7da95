"""HP2 — the tiered EmbeddingBag operator serving a RecShard sharding plan.

No reference implementation exists (the paper ran FBGEMM); this
is the operator SURVEY §8b names ``TieredEmbeddingBag{create; forward;
backward}``, whose forward accounting equals ``simulate()``
(core/src/simulator.cpp:86).  Rows live in the fast tier (HBM) or the slow
tier (pinned host memory read zero-copy over PCIe) as each table's remap
says; forward is a sum-pool, backward a deterministic row-wise SGD or
exact-row-wise-Adagrad update (csrc/emb.cu).  Rows are fp32 or fp16
(TableSpec.elem_bytes 2); arithmetic is fp32.  With an omit_unaccessed remap
only the profiled slow rows have storage; the others pool as zeros and drop
their gradients (counted by ``unbacked()``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .runtime import default_context, is_device, ptr
from .types import InvalidArgument

OPTIMIZERS = {"sgd": _lib.RS_OPT_SGD, "rowwise_adagrad": _lib.RS_OPT_ROWWISE_ADAGRAD}


class TieredEmbeddingBag:
    def __init__(self, specs, remaps, max_batch: int, max_lookups: int, optimizer: str = "sgd",
                 eps: float = 1e-8, ctx=None):
        if len(specs) != len(remaps):
            raise InvalidArgument("TieredEmbeddingBag: one remap per table")
        self.ctx = ctx or default_context()
        self.specs = list(specs)
        self.dims = [int(s.dim) for s in specs]
        self.total_dim = int(sum(self.dims))
        self.col_offsets = [int(x) for x in np.concatenate([[0], np.cumsum(self.dims)[:-1]])]
        self.max_batch = int(max_batch)
        self.optimizer = optimizer
        self.hbm_rows = [int(r.hbm_rows) for r in remaps]
        tabs = (_lib.rs_emb_table * len(specs))()
        hold = []
        self.unbacked_tables = 0
        for i, (s, r) in enumerate(zip(specs, remaps)):
            if s.elem_bytes not in (2, 4):  # inc/types.hpp:50-52
                raise InvalidArgument(f"table {s.table_id}: elem_bytes must be 2 or 4")
            # an omit_unaccessed remap (inc/remap.hpp:43-48) backs only its
            # slow_rows_allocated prefix; the rest pool as zero rows
            slow = int(s.hash_size - r.hbm_rows)
            alloc = int(r.slow_rows_allocated)
            unbacked = alloc < slow
            if unbacked:
                slow = alloc
                self.unbacked_tables += 1
            if is_device(r.entries):
                p, loc = ptr(r.entries), _lib.RS_MEM_DEVICE
            else:
                a = np.ascontiguousarray(r.entries, np.int32)
                hold.append(a)
                p, loc = ptr(a), _lib.RS_MEM_HOST
            tabs[i] = _lib.rs_emb_table(s.table_id, s.hash_size, s.dim, p, loc, r.hbm_rows, slow,
                                        s.elem_bytes, int(unbacked))
        h = C.c_void_p()
        _lib.check(_lib.lib().rs_emb_create(self.ctx.h, len(specs), tabs, C.c_uint64(max_batch),
                                            C.c_uint64(max_lookups), OPTIMIZERS[optimizer],
                                            C.c_float(eps), C.byref(h)))
        del hold
        self.h = h

    def init_weights(self, seed: int, scale: float = 0.1):
        _lib.check(_lib.lib().rs_emb_init_weights(self.h, C.c_uint64(seed), C.c_float(scale)))

    @staticmethod
    def _check_dev(*ts):
        for t in ts:
            if t is not None and (not is_device(t) or not t.is_contiguous()):
                raise InvalidArgument("TieredEmbeddingBag: batch tensors must be contiguous cuda tensors")

    def forward(self, offsets, indices, batch: int, out=None, hits=None):
        """offsets: [T*B+1] u32/i32, indices: u32/i32 original rows (cuda).  Returns
        pooled [B, sum(dim)] fp32.  ``hits`` (cuda u64/i64 [2T]) accumulates the
        per-table (fast, slow) lookup counts."""
        import torch

        self._check_dev(offsets, indices, out, hits)
        if out is None:
            out = torch.empty(batch, self.total_dim, dtype=torch.float32, device=offsets.device)
        _lib.check(_lib.lib().rs_emb_forward(self.h, C.c_uint64(batch), ptr(offsets), ptr(indices),
                                             ptr(out), ptr(hits)))
        return out

    def backward(self, offsets, indices, grad, batch: int, lr: float):
        self._check_dev(offsets, indices, grad)
        _lib.check(_lib.lib().rs_emb_backward(self.h, C.c_uint64(batch), ptr(offsets), ptr(indices),
                                              ptr(grad), C.c_float(lr)))

    def enable_uvm_cache(self, nslots: int):
        """HBM staging of slow-tier rows with side-stream prefetch/write-back
        (csrc/uvm_cache.cuh); nslots >= 4x the unique slow rows of a batch (up to four generations are live)."""
        _lib.check(_lib.lib().rs_emb_enable_uvm_cache(self.h, C.c_uint32(nslots)))

    def prefetch(self, offsets, indices, batch: int):
        """Stage the next batch's slow rows while the current batch runs."""
        self._check_dev(offsets, indices)
        _lib.check(_lib.lib().rs_emb_prefetch(self.h, C.c_uint64(batch), ptr(offsets), ptr(indices)))

    def flush(self):
        _lib.check(_lib.lib().rs_emb_flush(self.h))

    def read_rows(self, t: int, rows):
        rows = np.ascontiguousarray(rows, np.uint32)
        out = np.empty((rows.size, self.dims[t]), np.float32)
        mom = np.empty(rows.size, np.float32)
        _lib.check(_lib.lib().rs_emb_read_rows(self.h, t, ptr(rows), C.c_uint64(rows.size),
                                               ptr(out), ptr(mom)))
        return out, mom

    def kernel_times(self, reset: bool = False):
        """(fwd_ms, n_fwd, bwd_ms, n_bwd): summed kernel-only times of the
        forward / backward kernel sequences (CUDA events on the operator's
        stream, excluding staging waits) since the last reset."""
        f, nf, b, nb = C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()
        _lib.check(_lib.lib().rs_emb_kernel_times(self.h, C.byref(f), C.byref(nf), C.byref(b),
                                                  C.byref(nb), int(reset)))
        return float(f.value), int(nf.value), float(b.value), int(nb.value)

    def unbacked(self, reset: bool = False):
        """(lookups, rows) per table: lookups of rows an omit_unaccessed remap
        left without storage since the last reset (they pooled as zero rows),
        and how many remap entries are unbacked."""
        n = len(self.specs)
        lk = np.zeros(n, np.uint64)
        rw = np.zeros(n, np.uint64)
        _lib.check(_lib.lib().rs_emb_unbacked(self.h, ptr(lk), ptr(rw), int(reset)))
        return lk, rw

    def memory(self):
        a, b = C.c_uint64(), C.c_uint64()
        _lib.check(_lib.lib().rs_emb_memory(self.h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def close(self):
        if self.h:
            _lib.lib().rs_emb_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
