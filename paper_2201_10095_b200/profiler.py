"""HP1 — the profiler: Python mirror of include/shardplan/profiler.hpp over the C-ABI.

``profile`` / ``profile_raw`` / ``build_icdf`` / ``hash_utilization`` /
``hash_value`` keep the reference's names, argument meaning and errors
(core/src/profiler.cpp:49-174, inc/workload.hpp:28-31); the work runs in the
sm_100a kernels of csrc/profile.cu.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .runtime import default_context, is_device, ptr
from .types import FeatureStats, Trace


def hash_value(raw_id: int, hash_size: int) -> int:
    """inc/workload.hpp:28-31 — uint32(mix64(raw) % hash_size)."""
    out = C.c_uint32()
    _lib.check(_lib.lib().rs_hash_value(C.c_uint64(raw_id), C.c_uint64(hash_size), C.byref(out)))
    return int(out.value)


def hash_ids(raw, hash_size: int, ctx=None):
    """Batched hash_value on the GPU (K0).  numpy in -> numpy out; cuda tensor in -> cuda tensor out."""
    ctx = ctx or default_context()
    if is_device(raw):
        import torch

        out = torch.empty(raw.numel(), dtype=torch.int32, device=raw.device)
        loc = _lib.RS_MEM_DEVICE
    else:
        raw = np.ascontiguousarray(raw, np.uint64)
        out = np.empty(raw.size, np.uint32)
        loc = _lib.RS_MEM_HOST
    n = raw.numel() if is_device(raw) else raw.size
    _lib.check(_lib.lib().rs_hash_ids(ctx.h, ptr(raw), C.c_uint64(n), C.c_uint64(hash_size),
                                      ptr(out), loc))
    return out


def _spec_array(tables):
    arr = (_lib.rs_table_spec * max(1, len(tables)))()
    for i, t in enumerate(tables):
        arr[i] = _lib.rs_table_spec(t.table_id, t.cardinality, t.hash_size, t.dim, t.elem_bytes)
    return arr


def _host(a, dt):
    return None if a is None else np.ascontiguousarray(a, dt)


def trace_struct(trace: Trace):
    """Builds the rs_trace view; returns (struct, keepalive)."""
    dev = is_device(trace.rec_sample)
    ids = trace.ids
    raw = trace.raw_ids
    if dev:
        arrs = [trace.rec_sample, trace.rec_table, trace.rec_offset, trace.rec_len, ids, raw]
        for a, sz in zip(arrs, (8, 4, 8, 4, 4, 8)):
            if a is not None and (a.element_size() != sz or not a.is_contiguous()):
                raise TypeError("device trace arrays must be contiguous with u64/u32 element sizes")
        loc = _lib.RS_MEM_DEVICE
    else:
        arrs = [_host(trace.rec_sample, np.uint64), _host(trace.rec_table, np.uint32),
                _host(trace.rec_offset, np.uint64), _host(trace.rec_len, np.uint32),
                _host(ids, np.uint32), _host(raw, np.uint64)]
        loc = _lib.RS_MEM_HOST
    specs = _spec_array(trace.tables)
    n_ids = 0
    src = arrs[4] if arrs[4] is not None else arrs[5]
    if src is not None:
        n_ids = src.numel() if dev else src.size
    nrec = arrs[0].numel() if dev else arrs[0].size
    st = _lib.rs_trace(len(trace.tables), specs, trace.num_samples, nrec, ptr(arrs[0]),
                       ptr(arrs[1]), ptr(arrs[2]), ptr(arrs[3]), n_ids, ptr(arrs[4]),
                       ptr(arrs[5]), loc)
    return st, (arrs, specs)


class _Owner:
    """Owns one rs_profile; freed when the Profile and every array viewing its
    pinned buffers are gone (the stats arrays are zero-copy views)."""

    def __init__(self, h):
        self.h = h

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            if self.h:
                _lib.lib().rs_profile_destroy(self.h)
                self.h = None
        except Exception:
            pass


def _view(owner, p, n, ctype, dtype):
    """numpy view of n elements at ctypes pointer p that keeps `owner` alive."""
    if n == 0:
        return np.zeros(0, dtype)
    arr = (ctype * n).from_address(C.cast(p, C.c_void_p).value)
    arr._owner = owner
    return np.frombuffer(arr, dtype=dtype)


class Profile:
    """Handle of one profile() result.  ``stats`` hold zero-copy numpy views of
    the pinned host arrays the kernels wrote (no host-side copy of the
    per-row CDFs/rankings); ``device_rows_by_rank(j)`` exposes the device
    ranking (feeds build_remap)."""

    def __init__(self, h):
        self._owner = _Owner(h)
        self.h = h
        L = _lib.lib()
        n = C.c_uint32()
        _lib.check(L.rs_profile_num_tables(h, C.byref(n)))
        sel = C.c_uint64()
        _lib.check(L.rs_profile_selected(h, C.byref(sel)))
        self.selected = int(sel.value)
        self.stats = []
        self._dev = []
        for j in range(n.value):
            v = _lib.rs_feature_stats()
            _lib.check(L.rs_profile_get(h, j, C.byref(v)))
            d = int(v.distinct_rows_accessed)
            icdf = np.ctypeslib.as_array(v.icdf_steps, shape=(101,)).copy()
            cdf = _view(self._owner, v.access_cdf, d, C.c_double, np.float64)
            rbr = _view(self._owner, v.rows_by_rank, d, C.c_uint32, np.uint32)
            self.stats.append(FeatureStats(int(v.table_id), float(v.coverage),
                                           float(v.avg_pooling), d, int(v.total_accesses),
                                           icdf, cdf, rbr))
            self._dev.append(v.d_rows_by_rank)

    def device_rows_by_rank(self, j):
        if self._owner is None:
            raise ValueError("profile handle closed")
        return self._dev[j]

    def close(self):
        """Drops this handle's reference; the buffers are freed once no stats
        array views them any more."""
        self._owner = None
        self.h = None


def profile_handle(trace: Trace, sample_rate: float, seed: int, ctx=None) -> Profile:
    ctx = ctx or default_context()
    st, keep = trace_struct(trace)
    h = C.c_void_p()
    _lib.check(_lib.lib().rs_profile_run(ctx.h, C.byref(st), C.c_double(sample_rate),
                                         C.c_uint64(seed), C.byref(h)))
    del keep
    return Profile(h)


def profile(trace: Trace, sample_rate: float, seed: int, ctx=None) -> list:
    """core/src/profiler.cpp:60-161 — one FeatureStats per trace table, in trace order.

    A trace carrying ``raw_ids`` (and no ``ids``) is hashed on the GPU first
    (profile_raw)."""
    p = profile_handle(trace, sample_rate, seed, ctx)
    out = p.stats
    p.close()
    return out


def profile_raw(trace: Trace, sample_rate: float, seed: int, ctx=None) -> list:
    if trace.raw_ids is None:
        raise ValueError("profile_raw needs trace.raw_ids")
    return profile(trace, sample_rate, seed, ctx)


def build_icdf(counts_per_row, ctx=None) -> np.ndarray:
    """core/src/profiler.cpp:49-58 — 101-entry inverse CDF (GPU sort + scan)."""
    ctx = ctx or default_context()
    c = np.ascontiguousarray(counts_per_row, np.uint64)
    out = np.empty(101, np.uint64)
    _lib.check(_lib.lib().rs_build_icdf(ctx.h, ptr(c), C.c_uint64(c.size), _lib.RS_MEM_HOST,
                                        ptr(out)))
    return out


def count_distinct_raw(trace: Trace, ctx=None) -> np.ndarray:
    """GenStats.distinct_raw_ids (core/src/workload.cpp:195-223) of a raw trace,
    counted on the GPU: distinct raw values per table over every record."""
    if trace.raw_ids is None:
        raise ValueError("count_distinct_raw needs trace.raw_ids")
    ctx = ctx or default_context()
    st, keep = trace_struct(trace)
    out = np.zeros(max(1, len(trace.tables)), np.uint64)
    _lib.check(_lib.lib().rs_count_distinct_raw(ctx.h, C.byref(st), ptr(out)))
    del keep
    return out[:len(trace.tables)]


def hash_utilization(stats: FeatureStats, spec, distinct_raw_ids_seen: int):
    """core/src/profiler.cpp:163-174 — (sparsity_fraction, collision_fraction)."""
    s, c = C.c_double(), C.c_double()
    _lib.check(_lib.lib().rs_hash_utilization(C.c_uint64(stats.distinct_rows_accessed),
                                              C.c_uint64(spec.hash_size),
                                              C.c_uint64(distinct_raw_ids_seen), C.byref(s),
                                              C.byref(c)))
    return s.value, c.value
