"""Trace files: Python mirror of include/shardplan/trace_io.hpp on the GPU.

``read_trace`` / ``write_trace`` keep the reference's names, file format and
errors (core/src/trace_io.cpp:48-158; ".gz" paths through zlib as
core/src/line_io.cpp).  Parsing and formatting run in the kernels of
csrc/trace_io.cu; ``TraceFile`` keeps a loaded trace in device memory so it
can be profiled or simulated without a host round trip.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .profiler import trace_struct
from .runtime import default_context
from .types import TableSpec, Trace


class TraceFile:
    """A trace loaded on the GPU (``rs_trace_file``).  ``trace()`` returns it as a
    :class:`Trace` of cuda tensors (copies) or numpy arrays (``device=False``)."""

    def __init__(self, path, ctx=None, chunk_bytes: int = 0):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _lib.check(_lib.lib().rs_trace_read(self.ctx.h, str(path).encode(), C.c_uint64(chunk_bytes),
                                            C.byref(h)))
        self.h = h
        v = _lib.rs_trace()
        _lib.check(_lib.lib().rs_trace_file_view(self.h, C.byref(v)))
        self.view = v
        self.tables = [TableSpec(v.tables[i].table_id, v.tables[i].cardinality, v.tables[i].hash_size,
                                 v.tables[i].dim, v.tables[i].elem_bytes) for i in range(v.num_tables)]
        self.num_samples = int(v.num_samples)
        self.num_records = int(v.num_records)
        self.num_ids = int(v.num_ids)

    def trace(self, device: bool = True) -> Trace:
        R, N = self.num_records, self.num_ids
        if device:
            import torch

            dev = f"cuda:{self.ctx.device}"
            arrs = [torch.empty(R, dtype=torch.int64, device=dev), torch.empty(R, dtype=torch.int32, device=dev),
                    torch.empty(R, dtype=torch.int64, device=dev), torch.empty(R, dtype=torch.int32, device=dev),
                    torch.empty(N, dtype=torch.int32, device=dev)]
            loc = _lib.RS_MEM_DEVICE
            ptrs = [C.c_void_p(a.data_ptr()) if a.numel() else None for a in arrs]
        else:
            arrs = [np.empty(R, np.uint64), np.empty(R, np.uint32), np.empty(R, np.uint64),
                    np.empty(R, np.uint32), np.empty(N, np.uint32)]
            loc = _lib.RS_MEM_HOST
            ptrs = [C.c_void_p(a.ctypes.data) if a.size else None for a in arrs]
        _lib.check(_lib.lib().rs_trace_file_export(self.ctx.h, self.h, *ptrs, loc))
        return Trace(list(self.tables), self.num_samples, arrs[0], arrs[1], arrs[2], arrs[3], ids=arrs[4])

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().rs_trace_file_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass


def read_trace(path, device: bool = False, ctx=None) -> Trace:
    """include/shardplan/trace_io.hpp:35 — ``Trace read_trace(path)``."""
    f = TraceFile(path, ctx)
    try:
        return f.trace(device=device)
    finally:
        f.close()


def write_trace(trace: Trace, path, comments=(), ctx=None) -> None:
    """include/shardplan/trace_io.hpp:32-33 — ``write_trace(trace, path, comments)``;
    byte-identical to the reference writer.  Host or cuda-tensor traces."""
    ctx = ctx or default_context()
    st, keep = trace_struct(trace)
    cs = [str(c).encode() for c in comments]
    arr = (C.c_char_p * max(1, len(cs)))(*cs)
    _lib.check(_lib.lib().rs_trace_write(ctx.h, C.byref(st), str(path).encode(), arr, len(cs)))
    del keep
