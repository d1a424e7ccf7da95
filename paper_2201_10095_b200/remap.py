"""Remap tables: Python mirror of include/shardplan/remap.hpp (K3 on the GPU).

``build_remap`` keeps the reference's signature and errors
(core/src/remap.cpp:40-105); ``translate`` decodes the sign-bit encoding
(core/src/remap.cpp:107-116).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .runtime import default_context, is_device, ptr
from .types import TIER_FAST, TIER_SLOW, InvalidArgument, RemapTable


def build_remap(entry, stats, spec, omit_unaccessed: bool = False, ctx=None, device_rows=None,
                out=None) -> RemapTable:
    """The plan's ``entry.hbm_rows`` top-ranked rows go to the fast tier in rank
    order; the rest to the slow tier in ascending row order.

    ``device_rows``: optional device pointer of ``stats.rows_by_rank`` (from
    ``Profile.device_rows_by_rank``) to skip the upload.  ``out``: optional
    int32 cuda tensor of hash_size entries — then the entries stay on the GPU
    and ``RemapTable.entries`` is that tensor."""
    ctx = ctx or default_context()
    H = int(spec.hash_size)
    d = int(stats.distinct_rows_accessed)
    if device_rows is not None:
        rows_p, rows_loc = C.c_void_p(device_rows), _lib.RS_MEM_DEVICE
    else:
        rbr = np.ascontiguousarray(stats.rows_by_rank, np.uint32)
        if rbr.size != d:
            rows_p, rows_loc = None, _lib.RS_MEM_HOST  # reference: stats lack ranking
            if d == 0:
                rbr = np.zeros(1, np.uint32)
                rows_p = ptr(rbr)
        else:
            rows_p, rows_loc = ptr(rbr if rbr.size else np.zeros(1, np.uint32)), _lib.RS_MEM_HOST
    if out is not None:
        if not is_device(out) or out.numel() < H or out.element_size() != 4:
            raise InvalidArgument("build_remap: out must be an int32 cuda tensor of hash_size")
        ent, loc = out, _lib.RS_MEM_DEVICE
    else:
        ent, loc = np.empty(max(1, H), np.int32), _lib.RS_MEM_HOST
    slow = C.c_uint64()
    _lib.check(_lib.lib().rs_build_remap(ctx.h, C.c_uint32(spec.table_id), C.c_uint64(H),
                                         C.c_uint64(int(entry.hbm_rows)), rows_p, C.c_uint64(d),
                                         rows_loc, int(bool(omit_unaccessed)), ptr(ent), loc,
                                         C.byref(slow)))
    return RemapTable(int(spec.table_id), H, int(entry.hbm_rows), int(slow.value),
                      ent if loc == _lib.RS_MEM_DEVICE else ent[:H])


def translate(remap: RemapTable, original_index: int):
    """core/src/remap.cpp:107-116 — (Tier, offset)."""
    if original_index < 0 or original_index >= remap.hash_size:
        raise InvalidArgument(f"translate: index {original_index} out of range for table "
                              f"{remap.table_id}")
    v = int(remap.entries[original_index])
    return (TIER_FAST, v) if v >= 0 else (TIER_SLOW, -v - 1)


def write_remap(remap: RemapTable, path, ctx=None) -> None:
    """include/shardplan/remap.hpp:62 — SPRM binary file, byte-identical to the
    reference's write_remap.  Entries may be a numpy array or an int32 cuda
    tensor (streamed out through pinned memory)."""
    if len(remap.entries) != remap.hash_size:
        raise InvalidArgument(f"write_remap: table {remap.table_id} has {len(remap.entries)} "
                              f"entries for hash_size {remap.hash_size}")
    dev = is_device(remap.entries)
    if dev:
        ctx = ctx or default_context()
        ent, loc, h = remap.entries, _lib.RS_MEM_DEVICE, ctx.h
    else:
        ent = np.ascontiguousarray(remap.entries, np.int32)
        loc, h = _lib.RS_MEM_HOST, None
    _lib.check(_lib.lib().rs_remap_write(h, str(path).encode(), C.c_uint32(remap.table_id),
                                         C.c_uint64(remap.hash_size), C.c_uint64(remap.hbm_rows),
                                         ptr(ent) if remap.hash_size else None, loc))


def read_remap(path, device: bool = False, ctx=None) -> RemapTable:
    """include/shardplan/remap.hpp:63 — reads an SPRM file (the reference's
    errors: IoError, ParseError).  ``device``: entries land in an int32 cuda
    tensor, streamed through pinned memory; slow_rows_allocated is counted on
    the GPU."""
    tid, H, hbm = C.c_uint32(), C.c_uint64(), C.c_uint64()
    _lib.check(_lib.lib().rs_remap_read_header(str(path).encode(), C.byref(tid), C.byref(H),
                                               C.byref(hbm)))
    n = int(H.value)
    slow = C.c_uint64()
    if device:
        import torch

        ctx = ctx or default_context()
        out = torch.empty(max(1, n), dtype=torch.int32, device=f"cuda:{ctx.device}")
        _lib.check(_lib.lib().rs_remap_read(ctx.h, str(path).encode(), ptr(out), _lib.RS_MEM_DEVICE,
                                            C.c_uint64(out.numel()), C.byref(slow)))
        ent = out[:n]
    else:
        ent = np.empty(max(1, n), np.int32)
        _lib.check(_lib.lib().rs_remap_read(None, str(path).encode(), ptr(ent), _lib.RS_MEM_HOST,
                                            C.c_uint64(ent.size), C.byref(slow)))
        ent = ent[:n]
    return RemapTable(int(tid.value), n, int(hbm.value), int(slow.value), ent)
