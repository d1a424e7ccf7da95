"""simulate(): Python mirror of include/shardplan/simulator.hpp:45-47.

Tier counts come from the GPU pass in csrc/simulate.cu; the report is filled
exactly as core/src/simulator.cpp:96-137 writes it.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .profiler import trace_struct
from .runtime import default_context, is_device, ptr
from .types import GpuReport, SimReport


def simulate(trace, plan, remaps, system, batch_size: int, ctx=None) -> SimReport:
    ctx = ctx or default_context()
    st, keep = trace_struct(trace)
    ents = (_lib.rs_plan_entry * max(1, len(plan.entries)))()
    for i, e in enumerate(plan.entries):
        ents[i] = _lib.rs_plan_entry(e.table_id, e.gpu, e.step, e.hbm_rows, e.pct, e.mem_bytes)
    rv = (_lib.rs_remap_view * max(1, len(remaps)))()
    hold = []
    for i, r in enumerate(remaps):
        if is_device(r.entries):
            rv[i] = _lib.rs_remap_view(r.table_id, r.hash_size, r.hbm_rows, ptr(r.entries),
                                       _lib.RS_MEM_DEVICE)
        else:
            a = np.ascontiguousarray(r.entries, np.int32)
            hold.append(a)
            rv[i] = _lib.rs_remap_view(r.table_id, r.hash_size, r.hbm_rows, ptr(a),
                                       _lib.RS_MEM_HOST)
    sysc = _lib.rs_system_spec(system.num_gpus, system.batch_size, system.cap_hbm_bytes,
                               system.cap_dram_bytes, system.bw_hbm, system.bw_uvm)
    M = max(1, system.num_gpus)
    gh, gu, gc = np.zeros(M), np.zeros(M), np.zeros(M)
    tff = np.zeros(max(1, len(trace.tables)))
    rep = _lib.rs_sim_report()
    rep.gpu_hbm_accesses = gh.ctypes.data_as(C.POINTER(C.c_double))
    rep.gpu_uvm_accesses = gu.ctypes.data_as(C.POINTER(C.c_double))
    rep.gpu_est_iter_cost = gc.ctypes.data_as(C.POINTER(C.c_double))
    rep.table_fast_fraction = tff.ctypes.data_as(C.POINTER(C.c_double))
    _lib.check(_lib.lib().rs_simulate(ctx.h, C.byref(st), len(plan.entries), ents, len(remaps),
                                      rv, C.byref(sysc), C.c_uint64(batch_size), C.byref(rep)))
    del keep, hold
    out = SimReport()
    out.gpus = [GpuReport(float(gh[g]), float(gu[g]), float(gc[g])) for g in range(system.num_gpus)]
    out.batches = int(rep.batches)
    out.total_accesses = int(rep.total_accesses)
    out.min_cost, out.max_cost = float(rep.min_cost), float(rep.max_cost)
    out.mean_cost, out.stddev_cost = float(rep.mean_cost), float(rep.stddev_cost)
    out.uvm_access_fraction = float(rep.uvm_access_fraction)
    out.table_fast_fraction = [float(x) for x in tff[:len(trace.tables)]]
    return out
