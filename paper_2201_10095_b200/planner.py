"""Host-side sharder: the plans HP2 serves.

The cost model and every placement strategy run in ``libshardplan_gpu.so``'s
host planner (csrc/planner.cpp), restated from the reference with the same
floating-point order and tie-breaks, so plans are identical to the
reference's (tests/test_planner.py compares them field by field):

* ``table_fixed_cost``  core/src/baselines.cpp:44-67
* ``greedy_shard``      core/src/baselines.cpp:136-203 (the greedy/size plan)
* ``ldm_shard``         core/src/baselines.cpp:205-292
* ``build_instance`` + ``solve``  core/src/milp.cpp:20-56 +
  core/src/milp_solve.cpp:633-709 (RecShard's MILP: branch and bound with an
  LPT seed, move/swap local search and exact knapsack polish) — the local
  search evaluates its candidates on host threads (``threads``), with the
  reference's scan order, so the plan does not depend on the thread count.

``table_cost`` / ``rows_at_step`` / ``recompute_plan_costs`` restate
core/src/plan.cpp:25-63 in Python for reporting.  ``fill_spare_capacity`` is
OUR extension beyond the MILP (off unless asked for).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .runtime import ptr
from .types import InvalidArgument, PlanEntry, ShardingPlan

KPCT = 100
COST_KINDS = {"size": 0, "lookup": 1, "size-lookup": 2, "size-and-lookup": 2}


def table_cost(spec, stats, pct, system, use_pooling=True):
    """core/src/plan.cpp:25-33"""
    if not (0.0 <= pct <= 1.0):
        raise InvalidArgument("table_cost: pct must be in [0, 1]")
    pool = stats.avg_pooling if use_pooling else 1.0
    demand = pool * spec.dim * spec.elem_bytes * float(system.batch_size)
    return demand * (pct / system.bw_hbm + (1.0 - pct) / system.bw_uvm)


def rows_at_step(icdf_steps, step, step_count):
    """core/src/plan.cpp:35-44"""
    if step > step_count:
        raise InvalidArgument("rows_at_step: step exceeds step_count")
    pidx = (step * KPCT + step_count - 1) // step_count
    return int(icdf_steps[pidx])


def recompute_plan_costs(plan, specs, stats, system, use_coverage=True, use_pooling=True):
    """core/src/plan.cpp:46-63"""
    by_id = {s.table_id: (s, st) for s, st in zip(specs, stats)}
    plan.gpu_cost = [0.0] * system.num_gpus
    for e in plan.entries:
        if e.table_id not in by_id:
            raise InvalidArgument(f"plan entry for table {e.table_id} not in instance")
        s, st = by_id[e.table_id]
        w = st.coverage if use_coverage else 1.0
        plan.gpu_cost[e.gpu] += w * table_cost(s, st, e.pct, system, use_pooling)
    plan.objective = 0.0
    for c in plan.gpu_cost:
        plan.objective = max(plan.objective, c)
    return plan


def _spec(s):
    return _lib.rs_table_spec(s.table_id, s.cardinality, s.hash_size, s.dim, s.elem_bytes)


def _sys(system):
    return _lib.rs_system_spec(system.num_gpus, system.batch_size, system.cap_hbm_bytes,
                               system.cap_dram_bytes, system.bw_hbm, system.bw_uvm)


def table_fixed_cost(spec, stats, kind="size"):
    """core/src/baselines.cpp:44-67 (stats may be None for "size")."""
    if kind not in COST_KINDS:
        raise InvalidArgument("unknown cost function: " + str(kind))
    out = C.c_double()
    pool = None if stats is None else C.c_double(stats.avg_pooling)
    sp = _spec(spec)
    _lib.check(_lib.lib().rs_table_fixed_cost(C.byref(sp), None if pool is None else C.byref(pool),
                                              COST_KINDS[kind], C.byref(out)), planner=True)
    return out.value


@dataclass
class MilpInstance:
    """include/shardplan/plan.hpp:37-47 — aligned (spec, stats) pairs + system."""
    specs: list
    stats: list
    system: object
    use_pooling: bool = True
    use_coverage: bool = True
    step_count: int = 100


def build_instance(stats, specs, system, ablation=(True, True), step_count=100):
    """core/src/milp.cpp:20-56 — stats are matched to specs by table id."""
    if not specs:
        raise InvalidArgument("build_instance: no tables")
    if len(stats) != len(specs):
        raise InvalidArgument(f"build_instance: {len(stats)} stats for {len(specs)} specs")
    by_id = {st.table_id: st for st in stats}
    aligned = []
    for s in specs:
        if s.table_id not in by_id:
            raise InvalidArgument(f"build_instance: no stats for table {s.table_id}")
        aligned.append(by_id[s.table_id])
    return MilpInstance(list(specs), aligned, system, bool(ablation[0]), bool(ablation[1]), int(step_count))


def _tables(specs, stats):
    arr = (_lib.rs_plan_table * len(specs))()
    keep = []
    for i, (s, st) in enumerate(zip(specs, stats)):
        icdf = np.ascontiguousarray(st.icdf_steps, np.uint64)
        if icdf.size != 101:
            raise InvalidArgument(f"build_instance: table {s.table_id} stats lack the 101-entry icdf")
        keep.append(icdf)
        arr[i] = _lib.rs_plan_table(_spec(s), st.coverage, st.avg_pooling, ptr(icdf))
    return arr, keep


def _plan_out(call, specs, stats, system, strategy, step_count):
    """call(J, tables, system, entries, gpu_cost, summary) -> status"""
    J, M = len(specs), system.num_gpus
    tabs, keep = _tables(specs, stats)
    ents = (_lib.rs_plan_entry * max(1, J))()
    gc = np.zeros(max(1, M), np.float64)
    summ = _lib.rs_plan_summary()
    sysc = _sys(system)
    _lib.check(call(J, tabs, C.byref(sysc), ents, ptr(gc), C.byref(summ)), planner=True)
    del keep
    plan = ShardingPlan(strategy=strategy, step_count=step_count)
    plan.entries = [PlanEntry(e.table_id, e.gpu, e.step, e.hbm_rows, e.pct, e.mem_bytes)
                    for e in ents[:J]]
    plan.gpu_cost = [float(x) for x in gc[:M]]
    plan.objective = summ.objective
    plan.lower_bound = summ.lower_bound
    plan.proved_optimal = bool(summ.proved_optimal)
    return plan


def greedy_shard(costs, specs, stats, system, name="greedy"):
    """core/src/baselines.cpp:136-203"""
    c = np.ascontiguousarray(costs, np.float64)
    return _plan_out(lambda J, t, sy, e, g, su: _lib.lib().rs_plan_greedy(J, t, ptr(c), sy, e, g, su),
                     specs, stats, system, name, 1)


def ldm_shard(costs, specs, stats, system, name="ldm"):
    """core/src/baselines.cpp:205-292"""
    c = np.ascontiguousarray(costs, np.float64)
    return _plan_out(lambda J, t, sy, e, g, su: _lib.lib().rs_plan_ldm(J, t, ptr(c), sy, e, g, su),
                     specs, stats, system, name, 1)


def solve(instance, time_limit_seconds=math.inf, threads=0):
    """core/src/milp_solve.cpp:633-709 — the RecShard plan."""
    i = instance
    return _plan_out(lambda J, t, sy, e, g, su: _lib.lib().rs_plan_solve(
        J, t, sy, i.step_count, int(i.use_pooling), int(i.use_coverage), time_limit_seconds, threads,
        e, g, su), i.specs, i.stats, i.system, "milp", i.step_count)


def recshard_plan(specs, stats, system, step_count=100, time_limit_seconds=math.inf, threads=0):
    """RecShard: solve(build_instance(stats, specs, system))."""
    return solve(build_instance(stats, specs, system, step_count=step_count), time_limit_seconds, threads)


def unseen_mass(st):
    """Good-Turing estimate of the access probability mass on rows the
    profile never saw: (rows seen exactly once) / total accesses, read off the
    ranked CDF (count at rank r = (cdf[r] - cdf[r-1]) * total)."""
    if st.total_accesses == 0 or st.distinct_rows_accessed == 0:
        return 0.0
    cdf = np.asarray(st.access_cdf, np.float64)
    inc = np.diff(np.concatenate([[0.0], cdf])) * st.total_accesses
    n1 = int(np.count_nonzero(np.rint(inc) == 1))
    return n1 / float(st.total_accesses)


def fill_spare_capacity(plan, specs, stats, system):
    """Extension beyond the MILP (off by default in the solver): spend each
    GPU's leftover fast-tier bytes on never-profiled rows of tables whose whole
    profiled set is already fast, greedily by expected hits per byte
    (coverage * pooling * unseen mass / unseen rows / row bytes).  The extra
    rows are the reference remap's "never-accessed rows in ascending index
    order" (core/src/remap.cpp:71-78), so the plan format is unchanged."""
    M = system.num_gpus
    used = [0] * M
    for e in plan.entries:
        used[e.gpu] += e.mem_bytes
    cands = []
    for j, (s, st, e) in enumerate(zip(specs, stats, plan.entries)):
        unseen_rows = s.hash_size - st.distinct_rows_accessed
        if e.hbm_rows < st.distinct_rows_accessed or unseen_rows <= 0:
            continue
        m = unseen_mass(st)
        if m <= 0:
            continue
        rb = s.dim * s.elem_bytes
        dens = st.coverage * st.avg_pooling * m / unseen_rows / rb
        cands.append((-dens, s.table_id, j))
    cands.sort()
    for _, _, j in cands:
        e, s = plan.entries[j], specs[j]
        rb = s.dim * s.elem_bytes
        room = (system.cap_hbm_bytes - used[e.gpu]) // rb
        add = int(min(room, s.hash_size - e.hbm_rows))
        if add <= 0:
            continue
        e.hbm_rows += add
        e.mem_bytes = e.hbm_rows * rb
        used[e.gpu] += add * rb
    plan.strategy += "+fill"
    return plan
