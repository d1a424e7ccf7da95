"""Host-side sharders that produce the plans HP2 serves.

Out of the §8 hot-path scope (the planner is tiny host work): these exist so
the operator and bench have plans to serve.

* ``table_cost`` / ``rows_at_step`` / ``recompute_plan_costs`` restate
  core/src/plan.cpp:25-63.
* ``table_fixed_cost`` / ``greedy_shard`` restate core/src/baselines.cpp:44-203
  (the "greedy/size" baseline plan); tests check them against the reference.
* ``recshard_plan`` is OUR heuristic for RecShard's MILP (
  reference solver core/src/milp_solve.cpp): per-GPU multiple-choice knapsack
  over each table's ICDF step curve (convex-hull greedy) plus an LPT
  assignment refined by move/swap local search.  It is not the reference
  branch-and-bound, so placements are not bit-identical to ``solve``; tests
  bound its objective against the reference solver's.
"""
from __future__ import annotations

import math

import numpy as np

from .types import InfeasibleError, InvalidArgument, PlanEntry, ShardingPlan

KPCT = 100


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


def table_fixed_cost(spec, stats, kind="size"):
    """core/src/baselines.cpp:44-68"""
    if kind == "size":
        return float(spec.hash_size) * spec.dim
    if stats is None:
        raise InvalidArgument(f"{kind} cost needs feature stats")
    if kind == "lookup":
        return stats.avg_pooling * spec.dim
    if kind == "size-lookup":
        lt = math.log10(float(spec.hash_size))
        return stats.avg_pooling * spec.dim * max(0.0, lt)
    raise InvalidArgument("unknown cost function: " + kind)


def _validate_system(s):
    if s.num_gpus < 1:
        raise InvalidArgument("system: num_gpus must be >= 1")
    if s.batch_size < 1:
        raise InvalidArgument("system: batch_size must be >= 1")
    if s.cap_hbm_bytes < 1 or s.cap_dram_bytes < 1:
        raise InvalidArgument("system: capacities must be positive")
    if not (s.bw_hbm > 0 and s.bw_uvm > 0):
        raise InvalidArgument("system: bandwidths must be positive")
    if not s.bw_hbm > s.bw_uvm:
        raise InvalidArgument("system: bw_hbm must exceed bw_uvm")


def _check_aggregate(specs, system):
    total = sum(s.bytes() for s in specs)
    agg = system.num_gpus * (system.cap_hbm_bytes + system.cap_dram_bytes)
    if total > agg:
        raise InfeasibleError(f"total table bytes {total} exceed aggregate capacity {agg}")


def _assemble(specs, stats, system, gpu_of, in_hbm, strategy):
    """core/src/baselines.cpp:94-118 — whole-table plan, step grid of 1."""
    plan = ShardingPlan(strategy=strategy, step_count=1)
    for j, s in enumerate(specs):
        hb = s.hash_size if in_hbm[j] else 0
        plan.entries.append(PlanEntry(s.table_id, gpu_of[j], 1 if in_hbm[j] else 0, hb,
                                      1.0 if in_hbm[j] else 0.0, hb * s.dim * s.elem_bytes))
    return recompute_plan_costs(plan, specs, stats, system)


def greedy_shard(costs, specs, stats, system, name="greedy"):
    """core/src/baselines.cpp:136-203"""
    _validate_system(system)
    _check_aggregate(specs, system)
    if len(costs) != len(specs):
        raise InvalidArgument("baseline: costs and specs differ in length")
    if not specs:
        raise InvalidArgument("baseline: no tables")
    order = sorted(range(len(specs)), key=lambda i: (-costs[i], specs[i].table_id))
    M = system.num_gpus
    gpu_of = [0] * len(specs)
    in_hbm = [False] * len(specs)
    hbm_cost, tot_cost = [0.0] * M, [0.0] * M
    hbm_used, uvm_used = [0] * M, [0] * M
    uvm_scale = system.bw_hbm / system.bw_uvm
    hbm_phase = True
    for pos, j in enumerate(order):
        b = specs[j].bytes()
        if hbm_phase:
            pick = None
            if pos < M:
                if hbm_used[pos] + b <= system.cap_hbm_bytes:
                    pick = pos
            else:
                best = 0.0
                for g in range(M):
                    if hbm_used[g] + b > system.cap_hbm_bytes:
                        continue
                    if pick is None or hbm_cost[g] < best:
                        pick, best = g, hbm_cost[g]
            if pick is not None:
                gpu_of[j], in_hbm[j] = pick, True
                hbm_used[pick] += b
                hbm_cost[pick] += costs[j]
                tot_cost[pick] += costs[j]
                continue
            hbm_phase = False
        pick, best = None, 0.0
        for g in range(M):
            if uvm_used[g] + b > system.cap_dram_bytes:
                continue
            if pick is None or tot_cost[g] < best:
                pick, best = g, tot_cost[g]
        if pick is None:
            raise InfeasibleError(f"greedy: table {specs[j].table_id} ({b} bytes) fits no GPU's slow tier")
        gpu_of[j], in_hbm[j] = pick, False
        uvm_used[pick] += b
        tot_cost[pick] += costs[j] * uvm_scale
    return _assemble(specs, stats, system, gpu_of, in_hbm, name)


# ---------------------------------------------------------------- RecShard heuristic
class _Curve:
    """One table's step options: rows/bytes/cost per step, and the lower convex
    hull used for the marginal-gain knapsack."""

    def __init__(self, spec, st, system, S):
        self.spec, self.st, self.S = spec, st, S
        rb = spec.dim * spec.elem_bytes
        self.rows = np.array([rows_at_step(st.icdf_steps, i, S) for i in range(S + 1)], np.int64)
        self.bytes = self.rows * rb
        self.dram = (spec.hash_size - self.rows) * rb
        w = st.coverage
        self.cost = np.array([w * table_cost(spec, st, i / S, system) for i in range(S + 1)])
        # among equal-row steps keep the highest pct (plan.hpp: ties pin the highest pct)
        hull = [0]
        for i in range(1, S + 1):
            if self.rows[i] == self.rows[hull[-1]]:
                hull[-1] = i
                continue
            while len(hull) >= 2:
                a, b = hull[-2], hull[-1]
                s1 = (self.cost[a] - self.cost[b]) / max(1, self.bytes[b] - self.bytes[a])
                s2 = (self.cost[b] - self.cost[i]) / max(1, self.bytes[i] - self.bytes[b])
                if s2 >= s1:
                    hull.pop()
                else:
                    break
            hull.append(i)
        self.hull = hull


def _knapsack(curves, cap_hbm, cap_dram):
    """Greedy over hull segments by cost decrease per HBM byte; returns (steps, cost) or None."""
    steps = [c.hull[0] for c in curves]
    pos = [0] * len(curves)
    used = sum(int(c.bytes[s]) for c, s in zip(curves, steps))
    dram = sum(int(c.dram[s]) for c, s in zip(curves, steps))
    if used > cap_hbm:
        return None
    import heapq

    heap = []

    def push(k):
        c = curves[k]
        if pos[k] + 1 < len(c.hull):
            a, b = c.hull[pos[k]], c.hull[pos[k] + 1]
            db = int(c.bytes[b] - c.bytes[a])
            gain = (c.cost[a] - c.cost[b]) / max(1, db)
            heapq.heappush(heap, (-gain, c.spec.table_id, k))

    for k in range(len(curves)):
        push(k)
    while heap:
        _, _, k = heapq.heappop(heap)
        c = curves[k]
        a, b = c.hull[pos[k]], c.hull[pos[k] + 1]
        db = int(c.bytes[b] - c.bytes[a])
        if used + db <= cap_hbm:
            used += db
            dram -= int(c.dram[a] - c.dram[b])
            pos[k] += 1
            steps[k] = b
            push(k)
        else:
            # partial: best non-hull step of this table that still fits
            best = steps[k]
            for i in range(steps[k] + 1, c.S + 1):
                if used + int(c.bytes[i] - c.bytes[steps[k]]) <= cap_hbm and c.cost[i] < c.cost[best]:
                    best = i
            used += int(c.bytes[best] - c.bytes[steps[k]])
            dram -= int(c.dram[steps[k]] - c.dram[best])
            steps[k] = best
    if dram > cap_dram:
        return None
    return steps, float(sum(c.cost[s] for c, s in zip(curves, steps)))


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


def recshard_plan(specs, stats, system, step_count=100, iters=200):
    """Minimise max_m c_m with per-GPU HBM/DRAM capacities."""
    _validate_system(system)
    _check_aggregate(specs, system)
    M = system.num_gpus
    curves = [_Curve(s, st, system, step_count) for s, st in zip(specs, stats)]
    # LPT on the all-HBM access demand, balancing bytes as a secondary key
    order = sorted(range(len(specs)), key=lambda j: (-curves[j].cost[-1], specs[j].table_id))
    load = [0.0] * M
    bytes_on = [0] * M
    assign = [0] * len(specs)
    # a GPU can only take a table if its slow tier can hold what its fast tier
    # cannot: the fast tier holds profiled rows only (the curves end at the
    # distinct rows seen), so never-seen rows always count against DRAM
    acc_on = [0] * M
    acc = [int(c.bytes[-1]) for c in curves]

    def fits(m, j):
        b = bytes_on[m] + specs[j].bytes()
        return b - min(system.cap_hbm_bytes, acc_on[m] + acc[j]) <= system.cap_dram_bytes

    for j in order:
        ok = [m for m in range(M) if fits(m, j)]
        g = min(ok or range(M), key=lambda m: (load[m], bytes_on[m], m))
        assign[j] = g
        acc_on[g] += acc[j]
        load[g] += curves[j].cost[-1]
        bytes_on[g] += specs[j].bytes()

    def solve_gpu(g, asg):
        ks = [j for j in range(len(specs)) if asg[j] == g]
        r = _knapsack([curves[j] for j in ks], system.cap_hbm_bytes, system.cap_dram_bytes)
        if r is None:
            return None
        return dict(zip(ks, r[0])), r[1]

    sol = [solve_gpu(g, assign) for g in range(M)]
    if any(s is None for s in sol):
        raise InfeasibleError("recshard_plan: initial assignment infeasible")
    for _ in range(iters if M > 1 else 0):
        costs = [s[1] for s in sol]
        gmax = int(np.argmax(costs))
        best = None
        for j in [k for k in range(len(specs)) if assign[k] == gmax]:
            for g in range(M):
                if g == gmax:
                    continue
                trial = list(assign)
                trial[j] = g
                a, b = solve_gpu(gmax, trial), solve_gpu(g, trial)
                if a is None or b is None:
                    continue
                new_max = max([a[1], b[1]] + [costs[m] for m in range(M) if m not in (g, gmax)])
                if new_max < max(costs) * (1 - 1e-9) and (best is None or new_max < best[0]):
                    best = (new_max, j, g, a, b)
        if best is None:
            break
        _, j, g, a, b = best
        assign[j] = g
        sol[gmax], sol[g] = a, b
    plan = ShardingPlan(strategy="recshard", step_count=step_count)
    for j, s in enumerate(specs):
        step = sol[assign[j]][0][j]
        rows = int(curves[j].rows[step])
        plan.entries.append(PlanEntry(s.table_id, assign[j], step, rows, step / step_count,
                                      rows * s.dim * s.elem_bytes))
    return recompute_plan_costs(plan, specs, stats, system)
