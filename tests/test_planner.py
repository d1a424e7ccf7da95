"""Placements: the host planner (csrc/planner.cpp) against the UNMODIFIED
reference planners (oracle/_ref: greedy_shard, ldm_shard, solve) — every
plan field compared exactly (gpu, step, hbm_rows, mem_bytes, pct by bits,
objective by bits), on random instances in the exact-search regime
(J <= 10, M <= 3, step_count <= 12), on budgeted ones, and on RM1/RM2-like
table sets.  North star: "placements bit-exact vs the CPU oracle".
CPU-only (the planner is host code)."""
import math

import numpy as np
import pytest

import oracle
from paper_2201_10095_b200 import planner
from paper_2201_10095_b200 import workload as wl
from paper_2201_10095_b200.types import (FeatureStats, InfeasibleError, InvalidArgument, SystemSpec,
                                         TableSpec)

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")


def _stats(rng, s):
    """Random FeatureStats with a valid (monotone, <= hash_size) ICDF."""
    H = s.hash_size
    distinct = int(rng.integers(1, H + 1))
    shape = rng.choice(["zipf", "uniform", "point"])
    if shape == "point":
        icdf = np.concatenate([[0], np.ones(100, np.uint64)]).astype(np.uint64)
    elif shape == "uniform":
        icdf = np.ceil(np.arange(101) / 100.0 * distinct).astype(np.uint64)
    else:
        a = float(rng.uniform(1.5, 6.0))
        icdf = np.ceil((np.arange(101) / 100.0) ** a * distinct).astype(np.uint64)
        icdf = np.maximum.accumulate(icdf)
    icdf[0] = 0
    cov = float(rng.choice([1.0, rng.uniform(0.01, 1.0)]))
    pool = float(rng.choice([1.0, 3.0, rng.uniform(0.5, 80.0)]))
    return FeatureStats(s.table_id, cov, pool, distinct, int(distinct * 3), icdf,
                        np.zeros(0), np.zeros(0, np.uint32))


def _ref_plans(specs, stats, system, kind, cost_kind=0, step_count=100, time_limit=math.inf):
    R = oracle.Ref()
    e = np.zeros(0, np.uint64)
    tr = R.trace([oracle.Spec(s.table_id, s.cardinality, s.hash_size, s.dim, s.elem_bytes) for s in specs],
                 1, e, e.astype(np.uint32), e, e.astype(np.uint32), e.astype(np.uint32))
    h = R.stats_handle([dict(table_id=st.table_id, coverage=st.coverage, avg_pooling=st.avg_pooling,
                             distinct_rows_accessed=0,  # unused by the planners (no cdf arrays)
                             total_accesses=st.total_accesses, icdf_steps=st.icdf_steps,
                             access_cdf=np.zeros(0), rows_by_rank=np.zeros(0, np.uint32)) for st in stats])
    try:
        return R.plan(tr, h, kind, system, cost_kind=cost_kind, step_count=step_count, time_limit=time_limit)
    finally:
        R.free_stats(h)
        R.free_trace(tr)


def _assert_same(got, want):
    assert [e.table_id for e in got.entries] == list(want["table_id"])
    assert [e.gpu for e in got.entries] == list(want["gpu"])
    assert [e.step for e in got.entries] == list(want["step"])
    assert [e.hbm_rows for e in got.entries] == list(want["hbm_rows"])
    assert np.array_equal(np.array([e.pct for e in got.entries]).view(np.uint64),
                          np.asarray(want["pct"], np.float64).view(np.uint64))
    assert [e.mem_bytes for e in got.entries] == list(want["mem_bytes"])
    assert got.step_count == want["step_count"]
    assert np.float64(got.objective).view(np.uint64) == np.float64(want["objective"]).view(np.uint64)


def _instance(rng, J, M, frac_hbm=None, dims=(4, 8, 16, 64)):
    specs = []
    for j in range(J):
        H = int(rng.integers(10, 5000))
        specs.append(TableSpec(int(j * 3 + rng.integers(0, 3)), H, H, int(rng.choice(dims)),
                               int(rng.choice([2, 4]))))
    stats = [_stats(rng, s) for s in specs]
    total = sum(s.bytes() for s in specs)
    f = frac_hbm if frac_hbm is not None else float(rng.uniform(0.05, 0.9))
    cap_hbm = max(1, int(f * total / M))
    cap_dram = int(total * float(rng.uniform(0.6, 1.5)) / M) + 1
    system = SystemSpec(M, int(rng.choice([1, 512, 16384])), cap_hbm, cap_dram,
                        float(rng.choice([1.555e12, 6.5e12])), float(rng.choice([1.6e10, 5e10])))
    return specs, stats, system


def _both(fn_ours, fn_ref):
    try:
        want = fn_ref()
    except oracle.OracleError as e:
        with pytest.raises((InfeasibleError, InvalidArgument)):
            fn_ours()
        return e.status
    _assert_same(fn_ours(), want)
    return 0


@pytest.mark.parametrize("seed", range(40))
def test_baselines_match_reference(seed):
    rng = np.random.default_rng(seed)
    specs, stats, system = _instance(rng, int(rng.integers(1, 40)), int(rng.integers(1, 9)))
    for ck, name in enumerate(["size", "lookup", "size-lookup"]):
        costs = [planner.table_fixed_cost(s, st, name) for s, st in zip(specs, stats)]
        _both(lambda: planner.greedy_shard(costs, specs, stats, system),
              lambda: _ref_plans(specs, stats, system, "greedy", ck))
        _both(lambda: planner.ldm_shard(costs, specs, stats, system),
              lambda: _ref_plans(specs, stats, system, "ldm", ck))


@pytest.mark.parametrize("seed", range(40))
def test_solve_exact_regime_matches_reference(seed):
    """J <= 10, M <= 3, step_count <= 12: the reference proves optimality
    with its lexicographic exact search; the plans must be identical."""
    rng = np.random.default_rng(1000 + seed)
    specs, stats, system = _instance(rng, int(rng.integers(1, 11)), int(rng.integers(1, 4)))
    steps = int(rng.integers(1, 13))
    inst = planner.build_instance(stats, specs, system, step_count=steps)
    _both(lambda: planner.solve(inst), lambda: _ref_plans(specs, stats, system, "milp", step_count=steps))


@pytest.mark.parametrize("seed", range(12))
def test_solve_budgeted_matches_reference(seed):
    """Beyond exact scale (LPT seed, local search, budgeted branch and bound,
    polish): same plan for the same deterministic budget, any thread count."""
    rng = np.random.default_rng(2000 + seed)
    specs, stats, system = _instance(rng, int(rng.integers(11, 40)), int(rng.integers(2, 9)))
    tl = float(rng.choice([0.5, 2.0]))
    inst = planner.build_instance(stats, specs, system, step_count=int(rng.choice([20, 100])))
    ref = lambda: _ref_plans(specs, stats, system, "milp", step_count=inst.step_count, time_limit=tl)  # noqa: E731
    st = _both(lambda: planner.solve(inst, tl, threads=1), ref)
    if st == 0:
        _both(lambda: planner.solve(inst, tl, threads=8), ref)


def test_rm_like_plans_match_reference():
    """RM1-like tables (100 EMBs) with synthetic ICDFs on 8 GPUs: greedy/size,
    LDM/lookup and the budgeted solve (time limit 2 s of budget)."""
    rng = np.random.default_rng(7)
    specs = [w.table for w in wl.rm_specs("rm1")]
    stats = [_stats(rng, s) for s in specs]
    system = wl.system_for([type("W", (), {"table": s})() for s in specs], 8, 16384, 6.5e12, 5.1e10)
    costs = [planner.table_fixed_cost(s, None, "size") for s in specs]
    _assert_same(planner.greedy_shard(costs, specs, stats, system), _ref_plans(specs, stats, system, "greedy", 0))
    costs = [planner.table_fixed_cost(s, st, "lookup") for s, st in zip(specs, stats)]
    _assert_same(planner.ldm_shard(costs, specs, stats, system), _ref_plans(specs, stats, system, "ldm", 1))
    inst = planner.build_instance(stats, specs, system)
    _assert_same(planner.solve(inst, 2.0), _ref_plans(specs, stats, system, "milp", time_limit=2.0))


def test_planner_errors_match_reference():
    s = [TableSpec(0, 10, 10, 4, 4)]
    st = [FeatureStats(0, 1.0, 1.0, 10, 10, np.arange(101, dtype=np.uint64) // 10, np.zeros(0),
                       np.zeros(0, np.uint32))]
    bad = SystemSpec(1, 1, 1, 1, 1.0, 2.0)  # bw_hbm <= bw_uvm
    with pytest.raises(InvalidArgument, match="bw_hbm must exceed bw_uvm"):
        planner.greedy_shard([1.0], s, st, bad)
    tiny = SystemSpec(1, 1, 1, 1, 2.0, 1.0)  # 160 bytes of table, 2 bytes of capacity
    with pytest.raises(InfeasibleError, match="exceed aggregate capacity"):
        planner.solve(planner.build_instance(st, s, tiny))
    with pytest.raises(InvalidArgument, match="costs must be finite"):
        planner.greedy_shard([float("nan")], s, st, SystemSpec(1, 1, 100, 100, 2.0, 1.0))
    with pytest.raises(InvalidArgument, match="unknown cost function"):
        planner.table_fixed_cost(s[0], st[0], "bytes")
