"""GPU parity: K3 remap construction and simulate() accounting — bit-exact."""
import math

import numpy as np
import pytest

from conftest import golden_trace, load_golden

import paper_2201_10095_b200 as sp
from paper_2201_10095_b200.types import (FeatureStats, PlanEntry, RemapTable, ShardingPlan,
                                         SystemSpec, TableSpec)

pytestmark = pytest.mark.gpu


def _stats(rbr):
    return FeatureStats(0, 1.0, 1.0, len(rbr), 0, np.zeros(101, np.uint64), np.zeros(len(rbr)),
                        np.array(rbr, np.uint32))


def test_remap_goldens(cuda_ctx):
    for c in load_golden("remap.json")["cases"]:
        spec = TableSpec(0, c["hash_size"], c["hash_size"], 4, 4)
        r = sp.build_remap(PlanEntry(0, 0, 0, c["hbm_rows"]), _stats(c["rows_by_rank"]), spec,
                           omit_unaccessed=c["omit"], ctx=cuda_ctx)
        assert list(r.entries) == c["entries"]
        assert r.slow_rows_allocated == c["slow_rows_allocated"]


def test_remap_worked_example_and_translate(cuda_ctx):
    # tests/test_remap.cpp:73-85
    spec = TableSpec(0, 3, 3, 4, 4)
    r = sp.build_remap(PlanEntry(0, 0, 0, 2), _stats([2, 0]), spec, ctx=cuda_ctx)
    assert list(r.entries) == [1, -1, 0]
    assert sp.translate(r, 2) == (sp.TIER_FAST, 0)
    assert sp.translate(r, 1) == (sp.TIER_SLOW, 0)
    with pytest.raises(sp.InvalidArgument):
        sp.translate(r, 3)


def test_remap_errors(cuda_ctx):
    spec = TableSpec(0, 3, 3, 4, 4)
    with pytest.raises(sp.InvalidArgument):
        sp.build_remap(PlanEntry(0, 0, 0, 4), _stats([2, 1, 0]), spec, ctx=cuda_ctx)
    big = TableSpec(0, 1 << 31, 1 << 31, 4, 4)
    with pytest.raises(sp.InvalidArgument):
        sp.build_remap(PlanEntry(0, 0, 0, 0), _stats([2]), big, ctx=cuda_ctx)
    bare = FeatureStats(0, 1.0, 1.0, 2, 0)  # distinct 2, no rows_by_rank
    with pytest.raises(sp.InvalidArgument):
        sp.build_remap(PlanEntry(0, 0, 0, 1), bare, spec, ctx=cuda_ctx)


@pytest.mark.parametrize("omit", [False, True])
def test_remap_large_vs_oracle(cuda_ctx, coracle, omit):
    rng = np.random.default_rng(4)
    for H in (1, 1000, 3_000_000):
        counts = rng.integers(0, 3, H) * rng.integers(0, 2, H)
        rbr = sorted(np.nonzero(counts)[0].tolist(), key=lambda r: (-counts[r], r))
        for hbm in sorted({0, 1, len(rbr) // 2, len(rbr), min(H, len(rbr) + 17), H}):
            if hbm > H:
                continue
            got = sp.build_remap(PlanEntry(0, 0, 0, hbm), _stats(rbr), TableSpec(0, H, H, 4, 4),
                                 omit_unaccessed=omit, ctx=cuda_ctx)
            want, slow = coracle.build_remap(H, hbm, rbr, omit)
            assert np.array_equal(got.entries, want)
            assert got.slow_rows_allocated == slow


def _report_eq(got, want):
    f = lambda v: float.fromhex(v) if isinstance(v, str) else v  # noqa: E731
    assert got.batches == want["batches"] and got.total_accesses == want["total_accesses"]
    assert [g.hbm_accesses for g in got.gpus] == want["hbm_accesses"]
    assert [g.uvm_accesses for g in got.gpus] == want["uvm_accesses"]
    assert [g.est_iter_cost for g in got.gpus] == want["est_iter_cost"]
    for k in ("min_cost", "max_cost", "mean_cost", "stddev_cost", "uvm_access_fraction"):
        assert getattr(got, k) == f(want[k]), k
    for a, b in zip(got.table_fast_fraction, want["table_fast_fraction"]):
        assert (math.isnan(a) and math.isnan(b)) or a == b


def _sim_inputs(case):
    tr = golden_trace(case["trace"])
    p = case["plan"]
    plan = ShardingPlan("golden", 10, [PlanEntry(t, g, 0, h) for t, g, h in
                                       zip(p["table_id"], p["gpu"], p["hbm_rows"])])
    remaps = [RemapTable(r["table_id"], r["hash_size"], r["hbm_rows"], 0,
                         np.array(r["entries"], np.int32)) for r in case["remaps"]]
    return tr, plan, remaps, SystemSpec(**case["system"])


def test_simulate_goldens(cuda_ctx):
    for case in load_golden("simulate.json")["cases"]:
        tr, plan, remaps, system = _sim_inputs(case)
        rep = sp.simulate(tr, plan, remaps, system, case["batch_size"], ctx=cuda_ctx)
        _report_eq(rep, case["report"])


def test_simulate_errors(cuda_ctx):
    case = load_golden("simulate.json")["cases"][0]
    tr, plan, remaps, system = _sim_inputs(case)
    broken = ShardingPlan("x", 10, plan.entries[:-1])
    with pytest.raises(sp.InvalidArgument):
        sp.simulate(tr, broken, remaps, system, 128, ctx=cuda_ctx)
    with pytest.raises(sp.InvalidArgument):
        sp.simulate(tr, plan, remaps[:-1], system, 128, ctx=cuda_ctx)
    with pytest.raises(sp.InvalidArgument):  # batch larger than the trace
        sp.simulate(tr, plan, remaps, system, tr.num_samples + 1, ctx=cuda_ctx)
