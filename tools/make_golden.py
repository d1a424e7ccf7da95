#!/usr/bin/env python3
"""Generate tests/golden/*.json from the UNMODIFIED reference library.

Runs in the build container only (needs oracle/_ref/libshardplan_ref.so built
from /root/reference by `make -C oracle`).  The fixtures restate the
reference's own known-answer tests (tests/test_workload.cpp:50-57,
tests/test_profiler.cpp:30-101, tests/test_remap.cpp:73-163,
tests/test_simulator.cpp:75-104) plus seeded cases, with the reference's
outputs recorded so the GPU box (which has no /root/reference) can check
parity against them.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
R = oracle.Ref()
S = oracle.Spec


def arr(a):
    return [int(x) if np.issubdtype(np.asarray(a).dtype, np.integer) else float(x) for x in a]


def trace_json(t):
    return dict(tables=[vars(s) for s in t.tables], num_samples=int(t.num_samples),
                rec_sample=arr(t.rec_sample), rec_table=arr(t.rec_table),
                rec_offset=arr(t.rec_offset), rec_len=arr(t.rec_len), ids=arr(t.ids))


def stats_json(st):
    return [dict(table_id=s["table_id"], coverage=float(s["coverage"]).hex(),
                 avg_pooling=float(s["avg_pooling"]).hex(),
                 distinct_rows_accessed=s["distinct_rows_accessed"],
                 total_accesses=s["total_accesses"], icdf_steps=arr(s["icdf_steps"]),
                 access_cdf=[float(x).hex() for x in s["access_cdf"]],
                 rows_by_rank=arr(s["rows_by_rank"])) for s in st]


def worked_example():
    """tests/test_profiler.cpp:30-49"""
    tables = [S(0, 1000, 100, 4, 4), S(1, 1000, 100, 4, 4)]
    recs = [(0, 0, [1, 5, 9, 15]), (0, 1, [2, 4, 8]), (1, 0, [5, 7, 9, 30]), (2, 0, [1, 5, 9])]
    ids, rs, rt, ro, rl = [], [], [], [], []
    for s, t, v in recs:
        rs.append(s), rt.append(t), ro.append(len(ids)), rl.append(len(v))
        ids += v
    return R.trace(tables, 3, rs, rt, ro, rl, ids)


def point_mass():
    """tests/test_profiler.cpp:64-81"""
    tables = [S(0, 10, 50, 4, 4)]
    return R.trace(tables, 20, list(range(20)), [0] * 20, list(range(20)), [1] * 20, [0] * 20)


def main():
    os.makedirs(OUT, exist_ok=True)
    # ---------------------------------------------------------------- hashing
    hv = [(x, 1, 0) for x in (0, 1, 42, 0xFFFFFFFFFFFFFFFF)]
    hv += [(42, 1 << 32, 3564271138), (7, 1000, 604)]  # tests/test_workload.cpp:54-55
    rng = np.random.default_rng(11)
    for _ in range(200):
        raw = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        H = int(rng.choice([1, 2, 3, 97, 1000, 1 << 20, 1_000_000, 99_999_989, 0x7FFFFFFF]))
        hv.append((raw, H, R.hash_value(raw, H)))
    for raw, H, want in hv[:6]:
        assert R.hash_value(raw, H) == want, (raw, H)
    json.dump({"cases": [[str(a), str(b), str(c)] for a, b, c in hv]},
              open(os.path.join(OUT, "hash_value.json"), "w"))

    # ---------------------------------------------------------------- profiles
    prof = {}
    for name, tr, rate, seed in [("worked_example", worked_example(), 1.0, 0),
                                 ("point_mass", point_mass(), 1.0, 0)]:
        prof[name] = dict(trace=trace_json(tr), rate=rate, seed=seed,
                          stats=stats_json(R.profile(tr, rate, seed)))
    wl = [(S(0, 5000, 4000, 8, 4), (1.2, 6.0, 0.7, 1)), (S(3, 1000, 800, 4, 4), (0.5, 2.0, 0.9, 0)),
          (S(5, 20000, 30000, 16, 4), (1.05, 3.0, 0.5, 2))]
    tr = R.generate_trace(wl, 3000, 44, gen_stats=True)
    for rate, seed in [(1.0, 0), (0.25, 9), (0.01, 1)]:
        prof[f"generated_r{rate}_s{seed}"] = dict(trace=trace_json(tr), rate=rate, seed=seed,
                                                  stats=stats_json(R.profile(tr, rate, seed)),
                                                  distinct_raw=arr(tr.distinct_raw))
    rawt = R.generate_trace(wl, 1000, 45, raw=True)
    hashed = R.generate_trace(wl, 1000, 45)
    prof["raw_trace"] = dict(trace=trace_json(hashed), raw_ids=[str(int(x)) for x in rawt.raw_ids],
                             rate=1.0, seed=0, stats=stats_json(R.profile(hashed, 1.0, 0)))
    json.dump(prof, open(os.path.join(OUT, "profile.json"), "w"))

    # ---------------------------------------------------------------- build_icdf
    icdf = {"cases": []}
    icdf["cases"].append(dict(counts=[7] * 200, icdf=arr(R.build_icdf([7] * 200))))
    icdf["cases"].append(dict(counts=[90, 10], icdf=arr(R.build_icdf([90, 10]))))
    for _ in range(50):
        n = int(rng.integers(1, 1000))
        c = rng.integers(0, 100, n)
        if c.sum() == 0:
            c[0] = 1
        icdf["cases"].append(dict(counts=arr(c), icdf=arr(R.build_icdf(c))))
    json.dump(icdf, open(os.path.join(OUT, "build_icdf.json"), "w"))

    # ---------------------------------------------------------------- remap
    def rank_stats(counts):
        """tests/test_remap.cpp:27-45"""
        order = sorted([r for r in range(len(counts)) if counts[r]], key=lambda r: (-counts[r], r))
        return order

    rem = {"cases": []}
    cases = [([5, 1, 9], 2, False), ([3, 9, 0, 2, 0, 7], 0, False), ([3, 9, 0, 2, 0, 7], 6, False),
             ([0, 5, 0, 3, 0, 0, 2, 0], 1, True), ([0, 5, 0, 3, 0, 0, 2, 0], 1, False),
             ([0, 5, 0, 3, 0, 0, 2, 0], 6, True)]
    for _ in range(12):
        H = int(rng.integers(1, 300))
        c = [int(x) for x in rng.integers(0, 5, H)]
        cases.append((c, int(rng.integers(0, H + 1)), bool(rng.integers(0, 2))))
    for counts, hbm, omit in cases:
        rbr = rank_stats(counts)
        st = dict(table_id=0, coverage=1.0, avg_pooling=1.0, distinct_rows_accessed=len(rbr),
                  total_accesses=int(sum(counts)), icdf_steps=np.zeros(101, np.uint64),
                  access_cdf=np.zeros(len(rbr)), rows_by_rank=np.array(rbr, np.uint32))
        h = R.stats_handle([st])
        ent, slow = R.build_remap(h, 0, S(0, len(counts), len(counts), 4, 4), hbm, omit)
        R.free_stats(h)
        rem["cases"].append(dict(hash_size=len(counts), hbm_rows=hbm, omit=omit, rows_by_rank=rbr,
                                 entries=arr(ent), slow_rows_allocated=slow))
    json.dump(rem, open(os.path.join(OUT, "remap.json"), "w"))

    # ---------------------------------------------------------------- simulate
    # tests/test_simulator.cpp:40-58 make_pipeline, with MILP and greedy plans
    sim = {"cases": []}
    wl3 = [(S(0, 4000, 3000, 16, 4), (1.3, 6.0, 0.9, 1)), (S(1, 9000, 8000, 8, 4), (1.1, 3.0, 0.5, 1)),
           (S(2, 2000, 1500, 32, 2), (0.9, 2.0, 1.0, 0))]
    for samples, gpus, batch, cap_div in [(3000, 2, 512, 3), (2048, 2, 256, 1), (1500, 3, 100, 4)]:
        t3 = R.generate_trace(wl3, samples, 5)
        st3, h3 = R.profile(t3, 1.0, 0, keep_handle=True)
        total = sum(s.hash_size * s.dim * s.elem_bytes for s, _ in wl3)

        class Sys:
            pass
        sysd = Sys()
        sysd.num_gpus, sysd.batch_size = gpus, batch
        sysd.cap_hbm_bytes = (1 << 30) if cap_div == 1 else total // cap_div
        sysd.cap_dram_bytes = 1 << 30
        sysd.bw_hbm, sysd.bw_uvm = 1.555e12, 1.6e10
        for kind in ("milp", "greedy"):
            p = R.plan(t3, h3, kind, sysd, cost_kind=0, step_count=10, time_limit=5.0)
            remaps = []
            for j, (spec, _) in enumerate(wl3):
                k = list(p["table_id"]).index(spec.table_id)
                ent, _slow = R.build_remap(h3, j, spec, int(p["hbm_rows"][k]))
                remaps.append((spec.table_id, spec.hash_size, int(p["hbm_rows"][k]), ent))
            rep = R.simulate(t3, (p["table_id"], p["gpu"], p["hbm_rows"]), remaps, sysd, batch)
            sim["cases"].append(dict(
                trace=trace_json(t3), plan=dict(table_id=arr(p["table_id"]), gpu=arr(p["gpu"]),
                                                hbm_rows=arr(p["hbm_rows"])),
                remaps=[dict(table_id=r[0], hash_size=r[1], hbm_rows=r[2], entries=arr(r[3]))
                        for r in remaps],
                system=vars(sysd), batch_size=batch,
                report={k: (arr(v) if isinstance(v, np.ndarray) else
                            (float(v).hex() if isinstance(v, float) else v))
                        for k, v in rep.items()}))
        R.free_stats(h3)
    json.dump(sim, open(os.path.join(OUT, "simulate.json"), "w"))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
