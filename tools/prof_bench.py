#!/usr/bin/env python3
"""HP1 micro-bench: profile() over ~N hashed ids on the cfg1 tables (BASELINE
configs[4]), wall time end to end and the device-only time of the call.

    python tools/prof_bench.py [--ids 1e9] [--reps 3] [--raw]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--ids", type=float, default=1e9)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--rate", type=float, default=1.0)
    p.add_argument("--config", default="cfg1", help="cfg1 (BASELINE configs[4]) or rm1/rm2/rm3 table sets")
    p.add_argument("--samples", type=int, default=0, help="samples instead of --ids (e.g. 262144 = the "
                   "bench's 16 profiling batches of 16384)")
    a = p.parse_args()
    import torch

    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import workload as wl

    ctx = sp.default_context(0)
    specs = wl.cfg1_specs() if a.config == "cfg1" else wl.rm_specs(a.config, 20260809)
    per = sum(w.gen.mean_pooling * w.gen.coverage for w in specs)
    S = a.samples or int(a.ids // per)
    gen = wl.BatchGenerator(specs, S, 20260810)
    off, idx, n = gen.batch(0)
    tr = wl.kjt_to_trace(specs, off, idx, n, S, 0, ctx=ctx)
    sp.profile(tr, a.rate, 7, ctx=ctx)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        torch.cuda.nvtx.range_push("profile_call")
        t0 = time.perf_counter()
        h = sp.profiler.profile_handle(tr, a.rate, 7, ctx=ctx)
        ts.append(time.perf_counter() - t0)
        torch.cuda.nvtx.range_pop()
        h.close()
        del h  # its pinned result buffers go back to the pool before the next call
    ts.sort()
    print(json.dumps({"ids": int(n), "records": int(tr.rec_sample.numel()), "s": ts[len(ts) // 2], "all_s": ts,
                      "ids_per_s": n / ts[len(ts) // 2]}))


if __name__ == "__main__":
    main()
