#!/usr/bin/env python3
"""Trace-file micro-bench: write_trace / read_trace of ~N
hashed ids on the cfg1 tables through the GPU path, next to the unmodified
reference read_trace / write_trace (oracle/_ref, one thread) on a prefix.

    python tools/trace_bench.py [--ids 2e8] [--ref-ids 2e7] [--dir /tmp] [--gz]

The read is timed from the page cache (the file was just written), so it
measures parsing + host reads, not the disk.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(a):
    """a: namespace with ids, ref_ids, dir, gz, reps, chunk_mb.  Returns the result dict."""
    import torch

    import oracle
    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import workload as wl

    ctx = sp.default_context(0)
    specs = wl.cfg1_specs()
    per = sum(w.gen.mean_pooling for w in specs)
    S = int(a.ids // per)
    gen = wl.BatchGenerator(specs, S, 20260811)
    off, idx, n = gen.batch(0)
    tr = wl.kjt_to_trace(specs, off, idx, n, S, 0, ctx=ctx)
    R = int(tr.rec_sample.numel())
    # the batch's records are table-major; a trace file is sorted by (sample, table)
    order = torch.argsort((tr.rec_sample << 32) | (tr.rec_table.long() & 0xFFFFFFFF), stable=True)
    tr = sp.Trace(tr.tables, tr.num_samples, tr.rec_sample[order].contiguous(), tr.rec_table[order].contiguous(),
                  tr.rec_offset[order].contiguous(), tr.rec_len[order].contiguous(), ids=tr.ids)
    ext = ".trace.gz" if a.gz else ".trace"
    path = os.path.join(a.dir, f"rs_bench{ext}")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sp.write_trace(tr, path, ["trace_bench"], ctx=ctx)
    t_write = time.perf_counter() - t0
    size = os.path.getsize(path)
    times = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        f = sp.TraceFile(path, ctx=ctx, chunk_bytes=a.chunk_mb << 20)
        times.append(time.perf_counter() - t0)
        got_n = f.num_ids
        f.close()
    t_read = float(np.median(times))
    assert got_n == n, (got_n, n)
    out = {"workload": "cfg1 tables", "ids": int(n), "records": R, "file_bytes": size, "gz": a.gz,
           "write_s": t_write, "write_ids_per_s": n / t_write,
           "read_s": t_read, "read_ids_per_s": n / t_read, "read_text_gbs": size / t_read / 1e9}
    os.remove(path)
    if oracle.ref_available() and a.ref_ids > 0:
        # prefix of the same trace for the single-threaded reference
        m = int(a.ref_ids // per * len(specs) * 0.9)
        m = max(1, min(R, m))
        # re-pack the first m records' ids contiguously
        lens = tr.rec_len[:m].long()
        offs = torch.cumsum(lens, 0) - lens
        last = int(lens.sum().item())
        gather = (tr.rec_offset[:m].repeat_interleave(lens) + torch.arange(last, device=lens.device)
                  - offs.repeat_interleave(lens))
        sub = sp.Trace(tr.tables, int(tr.rec_sample[m - 1].item()) + 1, tr.rec_sample[:m].contiguous(),
                       tr.rec_table[:m].contiguous(), offs.contiguous(), tr.rec_len[:m].contiguous(),
                       ids=tr.ids[gather].contiguous())
        p2 = os.path.join(a.dir, f"rs_bench_prefix{ext}")
        sp.write_trace(sub, p2, ["trace_bench"], ctx=ctx)
        Rf = oracle.Ref()
        t0 = time.perf_counter()
        rt = Rf.read_trace(p2)
        t_ref = time.perf_counter() - t0
        ok = np.array_equal(rt.ids, sub.ids.cpu().numpy().view(np.uint32))
        p3 = os.path.join(a.dir, f"rs_bench_prefix_ref{ext}")
        t0 = time.perf_counter()
        Rf.write_trace(rt, p3, ["trace_bench"])
        t_refw = time.perf_counter() - t0
        same = a.gz or open(p2, "rb").read() == open(p3, "rb").read()
        Rf.free_trace(rt)
        out["cpu_reference"] = {"ids": last, "read_ids_per_s": last / t_ref, "write_ids_per_s": last / t_refw,
                                "cores": 1, "kind": "reference",
                                "sample": f"first {m} records ({last} ids) of the same trace, unmodified "
                                          "shardplan::read_trace / write_trace",
                                "ids_equal": bool(ok), "bytes_equal": bool(same)}
        os.remove(p2)
        os.remove(p3)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--ids", type=float, default=2e8)
    p.add_argument("--ref-ids", type=float, default=2e7)
    p.add_argument("--dir", default="/tmp")
    p.add_argument("--gz", action="store_true")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--chunk-mb", type=int, default=0)
    print(json.dumps(measure(p.parse_args())))


if __name__ == "__main__":
    main()
