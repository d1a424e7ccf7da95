#!/usr/bin/env python3
"""Kernel-level micro-bench of the tiered EmbeddingBag on an RM-like table set
with every row in HBM (identity remaps): forward and backward times per step.

    python tools/op_bench.py [--config rm1] [--iters 10] [--slow-frac 0.0]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="rm1")
    p.add_argument("--iters", type=int, default=10)
    p.add_argument("--batch", type=int, default=16384)
    p.add_argument("--optimizer", default="rowwise_adagrad")
    p.add_argument("--hash-scale", type=float, default=1.0, help="shrink every hash size (rm configs)")
    p.add_argument("--dma-mb", type=float, default=0.0,
                   help="background H2D + D2H copy-engine traffic (MB per step each way) during the timed steps")
    p.add_argument("--slow-frac", type=float, default=0.0,
                   help="fraction of each table's rows (highest ids) placed in the host tier")
    a = p.parse_args()
    import torch

    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import workload as wl

    specs = wl.rm_specs(a.config, hash_scale=a.hash_scale) if a.config != "cfg1" else wl.cfg1_specs()
    B = a.batch
    dev = torch.device("cuda", 0)
    remaps = []
    for w in specs:
        H = w.table.hash_size
        hb = int(round(H * (1 - a.slow_frac)))
        ent = torch.arange(H, dtype=torch.int32, device=dev)
        if hb < H:
            ent[hb:] = -torch.arange(1, H - hb + 1, dtype=torch.int32, device=dev)
        remaps.append(sp.RemapTable(w.table.table_id, H, hb, H - hb, ent))
    gen = wl.BatchGenerator(specs, B, 20260809)
    batches = [gen.batch(100 + i) for i in range(2)]
    cap = max(b[2] for b in batches)
    op = sp.TieredEmbeddingBag([w.table for w in specs], remaps, B, cap, a.optimizer)
    op.init_weights(1, 0.1)
    pooled = torch.empty(B, op.total_dim, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(a.iters)]
    for i in range(2):
        off, idx, n = batches[i % 2]
        op.forward(off, idx, B, out=pooled)
        op.backward(off, idx, pooled, B, 0.01)
    torch.cuda.synchronize()
    if a.dma_mb > 0:  # copy-engine traffic beside the kernels (staging's PCIe DMA, without the staging)
        nb = int(a.dma_mb * (1 << 20))
        hin = torch.empty(nb, dtype=torch.uint8).pin_memory()
        hout = torch.empty(nb, dtype=torch.uint8).pin_memory()
        din = torch.empty(nb, dtype=torch.uint8, device=dev)
        dout = torch.empty(nb, dtype=torch.uint8, device=dev)
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        for _ in range(a.iters + 2):
            with torch.cuda.stream(s_in):
                din.copy_(hin, non_blocking=True)
            with torch.cuda.stream(s_out):
                hout.copy_(dout, non_blocking=True)
    for i in range(a.iters):
        off, idx, n = batches[i % 2]
        flush.zero_()
        torch.cuda.nvtx.range_push("bench_step")
        ev[i][0].record()
        op.forward(off, idx, B, out=pooled)
        ev[i][1].record()
        op.backward(off, idx, pooled, B, 0.01)
        ev[i][2].record()
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    f = float(np.median([e[0].elapsed_time(e[1]) for e in ev]))
    b = float(np.median([e[1].elapsed_time(e[2]) for e in ev]))
    print(json.dumps({"config": a.config, "variant": os.environ.get("RS_FWD_VARIANT", "0"),
                      "slow_frac": a.slow_frac, "lookups": float(np.mean([x[2] for x in batches])),
                      "fwd_ms": f, "bwd_ms": b, "samples_per_s": B / ((f + b) / 1e3)}))


if __name__ == "__main__":
    main()
