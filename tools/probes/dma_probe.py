#!/usr/bin/env python3
"""Diagnostic: does copy-engine (DMA) PCIe traffic on a side stream slow the
all-HBM EmbeddingBag step?  Times fwd+bwd alone, then with 32 MB H2D + 32 MB
D2H cudaMemcpyAsync per step on a second stream."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import workload as wl

    specs = wl.rm_specs("rm1")
    B = 16384
    dev = torch.device("cuda", 0)
    remaps = []
    for w in specs:
        H = w.table.hash_size
        remaps.append(sp.RemapTable(w.table.table_id, H, H, 0, torch.arange(H, dtype=torch.int32, device=dev)))
    gen = wl.BatchGenerator(specs, B, 20260809)
    batches = [gen.batch(100 + i) for i in range(2)]
    op = sp.TieredEmbeddingBag([w.table for w in specs], remaps, B, max(b[2] for b in batches), "rowwise_adagrad")
    op.init_weights(1, 0.1)
    pooled = torch.empty(B, op.total_dim, device=dev)
    side = torch.cuda.Stream()
    h_src = torch.empty(32 << 20, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(32 << 20, dtype=torch.uint8).pin_memory()
    d_buf = torch.empty(32 << 20, dtype=torch.uint8, device=dev)
    d_buf2 = torch.empty(32 << 20, dtype=torch.uint8, device=dev)

    def run(n, dma):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ev[0].record()
        for i in range(n):
            off, idx, _ = batches[i % 2]
            if dma:
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    d_buf.copy_(h_src, non_blocking=True)
                    h_dst.copy_(d_buf2, non_blocking=True)
            op.forward(off, idx, B, out=pooled)
            op.backward(off, idx, pooled, B, 0.01)
        torch.cuda.current_stream().wait_stream(side)
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / n

    run(3, False)
    out = {"alone_ms": run(10, False), "with_dma_ms": run(10, True), "alone2_ms": run(10, False)}
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record(side)
    with torch.cuda.stream(side):
        for _ in range(10):
            d_buf.copy_(h_src, non_blocking=True)
            h_dst.copy_(d_buf2, non_blocking=True)
    e.record(side)
    torch.cuda.synchronize()
    out["dma_alone_ms"] = s.elapsed_time(e) / 10
    print(json.dumps(out))


if __name__ == "__main__":
    main()
