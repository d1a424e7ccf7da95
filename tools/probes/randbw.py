import torch, time
dev = torch.device("cuda", 0)
for D, rows in [(128, 20_000_000), (64, 40_000_000)]:
    W = torch.empty(rows, D, device=dev)
    for n in [1_000_000, 4_000_000]:
        idx = torch.randperm(rows, device=dev)[:n]
        out = torch.empty(n, D, device=dev)
        for _ in range(3):
            torch.index_select(W, 0, idx, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            torch.index_select(W, 0, idx, out=out)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        rd = n * D * 4
        print(f"gather D={D} n={n}: {ms:.3f} ms  {2*rd/ms/1e6:.0f} GB/s (read+write)  random-read {rd/ms/1e6:.0f} GB/s")
        # scatter back (random writes)
        s.record()
        for _ in range(10):
            W.index_copy_(0, idx, out)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(f"scatter D={D} n={n}: {ms:.3f} ms  {2*rd/ms/1e6:.0f} GB/s (read+write)")
    del W
