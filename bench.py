#!/usr/bin/env python3
"""EMB fwd+bwd samples/s of the tiered EmbeddingBag serving a RecShard plan
(vs the greedy/size plan), with the UVM access share — BASELINE.json's metric.

Default workload: RM1-like (100 EMBs, hash 1e5-1e7, dim 64/128 fp32, Zipf ids,
B = 16384, fast tier capped at 40% of table bytes so the rest sits in pinned
host memory read zero-copy over PCIe) — configs[1], which fits one B200.
A step = forward (sum-pool) + synthetic loss 0.5*||pooled||^2 (grad = pooled)
+ backward with the row-wise Adagrad update, over one batch of B samples.
N > 1 (torchrun): tables are model-parallel per the plan's GPU, pooled rows
and their gradients cross an NCCL all-to-all (strong scaling: fixed global B).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PROFILE_SEED = 7          # profile(trace, 1.0, seed) — SURVEY §8d profile seed
WORKLOAD_SEED = 20260809  # configs/example_2x.cfg:6
INIT_SEED = 1234
LR = 0.01


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="rm1", choices=["rm1", "rm2", "rm3", "cfg1"])
    p.add_argument("--batch", type=int, default=16384)
    p.add_argument("--nbatches", type=int, default=4, help="distinct batches cycled")
    p.add_argument("--profile-batches", type=int, default=16)
    p.add_argument("--pure", action="store_true",
                   help="headline serves the pure RecShard plan (the reference's solve, whose "
                        "1%%-of-accesses ICDF steps leave HBM unused); default: that plan + the "
                        "row-granular spare-capacity fill. The other one is measured alongside")
    p.add_argument("--no-variant", action="store_true", help="skip the alternate-plan run")
    p.add_argument("--optimizer", default="rowwise_adagrad", choices=["sgd", "rowwise_adagrad"])
    p.add_argument("--no-greedy", action="store_true")
    p.add_argument("--greedy-steps", type=int, default=3)
    p.add_argument("--no-flush", action="store_true", help="skip the L2 flush between steps")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--hbm-fraction", type=float, default=0.4,
                   help="M*cap_hbm as a fraction of all table bytes (configs/example_2x.cfg:2-3)")
    p.add_argument("--only", default=None, choices=[None, "recshard", "greedy"])
    p.add_argument("--profile-ids", type=float, default=1e9,
                   help="HP1 sweep size (BASELINE configs[4]); 0 disables")
    p.add_argument("--cpu-profile-ids", type=float, default=5e7)
    p.add_argument("--trace-ids", type=float, default=2e8,
                   help="trace-file write/read size (SURVEY §8f row 3, tools/trace_bench.py); 0 disables")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-uniform", action="store_true", help="skip the uniform-row (alpha=0) forward control")
    p.add_argument("--omit-unaccessed", action="store_true",
                   help="remaps with RemapOptions.omit_unaccessed (inc/remap.hpp:43-48): only profiled slow "
                        "rows get host storage, never-profiled rows pool as zeros (default for rm3)")
    p.add_argument("--no-prefetch", action="store_true",
                   help="headline in zero-copy mode only (no slow-row staging pipeline)")
    p.add_argument("--plan-gpus", type=int, default=0,
                   help="plan for M GPUs but run one of their shards here (with --as-rank; "
                        "one process, no all-to-all) — e.g. RM2 at 8 GPUs, rank 0's tables")
    p.add_argument("--as-rank", type=int, default=0)
    p.add_argument("--prefetch-depth", type=int, default=2, choices=[1, 2],
                   help="batches staged ahead (2: batch i+2's claim is queued behind forward i)")
    a = p.parse_args()
    if a.config == "rm3":
        a.omit_unaccessed = True  # 3.9 TB of fp16 rows: only profiled rows can be backed
    return a


# where the step queues batch i+2's prefetch (claim + host gather): after the
# backward (default) or after the forward (BENCH_PREFETCH_AT=fwd)
PREFETCH_AFTER_BWD = os.environ.get("BENCH_PREFETCH_AT", "bwd") != "fwd"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def specs_for(name):
    from paper_2201_10095_b200 import workload as wl

    return wl.cfg1_specs() if name == "cfg1" else wl.rm_specs(name, WORKLOAD_SEED)


class Clocks:
    """SM clock + throttle reasons sampled every few ms during the timed region
    (NVML — the same counters as the recipe's nvidia-smi clocks line)."""

    NAMES = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
             "sw_power_cap": 0x4}

    def __init__(self, device, period=0.005):
        import threading

        self.samples, self.reasons, self.mx = [], set(), None
        self.stop_ev = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            idx = device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[device])
                except ValueError:
                    idx = device
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None
            return

        def poll():
            while not self.stop_ev.is_set():
                try:
                    self.samples.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    for n, bit in self.NAMES.items():
                        if r & bit:
                            self.reasons.add(n)
                except Exception:
                    pass
                self.stop_ev.wait(period)

        self.th = threading.Thread(target=poll, daemon=True)
        self.th.start()

    def stop(self):
        if self.nv is None:
            return None
        self.stop_ev.set()
        self.th.join(timeout=2)
        if not self.samples:
            return None
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- reference arm
METRIC = "EMB fwd+bwd samples/s (RecShard plan; greedy-size plan alongside); UVM access %"


def line_config(args, n_tables, parallelism):
    """The `config` object both arms print (the driver pairs the lines by metric)."""
    return {"workload": f"{args.config}-like", "tables": n_tables, "global_batch": args.batch,
            "optimizer": args.optimizer, "parallelism": parallelism,
            "fast_tier_cap": f"{args.hbm_fraction:.0%} of table bytes",
            "l2": "256 MiB flush between steps" if not args.no_flush
            else f"{args.nbatches} distinct batches cycled",
            **({"remaps": "omit_unaccessed"} if args.omit_unaccessed else {})}


class RefEmbWorkload:
    """The CPU reference side of the EMB step, built WITHOUT the GPU library:
    a bounded table sample (every `every`-th table, full hash sizes) whose
    training batch comes from the unmodified reference generator
    (shardplan::generate_trace, core/src/workload.cpp:198-217, via oracle/_ref)
    regrouped into table-major CSR, and whose tables are initialised ONCE
    (oracle.c or_init_table, the same weights the GPU operator starts from).
    `step()` is one fwd + (grad = pooled) + bwd with the row-wise update over
    the sample on `threads` host threads (oracle.c — the reference has no
    EmbeddingBag); samples/s are scaled to the whole workload by
    expected lookups."""

    def __init__(self, specs, B, optimizer, threads, every=12):
        from concurrent.futures import ThreadPoolExecutor

        import oracle
        from paper_2201_10095_b200 import workload as wl  # pure Python (no .so)

        self.sub = specs[::every] if len(specs) > every else list(specs)
        self.B, self.threads, self.optimizer = B, threads, optimizer
        R = oracle.Ref()
        t0 = time.perf_counter()
        tr = R.generate_trace([(w.table, (w.gen.zipf_exponent, w.gen.mean_pooling, w.gen.coverage,
                                          w.gen.pooling_law)) for w in self.sub], B, WORKLOAD_SEED)
        self.gen_s = time.perf_counter() - t0
        self.offsets, self.indices = oracle.trace_to_csr(tr, [w.table.table_id for w in self.sub], B)
        n = int(self.offsets[-1])
        R.free_trace(tr)
        self.n = n
        c = oracle.C()
        self.dims = [w.table.dim for w in self.sub]
        self.Hs = [w.table.hash_size for w in self.sub]
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=threads) as ex:
            self.W = list(ex.map(lambda w: c.init_table(INIT_SEED, w.table.table_id, w.table.hash_size,
                                                        w.table.dim, 0.1), self.sub))
        self.init_s = time.perf_counter() - t0
        self.mom = [np.zeros(h, np.float32) for h in self.Hs] if optimizer != "sgd" else None
        self.full_lookups = wl.expected_lookups(specs, B)
        self.n_specs = len(specs)

    def step(self):
        import oracle

        oracle.emb_step_cpu(self.B, self.dims, self.Hs, self.offsets, self.indices, self.W, self.mom,
                            0 if self.optimizer == "sgd" else 1, LR, 1e-8, self.threads)

    def samples_per_s(self, step_s):
        return self.B / (step_s * self.full_lookups / self.n)

    def sample_text(self, reps, secs):
        return (f"oracle/oracle.c fwd+bwd ({self.optimizer}) on {len(self.sub)} of {self.n_specs} "
                f"tables (every 12th, full hash sizes; weights initialised once), 1 batch of {self.B} "
                f"samples = {self.n} lookups from the unmodified reference generate_trace; {reps} steps "
                f"in {secs:.1f}s, scaled to the full step by expected lookups ({self.full_lookups:.3g})")


def cpu_emb_baseline(specs, B, seconds, threads, optimizer, work=None):
    """cpu_baseline of our arm: RefEmbWorkload stepped for ~`seconds`."""
    w = work or RefEmbWorkload(specs, B, optimizer, threads)
    w.step()  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        w.step()
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return dict(value=w.samples_per_s(el / reps), unit="samples/s", cores=threads, kind="port",
                sample=w.sample_text(reps, el))


def loaded_native_libs():
    """Shared objects of this repo mapped into the process (evidence of which
    native code ran)."""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for ln in f:
                p = ln.split()[-1]
                if p.endswith(".so") and p.startswith(ROOT):
                    out.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(out)


def run_reference(args, rank, world):
    """`--impl reference`: the CPU implementation of the path on this host's
    cores (rank 0 only; other ranks exit without work).  Never loads
    libshardplan_gpu.so: inputs come from the unmodified reference generator."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    specs = specs_for(args.config)
    work = RefEmbWorkload(specs, args.batch, args.optimizer, threads)
    for _ in range(args.warmup):
        work.step()
    times = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s = time.perf_counter()
        work.step()
        times.append(time.perf_counter() - s)
    el = time.perf_counter() - t0
    v = work.samples_per_s(float(np.sum(times)) / len(times))
    M = world
    line = {"impl": "reference", "metric": METRIC, "value": v,
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * args.batch / v, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": line_config(args, len(specs), f"table-wise mp{M}"),
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": "port",
                             "sample": work.sample_text(args.steps, el)},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "setup_s": {"reference_generate_trace": work.gen_s, "init_tables": work.init_s},
            "native_libs_loaded": loaded_native_libs()}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
def ex_forward(op, ex, off, idx, hits):
    """K4 + K6 (rs_emb_forward_to_owners): this rank's tables pooled for the
    global batch, every row stored into its sample owner's block."""
    import ctypes as C

    from paper_2201_10095_b200 import _lib
    from paper_2201_10095_b200.runtime import ptr

    f = C.c_void_p()
    _lib.check(_lib.lib().rs_emb_forward_to_owners(op.h, ex.h, ptr(off), ptr(idx), ptr(hits), C.byref(f)))


def ex_backward(op, ex, off, idx, lr):
    """K6 + K5 (rs_emb_backward_from_owners): the owner block's gradient
    (in place) back to the table owners, overlapped with K5's sort."""
    import ctypes as C

    from paper_2201_10095_b200 import _lib
    from paper_2201_10095_b200.runtime import ptr

    _lib.check(_lib.lib().rs_emb_backward_from_owners(op.h, ex.h, ptr(off), ptr(idx), None, C.c_float(lr)))


def h2d_bandwidth(torch, dev):
    a = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    b = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    b.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(4):
        b.copy_(a, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    return 4 * a.numel() / (s.elapsed_time(e) / 1e3)


def run_plan(args, torch, dist, rank, world, dev, ctx, specs, stats, prof, plan, system, steps,
             warmup, do_e2e, B):
    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import _lib
    from paper_2201_10095_b200 import workload as wl

    local = [j for j, e in enumerate(plan.entries) if e.gpu == rank]
    lspecs = [specs[j] for j in local]
    remaps = []
    for j in local:
        s = specs[j].table
        out = torch.empty(s.hash_size, dtype=torch.int32, device=dev)
        remaps.append(sp.build_remap(plan.entries[j], stats[j], s, omit_unaccessed=args.omit_unaccessed, ctx=ctx,
                                     device_rows=prof.device_rows_by_rank(j), out=out))
    T = len(local)
    D_local = sum(s.table.dim for s in lspecs)
    dims_all = [sum(specs[j].table.dim for j, e in enumerate(plan.entries) if e.gpu == r)
                for r in range(world)]
    gen = wl.BatchGenerator(lspecs, B, WORKLOAD_SEED) if T else None
    batches = []
    for i in range(args.nbatches if T else 0):
        off, idx, n = gen.batch(100 + i)
        batches.append((off, idx[:max(1, n)].clone(), n))
        del idx
    cap = max([b[2] for b in batches] + [1])
    if os.environ.get("BENCH_MEM_DEBUG"):
        free, tot = torch.cuda.mem_get_info(dev)
        print(f"mem before operator: free {free / 1e9:.1f} GB of {tot / 1e9:.1f}, torch allocated "
              f"{torch.cuda.memory_allocated(dev) / 1e9:.1f} reserved {torch.cuda.memory_reserved(dev) / 1e9:.1f}, "
              f"lookups cap {cap}", file=sys.stderr, flush=True)
    op = sp.TieredEmbeddingBag([w.table for w in lspecs], remaps, B, cap, args.optimizer,
                               ctx=ctx) if T else None
    if op:
        op.init_weights(INIT_SEED, 0.1)
    hbm_b, host_b = op.memory() if op else (0, 0)
    # algorithmic bytes per batch (fwd: rows + index + remap entry per lookup,
    # offsets, pooled output; bwd: grad read once, indices, unique rows RMW +
    # Adagrad state).  Per-table lookup counts and unique rows from the batch.
    fwd_bytes, bwd_bytes, lookups, uniques = [], [], [], []
    for off, idx, n in batches:
        o = off.cpu().numpy().view(np.uint32).astype(np.int64)
        ih = idx[:n].cpu().numpy().view(np.uint32)
        fb = 4 * (T * B + 1) + 4 * B * D_local
        bb = 4 * B * D_local + 4 * n
        uq = 0
        for t, w in enumerate(lspecs):
            lt = int(o[(t + 1) * B] - o[t * B])
            rb = w.table.elem_bytes * w.table.dim
            fb += lt * (rb + 8 + 8)  # row + index + remap entry; + key/value written for the backward
            u = np.unique(ih[o[t * B]:o[(t + 1) * B]]).size
            uq += u
            bb += u * 2 * rb + (8 * u if args.optimizer != "sgd" else 0)
        fwd_bytes.append(fb)
        bwd_bytes.append(bb)
        lookups.append(n)
        uniques.append(uq)
    pooled = torch.empty(B, max(1, D_local), dtype=torch.float32, device=dev)
    hits = torch.zeros(2 * max(1, T), dtype=torch.int64, device=dev)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ex = None
    if world > 1:
        from paper_2201_10095_b200.sharded import Exchange

        ex = Exchange(plan, [w.table.dim for w in specs], world, rank, B,
                      transport=os.environ.get("BENCH_EXCHANGE", "peer"), ctx=ctx)
    # unique slow-tier rows per batch (sizes the HBM staging of the pipelined mode)
    slow_u = 0
    for off, idx, n in batches:
        o = off.cpu().numpy().view(np.uint32).astype(np.int64)
        u = 0
        for t in range(T):
            seg = idx[int(o[t * B]):int(o[(t + 1) * B])].long()
            if seg.numel():
                ent = remaps[t].entries[seg]
                u += int(torch.unique(seg[ent < 0]).numel())
        slow_u = max(slow_u, u)
    nvtx = os.environ.get("BENCH_NVTX") == "1"

    D = args.prefetch_depth

    prefetch_after_bwd = PREFETCH_AFTER_BWD

    def step(i, cache, ev=None):
        if nvtx:
            torch.cuda.nvtx.range_push("bench_step")
        off, idx, n = batches[i % len(batches)] if T else (None, None, 0)
        if D == 1 and cache and i + 1 < cache:  # stage batch i+1's slow rows while batch i runs
            nb = batches[(i + 1) % len(batches)]
            op.prefetch(nb[0], nb[1], B)
        if ev:
            ev[0].record()
        fused = ex is not None and T > 0
        if fused:  # K4 stores straight into the sample owners' blocks (K6)
            ex_forward(op, ex, off, idx, hits)
        elif T:
            op.forward(off, idx, B, out=pooled, hits=hits)
        if D == 2 and cache and i + 2 < cache and not prefetch_after_bwd:
            # batch i+2 (BENCH_PREFETCH_AT=fwd): its claim queues behind this
            # forward, so its host gather has this backward and the next step
            nb = batches[(i + 2) % len(batches)]
            op.prefetch(nb[0], nb[1], B)
        if ev:
            ev[1].record()
        g = pooled
        if ex is not None and not fused:  # a rank without tables: the unfused primitives
            g = ex.to_tables(ex.to_owners(pooled))
        if ev:
            ev[2].record()
        if fused:  # loss 0.5*||y||^2 on this rank's samples: the gradient is the owner block itself
            ex_backward(op, ex, off, idx, LR)
        elif T:
            op.backward(off, idx, g, B, LR)
        if D == 2 and cache and i + 2 < cache and prefetch_after_bwd:
            # batch i+2 (default): its claim queues behind this backward and
            # runs beside the next forward, not beside this backward (whose
            # kernels it slowed by ~0.1 ms); the host gather still has a step:
            # RM1 3.53 -> 3.46 ms/step, three same-box A/B pairs
            nb = batches[(i + 2) % len(batches)]
            op.prefetch(nb[0], nb[1], B)
        if ev:
            ev[3].record()
        if nvtx:
            torch.cuda.nvtx.range_pop()

    def timed(cache):
        """warmup + steps steps in one continuous run.  With `cache` the
        pipeline is filled before step 0 (batch 0's staging) and drained after
        the last step (every staged row written back).  The timed window is
        the last `steps` steps in steady state: each holds exactly one step's
        work (its forward + backward, the next batch's claim/stage-in, the
        eviction/stage-out of the batch two behind); the fill/drain costs are
        reported separately (ms_per_step_incl_warmup_fill_drain)."""
        nsteps = warmup + steps
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
        ta0, t0, t1, ta1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        clocks, L0 = None, 0
        ta0.record()
        if cache and T:
            for k in range(min(D, nsteps)):
                op.prefetch(batches[k % len(batches)][0], batches[k % len(batches)][1], B)
        for i in range(nsteps):
            if i == warmup:
                torch.cuda.synchronize()
                hits.zero_()
                if world > 1:
                    dist.barrier()
                if T:
                    op.kernel_times(reset=True)
                torch.cuda.synchronize()
                clocks = Clocks(dev.index)
                L0 = _lib.lib().rs_launch_counter()
                t0.record()
            if flush is not None:
                flush.zero_()
            step(i, nsteps if cache else 0, evs[i - warmup] if i >= warmup else None)
        t1.record()
        launches = int(_lib.lib().rs_launch_counter() - L0)
        if cache and T:
            op.flush()
        ta1.record()
        torch.cuda.synchronize()
        kf, nf, kb, nbk = op.kernel_times(reset=True) if T else (0.0, 1, 0.0, 1)
        if world > 1:
            dist.barrier()
        clk = clocks.stop() if clocks else None
        tot_ms = t0.elapsed_time(t1)
        all_ms = ta0.elapsed_time(ta1)
        fwd_ms = [e[0].elapsed_time(e[1]) for e in evs]
        a2a_ms = [e[1].elapsed_time(e[2]) for e in evs]
        bwd_ms = [e[2].elapsed_time(e[3]) for e in evs]
        h = hits.cpu().numpy()
        fast, slow = int(h[0::2][:T].sum()), int(h[1::2][:T].sum())
        if world > 1:
            mx = allreduce(dist, torch, [tot_ms, all_ms], dist.ReduceOp.MAX, dev)
            sm = allreduce(dist, torch, [fast, slow], dist.ReduceOp.SUM, dev)
            tot_ms, all_ms, fast, slow = mx[0], mx[1], int(sm[0]), int(sm[1])
        return dict(ms_per_step=tot_ms / steps, samples_per_s=B * steps / (tot_ms / 1e3),
                    ms_per_step_incl_warmup_fill_drain=all_ms / nsteps,
                    uvm_pct=100.0 * slow / max(1, fast + slow), fast=fast, slow=slow,
                    fwd_ms=float(np.mean(fwd_ms)), bwd_ms=float(np.mean(bwd_ms)),
                    fwd_kernel_ms=kf / max(1, nf), bwd_kernel_ms=kb / max(1, nbk),
                    a2a_ms=float(np.mean(a2a_ms)), launches=launches, clocks=clk)

    # zero-copy mode (the paper's UVM operator: slow rows read over PCIe inside
    # the kernels), then the pipelined mode (slow rows staged in HBM one batch
    # ahead on a side stream, written back behind the next batch)
    zc = timed(0)
    pipe = None
    if T and slow_u and not args.no_prefetch:
        op.enable_uvm_cache(int(4.5 * slow_u) + 4096)  # up to 4 live generations
        if os.environ.get("BENCH_PROBE") == "1":
            probe_cache(torch, op, batches, pooled, B)
        pipe = timed(steps)
    best = pipe if pipe is not None and pipe["samples_per_s"] > zc["samples_per_s"] else zc
    res = dict(best)
    res.update(mode="pipelined" if best is pipe else "zero-copy", zero_copy=zc, pipelined=pipe,
               slow_unique_rows=slow_u,
               fwd_bytes=float(np.mean([fwd_bytes[i % len(batches)] for i in range(steps)])) if T else 0,
               bwd_bytes=float(np.mean([bwd_bytes[i % len(batches)] for i in range(steps)])) if T else 0,
               lookups=float(np.mean(lookups)) if T else 0,
               unique_rows=float(np.mean(uniques)) if T else 0, hbm_bytes=hbm_b, host_bytes=host_b,
               tables=T)
    # accounting check: the forward's hit counters equal simulate() on the same batch
    if T and world == 1:
        off, idx, n = batches[0]
        hits.zero_()
        op.unbacked(reset=True)
        op.forward(off, idx, B, out=pooled, hits=hits)
        ulk, _ = op.unbacked(reset=True)
        res["unbacked_pct"] = 100.0 * float(ulk.sum()) / max(1, int(n))
        tr = wl.kjt_to_trace(lspecs, off, idx, n, B, 0, ctx=ctx)
        import copy

        ents = [copy.copy(plan.entries[j]) for j in local]
        for e in ents:  # this GPU's shard as a one-GPU system
            e.gpu = 0
        rep = sp.simulate(tr, sp.ShardingPlan("x", 1, ents), remaps,
                          sp.SystemSpec(1, B, system.cap_hbm_bytes, system.cap_dram_bytes,
                                        system.bw_hbm, system.bw_uvm), B, ctx=ctx)
        hh = hits.cpu().numpy()
        res["uvm_matches_simulate"] = bool(
            abs(rep.uvm_access_fraction - hh[1::2].sum() / max(1, hh.sum())) == 0.0
            and rep.total_accesses == int(hh.sum()))
    if do_e2e and T:
        res["e2e"] = run_e2e(torch, dist, world, op, batches, pooled, hits, B, steps, ex,
                             res["mode"] == "pipelined", args.prefetch_depth, flush)
    if op:
        op.close()
    del remaps, batches
    torch.cuda.empty_cache()
    return res


def traffic_record():
    """profiles/traffic.json (tools/make_traffic.py: ncu DRAM bytes per forward
    / backward / profile call) with `_matches` = whether it was measured on
    the library this run loaded (sha256), else None."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tp):
        return None
    try:
        tj = json.load(open(tp))
        import hashlib

        from paper_2201_10095_b200 import _lib

        h = hashlib.sha256()
        with open(_lib.LIB_PATH, "rb") as f:
            for b in iter(lambda: f.read(1 << 20), b""):
                h.update(b)
        tj["_matches"] = tj.get("library_sha256") == h.hexdigest()
        return tj
    except Exception:
        return None


def run_uniform_control(args, torch, ctx, specs, B, hbm_peak, reps=10):
    """The forward's L2-free control ("an alpha=0 uniform-row
    control"): the same tables (all rows in HBM, identity remaps) and the same
    bag structure as the headline batches, but every index drawn uniformly
    from its table, so there is no Zipf head to reuse from L1/L2 and the
    gather runs against DRAM.  Kernel-only time (CUDA events on the
    operator's stream) over `reps` forwards, each after a 256 MiB L2 flush;
    the same algorithmic bytes as the headline roofline."""
    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import workload as wl

    dev = torch.device("cuda", ctx.device)
    remaps = [sp.RemapTable(w.table.table_id, w.table.hash_size, w.table.hash_size, 0,
                            torch.arange(w.table.hash_size, dtype=torch.int32, device=dev)) for w in specs]
    gen = wl.BatchGenerator(specs, B, WORKLOAD_SEED)
    off, idx, n = gen.batch(100)
    o = off.cpu().numpy().view(np.uint32).astype(np.int64)
    T = len(specs)
    counts = torch.from_numpy(np.diff(o[::B][:T + 1]).astype(np.int64)).to(dev)
    H = torch.tensor([w.table.hash_size for w in specs], dtype=torch.float64, device=dev)
    hl = torch.repeat_interleave(H, counts)
    g = torch.Generator(device=dev)
    g.manual_seed(12345)
    uidx = (torch.rand(int(n), generator=g, device=dev, dtype=torch.float64) * hl).to(torch.int64)
    uidx = torch.minimum(uidx, (hl - 1).to(torch.int64)).to(torch.int32)
    del hl
    op = sp.TieredEmbeddingBag([w.table for w in specs], remaps, B, max(1, int(n)), args.optimizer, ctx=ctx)
    op.init_weights(INIT_SEED, 0.1)
    D = sum(w.table.dim for w in specs)
    pooled = torch.empty(B, D, dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        op.forward(off, uidx, B, out=pooled)
    torch.cuda.synchronize()
    op.kernel_times(reset=True)
    for _ in range(reps):
        flush.zero_()
        op.forward(off, uidx, B, out=pooled)
    torch.cuda.synchronize()
    fk, nf, _, _ = op.kernel_times(reset=True)
    ms = fk / max(1, nf)
    fb = 4 * (T * B + 1) + 4 * B * D
    for t, w in enumerate(specs):
        fb += int(o[(t + 1) * B] - o[t * B]) * (w.table.elem_bytes * w.table.dim + 16)
    op.close()
    del remaps, uidx, off, idx, pooled, flush
    torch.cuda.empty_cache()
    gbs = fb / (ms / 1e3) / 1e9
    return {"workload": f"{args.config}-like tables, headline bag structure, uniform row ids, all rows in HBM",
            "lookups": int(n), "kernel_ms": ms, "algorithmic_bytes": fb, "achieved": gbs, "peak": hbm_peak,
            "unit": "GB/s", "frac": gbs / hbm_peak}


def run_profile_sweep(args, torch, ctx, hbm_peak):
    """HP1 at scale (BASELINE configs[4]): profile() over ~args.profile_ids hashed
    ids on the cfg1 tables (8 x 1e6 rows, Zipf 1.05, pooling 20), timed end to
    end (device trace -> FeatureStats on the host), next to the unmodified
    reference profile() (oracle/_ref, 1 thread) on a bounded sample."""
    import oracle
    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import workload as wl

    specs = wl.cfg1_specs()
    per_sample = sum(w.gen.mean_pooling for w in specs)
    S = int(args.profile_ids // per_sample)
    gen = wl.BatchGenerator(specs, S, WORKLOAD_SEED + 1)
    off, idx, n = gen.batch(0)
    tr = wl.kjt_to_trace(specs, off, idx, n, S, 0, ctx=ctx)
    R = int(tr.rec_sample.numel())
    sp.profile(tr, 1.0, PROFILE_SEED, ctx=ctx)  # warm-up
    torch.cuda.synchronize()
    # host-side settle: the call is timed end to end on the host, and the
    # earlier legs free tens of GB of pinned host memory and HBM
    import gc

    gc.collect()
    time.sleep(1.0)
    times, dev_times = [], []
    for _ in range(15):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        p = sp.profiler.profile_handle(tr, 1.0, PROFILE_SEED, ctx=ctx)
        times.append(time.perf_counter() - t0)
        e1.record()  # the call returns with its results on the host: the stream is idle
        torch.cuda.synchronize()
        dev_times.append(e0.elapsed_time(e1) / 1e3)
        # release this result before the next call, so its pinned host buffers
        # return to the context's pool (a live result makes the next call pin
        # fresh pages: ~25 ms per 100 MB, which is host allocation, not profiling)
        p.close()
        del p
    secs = float(np.median(times))
    H = sum(w.table.hash_size for w in specs)
    alg = 4.0 * n + 24.0 * R + 8.0 * H  # id + record + (zero + read) per row
    out = {"workload": "cfg1 tables, rate 1.0", "ids": int(n), "records": R,
           "seconds": secs, "seconds_each": times,
           "device_seconds": float(np.median(dev_times)),  # the call's span on its stream (host jitter excluded)
           "ids_per_s": n / secs, "algorithmic_gbs": alg / secs / 1e9,
           "frac_of_hbm": alg / secs / 1e9 / hbm_peak}
    try:  # DRAM bytes of one such call from the committed ncu launch list
        tb = (traffic_record() or {}).get("cfg1_profile_1e9", {}).get("dram_bytes")
        if tb:
            tb = tb * n / 1e9
            out["traffic"] = {"dram_bytes": tb, "gbs": tb / secs / 1e9, "frac_of_hbm": tb / secs / 1e9 / hbm_peak,
                              "bound": "per-id instructions and per-tile barriers of the single-pass partition; the 2-byte "
                                       "bucket-local address stream written and re-read is ~4 of its ~9.6 B/id"}
    except Exception:
        pass
    if oracle.ref_available():
        m = min(R, int(args.cpu_profile_ids // 20))
        sub = (tr.rec_sample[:m].cpu().numpy().view(np.uint64), tr.rec_table[:m].cpu().numpy().view(np.uint32),
               tr.rec_offset[:m].cpu().numpy().view(np.uint64), tr.rec_len[:m].cpu().numpy().view(np.uint32))
        last = int(sub[2][-1] + sub[3][-1])
        ids_h = idx[:last].cpu().numpy().view(np.uint32)
        Rf = oracle.Ref()
        rt = Rf.trace([oracle.Spec(w.table.table_id, w.table.cardinality, w.table.hash_size,
                                   w.table.dim, w.table.elem_bytes) for w in specs],
                      int(sub[0].max()) + 1, *sub, ids_h)
        cs = Rf.time_profile(rt, 1.0, PROFILE_SEED)
        # parity on the same prefix: GPU profile() vs the reference's, every
        # FeatureStats field bit-exact (doubles compared as raw bits)
        want = Rf.profile(rt, 1.0, PROFILE_SEED)
        Rf.free_trace(rt)
        ptr = sp.Trace([w.table for w in specs], int(sub[0].max()) + 1, *sub, ids=ids_h)
        got = sp.profile(ptr, 1.0, PROFILE_SEED, ctx=ctx)
        out["cpu_reference"] = {"ids_per_s": last / cs, "cores": 1, "kind": "reference",
                                "sample": f"first {m} records ({last} ids) of the same trace, "
                                          "unmodified shardplan::profile (single-threaded)",
                                "bit_exact": stats_equal(got, want)}
    del tr, idx, off
    torch.cuda.empty_cache()
    return out


def stats_equal(got, want):
    """GPU FeatureStats list == the reference's (oracle.Ref dicts), bit for bit."""
    if len(got) != len(want):
        return False
    for g, w in zip(got, want):
        if (g.table_id != w["table_id"] or g.total_accesses != w["total_accesses"]
                or g.distinct_rows_accessed != w["distinct_rows_accessed"]
                or np.float64(g.coverage).view(np.uint64) != np.float64(w["coverage"]).view(np.uint64)
                or np.float64(g.avg_pooling).view(np.uint64) != np.float64(w["avg_pooling"]).view(np.uint64)
                or not np.array_equal(np.asarray(g.icdf_steps, np.uint64), w["icdf_steps"])
                or not np.array_equal(np.asarray(g.rows_by_rank, np.uint32), w["rows_by_rank"])
                or not np.array_equal(np.asarray(g.access_cdf, np.float64).view(np.uint64),
                                      w["access_cdf"].view(np.uint64))):
            return False
    return True


def run_profile_sweep_sharded(args, torch, dist, ctx, world, rank):
    """HP1 on N GPUs: the same ~args.profile_ids-id cfg1 trace on
    every rank, each rank profiling its tables' records (sharded.subtrace; no
    id exchange), the FeatureStats all-gathered.  Timed as the max over ranks
    of (sub-trace + profile + gather); weak in ids per table, strong in total."""
    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import workload as wl
    from paper_2201_10095_b200.sharded import profile_sharded

    specs = wl.cfg1_specs()
    per_sample = sum(w.gen.mean_pooling for w in specs)
    S = int(args.profile_ids // per_sample)
    gen = wl.BatchGenerator(specs, S, WORKLOAD_SEED + 1)
    off, idx, n = gen.batch(0)
    tr = wl.kjt_to_trace(specs, off, idx, n, S, 0, ctx=ctx)
    prof = lambda t, r, s: sp.profile(t, r, s, ctx=ctx)  # noqa: E731
    profile_sharded(tr, 1.0, PROFILE_SEED, profile_fn=prof)  # warm-up
    times = []
    for _ in range(3):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        profile_sharded(tr, 1.0, PROFILE_SEED, profile_fn=prof)
        torch.cuda.synchronize()
        times.append(allreduce(dist, torch, [time.perf_counter() - t0], dist.ReduceOp.MAX,
                               torch.device("cuda", ctx.device))[0])
    secs = float(np.median(times))
    del tr, idx, off
    torch.cuda.empty_cache()
    return {"workload": "cfg1 tables, rate 1.0, tables split over ranks", "ids": int(n), "n_gpus": world,
            "seconds": secs, "ids_per_s": n / secs}


def probe_cache(torch, op, batches, pooled, B):
    """Diagnostics: each stage of the staged pipeline timed alone (synchronised)."""
    def wall(f):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        return 1e3 * (time.perf_counter() - t0)
    for k in range(3):
        off, idx, n = batches[k % len(batches)]
        out = {}
        out["prefetch_ms"] = wall(lambda: op.prefetch(off, idx, B))
        out["fwd_staged_ms"] = wall(lambda: op.forward(off, idx, B, out=pooled))
        out["bwd_staged_ms"] = wall(lambda: op.backward(off, idx, pooled, B, LR))
        out["writeback_flush_ms"] = wall(lambda: op.flush())
        out["fwd_zero_copy_ms"] = wall(lambda: op.forward(off, idx, B, out=pooled))
        out["bwd_zero_copy_ms"] = wall(lambda: op.backward(off, idx, pooled, B, LR))
        print("probe", json.dumps(out), flush=True)


def modes(r):
    return {m: (None if r.get(k) is None else {x: r[k][x] for x in ("samples_per_s", "ms_per_step",
                                                                  "ms_per_step_incl_warmup_fill_drain",
                                                                  "fwd_ms", "bwd_ms", "fwd_kernel_ms",
                                                                  "bwd_kernel_ms")})
            for m, k in (("zero-copy", "zero_copy"), ("pipelined", "pipelined"))}


def run_e2e(torch, dist, world, op, batches, pooled, hits, B, steps, ex, cache, depth=2, flush=None):
    """Same step through the public API with host inputs: every step's offsets +
    indices are copied from pinned host memory (a copy stream, two batches
    ahead, triple-buffered — the data loader's overlap) and the hit counters
    (the step's UVM metric) are read back D2H.  With `cache`, batch k+1's slow
    rows are staged while batch k runs, as in the device-resident run; the
    same steady-state window (after 3 warm-up steps of the continuous run)."""
    dev = pooled.device
    host = [(off.cpu().pin_memory(), idx[:max(1, n)].cpu().pin_memory(), n) for off, idx, n in batches]
    nb = depth + 2  # in use: step i, the staged batches up to i + depth, the copy in flight
    ahead = depth + 1
    bufs = [(torch.empty_like(batches[0][0]),
             torch.empty(max(b[1].numel() for b in batches), dtype=torch.int32, device=dev))
            for _ in range(nb)]
    cs = torch.cuda.Stream(device=dev)
    main = torch.cuda.current_stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(nb)]
    ev_free = [torch.cuda.Event() for _ in range(nb)]
    used = [False] * nb
    h_hits = torch.empty(hits.numel(), dtype=torch.int64).pin_memory()
    bi = [0]

    def h2d(k, total):
        if k >= total:
            return
        b = k % nb
        if used[b]:
            cs.wait_event(ev_free[b])
        ho, hi, n = host[k % len(host)]
        with torch.cuda.stream(cs):
            bufs[b][0].copy_(ho, non_blocking=True)
            bufs[b][1][:hi.numel()].copy_(hi, non_blocking=True)
        ev_in[b].record(cs)
        bi[0] = ho.numel() * 4 + hi.numel() * 4

    def view(k):
        b = k % nb
        return bufs[b][0], bufs[b][1][:host[k % len(host)][1].numel()]

    warm = 3
    total = warm + steps
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run():
        for k in range(ahead):
            h2d(k, total)
        if cache:
            for k in range(min(depth, total)):
                main.wait_event(ev_in[k % nb])
                op.prefetch(*view(k), B)
        for i in range(total):
            if i == warm:  # steady state from here (same window as the device-resident run)
                torch.cuda.synchronize()
                s.record()
            h2d(i + ahead, total)
            if flush is not None:  # the same L2 flush between steps as the device-resident run
                flush.zero_()
            if cache and depth == 1 and i + 1 < total:
                main.wait_event(ev_in[(i + 1) % nb])
                op.prefetch(*view(i + 1), B)
            main.wait_event(ev_in[i % nb])
            d_off, d_idx = view(i)
            if ex is not None:
                ex_forward(op, ex, d_off, d_idx, hits)
            else:
                op.forward(d_off, d_idx, B, out=pooled, hits=hits)
            if cache and depth == 2 and i + 2 < total and not PREFETCH_AFTER_BWD:
                main.wait_event(ev_in[(i + 2) % nb])  # copied a step ago
                op.prefetch(*view(i + 2), B)
            if ex is not None:
                ex_backward(op, ex, d_off, d_idx, LR)
            else:
                op.backward(d_off, d_idx, pooled, B, LR)
            if cache and depth == 2 and i + 2 < total and PREFETCH_AFTER_BWD:
                main.wait_event(ev_in[(i + 2) % nb])  # copied a step ago
                op.prefetch(*view(i + 2), B)
            h_hits.copy_(hits, non_blocking=True)
            ev_free[i % nb].record(main)
            used[i % nb] = True
        e.record()
        if cache:
            op.flush()

    run()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    if world > 1:
        ms = allreduce(dist, torch, [ms], dist.ReduceOp.MAX, dev)[0]
    return {"value": B * steps / (ms / 1e3), "unit": "samples/s", "h2d_bytes_per_step": int(bi[0]),
            "d2h_bytes_per_step": int(h_hits.numel() * 8), "ms_per_step": ms / steps,
            "mode": "pipelined" if cache else "zero-copy"}


def allreduce(dist, torch, vals, op, dev):
    """All-reduce a few float64 scalars over the bench's process group (NCCL
    takes device tensors; the gloo group of a one-GPU multi-rank smoke takes
    host tensors)."""
    cpu = dist.get_backend() == "gloo"
    t = torch.tensor(vals, dtype=torch.float64, device="cpu" if cpu else dev)
    dist.all_reduce(t, op=op)
    return [float(x) for x in t.cpu()]


def free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` launched directly: spawn the N ranks the way the
        # driver does (torchrun, one process per GPU, rendezvous on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}; running {world} ranks",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        # one process per GPU over NCCL; BENCH_DIST_BACKEND=gloo lets ranks
        # share GPUs (a one-GPU smoke of the multi-rank path: the K6 peer
        # transport maps each rank's owner block with CUDA IPC either way)
        local_rank %= torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)

    import paper_2201_10095_b200 as sp
    from paper_2201_10095_b200 import planner
    from paper_2201_10095_b200 import workload as wl

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if os.environ.get("RS_BENCH_PRIO", "1") != "0":
        # the step's kernels on a high-priority stream: the operator's staging
        # kernels (claim, stage-in scatter) run on default-priority streams
        # beside them and yield SMs to the forward/backward
        torch.cuda.set_stream(torch.cuda.Stream(device=dev, priority=-100))
    ctx = sp.default_context(local_rank)
    specs = specs_for(args.config)
    B = args.batch
    hbm_peak, peak_kind = measured_peaks()
    bw_uvm = h2d_bandwidth(torch, dev)
    emulate = args.plan_gpus > 1 and world == 1
    M = args.plan_gpus if emulate else world
    prank = args.as_rank if emulate else rank
    if emulate and prank >= M:
        raise SystemExit("--as-rank outside [0, --plan-gpus)")
    system = wl.system_for(specs, M, B, hbm_peak * 1e9, bw_uvm, args.hbm_fraction)
    tables = [w.table for w in specs]

    # ---- HP1: profile the training data on the GPU (whole-sample rate 1.0)
    pgen = wl.BatchGenerator(specs, B * args.profile_batches, WORKLOAD_SEED)
    poff, pidx, pn = pgen.batch(0)
    ptrace = wl.kjt_to_trace(specs, poff, pidx, pn, B * args.profile_batches, 0, ctx=ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prof = sp.profiler.profile_handle(ptrace, 1.0, PROFILE_SEED, ctx=ctx)
    prof_cold_s = time.perf_counter() - t0  # includes first-use pinned result buffers
    prof.close()
    del prof  # its pinned result buffers return to the pool before the timed call
    t0 = time.perf_counter()
    prof = sp.profiler.profile_handle(ptrace, 1.0, PROFILE_SEED, ctx=ctx)
    prof_s = time.perf_counter() - t0
    stats = prof.stats
    del ptrace, pidx, poff
    torch.cuda.empty_cache()

    # HP1 at scale (the 1e9-id sweep) before any operator exists: its calls
    # are timed end to end on the host, which the later legs (tens of GB of
    # pinned host tiers allocated and freed) leave noisy for seconds
    sweep = None
    if world == 1 and args.profile_ids > 0:
        sweep = run_profile_sweep(args, torch, ctx, hbm_peak)
    elif world > 1 and args.profile_ids > 0:
        sweep = run_profile_sweep_sharded(args, torch, dist, ctx, world, rank)
    torch.cuda.empty_cache()

    # ---- plans (host): RecShard vs the greedy/size baseline
    t0 = time.perf_counter()
    rec_pure = planner.recshard_plan(tables, stats, system)  # the reference's solve, restated
    plan_s = time.perf_counter() - t0
    gre = planner.greedy_shard([planner.table_fixed_cost(t, None, "size") for t in tables], tables,
                               stats, system, "greedy-size")
    import copy

    rec_fill = planner.fill_spare_capacity(copy.deepcopy(rec_pure), tables, stats, system)
    rec = rec_pure if args.pure else rec_fill
    rec_var = rec_fill if args.pure else rec_pure
    # simulate() (GPU) on one training batch for each placement: the UVM share
    # the plans predict, before any operator is built
    sim_uvm = {}
    if world == 1:
        sgen = wl.BatchGenerator(specs, B, WORKLOAD_SEED)
        soff, sidx, sn = sgen.batch(100)
        strace = wl.kjt_to_trace(specs, soff, sidx, sn, B, 100 * B, ctx=ctx)
        strace.num_samples = B  # records carry sample ids 100B..101B-1; one batch of B
        strace.rec_sample = strace.rec_sample - 100 * B
        for name, pl in (("recshard", rec_pure), (rec_fill.strategy, rec_fill), ("greedy-size", gre)):
            rms = [sp.build_remap(pl.entries[j], stats[j], tables[j], omit_unaccessed=args.omit_unaccessed, ctx=ctx,
                                  device_rows=prof.device_rows_by_rank(j),
                                  out=torch.empty(tables[j].hash_size, dtype=torch.int32, device=dev))
                   for j in range(len(tables))]
            rep = sp.simulate(strace, pl, rms, system, B, ctx=ctx)
            sim_uvm[name] = 100.0 * rep.uvm_access_fraction
            del rms
        del strace, sidx, soff
        torch.cuda.empty_cache()

    if emulate and prank < 0:
        # every shard of the M-GPU plans, one after the other on this GPU: the
        # plan's step time is its slowest shard's (the all-to-all is not run)
        shards = []
        for q in range(M):
            rq = run_plan(args, torch, dist, q, world, dev, ctx, specs, stats, prof, rec, system,
                          args.steps, args.warmup, False, B)
            gq = run_plan(args, torch, dist, q, world, dev, ctx, specs, stats, prof, gre, system,
                          args.greedy_steps, 1, False, B)
            shards.append({"rank": q,
                           "tables": sum(1 for e in rec.entries if e.gpu == q),
                           "greedy_tables": sum(1 for e in gre.entries if e.gpu == q),
                           "recshard": {k: rq.get(k) for k in ("samples_per_s", "ms_per_step", "uvm_pct", "fast",
                                                               "slow", "mode", "unbacked_pct", "hbm_bytes",
                                                               "host_bytes")},
                           "greedy": {k: gq.get(k) for k in ("samples_per_s", "ms_per_step", "uvm_pct", "fast",
                                                             "slow", "mode", "unbacked_pct", "hbm_bytes",
                                                             "host_bytes")}})
            torch.cuda.empty_cache()
        prof.close()

        def system_of(key):
            ms = max(x[key]["ms_per_step"] for x in shards)
            slow = sum(x[key]["slow"] for x in shards)
            tot = slow + sum(x[key]["fast"] for x in shards)
            unb = sum((x[key].get("unbacked_pct") or 0.0) * (x[key]["fast"] + x[key]["slow"]) for x in shards)
            return {"samples_per_s": B / (ms / 1e3), "ms_per_step_slowest_shard": ms,
                    "uvm_access_pct": 100.0 * slow / max(1, tot),
                    "unbacked_access_pct": unb / max(1, tot)}

        rs_, gs_ = system_of("recshard"), system_of("greedy")
        print(json.dumps({
            "metric": "EMB fwd+bwd samples/s of an M-GPU plan, every shard run on this GPU in turn "
                      "(slowest shard sets the step; no all-to-all)",
            "config": {"workload": f"{args.config}-like", "tables": len(specs), "global_batch": B,
                       "plan_gpus": M, "fast_tier_cap": f"{args.hbm_fraction:.0%} of table bytes",
                       "optimizer": args.optimizer, "elem_bytes": sorted({w.table.elem_bytes for w in specs}),
                       **({"remaps": "omit_unaccessed"} if args.omit_unaccessed else {})},
            "recshard": rs_, "greedy": gs_, "recshard_vs_greedy": rs_["samples_per_s"] / gs_["samples_per_s"],
            "simulated_uvm_pct": sim_uvm, "planner_s": plan_s, "shards": shards}), flush=True)
        return

    first = gre if args.only == "greedy" else rec
    r = run_plan(args, torch, dist, prank, world, dev, ctx, specs, stats, prof, first, system,
                 args.steps, args.warmup, True, B)
    g = None
    if not args.no_greedy and args.only is None:
        g = run_plan(args, torch, dist, prank, world, dev, ctx, specs, stats, prof, gre, system,
                     args.greedy_steps, 1, False, B)
    v = None
    if not args.no_variant and args.only is None:
        v = run_plan(args, torch, dist, prank, world, dev, ctx, specs, stats, prof, rec_var, system,
                     args.greedy_steps, 1, False, B)
    prof.close()

    uniform = None
    if rank == 0 and world == 1 and not args.no_uniform:
        need = sum(w.table.hash_size * (w.table.dim * w.table.elem_bytes + 8) for w in specs)
        if need < 0.8 * torch.cuda.mem_get_info(dev)[0]:
            uniform = run_uniform_control(args, torch, ctx, specs, B, hbm_peak)
    trace_io = None
    if rank == 0 and world == 1 and args.trace_ids > 0:
        import importlib.util
        import tempfile
        from types import SimpleNamespace

        spec = importlib.util.spec_from_file_location("trace_bench", os.path.join(ROOT, "tools", "trace_bench.py"))
        tb = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(tb)
        with tempfile.TemporaryDirectory() as d:
            trace_io = tb.measure(SimpleNamespace(ids=args.trace_ids, ref_ids=2e6, dir=d, gz=False, reps=3,
                                                  chunk_mb=0))
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_emb_baseline(specs, B, args.cpu_seconds, os.cpu_count() or 1, args.optimizer)

    if rank == 0:
        # roofline: algorithmic bytes / kernel-only time (events around the
        # operator's kernels on its stream, staging waits excluded)
        fk, bk = r["fwd_kernel_ms"], r["bwd_kernel_ms"]
        fwd_gbs = r["fwd_bytes"] / (fk / 1e3) / 1e9 if fk > 0 else 0.0
        bwd_gbs = r["bwd_bytes"] / (bk / 1e3) / 1e9 if bk > 0 else 0.0
        traffic, traffic_src = None, None
        tj = traffic_record()
        if tj is not None:
            traffic = tj.get(args.config, {}).get("forward_dram_bytes")
            traffic_src = {k: tj.get(k) for k in ("commit", "date", "script", "library_sha256")}
            traffic_src["library_matches"] = tj.get("_matches")
        line = {
            "metric": METRIC,
            "value": r["samples_per_s"], "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (GPU Zipf generator, random-init weights)",
            "config": line_config(args, len(specs),
                                  f"one shard (rank {prank}) of a table-wise mp{M} plan, no all-to-all"
                                  if emulate else f"table-wise mp{world}"),
            "uvm_access_pct": r["uvm_pct"],
            **({"unbacked_access_pct": r.get("unbacked_pct"),
                "unbacked_note": "lookups of rows the omit_unaccessed remaps left without storage (never "
                                 "profiled); simulate() and uvm_access_pct count them as slow-tier accesses, "
                                 "the operator pools them as zero rows"} if args.omit_unaccessed else {}),
            "parity": {
                "profile_prefix_vs_reference": (sweep or {}).get("cpu_reference", {}).get("bit_exact"),
                "uvm_counts_vs_simulate": r.get("uvm_matches_simulate"),
                "tests": "tests/test_scale_gpu.py (cfg1 + RM1-slice fwd/bwd vs the fp64 oracle, full cfg1 "
                         "profile vs the reference), tests/test_pipeline_gpu.py (bundled configs end to end)"},
            "plan": first.strategy, "planner_s": plan_s,
            "simulated_uvm_pct": sim_uvm,
            "uvm_matches_simulate": r.get("uvm_matches_simulate"),
            "operator_mode": r["mode"],
            "recshard": dict({k: r[k] for k in ("samples_per_s", "ms_per_step", "fwd_ms", "bwd_ms",
                                                "fwd_kernel_ms", "bwd_kernel_ms",
                                                "lookups", "unique_rows", "slow_unique_rows",
                                                "a2a_ms", "uvm_pct", "hbm_bytes", "host_bytes")},
                             modes=modes(r)),
            "greedy": None if g is None else dict({k: g[k] for k in ("samples_per_s", "ms_per_step",
                                                                     "fwd_ms", "bwd_ms", "uvm_pct",
                                                                     "slow_unique_rows")},
                                                  mode=g["mode"], modes=modes(g)),
            "recshard_vs_greedy": None if g is None else r["samples_per_s"] / g["samples_per_s"],
            "plan_variant": None if v is None else dict({k: v[k] for k in ("samples_per_s", "ms_per_step",
                                                                           "uvm_pct", "slow_unique_rows")},
                                                        plan=rec_var.strategy, mode=v["mode"]),
            "recshard_vs_greedy_by_mode": None if g is None else {
                m: (r[k]["samples_per_s"] / g[k]["samples_per_s"]) if r.get(k) and g.get(k) else None
                for m, k in (("zero-copy", "zero_copy"), ("pipelined", "pipelined"))},
            "roofline": {"bound": "hbm", "kernel": "emb forward (gather-pool, both lane-class launches)",
                         "achieved": fwd_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": fwd_gbs / hbm_peak, "peak_kind": peak_kind,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "dram_frac": (traffic / (fk / 1e3) / 1e9 / hbm_peak) if traffic and fk > 0 else None,
                         "algorithmic_bytes": r["fwd_bytes"],
                         "kernel_ms": fk, "mode": r["mode"],
                         "backward": {"achieved": bwd_gbs, "frac": bwd_gbs / hbm_peak,
                                      "algorithmic_bytes": r["bwd_bytes"], "kernel_ms": bk},
                         "uniform_control": uniform},
            "cpu_baseline": cpu,
            "e2e": r.get("e2e"),
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
            "profile": {"ids": pn, "seconds_incl_host": prof_s, "ids_per_s": pn / prof_s,
                        "first_call_s": prof_cold_s},
            "profiler_sweep": sweep,
            "trace_io": trace_io,
            "bw_uvm_h2d_gbs": bw_uvm / 1e9,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
