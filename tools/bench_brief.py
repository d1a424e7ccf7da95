#!/usr/bin/env python3
"""One-line summary of a bench.py JSON line on stdin: value, ms/step, and per
operator mode the forward/backward wall and kernel times, e2e."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
out = [str(round(d["value"])), f"{d['ms_per_step']:.3f}ms"]
for name, m in (d.get("recshard", {}).get("modes") or {}).items():
    if m:
        out.append(f"{name}: fwd {m['fwd_ms']:.3f}/{m['fwd_kernel_ms']:.3f} bwd {m['bwd_ms']:.3f}/{m['bwd_kernel_ms']:.3f}"
                   f" step {m['ms_per_step']:.3f}")
if d.get("e2e"):
    out.append(f"e2e {round(d['e2e']['value'])}")
print(" | ".join(out))
