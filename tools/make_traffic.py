#!/usr/bin/env python3
"""Writes profiles/traffic.json — the measured DRAM traffic bench.py reports
as `roofline.traffic` — from ncu launch lists taken on the GPU box with the
SAME library build, and stamps it with that library's sha256 and the git
commit, so bench.py can tell a current measurement from a stale one.

    # on the GPU box (tools/round_full.sh runs these):
    BENCH_NVTX=1 ncu --nvtx --nvtx-include "bench_step/" --metrics \
        gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/launches_step.csv \
        python bench.py --steps 3 --warmup 1 --no-greedy --no-cpu --no-variant \
        --no-uniform --profile-ids 0 --trace-ids 0
    ncu --nvtx --nvtx-include "profile_call/" --metrics ... --csv \
        --log-file gpurun_out/launches_prof.csv python tools/prof_bench.py --ids 1e9 --reps 1
    # here:
    python tools/make_traffic.py gpurun_out/launches_step.csv gpurun_out/launches_prof.csv
"""
import collections
import csv
import datetime
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2201_10095_b200", "libshardplan_gpu.so")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in data:
        d = per.setdefault(r[ii], {"name": r[ki]})
        d[r[ni]] = float(r[vi].replace(",", ""))
    return list(per.values())


def dram(x):
    return x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)


def lib_sha256(path=LIB):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for b in iter(lambda: f.read(1 << 20), b""):
            h.update(b)
    return h.hexdigest()


def main(step_csv, prof_csv=None, config="rm1", out=os.path.join(ROOT, "profiles", "traffic.json")):
    L = launches(step_csv)
    fwd = [x for x in L if "forward_kernel" in x["name"]]
    classes = len({x["name"].split("(")[0] for x in fwd})
    nfwd = len(fwd) / max(1, classes)
    bwd_names = ("emb::bwd", "radix_", "scan_", "emb::keygen")
    bwd = [x for x in L if any(k in x["name"] for k in bwd_names)]
    res = {
        "library_sha256": lib_sha256(),
        "commit": subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                                 text=True).stdout.strip(),
        "date": datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ"),
        "script": "tools/make_traffic.py",
        config: {
            "forward_dram_bytes": sum(dram(x) for x in fwd) / max(1, nfwd),
            "backward_dram_bytes": sum(dram(x) for x in bwd) / max(1, nfwd),
            "per": "one operator forward (all lane-class launches) / one backward of the headline step",
            "forwards_in_list": nfwd,
            "source": os.path.basename(step_csv),
        },
    }
    if prof_csv:
        P = launches(prof_csv)
        res["cfg1_profile_1e9"] = {
            "dram_bytes": sum(dram(x) for x in P),
            "per": "one profile() call over 1e9 hashed ids on the cfg1 tables",
            "source": os.path.basename(prof_csv),
        }
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
