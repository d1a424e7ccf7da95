#!/usr/bin/env python3
"""Records the reference's bundled example configs (/root/reference/proj/
configs/example_{1,2,4}x.cfg — workload tables, [system], [planner],
[profiling]) as JSON fixtures under tests/golden/, so the GPU pipeline test
can rebuild them on a box without /root/reference.  Data only; the test
re-derives every expected output from the unmodified reference library."""
import json
import os
import re
import sys

SRC = "/root/reference/proj/configs"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
LAWS = {"constant": 0, "poisson": 1, "lognormal": 2}


def parse(path):
    sec, out = None, {"tables": []}
    for ln in open(path):
        ln = ln.split("#", 1)[0].strip()
        if not ln:
            continue
        m = re.match(r"\[(\w+)\]", ln)
        if m:
            sec = m.group(1)
            out.setdefault(sec, {})
            continue
        k, v = (x.strip() for x in ln.split("=", 1))
        if sec == "workload" and k == "table":
            f = v.split()
            out["tables"].append(dict(table_id=int(f[0]), cardinality=int(f[1]), hash_size=int(f[2]),
                                      dim=int(f[3]), elem_bytes=int(f[4]), zipf=float(f[5]),
                                      mean_pool=float(f[6]), coverage=float(f[7]), law=LAWS[f[8]]))
        else:
            out[sec][k] = v
    return out


if __name__ == "__main__":
    for n in ("1x", "2x", "4x"):
        p = os.path.join(SRC, f"example_{n}.cfg")
        if not os.path.exists(p):
            sys.exit(f"{p} missing (run where /root/reference exists)")
        with open(os.path.join(OUT, f"example_{n}.json"), "w") as f:
            json.dump(parse(p), f, indent=1)
        print("wrote", f"tests/golden/example_{n}.json")
