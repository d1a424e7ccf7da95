"""Summarise an ncu --csv launch list: per-kernel time share and DRAM bytes."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        per[r[ii]][r[ni]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki].split("(")[0][:60]
    agg = collections.OrderedDict()
    for i, m in per.items():
        a = agg.setdefault(names[i], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'ms':>8} {'share':>6} {'n':>4} {'DRAM MB':>9} {'GB/s':>7}  kernel")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t/1e6:8.3f} {100*t/tot:5.1f}% {n:4d} {b/1e6:9.1f} {b/t if t else 0:7.0f}  {k}")
    print(f"total {tot/1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
