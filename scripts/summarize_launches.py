"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])
into per-kernel count / mean / total, and each kernel's share of the total."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = defaultdict(dict)
    for r in rows[1:]:
        per[(r[ii], r[ki])][r[mi]] = float(r[vi].replace(",", ""))
    agg = defaultdict(lambda: defaultdict(float))
    for (_, k), m in per.items():
        a = agg[k.split("(")[0][:90]]
        a["n"] += 1
        for mk, mv in m.items():
            a[mk] += mv
    tot = sum(a.get("gpu__time_duration.sum", 0) for a in agg.values())
    print(f"{'kernel':90s} {'n':>5s} {'mean_us':>9s} {'share':>6s} {'MB/launch':>10s}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0)):
        t = a.get("gpu__time_duration.sum", 0)
        mb = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / a["n"] / 1e6
        print(f"{k:90s} {int(a['n']):5d} {t / a['n'] / 1e3:9.2f} {t / tot:6.1%} {mb:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
