"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_summary.py launches.csv [skip_first_n_launches]"""
import csv
import collections
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = collections.OrderedDict()
for r in rows[1 + skip:]:
    v = float(r[vi].replace(",", ""))
    v = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]] * v
    name = r[ki].split("(")[0].replace("void ", "")[:60]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{len(rows) - 1 - skip} launches, {tot / 1e3:.2f} ms total")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  x{n:<4d} {t / n:9.1f} us/launch  {k}")
