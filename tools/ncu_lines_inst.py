"""Per-source-line executed warp-instructions of an ncu report, sorted by instruction count,
with a per-function-range rollup (line ranges given as name:lo-hi ...).
usage: python tools/ncu_lines_inst.py report.ncu-rep N [file:name:lo-hi ...]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2])
ranges = []
for a in sys.argv[3:]:
    f, name, r = a.split(":"); lo, hi = r.split("-"); ranges.append((f, name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None; hdr = None; agg = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0].isdigit() and len(r) > 8 and r[2] == "-":
        try:
            agg.append((int(r[hdr.index("Instructions Executed")]), int(r[hdr.index("# Samples")]), cur, int(r[0]), r[1][:100]))
        except ValueError:
            pass
ti = sum(a[0] for a in agg) or 1; ts = sum(a[1] for a in agg) or 1
print(f"total warp-instructions {ti} samples {ts}")
for f, name, lo, hi in ranges:
    i = sum(a[0] for a in agg if a[2] == f and lo <= a[3] <= hi); s = sum(a[1] for a in agg if a[2] == f and lo <= a[3] <= hi)
    print(f"  {name:28s} {100*i/ti:5.1f}% inst {100*s/ts:5.1f}% samp   ({f}:{lo}-{hi})")
byfile = {}
for a in agg: byfile[a[2]] = byfile.get(a[2], 0) + a[0]
for f, i in sorted(byfile.items(), key=lambda kv: -kv[1]): print(f"  file {f:28s} {100*i/ti:5.1f}% inst")
for a in sorted(agg, reverse=True)[:n]:
    print(f"{100*a[0]/ti:5.1f}% inst {100*a[1]/ts:5.1f}% samp  {a[2]}:{a[3]}  {a[4]}")
