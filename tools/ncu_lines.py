"""Summarise an ncu report's source page by CUDA source line (samples, instructions).
usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
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
            agg.append((int(r[hdr.index("# Samples")]), int(r[hdr.index("Instructions Executed")]), cur, int(r[0]), r[1][:90]))
        except ValueError:
            pass
ts = sum(a[0] for a in agg) or 1; ti = sum(a[1] for a in agg) or 1
print(f"total samples {ts} warp-instructions {ti}")
for a in sorted(agg, reverse=True)[:n]:
    print(f"{100*a[0]/ts:5.1f}% samp {100*a[1]/ti:5.1f}% inst  {a[2]}:{a[3]}  {a[4]}")
