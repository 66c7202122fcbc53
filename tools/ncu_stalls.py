"""Stall-reason breakdown of an ncu report (source page, SASS): totals per
reason and the top SASS instructions with their dominant reasons.
usage: python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
extra = sys.argv[3:]
out = subprocess.run(["ncu", "-i", rep, *extra, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr, rows = rows[0], rows[1:]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ix = {h: i for i, h in enumerate(hdr)}
tot = {r: 0 for r in reasons}
per = []
for r in rows:
    try:
        s = {k: int(float(r[ix[k]] or 0)) for k in reasons}
    except (ValueError, IndexError):
        continue
    for k, v in s.items():
        tot[k] += v
    per.append((sum(s.values()), r[ix["Address"]], r[ix["Source"]].strip(), s))
T = sum(tot.values()) or 1
print("stall totals:")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"  {k:24s} {100 * v / T:5.1f}%")
print(f"top {top} instructions:")
for n, a, src, s in sorted(per, key=lambda x: -x[0])[:top]:
    dom = ", ".join(f"{k[6:]} {v}" for k, v in sorted(s.items(), key=lambda x: -x[1])[:3] if v)
    print(f"  {100 * n / T:5.1f}%  {a[-5:]}  {src[:60]:60s} {dom}")
