"""Write a text summary of an ncu --set full report (key metrics + hot source lines).
usage: python tools/ncu_summary.py report.ncu-rep out.txt"""
import io
import re
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Block Limit Registers", "Block Limit Shared Mem",
        "Grid Size", "Block Size", "Waves Per SM"]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
lines = [f"# ncu summary of {rep.split('/')[-1]}", ""]
kernel = None
for ln in det.splitlines():
    f = [x.strip('"') for x in re.findall(r'"((?:[^"]|"")*)"', ln)]
    if len(f) < 4:
        continue
    if kernel is None and "Kernel Name" not in ln:
        kernel = f[4] if len(f) > 4 else None
    if f[-3] in KEYS:
        lines.append(f"{f[-3]:35s} {f[-1]:>14s} {f[-2]}")
# raw metrics of interest
rows = [r for r in raw.splitlines()]
if len(rows) > 2:
    hdr = [x.strip('"') for x in rows[0].split('","')]
    units = [x.strip('"') for x in rows[1].split('","')]
    vals = [x.strip('"') for x in rows[2].split('","')]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "lts__t_bytes.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum"]
    lines.append("")
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            lines.append(f"{w:60s} {vals[i]:>16s} {units[i]}")
lines.append("")
src = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_lines.py"), rep, "25"],
                     capture_output=True, text=True).stdout
lines.append("## hot source lines (warp-stall samples, executed warp-instructions)")
lines.append(src)
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:40]))
