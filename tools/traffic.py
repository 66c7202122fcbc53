"""Per-side-pass DRAM traffic from an ncu metrics CSV of tools/profile_pass.py
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum).

    python tools/traffic.py launches.csv CONFIG out.json

The last `passes` user + item side passes of the capture are split at the
partial_gramian launches (k_gemm3_tf32 / k_slab_partial) and the projection
(k_project*, a tensor-core GEMM of the Gramian phase inside ials_epoch) is
left out; the JSON records the
DRAM bytes and kernel time per side pass (the unit bench.py's roofline is
quoted per), averaged over the user and the item pass."""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
        "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")})
    d[r[mi]] = float(r[vi].replace(",", "")) * unit.get(r[ui], 1.0)
L = list(launch.values())
# side passes: everything after a Gramian GEMM up to the next one
passes, cur = [], None
for d in L:
    n = d["name"]
    if "k_gemm3_tf32" in n or "k_slab_partial" in n or "k_reduce_splits" in n or "k_gram_reduce" in n:
        if cur and cur["kernels"]:
            passes.append(cur)
        cur = {"kernels": [], "bytes": 0.0, "seconds": 0.0}
        continue
    if cur is None or "k_project" in n:   # in ials_epoch the projection is a GEMM of the Gramian phase
        continue
    if "k_sym_eig" in n or "k_reduce_splits_strided" in n or "k_sync_copies" in n:
        continue   # side-stream eigendecompositions / GEMM-copy upkeep: not part of a side pass
    cur["kernels"].append(n)
    cur["bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    cur["seconds"] += d.get("gpu__time_duration.sum", 0)
if cur and cur["kernels"]:
    passes.append(cur)
last = passes[-2:]   # the user and the item pass of the profiled block
out = {"config": sys.argv[2], "source": sys.argv[1].split("/")[-1],
       "passes": [{"kernels": sorted(set(p["kernels"])), "dram_bytes": p["bytes"], "kernel_seconds": p["seconds"]}
                  for p in last],
       "dram_bytes_per_side_pass": sum(p["bytes"] for p in last) / len(last)}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out, indent=1))
