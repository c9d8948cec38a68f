"""Summarise an ncu launch list CSV (mean device time per kernel)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0].replace("void ", "")[:44]].append(float(r[vi].replace(",", "")))
tot = 0.0
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]) / len(x[1])):
    m = sum(v) / len(v) / 1e3
    if not k.startswith("at::"):
        tot += m * (len(v) / max(len(agg.get("tmb::k_tri_pass<long>", [1])), 1))
    print(f"{k:44s} n={len(v):3d} mean={m:9.1f} us")
