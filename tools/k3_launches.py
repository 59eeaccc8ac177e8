"""Per-iteration K3 launch times from an ncu launch list (tools/ncu_summary.py's CSV):
python tools/k3_launches.py gpurun_out/launches.csv [launches_per_step]"""
import csv
import sys

import numpy as np

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
pg = np.array([float(d["Metric Value"].replace(",", "")) for d in data
               if d["Metric Name"] == "gpu__time_duration.sum" and "k_pgd" in d["Kernel Name"]]) / 1e3
per = int(sys.argv[2]) if len(sys.argv) > 2 else None
step = pg[-per:] if per else pg
edges = [0, 1, 2, 3, 5, 10, 20, 50, 100, 200, 400, 800, 1600, 3200, 10000]
print("| launches | mean us | total ms |")
print("|---|---:|---:|")
for a, b in zip(edges[:-1], edges[1:]):
    if a >= len(step):
        break
    seg = step[a:b]
    print(f"| {a}-{min(b, len(step)) - 1} | {seg.mean():.1f} | {seg.sum() / 1e3:.2f} |")
print(f"\n{len(step)} launches, {step.sum() / 1e3:.1f} ms")
