"""profiles/r02_k3_traffic.json from an ncu capture of the two K3 launches of PGD iteration 1
(k_pgd<0> + k_pgd<1>: a full sweep, every editable processed, every row entry evaluated) on the
bench's default workload.  Usage: python tools/k3_traffic.py REP.ncu-rep E NPAIRS OUT.json"""
import csv
import io
import json
import subprocess
import sys

rep, E, npairs, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-3, "ms": 1.0, "ns": 1e-6, "usecond": 1e-3,
         "msecond": 1.0, "nsecond": 1e-6}
tot = {"dram_bytes_read": 0.0, "dram_bytes_write": 0.0, "duration_ms": 0.0}
names = []
for r in rows[2:]:
    names.append(r[h.index("Kernel Name")])
    for key, m in (("dram_bytes_read", "dram__bytes_read.sum"), ("dram_bytes_write", "dram__bytes_write.sum"),
                   ("duration_ms", "gpu__time_duration.sum")):
        i = h.index(m)
        tot[key] += float(r[i]) * scale[units[i]]
alg = 104.0 * E + 4.0 * 2 * npairs
d = {"kernel": "K3_pgd",
     "capture": f"ncu --set full --clock-control none, k_pgd launches #2-#3 (PGD iteration 1: k_pgd<0> + "
                f"k_pgd<1>, full sweep of all {E:,} editables) of `bench.py --steps 1 --warmup 0` on the default "
                f"workload",
     "launches": names,
     "duration_ms": tot["duration_ms"],
     "dram_bytes_read": tot["dram_bytes_read"], "dram_bytes_write": tot["dram_bytes_write"],
     "dram_bytes": tot["dram_bytes_read"] + tot["dram_bytes_write"],
     "algorithmic_bytes": alg,
     "algorithmic_note": "104 B per processed editable + 4 B per row entry (all 2|V| entries)",
     "traffic_over_algorithmic": (tot["dram_bytes_read"] + tot["dram_bytes_write"]) / alg,
     "achieved_GBps_algorithmic": alg / (tot["duration_ms"] * 1e-3) / 1e9,
     "source": rep}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
