"""Per-iteration K3 times from a sched_dump text log (the schedule's device timer column)."""
import sys

import numpy as np

rows = []
for ln in open(sys.argv[1]):
    f = ln.split()
    if len(f) == 9 and f[0].isdigit():
        rows.append([int(x) for x in f])
r = np.array(rows)
t, tm = r[:, 0], r[:, 8].astype(np.float64)
print(open(sys.argv[1]).readline()[:400])
edges = [1, 11, 51, 101, 111, 161, 661, 1161, 2161, 5161, 10001]
for a, b in zip(edges[:-1], edges[1:]):
    m = (t >= a) & (t <= b)
    idx = np.nonzero(m)[0]
    if len(idx) < 2:
        continue
    dt = (tm[idx[-1]] - tm[idx[0]]) / 1e6 / (t[idx[-1]] - t[idx[0]])
    print(f"t {a}..{b}: {dt:.3f} ms/iter  processed {r[idx, 3].mean():.0f} awake {r[idx, 4].mean():.0f} "
          f"moved-entries {r[idx, 5].mean():.0f} full-replay {r[idx, 6].mean():.0f} proven {r[idx, 7].mean():.0f}")
print("total", (tm[-1] - tm[0]) / 1e6, "ms over", t[-1] - t[0], "iterations")
