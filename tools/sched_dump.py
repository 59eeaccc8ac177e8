"""Dump K3's per-iteration schedule and convergence trace on a full-size workload (GPU
development tool): gpurun_out/sched_<cfg>.npz with trace (active, loss, violated) and schedule
(processed, awake, moved entries, full replay steps, proven-still replay steps)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_18801_b200 as cc  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = synth.CONFIGS[cfg]
if len(sys.argv) > 2:  # xi_rel override
    w = synth.Workload(w.name, w.kind, w.n, w.L, float(sys.argv[2]), eta=w.eta, b=w.b, seed=w.seed, extra=w.extra)
    cfg = f"{cfg}_{sys.argv[2]}"
REPS = int(os.environ.get("SCHED_REPS", "2"))
dev = torch.device("cuda", 0)
arrs = synth.make(w, device=dev)
p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, t_max=int(os.environ.get("CC_TMAX", "10000")), stop_mode=cc.STOP_RESTORED, profile=1)
c = cc.Corrector(p)
for rep in range(REPS):
    c.build_cells(*arrs)
    vp = c.find_vulnerable()
    c.kernel_stats(reset=True)
    torch.cuda.synchronize()
    t0 = time.time()
    out, info = c.correct()
    torch.cuda.synchronize()
    dt = time.time() - t0
    st = c.kernel_stats(reset=True)
    print(rep, "correct", info, f"{dt * 1e3:.1f} ms wall", {k: v for k, v in st.items() if "K3" in k}, flush=True)
a, l, v = c.trace()
sch = c.schedule()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez(os.path.join(ROOT, "gpurun_out", f"sched_{cfg}.npz"), active=a, loss=l, violated=v, schedule=sch,
         E=vp["n_editable"], V=vp["n_pairs"])
for t in list(range(0, 110)) + list(range(110, len(sch), 50)):
    if t < len(sch):
        print(t + 1, int(a[t]), int(v[t]), *sch[t].tolist())

# time of the first T iterations (STOP_NONE, t_max = T: the same computations as the full run's
# first T iterations) -> split of K3 time between the dense phase and the tail
for T in [int(x) for x in os.environ.get("SCHED_TMAX", "").split(",") if x]:
    pt = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, t_max=T, stop_mode=cc.STOP_NONE, profile=1)
    ct = cc.Corrector(pt)
    for rep in range(2):
        ct.build_cells(*arrs)
        ct.find_vulnerable()
        ct.kernel_stats(reset=True)
        _, it = ct.correct()
        st = ct.kernel_stats(reset=True)
    print(f"t_max={T}: iterations {it['iterations']} K3 {st['K3_pgd'][0]:.2f} ms", flush=True)
    ct.close()
