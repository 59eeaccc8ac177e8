"""Diagnostics on a full-size workload (GPU): convergence trace, FoF determinism and
label equality, halo catalogue equality.  Development tool, prints to stdout."""
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
xi_rel = float(sys.argv[2]) if len(sys.argv) > 2 else None
tmax = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
w = synth.CONFIGS[cfg]
if xi_rel is not None:
    w = synth.Workload(w.name, w.kind, w.n, w.L, xi_rel, eta=w.eta, b=w.b, seed=w.seed, extra=w.extra)
dev = torch.device("cuda", 0)
t0 = time.time()
arrs = synth.make(w, device=dev)
torch.cuda.synchronize()
print(f"{cfg} xi_rel={w.xi_rel} N={w.n} drawn in {time.time() - t0:.1f}s", flush=True)
stop = int(sys.argv[4]) if len(sys.argv) > 4 else cc.STOP_RESTORED
p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, t_max=tmax, stop_mode=stop)
c = cc.Corrector(p)
c.build_cells(*arrs)
vp = c.find_vulnerable()
print("vp", vp, flush=True)
t0 = time.time()
out, info = c.correct()
torch.cuda.synchronize()
print("corr", info, f"{time.time() - t0:.2f}s", flush=True)
a, l, v = c.trace()
idx = sorted(set([0, 1, 2, 5, 10, 20, 50, 100, 150, 200, 300, 500, 1000, 2000, 5000, len(a) - 1]))
print("trace (t, active, loss, violated)", [(i, int(a[i]), float(l[i]), int(v[i])) for i in idx if i < len(a)],
      flush=True)
sch = c.schedule()
print("schedule (t, processed, awake, moved entries, full replay steps, quick replay steps):")
for t in sorted(set(list(range(0, 12)) + list(range(12, len(sch), max(1, len(sch) // 40))) + [len(sch) - 1])):
    if t < len(sch):
        print("  ", t + 1, *sch[t].tolist())
gi, gj, fl = c.get_pairs()
deg = torch.bincount(torch.cat([gi.long(), gj.long()]), minlength=w.n)
dv, di = torch.sort(deg, descending=True)
print("row lengths: max", int(dv[0]), "top10", dv[:10].tolist(), "rows>32:", int((deg > 32).sum()),
      ">1000:", int((deg > 1000).sum()), ">10000:", int((deg > 10000).sum()), flush=True)
if os.environ.get("DIAG_ONLY_K3"):
    sys.exit(0)
m = c.mcc(cc.CC_CORR)
md = c.mcc(cc.CC_DECOMP)
print("mcc corr", m, "dec", md, flush=True)
l1, n1 = c.fof_label(cc.CC_ORIG)
l1 = l1.clone()
h1 = c.halo_sizes(cc.CC_ORIG)
l1b, n1b = c.fof_label(cc.CC_ORIG)
l1b = l1b.clone()
print("fof orig deterministic:", n1 == n1b, bool(torch.equal(l1, l1b)), flush=True)
l2, n2 = c.fof_label(cc.CC_CORR)
l2 = l2.clone()
h2 = c.halo_sizes(cc.CC_CORR)
diff = (l1 != l2).nonzero().flatten()
print("groups", n1, n2, "labels differ at", diff.numel(), "halos", len(h1), len(h2), "equal", np.array_equal(h1, h2),
      flush=True)
if diff.numel():
    print("first diffs", diff[:10].tolist(), l1[diff[:10]].tolist(), l2[diff[:10]].tolist())
    d = set(np.setxor1d(h1, h2).tolist())
    print("halo sizes only in one:", sorted(d)[:20])
l3, n3 = c.fof_label(cc.CC_DECOMP)
print("decomp groups", n3, flush=True)
st = c.kernel_stats()
print(st)
