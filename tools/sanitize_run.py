"""Small end-to-end run for compute-sanitizer (racecheck / synccheck / memcheck, one tool per
gpurun call): the C1 recipe through every ABI step (S1-S7, pairs, trace, edit log + pack), then
R = 2 virtual ranks through the multi-rank protocol.  Exits non-zero on any error."""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_18801_b200 as cc  # noqa: E402
import synth  # noqa: E402

N = int(os.environ.get("SAN_N", "12000"))
w = synth.Workload("san", "clumped", N, 1.0, 1e-3, seed=1)
dev = torch.device("cuda", 0)
arrs = synth.make(w, device=dev)
p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, stop_mode=cc.STOP_RESTORED, t_max=400)
c = cc.Corrector(p, device=0)
c.build_cells(*arrs)
vp = c.find_vulnerable()
gi, gj, fl = c.get_pairs()
out, info = c.correct()
for which in (cc.CC_ORIG, cc.CC_DECOMP, cc.CC_CORR):
    c.fof_label(which)
    c.halo_sizes(which, 20)
m = c.mcc(cc.CC_CORR)
c.trace()
c.schedule()
flags, q = c.edit_encode(*arrs, *out)
words = c.edit_pack(q)
assert torch.equal(c.edit_unpack(words, int(q.shape[0])), q)
c.edit_decode(*arrs[3:], flags, q)
torch.cuda.synchronize()
print("single", vp["n_pairs"], info["iterations"], m["mcc"], flush=True)
c.close()

# R = 2 virtual ranks (comm.cu transport) through the multi-rank protocol
vg = cc.VGroup(2)
owner = cc.slab_of(arrs[0].cpu(), 2, w.L)
gid_all = torch.arange(N, dtype=torch.int64)
errs = []


def rank(r):
    try:
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            mine = (owner == r).to(dev)
            loc = [a[mine].contiguous() for a in arrs]
            g = gid_all.to(dev)[mine].to(torch.int32)
            cr = cc.Corrector(p, device=0, stream=s, dist=(r, 2, None, vg))
            cr.build_cells(*loc, gid=g)
            cr.find_vulnerable()
            cr.correct()
            cr.fof_label(cc.CC_CORR)
            cr.halo_sizes(cc.CC_CORR, 20)
            cr.mcc(cc.CC_CORR)
            s.synchronize()
            cr.close()
    except Exception as e:  # pragma: no cover
        errs.append(repr(e))


th = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(2)]
for t in th:
    t.start()
for t in th:
    t.join(600)
vg.close()
assert not errs, errs
print("virtual ranks ok", flush=True)
