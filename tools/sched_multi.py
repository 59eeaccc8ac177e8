"""Per-iteration K3 timeline on several GPUs (development tool, run under torchrun): device
%globaltimer at the end of each PGD iteration's k_pgd<1> (cc_get_schedule column 5) on rank 0,
for the bench's default workload, printed as iteration periods."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_18801_b200 as cc  # noqa: E402
import synth  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
w = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
x, y, z, xh, yh, zh = synth.make(w, device=dev)
own = (cc.slab_of(x, world, w.L) == rank).nonzero().flatten()
arrs = [a[own].contiguous() for a in (x, y, z, xh, yh, zh)]
gid = own.to(torch.int32)
del x, y, z, xh, yh, zh, own
torch.cuda.empty_cache()
uid = [cc.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, profile=1)
c = cc.Corrector(p, device=local, dist=(rank, world, uid[0]))
for rep in range(3):
    c.build_cells(*arrs, gid=gid)
    c.find_vulnerable()
    _, info = c.correct()
sch = c.schedule()
if rank == 0:
    t = sch[:, 5].astype(np.float64)
    dt = np.diff(t) / 1e3
    print("iterations", info["iterations"], "processed/awake at t=1..5:", sch[:5, 0].tolist(), sch[:5, 1].tolist())
    for a, b in ((0, 5), (5, 20), (20, 60), (60, len(dt))):
        if b > a:
            print(f"iterations {a + 2}..{b + 1}: mean period {dt[a:b].mean():.1f} us (min {dt[a:b].min():.1f})")
    print("kernel stats", {k: v for k, v in c.kernel_stats().items() if k.startswith("K3")})
c.close()
dist.destroy_process_group()
