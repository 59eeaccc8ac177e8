"""CPU tests of the multi-GPU decomposition logic with torch.distributed (gloo, world size 2
and 3): slab ownership partitions the particles, the ghost shells of width
delta = b + 2 sqrt3 xi (§III-D) make every vulnerable pair with an owned endpoint visible
locally, and keeping each pair on the owner of its min-gid endpoint (R17) partitions the global
pair set exactly.  The pair search on each rank is the oracle's (no GPU here)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2604_18801_b200 as cc
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, xi_rel, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.Workload("g", "clumped", n, 1.0, xi_rel, seed=5)
        x, y, z, xh, yh, zh = synth.make(w)
        c = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi)
        th = oracle.thresholds(c)
        gw = max(th["band_hi"], math.sqrt(th["hi2"])) * (1 + 1e-5)
        owner = cc.slab_of(x, world, 1.0)
        mine = (owner == rank).nonzero().flatten()
        to_left, to_right = cc.shell_masks(x[mine], rank, world, 1.0, gw)
        left, right = (rank - 1) % world, (rank + 1) % world
        # exchange ghost index lists through gloo (the NCCL send/recv of dist.cu)
        send = {}
        send.setdefault(left, []).extend(mine[to_left].tolist())
        send.setdefault(right, []).extend(mine[to_right].tolist())
        lists = [None] * world
        dist.all_gather_object(lists, send)
        ghosts = []
        for r, obj in enumerate(lists):
            if r != rank:
                ghosts += obj.get(rank, [])
        loc = torch.cat([mine, torch.tensor(sorted(set(ghosts)), dtype=torch.long)])
        arr = [a[loc].numpy() for a in (x, y, z, xh, yh, zh)]
        gid = loc.numpy().astype(np.uint32)
        pi, pj, pf = oracle.find_pairs(*arr, c, gid=gid)
        gi, gj = gid[pi], gid[pj]          # gi < gj (canonical)
        owned = set(mine.tolist())
        keep = np.array([int(a) in owned for a in gi], bool)
        mine_pairs = sorted(zip(gi[keep].tolist(), gj[keep].tolist(), pf[keep].tolist()))
        # coverage: every global pair with an owned endpoint must be present locally
        allp = [None] * world
        dist.all_gather_object(allp, {"pairs": mine_pairs, "owned": sorted(owned)})
        if rank == 0:
            g = oracle.find_pairs(*(a.numpy() for a in (x, y, z, xh, yh, zh)), c)
            glob = sorted(zip(g[0].tolist(), g[1].tolist(), g[2].tolist()))
            union = sorted(p for d in allp for p in d["pairs"])
            owned_all = sorted(i for d in allp for i in d["owned"])
            q.put({"partition": owned_all == list(range(n)), "pairs_equal": union == glob,
                   "n_pairs": len(glob), "dup": len(union) != len(set(union))})
    except Exception as e:  # surface worker failures instead of hanging the queue
        q.put({"error": f"rank {rank}: {e!r}"})
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,xi", [(2, 12000, 1e-3), (3, 15000, 3e-3)])
def test_slab_ghost_protocol_partitions_pairs(world, n, xi):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, xi, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    assert "error" not in res, res
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert res["partition"], "slab ownership is not a partition"
    assert res["pairs_equal"] and not res["dup"], res
    assert res["n_pairs"] > 1000
