"""Multi-GPU parity worker (launched by tests/test_gpu_multi.py with torchrun, one rank per GPU).

Every rank draws the same seeded workload, keeps the particles of its x slab (cc_dist rule),
runs the distributed path (NCCL ghost exchange, per-iteration refresh + allreduce stop, FoF
label merge) and sends its owned results to rank 0, which runs the single-GPU path on the whole
set and requires bit-identical results (SURVEY §8e P11 / PAPER P:233 "results invariant to
process count")."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_18801_b200 as cc  # noqa: E402
import synth  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("MG_WATCHDOG", "240")), exit=True)
    n = int(os.environ.get("MG_N", "60000"))
    xi_rel = float(os.environ.get("MG_XI", "1e-3"))
    seed = int(os.environ.get("MG_SEED", "3"))
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    w = synth.Workload("mg", "clumped", n, 1.0, xi_rel, seed=seed)
    arrs = synth.make(w)  # host, identical on every rank
    gid_all = torch.arange(n, dtype=torch.int64)
    owner = cc.slab_of(arrs[0], world, w.L)
    mine = owner == rank
    loc = [a[mine].contiguous().to(dev) for a in arrs]
    gid = gid_all[mine].to(torch.int32).to(dev)
    uid = [cc.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi)
    def log(*a):
        print(f"[rank {rank}]", *a, file=sys.stderr, flush=True)

    c = cc.Corrector(p, device=local, dist=(rank, world, uid[0]))
    log("created, owned", int(mine.sum()))
    c.build_cells(*loc, gid=gid)
    log("cells built")
    vp = c.find_vulnerable()
    log("pairs", vp)
    out, info = c.correct()
    log("corrected", info)
    lab_o, ng_o = c.fof_label(cc.CC_ORIG)
    log("fof orig", ng_o)
    h_o = c.halo_sizes(cc.CC_ORIG, 20)
    lab_c, ng_c = c.fof_label(cc.CC_CORR)
    h_c = c.halo_sizes(cc.CC_CORR, 20)
    m_c = c.mcc(cc.CC_CORR)
    m_d = c.mcc(cc.CC_DECOMP)
    tr = c.trace()
    res = {"gid": gid.cpu().numpy().view(np.uint32), "out": [o.cpu().numpy() for o in out],
           "lab_o": lab_o.cpu().numpy().view(np.uint32), "lab_c": lab_c.cpu().numpy().view(np.uint32)}
    gathered = [None] * world
    dist.gather_object(res, gathered if rank == 0 else None, dst=0)
    ok = True
    msg = []
    if rank == 0:
        # single-GPU reference on the whole set (rank 0's GPU, separate context)
        full = [a.to(dev) for a in arrs]
        s = cc.Corrector(p, device=local)
        s.build_cells(*full, gid=gid_all.to(torch.int32).to(dev))
        vp1 = s.find_vulnerable()
        out1, info1 = s.correct()
        lo1, ngo1 = s.fof_label(cc.CC_ORIG)
        ho1 = s.halo_sizes(cc.CC_ORIG, 20)
        lc1, ngc1 = s.fof_label(cc.CC_CORR)
        hc1 = s.halo_sizes(cc.CC_CORR, 20)
        mc1 = s.mcc(cc.CC_CORR)
        md1 = s.mcc(cc.CC_DECOMP)
        tr1 = s.trace()
        o1 = [o.cpu().numpy() for o in out1]
        l1o = lo1.cpu().numpy().view(np.uint32)
        l1c = lc1.cpu().numpy().view(np.uint32)

        def check(cond, what):
            nonlocal ok
            if not cond:
                ok = False
                msg.append(what)

        check(vp["n_pairs"] == vp1["n_pairs"], f"n_pairs {vp['n_pairs']} vs {vp1['n_pairs']}")
        check(vp["n_editable"] == vp1["n_editable"], "n_editable")
        check(vp["n_violated0"] == vp1["n_violated0"], "violated0")
        check(info["iterations"] == info1["iterations"], f"iterations {info['iterations']} vs {info1['iterations']}")
        check(info["active0"] == info1["active0"] and info["active_final"] == info1["active_final"], "active")
        check(abs(info["loss0"] - info1["loss0"]) <= 1e-9 * max(info1["loss0"], 1e-300), "loss0")
        check(np.array_equal(tr[0], tr1[0]), "trace")
        check(ng_o == ngo1 and ng_c == ngc1, f"groups {ng_o}/{ngo1} {ng_c}/{ngc1}")
        check(np.array_equal(h_o, ho1) and np.array_equal(h_c, hc1), "halos")
        check((m_c["tp"], m_c["tn"], m_c["fp"], m_c["fn"]) == (mc1["tp"], mc1["tn"], mc1["fp"], mc1["fn"]), "mcc corr")
        check((m_d["tp"], m_d["tn"], m_d["fp"], m_d["fn"]) == (md1["tp"], md1["tn"], md1["fp"], md1["fn"]), "mcc dec")
        seen = 0
        for r in gathered:
            g = r["gid"].astype(np.int64)
            seen += len(g)
            for k in range(3):
                check(np.array_equal(r["out"][k].view(np.uint32), o1[k][g].view(np.uint32)), f"coords {k}")
            check(np.array_equal(r["lab_o"], l1o[g]), "labels orig")
            check(np.array_equal(r["lab_c"], l1c[g]), "labels corr")
        check(seen == n, "ownership partition")
        print(json.dumps({"ok": ok, "fail": msg, "world": world, "n": n, "pairs": vp1["n_pairs"],
                          "iterations": info1["iterations"], "groups": ngo1}), flush=True)
    c.close()  # collective teardown of libcc's NCCL communicator on every rank
    if rank == 0:
        s.close()
    okt = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(okt, src=0)
    dist.destroy_process_group()
    return 0 if int(okt.item()) == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
