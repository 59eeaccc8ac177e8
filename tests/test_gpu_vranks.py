"""Multi-rank correctness on ONE GPU: R = 2 / 4 / 8 virtual
ranks -- contexts of one process, one host thread each, exchanging through comm.cu's in-process
transport -- run the full x-slab protocol of dist.cu (ghost shells, refresh lists, per-iteration
refresh + allreduce stop, FoF label merge, MCC / halo reductions) and must be bit-identical to
one rank ("results invariant to process count") and equal to the oracle."""
import threading

import numpy as np
import pytest
import torch

import oracle  # noqa: F401  (the oracle pipeline below)
import paper_2604_18801_b200 as cc
import synth
from tests.parity import oracle_pipeline

pytestmark = pytest.mark.gpu


def _run_rank(rank, R, vg, arrs, gid_all, owner, p, res, errs):
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        stream = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(stream):
            mine = owner == rank
            loc = [a[mine].contiguous().to(dev) for a in arrs]
            gid = gid_all[mine].to(torch.int32).to(dev)
            stream.synchronize()
            c = cc.Corrector(p, device=0, stream=stream, dist=(rank, R, None, vg))
            c.build_cells(*loc, gid=gid)
            vp = c.find_vulnerable()
            out, info = c.correct()
            lo, ngo = c.fof_label(cc.CC_ORIG)
            ho = c.halo_sizes(cc.CC_ORIG, 20)
            ld, ngd = c.fof_label(cc.CC_DECOMP)
            lc, ngc = c.fof_label(cc.CC_CORR)
            hc = c.halo_sizes(cc.CC_CORR, 20)
            mc, md = c.mcc(cc.CC_CORR), c.mcc(cc.CC_DECOMP)
            tr = c.trace()
            stream.synchronize()
            res[rank] = {"gid": gid.cpu().numpy().view(np.uint32).astype(np.int64), "vp": vp, "info": info,
                         "out": [o.cpu().numpy() for o in out], "lo": lo.cpu().numpy().view(np.uint32),
                         "ld": ld.cpu().numpy().view(np.uint32), "lc": lc.cpu().numpy().view(np.uint32),
                         "ng": (ngo, ngd, ngc), "halos": (ho, hc), "mcc": (mc, md), "trace": tr}
            c.close()
    except Exception as e:  # pragma: no cover - reported by the test
        errs.append(f"rank {rank}: {type(e).__name__}: {e}")


def _virtual(R, arrs, p, L):
    vg = cc.VGroup(R)
    gid_all = torch.arange(arrs[0].shape[0], dtype=torch.int64)
    owner = cc.slab_of(arrs[0], R, L)
    res, errs = [None] * R, []
    th = [threading.Thread(target=_run_rank, args=(r, R, vg, arrs, gid_all, owner, p, res, errs), daemon=True)
          for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "virtual ranks hung"
    vg.close()
    assert not errs, errs
    return res


def _one_rank(arrs, p):
    dev = torch.device("cuda", 0)
    c = cc.Corrector(p, device=0)
    full = [a.to(dev) for a in arrs]
    c.build_cells(*full)
    vp = c.find_vulnerable()
    out, info = c.correct()
    lo, ngo = c.fof_label(cc.CC_ORIG)
    ho = c.halo_sizes(cc.CC_ORIG, 20)
    ld, ngd = c.fof_label(cc.CC_DECOMP)
    lc, ngc = c.fof_label(cc.CC_CORR)
    hc = c.halo_sizes(cc.CC_CORR, 20)
    r = {"vp": vp, "info": info, "out": [o.cpu().numpy() for o in out], "lo": lo.cpu().numpy().view(np.uint32),
         "ld": ld.cpu().numpy().view(np.uint32), "lc": lc.cpu().numpy().view(np.uint32), "ng": (ngo, ngd, ngc),
         "halos": (ho, hc), "mcc": (c.mcc(cc.CC_CORR), c.mcc(cc.CC_DECOMP)), "trace": c.trace()}
    c.close()
    return r


def _mcc_t(m):
    return (m["tp"], m["tn"], m["fp"], m["fn"])


@pytest.mark.parametrize("R,n,xi,kind", [(2, 60000, 1e-3, "clumped"), (4, 120000, 3e-4, "clumped"),
                                         (8, 200000, 1e-3, "clumped"), (4, 196066, 1e-3, "lattice")])
def test_virtual_ranks_bit_identical_to_one_rank(R, n, xi, kind):
    w = synth.Workload("vr", kind, n, 1.0, xi, seed=7)
    arrs = synth.make(w)
    p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi)
    one = _one_rank(arrs, p)
    res = _virtual(R, arrs, p, w.L)
    r0 = res[0]
    # global quantities (reduced over ranks) are the same on every rank and equal one rank's
    for r in res:
        assert r["vp"]["n_pairs"] == one["vp"]["n_pairs"] and r["vp"]["n_editable"] == one["vp"]["n_editable"]
        assert r["vp"]["n_violated0"] == one["vp"]["n_violated0"]
        assert r["info"]["iterations"] == one["info"]["iterations"], (r["info"], one["info"])
        assert r["info"]["active_final"] == one["info"]["active_final"]
        assert np.array_equal(r["trace"][0], one["trace"][0]) and np.array_equal(r["trace"][2], one["trace"][2])
        assert r["ng"] == one["ng"]
        assert all(np.array_equal(a, b) for a, b in zip(r["halos"], one["halos"]))
        assert [_mcc_t(m) for m in r["mcc"]] == [_mcc_t(m) for m in one["mcc"]]
    # per-particle results, gathered by gid: bit-identical
    seen = 0
    for r in res:
        g = r["gid"]
        seen += len(g)
        for k in range(3):
            assert np.array_equal(r["out"][k].view(np.uint32), one["out"][k][g].view(np.uint32)), f"coords {k}"
        for nm in ("lo", "ld", "lc"):
            assert np.array_equal(r[nm], one[nm][g]), nm
    assert seen == n
    assert r0["info"]["iterations"] > 0


def test_virtual_ranks_match_the_oracle():
    """R = 3 virtual ranks against the CPU oracle directly (pairs via MCC counts, corrected
    coordinates, FoF labels on all three position sets)."""
    w = synth.Workload("vr3", "clumped", 30000, 1.0, 1e-3, seed=9)
    arrs = synth.make(w)
    p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi)
    res = _virtual(3, arrs, p, w.L)
    o = oracle_pipeline([a.numpy() for a in arrs], p)
    for r in res:
        g = r["gid"]
        assert r["info"]["iterations"] == o["info"]["iterations"]
        for k in range(3):
            assert np.array_equal(r["out"][k].view(np.uint32), o["out"][k][g].view(np.uint32))
        assert np.array_equal(r["lo"], o["lab_orig"][g]) and np.array_equal(r["lc"], o["lab_cor"][g])
        assert np.array_equal(r["ld"], o["lab_dec"][g])
        assert _mcc_t(r["mcc"][0]) == tuple(o["mcc_cor"]) and _mcc_t(r["mcc"][1]) == tuple(o["mcc_dec"])
        assert r["ng"] == (o["ng_orig"], o["ng_dec"], o["ng_cor"])
