"""Shared harness of the GPU parity tests: run the CUDA path through the C ABI and the CPU
oracle on the SAME seeded inputs and compare element by element.

Acceptance (BASELINE.json north_star):
  pairs + both link flags, FoF labels (min gid), MCC counts, halo sizes, iteration count:
  bit-exact / exact.  Corrected coordinates: bit-exact (the pinned fp32 schedule is the same),
  the north_star floor being <= 1e-6 relative.  L_tight loss (fp64 sums in a different order):
  relative 1e-9.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
import paper_2604_18801_b200 as cc


def to_np(t):
    return t.detach().cpu().numpy()


def gpu_pipeline(arrs, params: cc.Params, gid=None, fof=True):
    dev = torch.device("cuda", 0)
    ts = [torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32).to(dev) for a in arrs]
    g = None if gid is None else torch.as_tensor(np.asarray(gid, dtype=np.uint32).view(np.int32)).to(dev)
    c = cc.Corrector(params, device=0)
    c.build_cells(*ts, gid=g)
    vp = c.find_vulnerable()
    gi, gj, fl = c.get_pairs()
    # §8(b): canonical (gi < gj) and sorted by (gi, gj)
    a_, b_ = to_np(gi).view(np.uint32).astype(np.int64), to_np(gj).view(np.uint32).astype(np.int64)
    assert np.all(a_ < b_), "cc_get_pairs: not canonical"
    key = (a_ << 32) | b_
    assert np.all(np.diff(key) > 0), "cc_get_pairs: not sorted by (gi, gj)"
    out, info = c.correct()
    res = {"vp": vp, "info": info, "pairs": (to_np(gi).view(np.uint32), to_np(gj).view(np.uint32), to_np(fl)),
           "out": [to_np(o) for o in out]}
    res["mcc_dec"] = c.mcc(cc.CC_DECOMP)
    res["mcc_cor"] = c.mcc(cc.CC_CORR)
    res["trace"] = c.trace()
    if fof:
        for name, which in (("orig", cc.CC_ORIG), ("dec", cc.CC_DECOMP), ("cor", cc.CC_CORR)):
            lab, ng = c.fof_label(which)
            res["lab_" + name] = to_np(lab).view(np.uint32).copy()
            res["ng_" + name] = ng
            res["halo_" + name] = c.halo_sizes(which, 20)
    res["ctx"] = c
    return res


def oracle_cfg(params: cc.Params, n: int):
    return oracle.cfg(L=params.box, b=params.b if params.b > 0 else None, xi=params.xi, periodic=bool(params.periodic),
                      m=params.m, alpha=params.alpha, beta1=params.beta1, beta2=params.beta2,
                      eps_adam=params.eps_adam, t_max=params.t_max, eps_loss=params.eps_loss,
                      stop_mode=params.stop_mode, optimizer=params.optimizer, vanilla_step=params.vanilla_step,
                      n=n, eta=params.eta)


def oracle_pipeline(arrs, params: cc.Params, gid=None, fof=True):
    x, y, z, xh, yh, zh = [np.ascontiguousarray(a, dtype=np.float32) for a in arrs]
    c = oracle_cfg(params, len(x))
    pairs = oracle.find_pairs(x, y, z, xh, yh, zh, c, gid=gid)
    xo, yo, zo, info, tr = oracle.correct(x, y, z, xh, yh, zh, pairs, c, gid=gid, trace=True)
    g = np.arange(len(x), dtype=np.uint32) if gid is None else np.asarray(gid, np.uint32)
    res = {"pairs": (g[pairs[0]], g[pairs[1]], pairs[2]), "info": info, "out": [xo, yo, zo], "trace": tr}
    ol = (pairs[2] & 1).astype(bool)
    res["mcc_dec"] = oracle.mcc_counts(ol, (pairs[2] & 2).astype(bool))
    res["mcc_cor"] = oracle.mcc_counts(ol, oracle.pair_links(pairs[0], pairs[1], xo, yo, zo, c))
    if fof:
        for name, P in (("orig", (x, y, z)), ("dec", (xh, yh, zh)), ("cor", (xo, yo, zo))):
            lab, ng = oracle.fof(*P, c, gid=gid)
            res["lab_" + name] = lab
            res["ng_" + name] = ng
            res["halo_" + name] = oracle.halo_catalog(lab, 20)
    return res


def sorted_pairs(p):
    gi, gj, fl = [np.asarray(a) for a in p]
    order = np.lexsort((gj, gi))
    return gi[order].astype(np.int64), gj[order].astype(np.int64), fl[order].astype(np.uint8)


def assert_parity(g, o, fof=True, exact_positions=True):
    gp, op = sorted_pairs(g["pairs"]), sorted_pairs(o["pairs"])
    assert len(gp[0]) == len(op[0]), f"|V| gpu {len(gp[0])} oracle {len(op[0])}"
    assert np.array_equal(gp[0], op[0]) and np.array_equal(gp[1], op[1]), "pair sets differ"
    assert np.array_equal(gp[2], op[2]), "link flags differ"
    gi, oi = g["info"], o["info"]
    assert gi["iterations"] == oi["iterations"], (gi, oi)
    assert gi["active0"] == oi["active0"] and gi["active_final"] == oi["active_final"], (gi, oi)
    assert gi["converged"] == oi["converged"]
    for a, b in ((gi["loss0"], oi["loss0"]), (gi["loss_final"], oi["loss_final"])):
        assert abs(a - b) <= 1e-9 * max(abs(b), 1e-300), (a, b)
    assert g["vp"]["n_editable"] == oi["n_editable"]
    for k in range(3):
        a, b = g["out"][k], o["out"][k]
        if exact_positions:
            bad = np.nonzero(a.view(np.uint32) != b.view(np.uint32))[0]
            assert bad.size == 0, f"coord {k}: {bad.size} differ, first {bad[:5]} gpu {a[bad[:5]]} oracle {b[bad[:5]]}"
        else:
            assert np.allclose(a, b, rtol=1e-6, atol=0)
    md, mc = g["mcc_dec"], g["mcc_cor"]
    assert (md["tp"], md["tn"], md["fp"], md["fn"]) == tuple(o["mcc_dec"])
    assert (mc["tp"], mc["tn"], mc["fp"], mc["fn"]) == tuple(o["mcc_cor"])
    ta, tl, tv = g["trace"]
    oa, ol, ov = o["trace"]
    assert np.array_equal(ta, oa), (ta[:10], oa[:10])
    assert np.array_equal(tv, ov), (tv[:10], ov[:10])
    assert gi["violated0"] == oi["violated0"] and gi["violated_final"] == oi["violated_final"]
    if fof:
        for name in ("orig", "dec", "cor"):
            assert g["ng_" + name] == o["ng_" + name], name
            assert np.array_equal(g["lab_" + name], o["lab_" + name]), name
            assert np.array_equal(g["halo_" + name], o["halo_" + name]), name


def check_invariants(arrs, out, params: cc.Params, info):
    """T2: |x' - x| <= xi_f exactly everywhere."""
    xi_f = np.float64(np.float32(params.xi))
    for a, b in zip(arrs[:3], out):
        assert np.all(np.abs(np.asarray(b, np.float64) - np.asarray(a, np.float64)) <= xi_f)
