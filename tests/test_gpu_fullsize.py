"""Full-size parity in the bench launch configuration (configs[3] = C4, N = 280,953,867, one
GPU): the oracle cannot run the whole set, so it checks sampled outputs one by one and the
properties that hold at any size:

* sampled particles: their vulnerable partners and link flags, found by the oracle's brute
  force against all N particles, equal the GPU's (bit-exact);
* sampled vulnerable-graph components: the oracle's PGD on the component alone, run for the
  same number of updates, gives bit-identical corrected coordinates (components are
  independent under Alg. 1; only the global stop couples them) and no active pair;
* everywhere: |x' - x| <= xi_f, non-editable particles untouched, MCC over V = 1 and FoF labels
  of corrected = original when converged; the fixed-T run with T = the converged iteration count
  reproduces the converged run bit-exactly (the speculative stop is exact at full size).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2604_18801_b200 as cc
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _gpu_run(arrs, p):
    c = cc.Corrector(p)
    c.build_cells(*arrs)
    vp = c.find_vulnerable()
    out, info = c.correct()
    return c, vp, out, info


@pytest.mark.parametrize("xi_rel", [1e-6, 1e-5])
def test_c4_full_size_sampled_parity(xi_rel):
    """C4 at full size in the bench configuration: xi_rel = 1e-6 (the bench default)
    and 1e-5 (round 1's default: a 50M-editable frontier and the long tail)."""
    if torch.cuda.get_device_properties(0).total_memory < 120e9:
        pytest.skip("needs a B200-class GPU")
    w0 = synth.CONFIGS["C4"]
    w = synth.Workload(w0.name, w0.kind, w0.n, w0.L, xi_rel, seed=w0.seed)
    dev = torch.device("cuda", 0)
    arrs = synth.make(w, device=dev)
    p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, stop_mode=cc.STOP_RESTORED)  # bench config
    c, vp, out, info = _gpu_run(arrs, p)
    assert info["converged"] and info["violated_final"] == 0
    # invariants everywhere
    xi_f = float(np.float32(w.xi))
    for a, o in zip(arrs[:3], out):
        assert float((o.double() - a.double()).abs().max()) <= xi_f
    m = c.mcc(cc.CC_CORR)
    assert m["fp"] == 0 and m["fn"] == 0 and m["mcc"] == 1.0
    lo, ng_o = c.fof_label(cc.CC_ORIG)
    lo = lo.clone()
    lc, ng_c = c.fof_label(cc.CC_CORR)
    assert ng_o == ng_c and torch.equal(lo, lc)
    gi, gj, fl = c.get_pairs()
    assert gi.shape[0] == vp["n_pairs"]
    T = info["iterations"]

    # host copies for the oracle
    H = [a.cpu().numpy() for a in arrs]
    O = [o.cpu().numpy() for o in out]
    gi = gi.cpu().numpy().view(np.uint32).astype(np.int64)
    gj = gj.cpu().numpy().view(np.uint32).astype(np.int64)
    fl = fl.cpu().numpy()
    # non-editable particles are untouched
    ed = np.zeros(w.n, bool)
    ed[gi] = True
    ed[gj] = True
    for k in range(3):
        assert np.array_equal(O[k][~ed].view(np.uint32), H[3 + k][~ed].view(np.uint32))
    order = np.argsort(gi, kind="stable")
    gi_s, gj_s, fl_s = gi[order], gj[order], fl[order]
    order_j = np.argsort(gj, kind="stable")
    gj_j, gi_j, fl_j = gj[order_j], gi[order_j], fl[order_j]
    c_or = oracle.cfg(L=w.L, b=w.linking_length, xi=w.xi, t_max=T, stop_mode=oracle.STOP_NONE)
    th = oracle.thresholds(c_or)
    rad = max(th["band_hi"], math.sqrt(th["hi2"])) * (1 + 1e-5)

    xs_t, xo_t = torch.sort(arrs[0], stable=True)  # the index only narrows the scan (device sort)
    xsorted, xorder = xs_t.cpu().numpy(), xo_t.cpu().numpy()
    del xs_t, xo_t

    def xwindow(lo, hi):
        # fp32 keys widened outward by one ulp (a float64 key would make numpy cast the array)
        lo32 = np.nextafter(np.float32(lo), np.float32(-np.inf))
        hi32 = np.nextafter(np.float32(hi), np.float32(np.inf))
        return xorder[np.searchsorted(xsorted, lo32, "left"):np.searchsorted(xsorted, hi32, "right")]

    def partners_oracle(i):
        """all N particles within the band radius per axis (min image; an x-sorted index only
        narrows the scan, every candidate is tested), then the oracle's own brute-force pair
        test on {i} U candidates"""
        xi_ = float(H[0][i])
        cand = [xwindow(xi_ - rad, xi_ + rad)]
        if xi_ - rad < 0:
            cand.append(xwindow(xi_ - rad + w.L, w.L))
        if xi_ + rad >= w.L:
            cand.append(xwindow(0.0, xi_ + rad - w.L))
        cand = np.unique(np.concatenate(cand))
        d = [np.abs(H[k][cand] - H[k][i]) for k in range(3)]
        d = [np.minimum(dk, w.L - dk) for dk in d]
        cand = cand[(d[0] <= rad) & (d[1] <= rad) & (d[2] <= rad)]
        idx = np.concatenate([[i], cand[cand != i]])
        pi, pj, pf = oracle.find_pairs(*(h[idx] for h in H), c_or, gid=idx.astype(np.uint32), brute=True)
        a, b = idx[pi], idx[pj]
        sel = (a == i) | (b == i)
        return {(int(min(x, y)), int(max(x, y))): int(f) for x, y, f in zip(a[sel], b[sel], pf[sel])}

    def partners_gpu(i):
        res = {}
        s, e = np.searchsorted(gi_s, i), np.searchsorted(gi_s, i, side="right")
        for k in range(s, e):
            res[(int(i), int(gj_s[k]))] = int(fl_s[k])
        s, e = np.searchsorted(gj_j, i), np.searchsorted(gj_j, i, side="right")
        for k in range(s, e):
            res[(int(gi_j[k]), int(i))] = int(fl_j[k])
        return res

    rng = np.random.default_rng(0)
    sample = np.concatenate([rng.choice(np.nonzero(ed)[0], 12, replace=False), rng.choice(w.n, 4, replace=False)])
    for i in sample:
        assert partners_oracle(int(i)) == partners_gpu(int(i)), f"particle {i}"

    # sampled components: BFS on the oracle's pairs, then the oracle's PGD on the component
    done = 0
    for i in rng.choice(np.nonzero(ed)[0], 40, replace=False):
        comp, frontier, pairs = {int(i)}, [int(i)], {}
        too_big = False
        while frontier and not too_big:
            nxt = []
            for a in frontier:
                for (u, v), f in partners_oracle(a).items():
                    pairs[(u, v)] = f
                    for q in (u, v):
                        if q not in comp:
                            comp.add(q)
                            nxt.append(q)
            frontier = nxt
            too_big = len(comp) > 60
        if too_big:
            continue
        idx = np.array(sorted(comp), np.int64)
        pos = {g: k for k, g in enumerate(idx)}
        keys = sorted(pairs)
        pi = np.array([pos[u] for u, v in keys], np.int64)
        pj = np.array([pos[v] for u, v in keys], np.int64)
        pf = np.array([pairs[k] for k in keys], np.uint8)
        xo, yo, zo, inf = oracle.correct(*(h[idx] for h in H), (pi, pj, pf), c_or, gid=idx.astype(np.uint32))
        assert inf["violated_final"] == 0
        for k, o in enumerate((xo, yo, zo)):
            assert np.array_equal(o.view(np.uint32), O[k][idx].view(np.uint32)), f"component of {i}, coord {k}"
        done += 1
        if done >= 8:
            break
    assert done >= 3

    # the fixed-T run reproduces the converged run bit-exactly
    pN = cc.Params(box=w.L, b=w.linking_length, xi=w.xi, t_max=T, stop_mode=cc.STOP_NONE)
    c2, _, out2, info2 = _gpu_run(arrs, pN)
    assert info2["iterations"] == T
    for a, b in zip(out, out2):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
