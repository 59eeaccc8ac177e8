"""Pins for the oracle's correction loop (O4/O5): losses (Eq. 1, Eq. 3), gradient, Adam,
projection, stop rule and the loop-level claims of the paper.

PAPER.md §III-A Eq. (1); Eq. (2); Alg. 1; §III-B
(Eq. 3, Adam P:458, convergence analysis P:458); §III-E budget P:471.
Pinned against worked values, central finite differences in fp64,
torch.optim.Adam in fp64, closed forms, and invariants (|x'-x| <= xi, MCC = 1, FoF equality).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


def _pair_positions(d_orig, d_dec, L=10.0):
    """two particles on the x axis at original distance d_orig and decompressed d_dec"""
    x = np.array([4.0, 4.0 + d_orig], np.float64)
    xh = np.array([4.0, 4.0 + d_dec], np.float64)
    return x, xh


def test_eq1_worked_values():
    """d=0.99, b=1, d_hat=1.05 -> 2.5e-3; d=1.01, d_hat=0.97 -> 9e-4."""
    for d, dh, want in ((0.99, 1.05, 2.5e-3), (1.01, 0.97, 9e-4), (0.99, 0.98, 0.0), (1.01, 1.02, 0.0)):
        x, xh = _pair_positions(d, dh)
        P = np.zeros((2, 3)); P[:, 0] = xh
        pairs = (np.array([0]), np.array([1]), np.array([1 if d <= 1 else 0], np.uint8))
        assert abs(oracle.loss_eq1_f64(P, pairs, 1.0, L=10.0) - want) < 1e-12


def test_tight_loss_reductions():
    """eps_q = 0 reduces L_tight to L; d_hat = b - 2 sqrt3 eps_q contributes 0;
    d_hat = b contributes (2 sqrt3 eps_q)^2."""
    rng = np.random.default_rng(2)
    for _ in range(50):
        d, dh = rng.uniform(0.9, 1.1, 2)
        P = np.zeros((2, 3)); P[1, 0] = dh
        pairs = (np.array([0]), np.array([1]), np.array([int(d <= 1.0)], np.uint8))
        assert abs(oracle.tight_f64(P, pairs, 1.0, 0.0, L=10.0) - oracle.loss_eq1_f64(P, pairs, 1.0, L=10.0)) < 1e-15
    eps_q = 1e-3
    mu = 2 * math.sqrt(3) * eps_q
    P = np.zeros((2, 3)); P[1, 0] = 1.0 - mu
    lk = (np.array([0]), np.array([1]), np.array([1], np.uint8))
    assert oracle.tight_f64(P, lk, 1.0, eps_q, L=10.0) == 0.0
    P[1, 0] = 1.0
    assert abs(oracle.tight_f64(P, lk, 1.0, eps_q, L=10.0) - mu * mu) < 1e-15


def test_gradient_matches_finite_differences_fp64():
    """SPEC acceptance 3: analytic grad of L_tight == central differences, rel < 1e-5,
    50 random configurations with active pairs of both kinds."""
    rng = np.random.default_rng(8)
    b, xi = 0.05, 2e-3
    eps_q = 2 * xi / (2 ** 16 - 1) * 50     # enlarge the margin so both terms are exercised
    done = 0
    while done < 50:
        n = 6
        P = rng.random((n, 3)) * 0.08 + 0.4
        ii, jj = np.triu_indices(n, 1)
        d = np.linalg.norm(P[ii] - P[jj], axis=1)
        flags = (rng.random(len(ii)) < 0.5).astype(np.uint8)
        pairs = (ii, jj, flags)
        f, g = oracle.tight_f64(P, pairs, b, eps_q, grad=True)
        mu = 2 * math.sqrt(3) * eps_q
        act_b = (flags == 1) & (d > b - mu)
        act_f = (flags == 0) & (d <= b + mu)
        # keep configurations away from activity switches (the loss is C1, FD needs smoothness)
        if not (act_b.any() and act_f.any()) or np.min(np.abs(d - (b - mu))) < 1e-4 or np.min(np.abs(d - (b + mu))) < 1e-4:
            continue
        h = 1e-6 * xi
        fd = np.zeros_like(P)
        for k in range(n):
            for q in range(3):
                Pp = P.copy(); Pp[k, q] += h
                Pm = P.copy(); Pm[k, q] -= h
                fd[k, q] = (oracle.tight_f64(Pp, pairs, b, eps_q) - oracle.tight_f64(Pm, pairs, b, eps_q)) / (2 * h)
        rel = np.linalg.norm(fd - g) / max(np.linalg.norm(g), 1e-300)
        assert rel < 1e-5, rel
        done += 1


def test_pinned_fp32_terms_match_fp64():
    """The fp32 pinned L_tight used by the PGD agrees with the fp64 Eq. (3) at generic points
    (same active set, loss and gradient to fp32 accuracy)."""
    w = synth.Workload("t", "clumped", 6000, 1.0, 1e-3, seed=21)
    x, y, z, xh, yh, zh = [t.numpy() for t in synth.make(w)]
    c = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi)
    th = oracle.thresholds(c)
    pairs = oracle.find_pairs(x, y, z, xh, yh, zh, c)
    act, loss32, g32 = oracle.tight_eval_f32(xh, yh, zh, pairs, c)
    P = np.stack([xh, yh, zh], 1).astype(np.float64)
    loss64, g64 = oracle.tight_f64(P, pairs, w.linking_length, th["eps_q"], grad=True)
    assert act > 100
    assert abs(loss32 - loss64) <= 1e-4 * loss64
    big = np.abs(g64) > 1e-3 * np.abs(g64).max()
    assert np.allclose(g32[big], g64[big], rtol=2e-3)


def test_gradient_directions():
    """a single broken pair along x is pulled together along x only; R15: a coincident
    active false pair is pushed apart along +-x (lower gid along +x after the descent step)."""
    c = oracle.cfg(L=1.0, b=0.125, xi=0.01)
    xh = np.array([0.25, 0.25 + 0.13], np.float32)
    h = np.full(2, 0.5, np.float32)
    pairs = (np.array([0]), np.array([1]), np.array([1], np.uint8))   # linked originally
    act, loss, g = oracle.tight_eval_f32(xh, h, h, pairs, c)
    assert act == 1 and g[0, 0] < 0 < g[1, 0] and np.all(g[:, 1:] == 0)
    xh = np.array([0.25, 0.25], np.float32)
    pairs = (np.array([0]), np.array([1]), np.array([0], np.uint8))   # unlinked originally
    act, loss, g = oracle.tight_eval_f32(xh, h, h, pairs, c)
    assert act == 1 and g[0, 0] < 0 < g[1, 0] and np.all(g[:, 1:] == 0)


def _bound_ok(x, xo, c):
    xi_f = np.float32(oracle.thresholds(c)["xi_f"])
    return np.all(np.abs(xo.astype(np.float64) - x.astype(np.float64)) <= np.float64(xi_f))


def test_adam_trajectory_matches_torch_adam():
    """P4: the oracle's fp32 Adam + projection follows torch.optim.Adam (fp64) on the same
    objective for a broken pair, to fp32 accuracy; first step is alpha*sign(g)."""
    b, xi, alpha = 0.1, 0.01, 1e-4
    x = np.array([0.40, 0.40 + 0.099], np.float32)
    xh = np.array([0.40 - 0.004, 0.40 + 0.099 + 0.004], np.float32)
    o = np.full(2, 0.5, np.float32)
    pairs = (np.array([0]), np.array([1]), np.array([1], np.uint8))
    th = oracle.thresholds(oracle.cfg(L=1.0, b=b, xi=xi))
    for T in (1, 2, 5, 12):
        c = oracle.cfg(L=1.0, b=b, xi=xi, alpha=alpha, t_max=T, stop_mode=oracle.STOP_NONE)
        xo, yo, zo, info = oracle.correct(x, o, o, xh, o, o, pairs, c)
        assert info["iterations"] == T
        p = torch.tensor(np.stack([xh, o, o], 1).astype(np.float64), requires_grad=True)
        opt = torch.optim.Adam([p], lr=alpha, betas=(0.9, 0.999), eps=1e-8)
        lo = torch.tensor(np.stack([x, o, o], 1).astype(np.float64)) - th["xip_f"]
        hi = lo + 2 * th["xip_f"]
        for _ in range(T):
            opt.zero_grad()
            _, g = oracle.tight_f64(p.detach().numpy(), pairs, b, th["eps_q"], grad=True)
            p.grad = torch.tensor(g)
            opt.step()
            with torch.no_grad():
                p.copy_(torch.minimum(torch.maximum(p, lo), hi))
        ref = p.detach().numpy()
        assert np.allclose(xo, ref[:, 0], atol=2e-7), (T, xo, ref[:, 0])
        if T == 1:
            assert np.allclose(xo - xh, [alpha, -alpha], rtol=1e-4)


def test_projection_clamps_exactly_and_never_exceeds_bound():
    """P5: a huge step lands exactly on the B(xi') face; |x' - x| <= xi' < xi_f holds exactly."""
    b, xi = 0.1, 1e-3
    x = np.array([0.40, 0.40 + 0.0995], np.float32)
    xh = np.array([0.40 - 0.0009, 0.40 + 0.0995 + 0.0009], np.float32)
    o = np.full(2, 0.5, np.float32)
    pairs = (np.array([0]), np.array([1]), np.array([1], np.uint8))
    c = oracle.cfg(L=1.0, b=b, xi=xi, alpha=1.0, t_max=1, stop_mode=oracle.STOP_NONE)
    th = oracle.thresholds(c)
    xo, _, _, _ = oracle.correct(x, o, o, xh, o, o, pairs, c)
    xip = np.float64(np.float32(th["xip_f"]))
    assert np.float64(xo[0]) - np.float64(x[0]) <= xip and np.float64(x[1]) - np.float64(xo[1]) <= xip
    assert xo[0] == np.float32(np.float64(x[0]) + xip) or np.float64(xo[0]) <= np.float64(x[0]) + xip
    # idempotence: a second projected step that is again clamped gives the same point
    c2 = oracle.cfg(L=1.0, b=b, xi=xi, alpha=1.0, t_max=2, stop_mode=oracle.STOP_NONE)
    xo2, _, _, _ = oracle.correct(x, o, o, xh, o, o, pairs, c2)
    assert np.array_equal(xo2, xo)
    assert _bound_ok(x, xo, c)


def test_zero_work_floor():
    """Alg. 1 early break (tab:iteration rows with 0 iterations): no active
    pair -> 0 iterations and output == input bit-exactly."""
    w = synth.Workload("t", "clumped", 4000, 1.0, 1e-3, seed=13)
    x, y, z, *_ = [t.numpy() for t in synth.make(w)]
    c = oracle.cfg(L=1.0, b=w.linking_length, xi=1e-6)
    pairs = oracle.find_pairs(x, y, z, x, y, z, c)
    keep = np.ones(len(pairs[0]), bool)
    # drop pairs inside the +-mu margin of b (they are active even when uncompressed)
    th = oracle.thresholds(c)
    P = np.stack([x, y, z], 1).astype(np.float64)
    d = P[pairs[1]] - P[pairs[0]]; d -= np.round(d); d = np.sqrt((d * d).sum(1))
    keep = np.abs(d - w.linking_length) > 10 * th["mu"]
    pairs = tuple(a[keep] for a in pairs)
    xo, yo, zo, info = oracle.correct(x, y, z, x, y, z, pairs, c)
    assert info["iterations"] == 0 and info["converged"]
    assert np.array_equal(xo, x) and np.array_equal(yo, y) and np.array_equal(zo, z)
    e = np.zeros(0, np.float32)
    _, _, _, info = oracle.correct(e, e, e, e, e, e, (np.zeros(0, np.int64),) * 2 + (np.zeros(0, np.uint8),), c)
    assert info["iterations"] == 0 and info["converged"]


def test_input_bound_violation_is_rejected():
    """the decompressed input must satisfy |x_hat - x| <= xi (status 66)."""
    c = oracle.cfg(L=1.0, b=0.1, xi=1e-3)
    x = np.array([0.5], np.float32)
    xh = np.array([0.5 + 2e-3], np.float32)
    with pytest.raises(RuntimeError, match="66"):
        oracle.correct(x, x, x, xh, x, x, (np.zeros(0, np.int64),) * 2 + (np.zeros(0, np.uint8),), c)


@pytest.mark.parametrize("xi_rel,dither", [(1e-3, True), (1e-4, True), (1e-3, False)])
def test_convergence_restores_clusters(xi_rel, dither):
    """P:15, P:138 / SPEC acceptance 4: run to convergence -> MCC over V = 1, FoF labels of the
    corrected data equal the original's, |x' - x| <= xi_f everywhere, non-editable untouched,
    and the iteration count respects the budget of §III-E in eps_L mode."""
    w = synth.Workload("t", "clumped", 12000, 1.0, xi_rel, seed=31)
    x, y, z, xh, yh, zh = [t.numpy() for t in synth.make(w, dither=dither)]
    c = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi)
    r = oracle.pipeline(x, y, z, xh, yh, zh, c)
    assert r.info["converged"] and r.info["active_final"] == 0
    tp, tn, fp, fn = r.mcc_after
    assert fp == 0 and fn == 0 and oracle.mcc(*r.mcc_after) == 1.0
    assert np.array_equal(r.labels_orig, r.labels_corr)
    for a, o in ((x, r.xo), (y, r.yo), (z, r.zo)):
        assert _bound_ok(a, o, c)
    ed = np.zeros(len(x), bool); ed[r.pairs[0]] = True; ed[r.pairs[1]] = True
    assert np.array_equal(r.xo[~ed], xh[~ed]) and np.array_equal(r.zo[~ed], zh[~ed])
    assert np.array_equal(oracle.halo_catalog(r.labels_orig), oracle.halo_catalog(r.labels_corr))
    ce = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi, stop_mode=oracle.STOP_EPS, eps_loss=1e-10)
    _, _, _, info = oracle.correct(x, y, z, xh, yh, zh, r.pairs, ce)
    assert info["iterations"] <= oracle.iteration_budget(oracle.thresholds(c)["xi"], info["active0"], 1e-10)
    # the bench's stop (Alg. 1 eps_L test + every link status restored): MCC = 1 at the stop
    cr = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi, stop_mode=oracle.STOP_RESTORED, eps_loss=1e-10)
    xr, yr, zr, ir = oracle.correct(x, y, z, xh, yh, zh, r.pairs, cr)
    assert ir["converged"] and ir["violated_final"] == 0 and ir["loss_final"] <= 1e-10
    assert ir["iterations"] <= r.info["iterations"]
    ol = (r.pairs[2] & 1).astype(bool)
    assert oracle.mcc(*oracle.mcc_counts(ol, oracle.pair_links(r.pairs[0], r.pairs[1], xr, yr, zr, cr))) == 1.0


def test_vanilla_pgd_monotone():
    """§III-B convergence analysis: vanilla PGD with step <= 1/Lip is monotone in
    L_tight; Lip <= 4 * max degree for sums of (|r|-c)^2 terms."""
    w = synth.Workload("t", "clumped", 6000, 1.0, 1e-3, seed=41)
    x, y, z, xh, yh, zh = [t.numpy() for t in synth.make(w)]
    c0 = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi)
    pairs = oracle.find_pairs(x, y, z, xh, yh, zh, c0)
    deg = np.bincount(np.concatenate([pairs[0], pairs[1]]), minlength=len(x)).max()
    step = 1.0 / (4.0 * deg)
    c = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi, optimizer=1, vanilla_step=step, t_max=60,
                   stop_mode=oracle.STOP_NONE)
    _, _, _, info, (ta, tl, tv) = oracle.correct(x, y, z, xh, yh, zh, pairs, c, trace=True)
    assert tl[-1] < tl[0]
    assert np.all(np.diff(tl) <= 1e-7 * tl[0]), np.diff(tl).max()


def test_adam_keeps_moving_after_zero_gradient_and_stop_is_exact():
    """R11: the loop stops at the first iteration whose state has no active pair; running
    exactly that many updates with stop disabled gives the same positions bit-exactly, one
    more update (Adam momentum, zero gradient) moves them."""
    w = synth.Workload("t", "clumped", 5000, 1.0, 1e-3, seed=51)
    x, y, z, xh, yh, zh = [t.numpy() for t in synth.make(w)]
    c = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi)
    pairs = oracle.find_pairs(x, y, z, xh, yh, zh, c)
    xo, yo, zo, info = oracle.correct(x, y, z, xh, yh, zh, pairs, c)
    T = info["iterations"]
    assert T > 0 and info["converged"]
    cn = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi, t_max=T, stop_mode=oracle.STOP_NONE)
    xn, yn, zn, _ = oracle.correct(x, y, z, xh, yh, zh, pairs, cn)
    assert np.array_equal(xn, xo) and np.array_equal(yn, yo) and np.array_equal(zn, zo)
    cn1 = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi, t_max=T + 1, stop_mode=oracle.STOP_NONE)
    xn1, _, _, _ = oracle.correct(x, y, z, xh, yh, zh, pairs, cn1)
    assert not np.array_equal(xn1, xo)
