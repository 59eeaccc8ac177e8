"""Pins for the oracle's vulnerable-pair search (O1/O2) against things other than itself:
brute force O(N^2), scipy's cKDTree in fp64, hand-built fp32 threshold cases, SPEC worked
examples, band nesting and permutation invariance.

Definition under test (§III-A; Alg. 1 line 3 P:421): (i,j) is vulnerable iff
its original distance lies in (b - 2 sqrt3 xi, b + 2 sqrt3 xi]; evaluated as lo2 < d2 <= hi2 on
the pinned fp32 squared distance (R2, R4).
"""
import numpy as np
import pytest
from scipy.spatial import cKDTree

import oracle
import synth


def _rand_instance(rng, n, L=1.0, clustered=False):
    if clustered:
        k = max(1, n // 100)
        c = rng.random((k, 3)) * L
        p = c[rng.integers(0, k, n)] + rng.normal(0, 0.02 * L, (n, 3))
        p = np.mod(p, L)
    else:
        p = rng.random((n, 3)) * L
    p = p.astype(np.float32)
    p = np.where(p >= L, np.nextafter(np.float32(L), np.float32(0)), p)
    return p[:, 0].copy(), p[:, 1].copy(), p[:, 2].copy()


def _np_d2(a, b, L):
    """fp32 squared min-image distance written independently with numpy float32 (no FMA)."""
    Lf, hL = np.float32(L), np.float32(L / 2)
    d = (b - a).astype(np.float32)
    d = np.where(d > hL, d - Lf, np.where(d < -hL, d + Lf, d)).astype(np.float32)
    s = (d[..., 0] * d[..., 0]).astype(np.float32)
    s = (s + (d[..., 1] * d[..., 1]).astype(np.float32)).astype(np.float32)
    s = (s + (d[..., 2] * d[..., 2]).astype(np.float32)).astype(np.float32)
    return s


def _pairset(p):
    pi, pj, pf = p
    return {(int(a), int(b)): int(f) for a, b, f in zip(pi, pj, pf)}


def test_grid_equals_brute_force_100_instances():
    """SPEC acceptance 1: grid search == brute force exactly (pairs + both link bits)."""
    rng = np.random.default_rng(123)
    for k in range(100):
        n = int(rng.integers(0, 1500))
        x, y, z = _rand_instance(rng, n, clustered=bool(k % 2))
        xi = 10 ** rng.uniform(-6, -2)
        b = 10 ** rng.uniform(-2.3, -1.2)
        noise = [(a + rng.uniform(-xi, xi, n)).astype(np.float32) for a in (x, y, z)]
        c = oracle.cfg(L=1.0, b=b, xi=xi)
        g = oracle.find_pairs(x, y, z, *noise, c)
        bf = oracle.find_pairs(x, y, z, *noise, c, brute=True)
        assert _pairset(g) == _pairset(bf), f"instance {k}: n={n} b={b} xi={xi}"


def test_pairs_match_scipy_ckdtree_fp64():
    """Independent library: periodic cKDTree(boxsize) enumerates all pairs within the band's
    outer radius in fp64; away from the fp32 rounding of the thresholds the sets agree."""
    rng = np.random.default_rng(7)
    for k in range(6):
        n = 3000
        x, y, z = _rand_instance(rng, n, clustered=bool(k % 2))
        b, xi = 0.04, [1e-4, 1e-3, 4e-3][k % 3]
        c = oracle.cfg(L=1.0, b=b, xi=xi)
        th = oracle.thresholds(c)
        lo, hi = th["band_lo"], th["band_hi"]
        P = np.stack([x, y, z], 1).astype(np.float64)
        tree = cKDTree(P, boxsize=1.0)
        cand = tree.query_pairs(hi * (1 + 1e-4), output_type="ndarray")
        d = P[cand[:, 1]] - P[cand[:, 0]]
        d = d - np.round(d)
        r = np.sqrt((d * d).sum(1))
        near = lambda v, t: np.abs(v - t) <= 1e-5 * t
        amb = near(r, hi) | near(r, max(lo, 1e-30)) | near(r, b)
        want = {(int(a), int(bb)) for (a, bb), rr, am in zip(cand, r, amb) if (lo < rr <= hi) and not am}
        ambig = {(int(a), int(bb)) for (a, bb), am in zip(cand, amb) if am}
        got = oracle.find_pairs(x, y, z, x, y, z, c)
        got_set = {(int(a), int(bb)) for a, bb in zip(got[0], got[1])}
        assert got_set - ambig == want
        # original-link bit agrees with fp64 d <= b away from b
        rmap = {(int(a), int(bb)): rr for (a, bb), rr in zip(cand, r)}
        for a, bb, f in zip(*got):
            rr = rmap[(int(a), int(bb))]
            if not near(rr, b):
                assert bool(f & 1) == (rr <= b)
            assert bool(f & 1) == bool(f & 2)       # decompressed == original here


def _boundary_pair(T, L=1.0, x0=0.25):
    """fp32 coordinates (x0, x1) on the x axis whose pinned fp32 d2 is the largest value <= T
    and the smallest value > T (found by walking representable x1)."""
    x0 = np.float32(x0)
    x1 = np.float32(x0 + np.float32(np.sqrt(T)))
    d2 = lambda a: np.float32(np.float32(a - x0) * np.float32(a - x0))
    while d2(x1) > T:
        x1 = np.nextafter(x1, np.float32(-1))
    below = x1
    while d2(x1) <= T:
        x1 = np.nextafter(x1, np.float32(2))
    above = x1
    return x0, below, above, d2(below), d2(above)


@pytest.mark.parametrize("xi", [1e-4, 1e-3])
def test_fp32_threshold_boundaries(xi):
    """Half-open band (R2) and link at equality (R3) at the exact fp32 thresholds."""
    b = 0.05
    c = oracle.cfg(L=1.0, b=b, xi=xi)
    th = oracle.thresholds(c)
    for name in ("lo2", "hi2", "b2"):
        T = np.float32(th[name])
        x0, below, above, d_below, d_above = _boundary_pair(T)
        assert d_below <= T < d_above
        for x1, d2v in ((below, d_below), (above, d_above)):
            xs = np.array([x0, x1], np.float32)
            zs = np.array([0.5, 0.5], np.float32)
            pi, pj, pf = oracle.find_pairs(xs, zs, zs, xs, zs, zs, c)
            in_band = (np.float32(th["lo2"]) < d2v) and (d2v <= np.float32(th["hi2"]))
            assert len(pi) == int(in_band), (name, float(d2v))
            if in_band:
                assert bool(pf[0] & 1) == bool(d2v <= np.float32(th["b2"]))
            assert oracle.dist2([x0, .5, .5], [x1, .5, .5], c) == d2v


def test_spec_worked_examples():
    """d = b -> one linked pair; d = b - 2 sqrt3 xi -> none; three collinear
    particles b apart -> (0,1),(1,2) only; N = 0 and N = 1 -> empty."""
    b = 0.125                              # exactly representable; 0.25 -> 0.375 exact in fp32
    c = oracle.cfg(L=1.0, b=b, xi=1e-3)
    xs = np.array([0.25, 0.375], np.float32); h = np.array([0.5, 0.5], np.float32)
    pi, pj, pf = oracle.find_pairs(xs, h, h, xs, h, h, c)
    assert list(zip(pi, pj)) == [(0, 1)] and pf[0] & 1
    th = oracle.thresholds(c)
    x0, below, above, d_below, _ = _boundary_pair(np.float32(th["lo2"]))
    xs = np.array([x0, below], np.float32)
    assert len(oracle.find_pairs(xs, h, h, xs, h, h, c)[0]) == 0
    xs = np.array([0.25, 0.375, 0.5], np.float32); h3 = np.full(3, 0.5, np.float32)
    pi, pj, pf = oracle.find_pairs(xs, h3, h3, xs, h3, h3, c)
    assert list(zip(pi.tolist(), pj.tolist())) == [(0, 1), (1, 2)]
    e = np.zeros(0, np.float32)
    assert len(oracle.find_pairs(e, e, e, e, e, e, c)[0]) == 0
    o = np.array([0.3], np.float32)
    assert len(oracle.find_pairs(o, o, o, o, o, o, c)[0]) == 0


def test_periodic_minimum_image_pairs():
    """A pair straddling the periodic face is found through the minimum image."""
    b = 0.125
    c = oracle.cfg(L=1.0, b=b, xi=1e-3)
    xs = np.array([0.0625, 0.9375], np.float32)   # min-image distance 0.125 = b
    h = np.array([0.5, 0.5], np.float32)
    pi, pj, pf = oracle.find_pairs(xs, h, h, xs, h, h, c)
    assert len(pi) == 1 and pf[0] & 1
    cn = oracle.cfg(L=1.0, b=b, xi=1e-3, periodic=False)
    assert len(oracle.find_pairs(xs, h, h, xs, h, h, cn)[0]) == 0


def test_band_nesting_and_permutation_invariance():
    """SPEC S:138 (V(xi1) subset of V(xi2) for xi1 < xi2) and S:141 (relabelling)."""
    x, y, z, *_ = [t.numpy() for t in synth.make(synth.Workload("t", "clumped", 3000, 1.0, 1e-3, seed=9))]
    b = oracle.linking_length(0.2, 1.0, 3000)
    prev = set()
    for xi in (1e-5, 1e-4, 1e-3, 5e-3):
        c = oracle.cfg(L=1.0, b=b, xi=xi)
        s = set(zip(*oracle.find_pairs(x, y, z, x, y, z, c)[:2]))
        assert prev <= s
        prev = s
    rng = np.random.default_rng(3)
    perm = rng.permutation(3000)
    gid = np.arange(3000, dtype=np.uint32)
    c = oracle.cfg(L=1.0, b=b, xi=1e-3)
    a = oracle.find_pairs(x, y, z, x, y, z, c, gid=gid)
    p = oracle.find_pairs(x[perm], y[perm], z[perm], x[perm], y[perm], z[perm], c, gid=gid[perm])
    ga = sorted((int(gid[i]), int(gid[j])) for i, j in zip(a[0], a[1]))
    gp = sorted((int(gid[perm][i]), int(gid[perm][j])) for i, j in zip(p[0], p[1]))
    assert ga == gp


def test_decompressed_link_bit_and_zero_error():
    """P2: dec-link bit is d2(p_hat) <= b2; with p_hat = p no pair is violated."""
    rng = np.random.default_rng(11)
    x, y, z = _rand_instance(rng, 2000)
    c = oracle.cfg(L=1.0, b=0.03, xi=1e-3)
    pi, pj, pf = oracle.find_pairs(x, y, z, x, y, z, c)
    assert np.all((pf & 1) == ((pf >> 1) & 1))
    xh = (x + np.float32(5e-4)).astype(np.float32)
    pi, pj, pf = oracle.find_pairs(x, y, z, xh, y, z, c)
    P = np.stack([xh, y, z], 1)
    d2 = _np_d2(P[pi], P[pj], 1.0)
    assert np.array_equal(((pf >> 1) & 1).astype(bool), d2 <= np.float32(oracle.thresholds(c)["b2"]))
