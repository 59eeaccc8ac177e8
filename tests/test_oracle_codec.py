"""Pins for the oracle's edit log: compaction, m-bit quantisation and
reconstruction -- Alg. 1 lines 11-13, §III-B P:446-448 ("Compaction,
quantization, and lossless compression"), P:456 ("Reconstruction"); readings R29-R31
(DESIGN.md §3).

Pinned against: the hand-built bit layout of SPEC's worked example, lattice points and
half-way cases of the quantiser worked by hand, exact rational arithmetic (fractions) for the
quantisation error bound s/2 = xi 2^-m = xi - xi', numpy's own bit unpacking for the
flag mask, and the paper's end-to-end claim that quantisation re-introduces no violation
 on a converged oracle correction, with |x_rec - x| <= xi_f (Eq. 2).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


def _cfg(xi=1e-3, m=16, L=1.0):
    return oracle.cfg(L=L, b=0.01, xi=xi, m=m)


def test_worked_bit_layout():
    """edits at coordinates k=0 and k=5 -> flags byte0 = 0b00100001, values in
    ascending k.  k = 3i + a (R29): k=0 is x of particle 0, k=5 is z of particle 1."""
    c = _cfg()
    s = oracle.edit_step(c)
    h = [np.full(3, 0.25, np.float32) for _ in range(3)]
    p = [a.copy() for a in h]
    p[0][0] = np.float32(0.25 + 3 * s)     # k = 0, q = +3
    p[2][1] = np.float32(0.25 - 7 * s)     # k = 5, q = -7
    flags, q = oracle.edit_encode(*p, *h, *p, c)
    assert flags.tolist() == [0b00100001, 0]          # ceil(9/8) = 2 bytes
    assert q.tolist() == [3, -7]
    r = oracle.edit_decode(*h, flags, q, c)
    for a in range(3):
        assert np.array_equal(r[a], p[a])


def test_empty_and_zero():
    c = _cfg()
    h = [np.arange(5, dtype=np.float32) / 7 for _ in range(3)]
    flags, q = oracle.edit_encode(*h, *h, *h, c)
    assert flags.tolist() == [0, 0] and q.size == 0
    r = oracle.edit_decode(*h, flags, q, c)
    assert all(np.array_equal(r[a], h[a]) for a in range(3))
    f0, q0 = oracle.edit_encode(*[np.zeros(0, np.float32)] * 9, c)
    assert f0.size == 0 and q0.size == 0


def test_lattice_and_half_even():
    """s = xi_f 2^(1-m) (R30); lattice points map to their index, half-way values round to
    even (IEEE rint), with xi = 2^-10 so that k s is exact: 0.5s -> 0, 1.5s -> 2, 2.5s -> 2, -0.5s -> 0, -1.5s -> -2."""
    for m in (8, 16):
        c = _cfg(xi=2.0 ** -10, m=m)          # power-of-2 xi: every k s below is an fp32
        s = oracle.edit_step(c)
        assert s == 2.0 ** (-9 - m)
        ks = [1, -1, 5, 2 ** m, -(2 ** m), 0.5, 1.5, 2.5, -0.5, -1.5]
        want = [1, -1, 5, 2 ** m, -(2 ** m), 0, 2, 2, 0, -2]
        h = [np.zeros(len(ks), np.float32) for _ in range(3)]
        p = [np.zeros(len(ks), np.float32) for _ in range(3)]
        p[1][:] = np.array([k * s for k in ks], np.float32)     # exact in fp32 (power-of-2 scale)
        assert all(Fraction(float(v)) == Fraction(k) * Fraction(s) for v, k in zip(p[1], ks))
        flags, q = oracle.edit_encode(*p, *h, *p, c)
        assert q.tolist() == want


def test_quantisation_error_bound_exact():
    """|q s - Delta| <= s/2 = xi_f 2^-m in exact rational arithmetic, on 20k random
    edits spanning [-2 xi, 2 xi] at several magnitudes of the base coordinate."""
    rng = np.random.default_rng(7)
    for m, L in ((16, 1.0), (8, 1.0), (16, 256.0), (32, 1.0)):
        xi = 1e-3 * L
        c = _cfg(xi=xi, m=m, L=L)
        s = Fraction(oracle.edit_step(c))
        xi_f = float(np.float32(xi))
        n = 20000
        h = [rng.uniform(0, L, n).astype(np.float32) for _ in range(3)]
        p = [(a.astype(np.float64) + rng.uniform(-2 * xi_f, 2 * xi_f, n)).astype(np.float32) for a in h]
        for a in range(3):                   # keep |Delta| <= 2 xi_f after fp32 rounding
            d = p[a].astype(np.float64) - h[a]
            bad = np.abs(d) > 2 * xi_f
            p[a][bad] = h[a][bad]
        flags, q = oracle.edit_encode(*p, *h, *p, c)
        bits = np.unpackbits(flags, bitorder="little")[: 3 * n].reshape(n, 3)
        want_bits = np.stack([p[a] != h[a] for a in range(3)], 1)
        assert np.array_equal(bits.astype(bool), want_bits)
        deltas = np.stack([p[a].astype(np.float64) - h[a].astype(np.float64) for a in range(3)], 1)[want_bits]
        assert q.size == deltas.size == int(bits.sum())
        for k in range(0, q.size, 37):
            err = abs(Fraction(int(q[k])) * s - Fraction(float(deltas[k])))
            assert err <= s / 2
        assert np.abs(q).max() <= 2 ** (m + 1)
        r = oracle.edit_decode(*h, flags, q, c)
        for a in range(3):
            if L == 256.0:
                # xi = 0.256: s = 0.256 * 2^-15 = 7.8e-6 < ulp(x) = 2^-16 for x > 128, so the
                # reconstruction is the corrected fp32 value itself wherever ulp exceeds s
                big = np.abs(p[a]) > 128.0
                assert np.array_equal(r[a][big], p[a][big])
            # the rounded sum stays within s/2 + half an ulp of the corrected value
            tol = float(s) / 2 + np.spacing(np.abs(p[a])).astype(np.float64) / 2
            assert np.all(np.abs(r[a].astype(np.float64) - p[a]) <= tol)


def test_bound_violation_rejected():
    c = _cfg()
    h = [np.zeros(2, np.float32) for _ in range(3)]
    p = [a.copy() for a in h]
    p[0][1] = np.float32(2.01e-3)
    with pytest.raises(ValueError, match="66"):
        oracle.edit_encode(*h, *h, *p, c)


@pytest.mark.parametrize("xi_rel", [1e-3, 1e-4])
def test_no_violation_reintroduced(xi_rel):
    """"zero violations are re-introduced by quantization"; the quantised
    reconstruction still satisfies the box constraint of Eq. 2.  On a converged oracle
    correction (R11 stop): every vulnerable pair's original link status holds on x_rec, FoF
    labels of x_rec equal the original's, |x_rec - x| <= xi_f, non-flagged coordinates are the
    decompressed ones bit for bit."""
    w = synth.Workload("t", "clumped", 8000, 1.0, xi_rel, seed=41)
    x, y, z, xh, yh, zh = [t.numpy() for t in synth.make(w)]
    c = oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi)
    r = oracle.pipeline(x, y, z, xh, yh, zh, c)
    assert r.info["converged"]
    flags, q = oracle.edit_encode(x, y, z, xh, yh, zh, r.xo, r.yo, r.zo, c)
    xr, yr, zr = oracle.edit_decode(xh, yh, zh, flags, q, c)
    ol = (r.pairs[2] & 1).astype(bool)
    assert np.array_equal(oracle.pair_links(r.pairs[0], r.pairs[1], xr, yr, zr, c), ol)
    lr, _ = oracle.fof(xr, yr, zr, c)
    assert np.array_equal(lr, r.labels_orig)
    xi_f = float(np.float32(w.xi))
    for a, o in ((x, xr), (y, yr), (z, zr)):
        assert np.all(np.abs(o.astype(np.float64) - a) <= xi_f)
    bits = np.unpackbits(flags, bitorder="little")[: 3 * len(x)].reshape(-1, 3).astype(bool)
    for k, (o, h) in enumerate(((xr, xh), (yr, yh), (zr, zh))):
        assert np.array_equal(o[~bits[:, k]], h[~bits[:, k]])
    # at most 3|E| edits
    ed = np.zeros(len(x), bool); ed[r.pairs[0]] = True; ed[r.pairs[1]] = True
    assert q.size <= 3 * int(ed.sum())


def test_bound_safe_index_near_origin():
    """R32: where ulp(x) < s the fp32 rounding of x_hat0 + q s can leave the box by up to half an
    ulp when the correction sits on the projection box (xi' + s/2 = xi).  Brute force over
    box-saturated corrections near the origin: every reconstruction lies within xi_f of the
    original (exact fp64 test of fp32 values), each index is within one lattice step of the
    nearest one (exact rationals), and the plain nearest index would have failed on some."""
    rng = np.random.default_rng(11)
    n, xi = 20000, 1e-3
    c = _cfg(xi=xi)
    s = Fraction(oracle.edit_step(c))
    th = oracle.thresholds(c)
    xi_f, xip = th["xi_f"], th["xip_f"]
    x = rng.uniform(0.0, 0.3, n).astype(np.float32)
    sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    h = (x.astype(np.float64) - sign * rng.uniform(0, xi_f, n)).astype(np.float32)
    p = (x.astype(np.float64) + sign * float(xip)).astype(np.float32)     # on the B(xi') box
    ok = np.abs(p.astype(np.float64) - x) <= float(xip)
    ok &= np.abs(h.astype(np.float64) - x) <= xi_f
    x, h, p = x[ok], h[ok], p[ok]
    z = np.zeros_like(x)
    flags, q = oracle.edit_encode(x, z, z, h, z, z, p, z, z, c)
    assert q.size == int((p != h).sum())
    xr, _, _ = oracle.edit_decode(h, z, z, flags, q, c)
    assert np.all(np.abs(xr.astype(np.float64) - x) <= xi_f)
    moved = np.nonzero(p != h)[0]
    plain_bad = 0
    for k, i in enumerate(moved):
        d = Fraction(float(p[i])) - Fraction(float(h[i]))
        q0 = round(d / s)                                   # nearest lattice index (half even)
        assert abs(int(q[k]) - q0) <= 1
        r0 = np.float32(float(Fraction(float(h[i])) + q0 * s))
        plain_bad += abs(Fraction(float(r0)) - Fraction(float(x[i]))) > Fraction(xi_f)
    assert plain_bad > 0


# --------------------------------------------------------------------------------------------
# m-bit packing of the edits (Alg. 1 l.13; reading R33: (m+2)-bit two's-complement fields,
# LSB first in 32-bit words)
def test_edit_pack_worked_layout():
    """Hand-derived: m = 2 -> 4-bit fields; q = 1,-1,3,-4,0,2,-2,4 -> nibbles 1,F,3,C,0,2,E,4 from
    the least significant end: one word 0x4E20C3F1.  m = 8 -> 10-bit fields straddle words:
    q = 255 (0x0FF), -1 (0x3FF), -256 (0x300), 7 -> bits 0..9, 10..19, 20..29, 30..39."""
    w = oracle.edit_pack(np.array([1, -1, 3, -4, 0, 2, -2, 4]), 2)
    assert w.tolist() == [0x4E20C3F1]
    w = oracle.edit_pack(np.array([255, -1, -256, 7]), 8)
    want = 0x0FF | (0x3FF << 10) | (0x300 << 20) | (7 << 30)
    assert w.tolist() == [want & 0xFFFFFFFF, want >> 32]
    assert oracle.edit_unpack(w, 4, 8).tolist() == [255, -1, -256, 7]


@pytest.mark.parametrize("m", [2, 8, 16, 24, 32, 40])
def test_edit_pack_round_trip_and_size(m):
    rng = np.random.default_rng(m)
    lim = 2 ** m
    q = rng.integers(-lim, lim + 1, 997)
    q[:4] = [-lim, lim, 0, -1]
    w = oracle.edit_pack(q, m)
    assert w.size == (q.size * (m + 2) + 31) // 32          # (m+2)/8 bytes per edit
    assert np.array_equal(oracle.edit_unpack(w, q.size, m), q)
    assert oracle.edit_pack(np.zeros(0, np.int64), m).size == 0


def test_edit_pack_rejects_out_of_range():
    with pytest.raises(ValueError):
        oracle.edit_pack(np.array([2 ** 8 + 1]), 8)
