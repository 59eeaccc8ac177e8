"""Hand-built adversarial inputs for the boundary parity tests (tests/test_gpu_edges.py).

Inputs only: every expected value comes from the oracle.  The pinned fp32 distance of DESIGN.md
R4 is retyped here in numpy solely to SELECT geometries where fp32 rounding decides a link."""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from tests import paper_s0

F32 = np.float32


def d2_pinned(p, q, L, periodic=True):
    Lf, hL = F32(L), paper_s0.fl32(Fraction(L) / 2)
    s = F32(0)
    for a in range(3):
        d = F32(q[a] - p[a])
        if periodic:
            if d > hL:
                d = F32(d - Lf)
            elif d < -hL:
                d = F32(d + Lf)
        s = F32(s + F32(d * d)) if a else F32(d * d)
    return s


def _toward(v, x, xi_f):
    """fp32 v moved one ulp at a time toward x until |v - x| <= xi_f (the input contract)."""
    while abs(float(v) - float(x)) > float(xi_f):
        v = np.nextafter(v, x)
    return v


def displaced(p, sgn, xi_f, L=None):
    """p + sgn * xi_f per coordinate, rounded to fp32 and kept inside the bound."""
    out = np.empty(3, F32)
    for a in range(3):
        v = F32(float(p[a]) + sgn[a] * float(xi_f))
        out[a] = _toward(v, p[a], xi_f)
    return out


def isolated_pairs(kind, b, xi, L, n_want, rng, wrap=False, tries=400000):
    """Pairs of particles (orig p, q; decompressed ph, qh) that are NOT vulnerable and whose link
    is nevertheless flipped by fp32 rounding under a diagonal +-xi_f displacement:
      kind 'lo': original d2 <= lo2 (linked; stable in exact arithmetic), decompressed moved
                 apart along the diagonal -> pinned d_hat2 > b2 (broken)
      kind 'hi': original d2 > hi2 (unlinked), moved together -> d_hat2 <= b2 (linked)
    wrap: the pair straddles the periodic x face (the minimum image rounds at ulp(L))."""
    e = paper_s0.thresholds(b, xi, 16, L)
    xi_f = e["xi_f"]
    D0 = float(e["band_lo"] if kind == "lo" else e["band_hi"])
    found = []
    for _ in range(tries):
        if len(found) >= n_want:
            break
        sgn = rng.choice([-1.0, 1.0], 3)
        u = sgn / np.sqrt(3.0)
        D = D0 * (1 + (rng.integers(-3, 4) * 2.0 ** -24 if not wrap else rng.uniform(-3e-4, 3e-4)))
        if wrap:
            c = np.array([rng.uniform(0, 0.5 * D), rng.uniform(0.3, 0.7), rng.uniform(0.3, 0.7)])
            if u[0] > 0:
                u = -u
                sgn = -sgn
        else:
            c = rng.uniform(0.3, 0.7, 3) * L
        p = c.astype(F32)
        q = (c + D * u)
        q[0] = q[0] % L
        q = q.astype(F32)
        if q[0] >= F32(L):
            continue
        d2 = d2_pinned(p, q, L)
        if kind == "lo" and not (d2 <= e["lo2"]):
            continue
        if kind == "hi" and not (d2 > e["hi2"]):
            continue
        move = -1.0 if kind == "lo" else 1.0   # lo: apart (p against u), hi: together
        ph = displaced(p, move * sgn, xi_f)
        qh = displaced(q, -move * sgn, xi_f)
        dh2 = d2_pinned(ph, qh, L)
        if (kind == "lo" and dh2 > e["b2"]) or (kind == "hi" and dh2 <= e["b2"]):
            found.append((p, q, ph, qh))
    return found


def place_pairs(pairs, L, rng, n_background=0, b=None, xi=None):
    """Arrays (x, y, z, xh, yh, zh) holding the given pairs plus background particles far away
    (x in the middle third, no two background particles within 3 b + 4 xi)."""
    P, H = [], []
    for p, q, ph, qh in pairs:
        P += [p, q]
        H += [ph, qh]
    P = np.array(P, F32).reshape(-1, 3)
    H = np.array(H, F32).reshape(-1, 3)
    return tuple(P[:, a].copy() for a in range(3)) + tuple(H[:, a].copy() for a in range(3))
