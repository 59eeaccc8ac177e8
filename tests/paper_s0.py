"""S0 written out from the paper in exact arithmetic, for the pins (test-side only).

Neither the oracle (oracle/cc_oracle.c) nor the CUDA path (csrc/api.cu) is used here: every
threshold is the paper's formula evaluated with 60-digit decimals and rounded ONCE to the
nearest fp32 (ties to even) with exact rational arithmetic, so a dropped factor, a wrong
constant or a double rounding in either implementation shows up as a mismatch.

  Alg. 1 l.1   eps_q = 2 xi / (2^m - 1)
  Alg. 1 l.2   xi'   = xi (1 - 2^-m)                      -> RD32 (R8)
  Alg. 1 l.3   band  (b - 2 sqrt3 xi, b + 2 sqrt3 xi]     -> lo2, hi2 = fl32(edge^2) (R2)
  P:362                link  d <= b                               -> b2 = fl32(b^2) (R3)
  Eq. 3    c_b = b - 2 sqrt3 eps_q, c_f = b + 2 sqrt3 eps_q -> fl32 (R13)
  R6                   xi_f = fl32(xi) is the bound everything derives from
"""
from __future__ import annotations

from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np

getcontext().prec = 60
SQRT3 = Fraction(Decimal(3).sqrt())     # 60 significant digits: far beyond fp32's 24 bits


def _f32_floor(q: Fraction) -> np.float32:
    f = np.float32(float(q))
    while Fraction(float(f)) > q:
        f = np.nextafter(f, np.float32(-np.inf))
    while Fraction(float(np.nextafter(f, np.float32(np.inf)))) <= q:
        f = np.nextafter(f, np.float32(np.inf))
    return f


def fl32(q: Fraction) -> np.float32:
    """Round an exact rational to the nearest fp32, ties to even (one rounding)."""
    lo = _f32_floor(q)
    if Fraction(float(lo)) == q:
        return lo
    hi = np.nextafter(lo, np.float32(np.inf))
    dl, dh = q - Fraction(float(lo)), Fraction(float(hi)) - q
    if dl < dh:
        return lo
    if dh < dl:
        return hi
    return lo if (int(lo.view(np.uint32)) & 1) == 0 else hi


def rd32(q: Fraction) -> np.float32:
    return _f32_floor(q)


def thresholds(b: float, xi: float, m: int = 16, L: float = 1.0) -> dict:
    """S0 from the paper's formulas; b, xi, L are the double parameters as given."""
    xi_f = np.float32(xi)
    X = Fraction(float(xi_f))
    B = Fraction(b)
    eps_q = 2 * X / (2 ** m - 1)
    mu = 2 * SQRT3 * eps_q
    lo = B - 2 * SQRT3 * X
    hi = B + 2 * SQRT3 * X
    return {
        "xi_f": xi_f,
        "xip_f": rd32(X * (1 - Fraction(1, 2 ** m))),
        "eps_q": eps_q,
        "mu": mu,
        "c_b": fl32(B - mu),
        "c_f": fl32(B + mu),
        "lo2": fl32(lo * lo) if lo > 0 else np.float32(-1.0),
        "hi2": fl32(hi * hi),
        "b2": fl32(B * B),
        "band_lo": lo,
        "band_hi": hi,
        "Lf": np.float32(L),
        "hLf": fl32(Fraction(L) / 2),
    }
