"""Pins for S0 (Alg. 1 lines 1-3; §III-B) and for the synthetic input
generators (shape checks of SURVEY.md §8(d), BASELINE.json configs)."""
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import synth


def _largest_f32_le(q: Fraction) -> np.float32:
    f = np.float32(float(q))
    while Fraction(float(f)) > q:
        f = np.nextafter(f, np.float32(-np.inf))
    while Fraction(float(np.nextafter(f, np.float32(np.inf)))) <= q:
        f = np.nextafter(f, np.float32(np.inf))
    return f


@pytest.mark.parametrize("xi,m", [(1e-3, 16), (2.56e-3, 16), (1e-4, 8), (3.7e-5, 32)])
def test_margins_exact(xi, m):
    """eps_q = 2 xi/(2^m-1); xi' = RD(xi(1-2^-m)) exactly; 0 < xi' < xi; eps_q > xi 2^-m
    (SPEC S:222 invariants); c_b < b < c_f; lo2 < b2 < hi2."""
    b = 0.0496
    t = oracle.thresholds(oracle.cfg(L=1.0, b=b, xi=xi, m=m))
    xi_f = Fraction(float(np.float32(xi)))
    assert t["xi"] == float(xi_f)
    assert np.float32(t["xip_f"]) == _largest_f32_le(xi_f * (1 - Fraction(1, 2 ** m)))
    assert 0 < t["xip_f"] < t["xi_f"]
    assert abs(t["eps_q"] - 2 * float(xi_f) / (2 ** m - 1)) <= 1e-18
    assert t["eps_q"] > float(xi_f) * 2.0 ** -m
    assert t["c_b"] <= np.float32(b) <= t["c_f"]
    assert t["lo2"] < t["b2"] < t["hi2"]


def test_lower_band_vacuous_when_xi_large():
    """b - 2 sqrt3 xi <= 0 -> the lower band test is vacuous (R2)."""
    t = oracle.thresholds(oracle.cfg(L=1.0, b=0.005, xi=2e-3))
    assert t["lo2"] < 0


def test_generators_deterministic_exact_counts_and_bounded():
    for w in (synth.Workload("a", "clumped", 5000, 1.0, 1e-3, seed=3),
              synth.Workload("b", "lattice", 4000, 1.0, 1e-4, seed=4),
              synth.Workload("c", "fcc", 4 * 6 ** 3 - 10, 1.0, 1e-4, b=0.1, seed=5,
                             extra={"cells": 6, "n_vac": 10})):
        a = synth.make(w)
        b = synth.make(w)
        for u, v in zip(a, b):
            assert torch.equal(u, v)
        x, y, z, xh, yh, zh = a
        assert x.shape[0] == w.n and x.dtype == torch.float32
        for o in (x, y, z):
            assert float(o.min()) >= 0 and float(o.max()) < w.L
        xi_f = float(np.float32(w.xi))
        for o, h in ((x, xh), (y, yh), (z, zh)):
            assert float((h.double() - o.double()).abs().max()) <= xi_f


def test_dither_error_uniform_and_plain_quantiser_grid():
    x = torch.rand(200_000, dtype=torch.float64).float()
    xi = 1e-3
    e = (synth.quantise(x, xi, 1).double() - x.double()).numpy()
    assert abs(e.mean()) < 2e-5 and abs(e.std() - xi / np.sqrt(3)) < 2e-5
    q = synth.quantise(x, xi, 1, dither=False).double().numpy()
    k = q / (2 * float(np.float32(xi)))
    assert np.max(np.abs(k - np.round(k))) < 1e-3


def test_clumped_halo_fraction_shape():
    """P10: G1 puts ~15% of particles in FoF groups >= 20 (paper HACC: 15.7%)."""
    w = synth.Workload("t", "clumped", 65536, 1.0, 1e-3, seed=1)
    x, y, z, *_ = [t.numpy() for t in synth.make(w)]
    lab, ng = oracle.fof(x, y, z, oracle.cfg(L=1.0, b=w.linking_length, xi=0.0))
    sizes = oracle.halo_catalog(lab, 20)
    frac = sizes.sum() / w.n
    assert 0.08 < frac < 0.3
