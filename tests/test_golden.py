"""Worked values printed in PAPER.md / SPEC.md (tests/golden/worked_examples.json, each entry
with its citation) checked against the oracle."""
import json
import math
import os
from fractions import Fraction

import numpy as np

import oracle

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _pair(d, dh):
    P = np.zeros((2, 3))
    P[1, 0] = dh
    return P, (np.array([0]), np.array([1]), np.array([1 if d <= 1.0 else 0], np.uint8))


def test_eq1_worked_values():
    for e in G["eq1_loss"]:
        P, pairs = _pair(e["d"], e["d_hat"])
        pairs = (pairs[0], pairs[1], np.array([1 if e["d"] <= e["b"] else 0], np.uint8))
        assert abs(oracle.loss_eq1_f64(P, pairs, e["b"], L=10.0) - e["loss"]) < 1e-12, e["cite"]


def test_tight_worked_values():
    for e in G["tight_loss"]:
        mu = 2 * math.sqrt(3) * e["eps_q"]
        P, pairs = _pair(e["d"], e["b"] + e["d_hat_minus_b_over_mu"] * mu)
        got = oracle.tight_f64(P, pairs, e["b"], e["eps_q"], L=10.0)
        assert abs(got - e["loss_over_mu2"] * mu * mu) < 1e-15, e["cite"]


def test_mcc_worked_values():
    for e in G["mcc"]:
        assert abs(oracle.mcc(e["tp"], e["tn"], e["fp"], e["fn"]) - e["mcc"]) < 1e-12, e["cite"]


def test_hmf_and_catalog_worked_values():
    for e in G["hmf"]:
        sizes = [2 ** k for k in e["log2_sizes"]]
        edges, dens = oracle.hmf(sizes, e["vol"], e["bins"])
        width = edges[1] - edges[0]
        assert np.allclose(dens * e["vol"] * width, e["counts_per_bin"]), e["cite"]
    for e in G["halo_catalog"]:
        lab = np.concatenate([np.full(k, i) for i, k in enumerate(e["components"])])
        assert list(oracle.halo_catalog(lab, e["min_size"])) == e["sizes"], e["cite"]


def test_alg1_constants_and_budget():
    for e in G["alg1_constants"]:
        xi = 0.015625   # exact in fp32 and fp64
        t = oracle.thresholds(oracle.cfg(L=1.0, b=0.5, xi=xi, m=e["m"]))
        want = Fraction(xi) * Fraction(*e["eps_q_over_xi"])
        assert abs(Fraction(t["eps_q"]) - want) <= want * Fraction(1, 2 ** 52), e["cite"]
        assert Fraction(float(t["xip_f"])) == Fraction(xi) * Fraction(*e["xip_over_xi"]), e["cite"]
    for e in G["budget"]:
        assert oracle.iteration_budget(e["xi"], e["v_tight"], e["eps_loss"]) == e["bound"], e["cite"]
