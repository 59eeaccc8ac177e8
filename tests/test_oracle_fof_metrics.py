"""Pins for the oracle's FoF labelling (O6) and the MCC / HMF checks (O7).

FoF: PAPER.md §II-B P:362 (edge iff d <= b, clusters = connected components), Fig. 1.
MCC: §IV-A P:12-15.  HMF: §II-B-2 P:387 (B log bins normalised by volume and bin width).
Pinned against scipy.sparse.csgraph.connected_components, sklearn's matthews_corrcoef and the
SPEC worked examples.
"""
import numpy as np
from scipy.sparse import coo_matrix
from scipy.sparse.csgraph import connected_components
from sklearn.metrics import matthews_corrcoef

import oracle
import synth
from tests.test_oracle_pairs import _np_d2, _rand_instance


def _canon(labels_by_root):
    """canonical min-index labels from arbitrary component ids"""
    lab = np.asarray(labels_by_root)
    out = np.empty(lab.shape[0], np.int64)
    first = {}
    for i, l in enumerate(lab):
        if l not in first:
            first[l] = i
        out[i] = first[l]
    return out


def test_fof_vs_scipy_connected_components():
    rng = np.random.default_rng(5)
    for k in range(12):
        n = int(rng.integers(1, 1200))
        x, y, z = _rand_instance(rng, n, clustered=bool(k % 2))
        b = 10 ** rng.uniform(-2, -1.2)
        c = oracle.cfg(L=1.0, b=b, xi=0.0)
        P = np.stack([x, y, z], 1)
        d2 = _np_d2(P[:, None, :], P[None, :, :], 1.0)
        adj = d2 <= np.float32(oracle.thresholds(c)["b2"])
        ii, jj = np.nonzero(np.triu(adj, 1))
        A = coo_matrix((np.ones(len(ii)), (ii, jj)), shape=(n, n))
        ng, comp = connected_components(A, directed=False)
        lab, ng2 = oracle.fof(x, y, z, c)
        labb, ng3 = oracle.fof(x, y, z, c, brute=True)
        assert ng == ng2 == ng3
        assert np.array_equal(lab, _canon(comp)) and np.array_equal(labb, lab)


def test_fof_spec_examples():
    b = 0.125
    c = oracle.cfg(L=1.0, b=b, xi=0.0)
    h2 = np.full(2, 0.5, np.float32)
    # d = b -> one component; d = next float above -> two
    for brute in (False, True):
        lab, ng = oracle.fof(np.array([0.25, 0.375], np.float32), h2, h2, c, brute=brute)
        assert ng == 1 and list(lab) == [0, 0]
        lab, ng = oracle.fof(np.array([0.25, np.nextafter(np.float32(0.375), np.float32(1))], np.float32), h2, h2, c,
                             brute=brute)
        assert ng == 2 and list(lab) == [0, 1]
    # chain p0-p1-p2 each link <= b, d(p0,p2) > b -> one component of size 3
    h3 = np.full(3, 0.5, np.float32)
    lab, ng = oracle.fof(np.array([0.25, 0.375, 0.5], np.float32), h3, h3, c)
    assert ng == 1 and list(lab) == [0, 0, 0]
    # labels are the min gid of the component (R20)
    lab, ng = oracle.fof(np.array([0.25, 0.375, 0.5], np.float32), h3, h3, c,
                         gid=np.array([7, 3, 9], np.uint32))
    assert list(lab) == [3, 3, 3]


def test_fof_monotone_in_b():
    x, y, z, *_ = [t.numpy() for t in synth.make(synth.Workload("t", "clumped", 5000, 1.0, 1e-3, seed=4))]
    prev = None
    for b in (0.002, 0.004, 0.006, 0.01):
        _, ng = oracle.fof(x, y, z, oracle.cfg(L=1.0, b=b, xi=0.0))
        assert prev is None or ng <= prev
        prev = ng


def test_mcc_vs_sklearn_and_spec():
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(10, 500))
        o = rng.random(n) < rng.random()
        l = np.where(rng.random(n) < 0.2, ~o, o)
        tp, tn, fp, fn = oracle.mcc_counts(o, l)
        assert tp + tn + fp + fn == n
        want = matthews_corrcoef(o, l)
        got = oracle.mcc(tp, tn, fp, fn)
        if (tp + fp) * (tp + fn) * (tn + fp) * (tn + fn) > 0:
            assert abs(got - want) < 1e-12
    assert abs(oracle.mcc(40, 40, 10, 10) - 0.6) < 1e-15
    assert oracle.mcc(0, 0, 25, 25) == -1.0                       # S:445 all flipped
    assert oracle.mcc(30, 0, 0, 0) == 1.0                         # R21 degenerate, perfect
    assert oracle.mcc(30, 0, 0, 5) == 0.0                         # R21 degenerate, imperfect


def test_halo_catalog_and_hmf_spec_examples():
    lab = np.zeros(100, np.int64)
    assert list(oracle.halo_catalog(lab, 20)) == [100]
    lab = np.concatenate([np.full(3, 0), np.full(5, 1), np.full(50, 2)])
    assert list(oracle.halo_catalog(lab, 20)) == [50]
    e, d = oracle.hmf([64], vol=2.0, n_bins=5)                                    # one halo
    assert np.count_nonzero(d) == 1 and np.isclose(d.max(), 1.0 / (2.0 * (e[1] - e[0])))
    sizes = [2 ** k for k in range(5, 15)]
    e, d = oracle.hmf(sizes, vol=1.0, n_bins=10)
    assert np.allclose(d, d[0]) and np.all(d > 0)
    e2, d2 = oracle.hmf(sizes, vol=2.0, n_bins=10)
    assert np.allclose(d2, d / 2)
    # total count reconstructs the catalogue
    assert np.isclose((d * 1.0 * (e[1] - e[0])).sum(), len(sizes))


def test_iteration_budget_examples():
    assert abs(oracle.iteration_budget(1e-3, 100, 1e-10) - 12_000_000) <= 1
    assert oracle.iteration_budget(1e-3, 0, 1e-10) == 0
    assert oracle.iteration_budget(2e-3, 100, 1e-10) >= oracle.iteration_budget(1e-3, 100, 1e-10)


def test_linking_length_examples():
    assert abs(oracle.linking_length(0.2, 1.0, 10**6) - 0.002) < 1e-15
    assert abs(oracle.linking_length(0.2, 8.0, 8) - 0.2) < 1e-15
