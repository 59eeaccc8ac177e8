"""GPU parity tests: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded
inputs, element by element (tests/parity.py states the bar).  Sizes span several tiles and a
ragged tail; edge cases: empty and tiny inputs, everything in one cell, coincident particles,
coordinates at 0 and L-, exact fp32 thresholds, all stop modes, both optimisers, and CUDA-graph
batch sizes that force speculative overrun."""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_18801_b200 as cc
import synth
from tests.parity import assert_parity, check_invariants, gpu_pipeline, oracle_pipeline

pytestmark = pytest.mark.gpu


def _arrs(w, dither=True):
    return [t.numpy() for t in synth.make(w, dither=dither)]


def _params(w, **kw):
    return cc.Params(box=w.L, b=w.linking_length, xi=w.xi, **kw)


@pytest.mark.parametrize("xi_rel,dither", [(1e-3, True), (1e-4, True), (1e-3, False), (3e-3, True)])
def test_c1_full_pipeline_bit_exact(xi_rel, dither):
    """configs[0]: clumped N = 65,536, b = 0.2 mean spacing."""
    w = synth.Workload("C1", "clumped", 65_536, 1.0, xi_rel, seed=1)
    arrs = _arrs(w, dither)
    p = _params(w)
    g = gpu_pipeline(arrs, p)
    o = oracle_pipeline(arrs, p)
    assert_parity(g, o)
    check_invariants(arrs, g["out"], p, g["info"])
    if g["info"]["converged"]:
        assert g["mcc_cor"]["mcc"] == 1.0
        assert np.array_equal(g["lab_orig"], g["lab_cor"])


@pytest.mark.parametrize("xi_rel", [1e-4, 1e-3])
def test_c2_lattice_bit_exact(xi_rel):
    """configs[1]: FPM-shaped N = 196,066 quasi-uniform cloud."""
    w = synth.Workload("C2", "lattice", 196_066, 1.0, xi_rel, seed=2)
    arrs = _arrs(w)
    p = _params(w)
    assert_parity(gpu_pipeline(arrs, p), oracle_pipeline(arrs, p))


def test_c3_fcc_bit_exact():
    """configs[2] shape (EXAALT FCC crystal, b = 0.8 a, 1.6 % vacancies, xi = 1e-5 a*90) on a
    30^3-cell block (N = 106,272) so the oracle finishes in seconds; the full 90^3 crystal is
    C3 itself (same lattice constant, jitter, vacancy fraction and absolute xi)."""
    c3 = synth.CONFIGS["C3"]
    cells = 30
    L = c3.L * cells / c3.extra["cells"]
    n_vac = round(c3.extra["n_vac"] * (cells / c3.extra["cells"]) ** 3)
    w = synth.Workload("C3s", "fcc", 4 * cells ** 3 - n_vac, L, 1e-5 / L, b=c3.b, seed=c3.seed,
                       extra={"cells": cells, "n_vac": n_vac})
    arrs = _arrs(w)
    p = _params(w)
    assert_parity(gpu_pipeline(arrs, p), oracle_pipeline(arrs, p))


@pytest.mark.parametrize("mode,tmax", [(cc.STOP_NONE, 7), (cc.STOP_NONE, 40), (cc.STOP_EPS, 10000), (cc.STOP_ACTIVE, 5),
                                       (cc.STOP_RESTORED, 10000)])
def test_stop_modes_bit_exact(mode, tmax):
    """Alg. 1 stop variants: truncated (exactly t_max updates), eps_L, active-count with a cap
    that ends the loop unconverged."""
    w = synth.Workload("t", "clumped", 20_000, 1.0, 1e-3, seed=7)
    arrs = _arrs(w)
    p = _params(w, stop_mode=mode, t_max=tmax)
    g = gpu_pipeline(arrs, p, fof=False)
    o = oracle_pipeline(arrs, p, fof=False)
    assert_parity(g, o, fof=False)
    if mode == cc.STOP_NONE:
        assert g["info"]["iterations"] == tmax


@pytest.mark.parametrize("frontier,mode", [(0, cc.STOP_ACTIVE), (0, cc.STOP_RESTORED), (1, cc.STOP_RESTORED)])
def test_frontier_is_exact(frontier, mode):
    """K3's frontier skipping (frozen particles replayed lazily) changes no result: both
    settings equal the oracle bit-exactly (the oracle sweeps every editable every iteration)."""
    w = synth.Workload("t", "clumped", 16_000, 1.0, 3e-3, seed=15)
    arrs = _arrs(w)
    p = _params(w, frontier=frontier, stop_mode=mode)
    assert_parity(gpu_pipeline(arrs, p, fof=False), oracle_pipeline(arrs, p, fof=False), fof=False)


@pytest.mark.parametrize("batch", [1, 3, 16, 64])
def test_graph_batch_does_not_change_result(batch):
    """The speculative device-side stop is exact for any graph batch (R11, S5)."""
    w = synth.Workload("t", "clumped", 30_000, 1.0, 1e-3, seed=8)
    arrs = _arrs(w)
    p = _params(w, graph_batch=batch)
    assert_parity(gpu_pipeline(arrs, p, fof=False), oracle_pipeline(arrs, p, fof=False), fof=False)


def test_vanilla_pgd_bit_exact():
    w = synth.Workload("t", "clumped", 20_000, 1.0, 1e-3, seed=9)
    arrs = _arrs(w)
    p = _params(w, optimizer=1, vanilla_step=2e-3, t_max=50, stop_mode=cc.STOP_NONE)
    assert_parity(gpu_pipeline(arrs, p, fof=False), oracle_pipeline(arrs, p, fof=False), fof=False)


@pytest.mark.parametrize("xi_rel,cells_per_particle", [(1e-3, 2.0), (3e-3, 0.05)])
def test_nonperiodic_domain_bit_exact(xi_rel, cells_per_particle):
    """the paper's own non-periodic domain (no minimum image, R5) on the
    clumped recipe: pairs across the faces must vanish, everything else bit-exact vs the oracle
    in the same mode."""
    w = synth.Workload("t", "clumped", 30_000, 1.0, xi_rel, seed=12)
    arrs = _arrs(w)
    p = _params(w, periodic=0, cells_per_particle=cells_per_particle)
    g = gpu_pipeline(arrs, p)
    o = oracle_pipeline(arrs, p)
    assert_parity(g, o)
    check_invariants(arrs, g["out"], p, g["info"])
    gi, gj, _ = g["pairs"]
    x = arrs[0]
    assert np.all(np.abs(x[gi].astype(np.float64) - x[gj]) < 0.5)     # no pair across the x faces


@pytest.mark.parametrize("cells_per_particle", [0.05, 1.0, 64.0])
def test_grid_resolution_does_not_change_result(cells_per_particle):
    """The pair set is grid-independent (R1): coarse and fine grids give identical results."""
    w = synth.Workload("t", "clumped", 25_000, 1.0, 1e-3, seed=10)
    arrs = _arrs(w)
    p = _params(w, cells_per_particle=cells_per_particle)
    assert_parity(gpu_pipeline(arrs, p), oracle_pipeline(arrs, p))


def _rand(rng, n, L=1.0):
    p = (rng.random((n, 3)) * L).astype(np.float32)
    p = np.where(p >= L, np.nextafter(np.float32(L), np.float32(0)), p)
    return [p[:, 0].copy(), p[:, 1].copy(), p[:, 2].copy()]


@pytest.mark.parametrize("n", [0, 1, 2, 3, 255, 256, 257, 4099])
def test_tiny_and_ragged_sizes(n):
    rng = np.random.default_rng(n)
    x, y, z = _rand(rng, n)
    xi = 2e-3
    noise = [(a + rng.uniform(-xi * 0.99, xi * 0.99, n)).astype(np.float32) for a in (x, y, z)]
    p = cc.Params(box=1.0, b=0.06, xi=xi)
    arrs = [x, y, z, *noise]
    assert_parity(gpu_pipeline(arrs, p), oracle_pipeline(arrs, p))


def test_everything_in_one_cell_and_coincident_points():
    """A dense blob (one cell holds most particles) with exact duplicates and the coincident
    false-pair rule (R15); coordinates at 0 and L-."""
    rng = np.random.default_rng(5)
    n = 3000
    c = np.float32(0.5)
    p = (c + rng.normal(0, 0.01, (n, 3))).astype(np.float32)
    p[100:200] = p[0:100]          # exact duplicates
    p[200:210] = 0.0
    p[210:220] = np.nextafter(np.float32(1.0), np.float32(0))
    x, y, z = p[:, 0].copy(), p[:, 1].copy(), p[:, 2].copy()
    xi = 1e-3
    noise = [np.clip(a + rng.uniform(-xi * 0.99, xi * 0.99, n).astype(np.float32), a - np.float32(xi * 0.99),
                     a + np.float32(xi * 0.99)).astype(np.float32) for a in (x, y, z)]
    pr = cc.Params(box=1.0, b=0.02, xi=xi, t_max=300)
    arrs = [x, y, z, *noise]
    assert_parity(gpu_pipeline(arrs, pr), oracle_pipeline(arrs, pr))


def test_giant_rows_bit_exact():
    """Rows beyond shared memory on both sorts: two tight clusters of 4,200 particles one linking
    length apart along x share one K1 row (8,400 records > 4,096) and every cross pair is in the
    band, so each editable's K2 row holds 4,200 entries (> 4,096): the in-place global bitonic
    paths of K1 and K2, and the K2 count's over-capacity strip, against the oracle (3 fixed
    iterations keep the oracle's 17.6M-pair loop to seconds)."""
    rng = np.random.default_rng(21)
    m, b, xi = 4200, 0.02, 1e-3
    h = 1.5e-4
    A = np.array([0.3, 0.5, 0.5]) + rng.uniform(-h, h, (m, 3))
    B = np.array([0.3 + b, 0.5, 0.5]) + rng.uniform(-h, h, (m, 3))
    P = np.concatenate([A, B]).astype(np.float32)
    perm = rng.permutation(2 * m)
    P = P[perm]
    x, y, z = P[:, 0].copy(), P[:, 1].copy(), P[:, 2].copy()
    noise = [np.clip(a + rng.uniform(-xi * 0.99, xi * 0.99, 2 * m).astype(np.float32), a - np.float32(xi * 0.99),
                     a + np.float32(xi * 0.99)).astype(np.float32) for a in (x, y, z)]
    pr = cc.Params(box=1.0, b=b, xi=xi, t_max=3, stop_mode=cc.STOP_NONE)
    arrs = [x, y, z, *noise]
    g, o = gpu_pipeline(arrs, pr), oracle_pipeline(arrs, pr)
    assert_parity(g, o)
    assert g["info"]["iterations"] == 3
    assert len(o["pairs"][0]) >= m * m


def test_gid_permutation():
    """User-supplied gids: results are keyed by gid (R14, R20)."""
    w = synth.Workload("t", "clumped", 10_000, 1.0, 1e-3, seed=12)
    arrs = _arrs(w)
    gid = np.random.default_rng(1).permutation(10_000).astype(np.uint32) * 3 + 7
    p = _params(w)
    assert_parity(gpu_pipeline(arrs, p, gid=gid), oracle_pipeline(arrs, p, gid=gid))


def test_bound_violation_rejected():
    x = torch.rand(100, device="cuda")
    xh = x + 0.01
    c = cc.Corrector(cc.Params(box=1.0, b=0.05, xi=1e-3))
    with pytest.raises(cc.CCError, match="CC_E_BOUND"):
        c.build_cells(x, x, x, xh, x, x)


def test_state_machine():
    c = cc.Corrector(cc.Params(box=1.0, b=0.05, xi=1e-3))
    with pytest.raises(cc.CCError, match="CC_E_STATE"):
        c.find_vulnerable()


def test_run_host_buffers_equal_device_path():
    """cc_run with HOST buffers (the e2e call) == the step-by-step device path."""
    w = synth.Workload("t", "clumped", 40_000, 1.0, 1e-3, seed=13)
    arrs = _arrs(w)
    p = _params(w)
    g = gpu_pipeline(arrs, p, fof=False)
    host = [torch.as_tensor(a).pin_memory() for a in arrs]
    out = [torch.empty(w.n, dtype=torch.float32).pin_memory() for _ in range(3)]
    c = cc.Corrector(p)
    r = c.run(*host, out=out, host=True)
    assert r["corr"]["iterations"] == g["info"]["iterations"]
    for a, b in zip(out, g["out"]):
        assert np.array_equal(a.numpy().view(np.uint32), b.view(np.uint32))
    dev = [torch.as_tensor(a).cuda() for a in arrs]
    dout = [torch.empty(w.n, dtype=torch.float32, device="cuda") for _ in range(3)]
    r2 = c.run(*dev, out=dout)
    for a, b in zip(dout, g["out"]):
        assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32))


def test_repeat_runs_bit_identical():
    w = synth.Workload("t", "clumped", 30_000, 1.0, 1e-3, seed=14)
    arrs = _arrs(w)
    p = _params(w)
    a = gpu_pipeline(arrs, p, fof=False)
    b = gpu_pipeline(arrs, p, fof=False)
    for u, v in zip(a["out"], b["out"]):
        assert np.array_equal(u.view(np.uint32), v.view(np.uint32))
    assert a["info"]["loss_final"] == b["info"]["loss_final"]


def test_hmf_on_gpu_catalogue_matches_oracle():
    w = synth.Workload("t", "clumped", 65_536, 1.0, 1e-3, seed=1)
    arrs = _arrs(w)
    p = _params(w)
    g = gpu_pipeline(arrs, p)
    e1, d1 = cc.hmf(g["halo_orig"], 1.0, 50)
    e2, d2 = oracle.hmf(oracle.halo_catalog(oracle.fof(*arrs[:3], oracle.cfg(L=1.0, b=w.linking_length, xi=w.xi))[0]),
                        1.0, 50)
    assert np.allclose(d1, d2, rtol=1e-12) and np.allclose(e1, e2, atol=1e-12)
    lo, hi = float(np.log10(g["halo_orig"].min())), float(np.log10(g["halo_orig"].max()))
    _, d4 = cc.hmf(g["halo_orig"], 1.0, 50, lo=lo, hi=hi)
    _, d3 = cc.hmf(g["halo_cor"], 1.0, 50, lo=lo, hi=hi)
    assert np.array_equal(d4, d3)   # converged -> identical HMF on the original's bins (R22)


@pytest.mark.parametrize("frontier", [1, 0])
def test_margin_below_fp32_resolution_violated_but_inactive(frontier):
    """configs[2] (C3, full size) at xi_rel = 1e-6: the Eq. 3 margin 2 sqrt3 eps_q (1.06e-10) is
    below half an ulp of b, so c_b = fl32(b) and one pair stays violated (d_hat^2 > b2) yet
    L_tight-inactive from iteration 3 on (oracle trace: active 2753, 9, 0, ...; violated 2754,
    10, 1, 1, ...).  The frontier must not freeze its endpoints (round 1 did, ending the RESTORED
    loop at t = 2): GPU trace and iteration count == oracle, not converged at T_max."""
    w0 = synth.CONFIGS["C3"]
    w = synth.Workload(w0.name, w0.kind, w0.n, w0.L, 1e-6, b=w0.b, seed=w0.seed, extra=w0.extra)
    arrs = _arrs(w)
    p = _params(w, stop_mode=cc.STOP_RESTORED, t_max=30, frontier=frontier)
    g = gpu_pipeline(arrs, p, fof=False)
    o = oracle_pipeline(arrs, p, fof=False)
    assert_parity(g, o, fof=False)
    assert o["info"]["violated_final"] > 0 and not g["info"]["converged"]


def test_torch_caching_allocator_scratch():
    """cc_params.alloc_fn/free_fn (§8(b)): scratch from torch's caching allocator on the
    context's stream gives the same bit-exact results."""
    w = synth.Workload("C1", "clumped", 30_000, 1.0, 1e-3, seed=2)
    arrs = _arrs(w)
    p = _params(w, torch_allocator=True)
    assert_parity(gpu_pipeline(arrs, p), oracle_pipeline(arrs, p))


def test_output_into_the_decompressed_input_arrays():
    """cc_correct copies every non-editable particle's decompressed input and scatters the
    editables (cc.h): writing the outputs over xh, yh, zh themselves gives the same corrected
    positions as separate outputs (and the oracle's)."""
    w = synth.Workload("alias", "clumped", 20_000, 1.0, 1e-3, seed=14)
    arrs = _arrs(w)
    p = _params(w)
    o = oracle_pipeline(arrs, p, fof=False)
    dev = torch.device("cuda", 0)
    ts = [torch.as_tensor(a).to(dev) for a in arrs]
    c = cc.Corrector(p, device=0)
    c.build_cells(*ts)
    c.find_vulnerable()
    out, info = c.correct(out=(ts[3], ts[4], ts[5]))
    torch.cuda.synchronize()
    for k in range(3):
        assert np.array_equal(out[k].cpu().numpy().view(np.uint32), o["out"][k].view(np.uint32))
    assert info["iterations"] == o["info"]["iterations"]
    c.close()
