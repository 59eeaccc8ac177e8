"""GPU parity of the f1 edit log (cc_edit_encode / cc_edit_decode through the C ABI) against
the oracle's oc_edit_encode / oc_edit_decode: Alg. 1 lines 11-13, §III-B
and P:456, readings R29-R32.  Flags bytes, quantisation indices and reconstructed coordinates
are bit-exact (integer/byte work; the fp64 quantiser and the single fp32 rounding of the
reconstruction are the same IEEE operations on both sides).  Inputs: seeded synthetic edit sets
(sparse, ragged sizes, several magnitudes and bit depths) and the C1 correction of each side;
plus the paper's quantisation-safety re-check through cc_find_vulnerable."""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_18801_b200 as cc
import synth
from tests.parity import oracle_cfg

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def _edits(n, L, xi, seed, frac=0.3):
    """seeded synthetic (decompressed, corrected) pair: a fraction of the coordinates moved by
    a uniform amount in [-2 xi_f, 2 xi_f] (clipped after fp32 rounding), the rest untouched"""
    rng = np.random.default_rng(seed)
    xi_f = float(np.float32(xi))
    h = [rng.uniform(0, L, n).astype(np.float32) for _ in range(3)]
    p = []
    for a in range(3):
        mv = rng.random(n) < frac
        v = (h[a].astype(np.float64) + rng.uniform(-2 * xi_f, 2 * xi_f, n)).astype(np.float32)
        bad = np.abs(v.astype(np.float64) - h[a]) > 2 * xi_f
        v[bad] = h[a][bad]
        p.append(np.where(mv, v, h[a]).astype(np.float32))
    return h, p


def _dev(a):
    return torch.as_tensor(np.ascontiguousarray(a)).to(DEV)


def _check(h, p, L, xi, m):
    params = cc.Params(box=L, b=0.01 * L, xi=xi, m=m)
    ctx = cc.Corrector(params, device=0)
    hd, pd = [_dev(a) for a in h], [_dev(a) for a in p]
    flags, q = ctx.edit_encode(*pd, *hd, *pd)
    oc = oracle.cfg(L=L, b=0.01 * L, xi=xi, m=m)
    of, oq = oracle.edit_encode(*p, *h, *p, oc)
    assert np.array_equal(flags.cpu().numpy(), of)
    assert np.array_equal(q.cpu().numpy(), oq)
    rec = ctx.edit_decode(*hd, flags, q)
    orec = oracle.edit_decode(*h, of, oq, oc)
    for a in range(3):
        assert np.array_equal(rec[a].cpu().numpy().view(np.uint32), orec[a].view(np.uint32))
    ctx.close()
    return of, oq


@pytest.mark.parametrize("n", [1, 2, 3, 31, 32, 33, 255, 256, 257, 1000, 65_537])
def test_ragged_sizes_bit_exact(n):
    _check(*_edits(n, 1.0, 1e-3, seed=n), 1.0, 1e-3, 16)


@pytest.mark.parametrize("m,L,frac", [(8, 1.0, 0.3), (16, 256.0, 0.05), (32, 1.0, 1.0), (16, 1.0, 0.0)])
def test_bit_depths_and_magnitudes(m, L, frac):
    n = 200_003
    xi = 1e-3 * L
    _check(*_edits(n, L, xi, seed=m + int(L), frac=frac), L, xi, m)


def test_multi_million_block_offsets():
    """several thousand blocks: the block-sum scan spans many 1024-chunks (u64 offsets)"""
    n = 5_000_011
    of, oq = _check(*_edits(n, 1.0, 1e-3, seed=99, frac=0.45), 1.0, 1e-3, 16)
    assert oq.size > 4 * 1024 * 256


def test_errors():
    params = cc.Params(box=1.0, b=0.01, xi=1e-3)
    ctx = cc.Corrector(params, device=0)
    h = [torch.zeros(100, dtype=torch.float32, device=DEV) for _ in range(3)]
    p = [t.clone() for t in h]
    p[1][7] = 2.5e-3                                         # |Delta| > 2 xi_f
    with pytest.raises(cc.CCError, match="CC_E_BOUND"):
        ctx.edit_encode(*p, *h, *p)
    p[1][7] = 1e-3
    p[2][9] = -1e-3
    with pytest.raises(cc.CCError, match="CC_E_OOM"):
        ctx.edit_encode(*p, *h, *p, cap=1)
    flags, q = ctx.edit_encode(*p, *h, *p)
    assert q.shape[0] == 2
    with pytest.raises(cc.CCError, match="CC_E_DATA"):
        ctx.edit_decode(*h, flags, q[:1])
    e = [torch.zeros(0, dtype=torch.float32, device=DEV) for _ in range(3)]
    f0, q0 = ctx.edit_encode(*e, *e, *e)
    assert f0.numel() == 0 and q0.numel() == 0
    ctx.close()


@pytest.mark.parametrize("xi_rel", [1e-3, 1e-4])
def test_c1_correction_edit_log_and_recheck(xi_rel):
    """configs[0]: each side encodes its own C1 correction (the GPU path's cc_correct output,
    the oracle's oc_correct output) -> identical flags and indices; the GPU reconstruction
    re-checked through cc_find_vulnerable on (P, x_rec): no violated pair, no bound
    error, FoF labels of x_rec equal the original's."""
    w = synth.Workload("C1", "clumped", 65_536, 1.0, xi_rel, seed=1)
    arrs = [t.numpy() for t in synth.make(w)]
    params = cc.Params(box=w.L, b=w.linking_length, xi=w.xi)
    ts = [_dev(a) for a in arrs]
    ctx = cc.Corrector(params, device=0)
    ctx.build_cells(*ts)
    ctx.find_vulnerable()
    out, info = ctx.correct()
    assert info["converged"]
    flags, q = ctx.edit_encode(*ts, *out)
    rec = ctx.edit_decode(*ts[3:], flags, q)
    ctx.close()

    c = oracle_cfg(params, len(arrs[0]))
    r = oracle.pipeline(*arrs, c)
    of, oq = oracle.edit_encode(*arrs, r.xo, r.yo, r.zo, c)
    assert np.array_equal(flags.cpu().numpy(), of)
    assert np.array_equal(q.cpu().numpy(), oq)

    chk = cc.Corrector(params, device=0)
    chk.build_cells(*ts[:3], *rec)                          # raises CC_E_BOUND if |x_rec - x| > xi_f
    vp = chk.find_vulnerable()
    assert vp["n_violated0"] == 0
    assert chk.mcc(cc.CC_DECOMP)["mcc"] == 1.0
    lo, _ = chk.fof_label(cc.CC_ORIG)
    lo = lo.cpu().numpy().copy()
    ld, _ = chk.fof_label(cc.CC_DECOMP)
    assert np.array_equal(lo, ld.cpu().numpy())
    chk.close()


def test_bound_safe_index_near_origin():
    """R32 on the GPU: box-saturated corrections near the origin (ulp(x) < s), where the plain
    nearest index can reconstruct up to half an ulp outside xi_f; bit-exact vs the oracle and
    every reconstruction within xi_f of the original."""
    rng = np.random.default_rng(12)
    n, xi = 300_001, 1e-3
    oc = oracle.cfg(L=1.0, b=0.01, xi=xi)
    th = oracle.thresholds(oc)
    x = rng.uniform(0.0, 0.3, n).astype(np.float32)
    sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    h = (x.astype(np.float64) - sign * rng.uniform(0, th["xi_f"], n)).astype(np.float32)
    p = (x.astype(np.float64) + sign * float(th["xip_f"])).astype(np.float32)
    ok = (np.abs(p.astype(np.float64) - x) <= float(th["xip_f"])) & (np.abs(h.astype(np.float64) - x) <= th["xi_f"])
    x, h, p = x[ok], h[ok], p[ok]
    y = np.full_like(x, 0.5)
    ctx = cc.Corrector(cc.Params(box=1.0, b=0.01, xi=xi), device=0)
    d = [_dev(a) for a in (x, y, y, h, y, y, p, y, y)]
    flags, q = ctx.edit_encode(*d)
    of, oq = oracle.edit_encode(x, y, y, h, y, y, p, y, y, oc)
    assert np.array_equal(flags.cpu().numpy(), of) and np.array_equal(q.cpu().numpy(), oq)
    xr, _, _ = ctx.edit_decode(d[3], d[4], d[5], flags, q)
    xr = xr.cpu().numpy()
    assert np.all(np.abs(xr.astype(np.float64) - x) <= th["xi_f"])
    ctx.close()


@pytest.mark.parametrize("path", ["vector", "scalar_env", "misaligned"])
def test_vector_and_scalar_paths(path, monkeypatch):
    """the float4 kernels (16-byte aligned buffers) and the scalar ones (CC_CODEC_SCALAR=1, or
    views that start one float in) give the oracle's bytes"""
    n = 100_003
    h, p = _edits(n + 1, 1.0, 1e-3, seed=5, frac=0.4)
    if path == "scalar_env":
        monkeypatch.setenv("CC_CODEC_SCALAR", "1")
    off = 1 if path == "misaligned" else 0
    h = [a[off:off + n] for a in h]
    p = [a[off:off + n] for a in p]
    params = cc.Params(box=1.0, b=0.01, xi=1e-3)
    ctx = cc.Corrector(params, device=0)
    hd = [_dev(np.concatenate([np.zeros(off, np.float32), a]))[off:] for a in h]
    pd = [_dev(np.concatenate([np.zeros(off, np.float32), a]))[off:] for a in p]
    assert all((t.data_ptr() % 16 == 0) == (off == 0) for t in hd + pd)
    flags, q = ctx.edit_encode(*pd, *hd, *pd)
    oc = oracle.cfg(L=1.0, b=0.01, xi=1e-3)
    of, oq = oracle.edit_encode(*p, *h, *p, oc)
    assert np.array_equal(flags.cpu().numpy(), of) and np.array_equal(q.cpu().numpy(), oq)
    out = [torch.empty(n + off, dtype=torch.float32, device=DEV)[off:] for _ in range(3)]
    rec = ctx.edit_decode(*hd, flags, q, out=tuple(out))
    orec = oracle.edit_decode(*h, of, oq, oc)
    for a in range(3):
        assert np.array_equal(rec[a].cpu().numpy().view(np.uint32), orec[a].view(np.uint32))
    ctx.close()


@pytest.mark.parametrize("m", [2, 8, 16, 32, 40])
def test_edit_pack_bit_exact(m):
    """cc_edit_pack / cc_edit_unpack (R33): (m+2)-bit fields bit-exact against the oracle's
    packer, ragged counts (fields straddling 2-3 words), and the round trip."""
    rng = np.random.default_rng(100 + m)
    c = cc.Corrector(cc.Params(box=1.0, xi=1e-3, m=m), device=0)
    for n in (0, 1, 31, 32, 33, 1000, 65537):
        q = rng.integers(-(2 ** m), 2 ** m + 1, n).astype(np.int64)
        if n >= 2:
            q[:2] = [-(2 ** m), 2 ** m]
        w = c.edit_pack(_dev(q))
        want = oracle.edit_pack(q, m)
        assert np.array_equal(w.cpu().numpy().view(np.uint32), want), (m, n)
        assert np.array_equal(c.edit_unpack(w, n).cpu().numpy(), q)
    with pytest.raises(cc.CCError):
        c.edit_pack(_dev(np.array([2 ** m + 1], np.int64)))


def test_edit_pack_of_a_correction_matches_oracle():
    """The packed index stream of a real correction (C1 recipe): GPU encode + pack == oracle
    encode + pack, (m+2)/8 bytes per edit."""
    w = synth.Workload("C1", "clumped", 20000, 1.0, 1e-3, seed=1)
    arrs = [t.numpy() for t in synth.make(w)]
    p = cc.Params(box=w.L, b=w.linking_length, xi=w.xi)
    c = cc.Corrector(p, device=0)
    d = [_dev(a) for a in arrs]
    c.build_cells(*d)
    c.find_vulnerable()
    out, _ = c.correct()
    fl, q = c.edit_encode(*d, *out)
    words = c.edit_pack(q)
    oc = oracle_cfg(p, w.n)
    of, oq = oracle.edit_encode(*arrs, *[o.cpu().numpy() for o in out], oc)
    assert np.array_equal(words.cpu().numpy().view(np.uint32), oracle.edit_pack(oq, p.m))
    assert words.numel() * 4 == (len(oq) * (p.m + 2) + 31) // 32 * 4
