"""CPU oracle for the FoF-connectivity correction of arXiv 2604.18801.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this package.  The product path (paper_2604_18801_b200)
never imports it and shares no code with it.

The heavy steps (pairs, PGD, FoF) are the plain single-threaded C in ``cc_oracle.c`` loaded with
ctypes; the closed-form metrics (MCC, HMF) are written out here in plain Python.  Every
function cites the PAPER.md passage it follows ("P:n" = line n) and the DESIGN.md §3 reading
("R<k>") where the paper is silent.  Parity pins live in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cc_oracle.c")
_LIB = os.path.join(_HERE, "libcc_oracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-Wall", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Cfg(C.Structure):
    _fields_ = [("L", C.c_double), ("periodic", C.c_int), ("b", C.c_double), ("xi", C.c_double),
                ("m", C.c_int), ("alpha", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps_adam", C.c_double), ("t_max", C.c_int),
                ("eps_loss", C.c_double), ("stop_mode", C.c_int), ("optimizer", C.c_int),
                ("vanilla_step", C.c_double)]


class Th(C.Structure):
    _fields_ = [("Lf", C.c_float), ("hLf", C.c_float), ("xi_f", C.c_float), ("xip_f", C.c_float),
                ("b2", C.c_float), ("lo2", C.c_float), ("hi2", C.c_float), ("c_b", C.c_float),
                ("c_f", C.c_float), ("pad", C.c_float), ("xi", C.c_double), ("eps_q", C.c_double),
                ("mu", C.c_double), ("band_lo", C.c_double), ("band_hi", C.c_double)]


class CorrInfo(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("active0", C.c_int64), ("active_final", C.c_int64),
                ("violated0", C.c_int64), ("violated_final", C.c_int64), ("loss0", C.c_double),
                ("loss_final", C.c_double), ("n_editable", C.c_int64), ("converged", C.c_int),
                ("pad", C.c_int)]


STOP_ACTIVE, STOP_EPS, STOP_NONE, STOP_RESTORED = 0, 1, 2, 3

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        f32p, u32p, i64p, u8p, f64p = P(C.c_float), P(C.c_uint32), P(C.c_int64), P(C.c_uint8), P(C.c_double)
        L.oc_thresholds.argtypes = [P(Cfg), P(Th)]
        L.oc_dist2.argtypes = [f32p, f32p, P(Cfg)]
        L.oc_dist2.restype = C.c_float
        L.oc_find_pairs.argtypes = [C.c_int64, f32p, f32p, f32p, f32p, f32p, f32p, u32p, P(Cfg), C.c_int,
                                    P(i64p), P(i64p), P(u8p)]
        L.oc_find_pairs.restype = C.c_int64
        L.oc_free.argtypes = [C.c_void_p]
        L.oc_pair_links.argtypes = [C.c_int64, i64p, i64p, f32p, f32p, f32p, P(Cfg), u8p]
        L.oc_fof.argtypes = [C.c_int64, f32p, f32p, f32p, u32p, P(Cfg), C.c_int, u32p]
        L.oc_fof.restype = C.c_int64
        L.oc_tight_eval_f32.argtypes = [C.c_int64, f32p, f32p, f32p, u32p, C.c_int64, i64p, i64p, u8p,
                                        P(Cfg), i64p, f64p, f32p]
        L.oc_loss_eq1_f64.argtypes = [f64p, C.c_int64, i64p, i64p, u8p, C.c_double, C.c_double, C.c_int]
        L.oc_loss_eq1_f64.restype = C.c_double
        L.oc_tight_f64.argtypes = [f64p, C.c_int64, i64p, i64p, u8p, C.c_double, C.c_double, C.c_double,
                                   C.c_int, f64p]
        L.oc_tight_f64.restype = C.c_double
        L.oc_correct.argtypes = [C.c_int64, f32p, f32p, f32p, f32p, f32p, f32p, u32p, C.c_int64, i64p, i64p,
                                 u8p, P(Cfg), f32p, f32p, f32p, P(CorrInfo), i64p, f64p, i64p]
        L.oc_edit_encode.argtypes = [C.c_int64, f32p, f32p, f32p, f32p, f32p, f32p, f32p, f32p, f32p, P(Cfg), u8p, i64p,
                                     C.c_int64, i64p]
        L.oc_edit_decode.argtypes = [C.c_int64, f32p, f32p, f32p, u8p, i64p, C.c_int64, P(Cfg),
                                     f32p, f32p, f32p]
        L.oc_edit_packed_words.argtypes = [C.c_int64, C.c_int]
        L.oc_edit_packed_words.restype = C.c_int64
        L.oc_edit_pack.argtypes = [i64p, C.c_int64, C.c_int, u32p]
        L.oc_edit_unpack.argtypes = [u32p, C.c_int64, C.c_int, i64p]
        _lib = L
    return _lib


# ------------------------------------------------------------------------------------------
def cfg(L=1.0, b=None, xi=0.0, periodic=True, m=16, alpha=1e-3, beta1=0.9, beta2=0.999,
        eps_adam=1e-8, t_max=10_000, eps_loss=1e-10, stop_mode=STOP_ACTIVE, optimizer=0,
        vanilla_step=0.0, n=None, eta=0.2) -> Cfg:
    """Alg. 1 REQUIRE line plus the box.  b defaults to eta*(V/N)^(1/3)
    (§II-B); Adam constants per P:75/P:458."""
    if b is None:
        b = linking_length(eta, L ** 3, n)
    return Cfg(L, int(periodic), b, xi, m, alpha, beta1, beta2, eps_adam, t_max, eps_loss,
               stop_mode, optimizer, vanilla_step)


def linking_length(eta: float, vol: float, n: int, d: int = 3) -> float:
    """b = eta * Delta_p, Delta_p = (V/N)^(1/d)  (§II-B)."""
    if n is None or n <= 0 or vol <= 0:
        raise ValueError("need n > 0 and vol > 0")
    return eta * (vol / n) ** (1.0 / d)


def thresholds(c: Cfg) -> dict:
    t = Th()
    st = lib().oc_thresholds(C.byref(c), C.byref(t))
    if st:
        raise ValueError(f"oc_thresholds status {st}")
    return {k: getattr(t, k) for k, _ in Th._fields_ if k != "pad"}


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def dist2(pi, pj, c: Cfg) -> np.float32:
    a, b = _f32(pi), _f32(pj)
    return np.float32(lib().oc_dist2(_ptr(a, C.c_float), _ptr(b, C.c_float), C.byref(c)))


def find_pairs(x, y, z, xh, yh, zh, c: Cfg, gid=None, brute=False):
    """Canonical vulnerable pairs (Alg. 1 line 3).  Returns (pi, pj, flags) as input
    indices with gid[pi] < gid[pj], sorted by (gid[pi], gid[pj]); flags bit0 = linked in the
    original, bit1 = linked in the decompressed positions."""
    arrs = [_f32(a) for a in (x, y, z, xh, yh, zh)]
    n = arrs[0].shape[0]
    g = None if gid is None else np.ascontiguousarray(np.asarray(gid, dtype=np.uint32))
    oi, oj, of = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_uint8)()
    cnt = lib().oc_find_pairs(n, *[_ptr(a, C.c_float) for a in arrs],
                              None if g is None else _ptr(g, C.c_uint32), C.byref(c), int(brute),
                              C.byref(oi), C.byref(oj), C.byref(of))
    if cnt < 0:
        raise RuntimeError(f"oc_find_pairs status {-cnt}")
    pi = np.ctypeslib.as_array(oi, shape=(cnt,)).copy() if cnt else np.zeros(0, np.int64)
    pj = np.ctypeslib.as_array(oj, shape=(cnt,)).copy() if cnt else np.zeros(0, np.int64)
    pf = np.ctypeslib.as_array(of, shape=(cnt,)).copy() if cnt else np.zeros(0, np.uint8)
    for p in (oi, oj, of):
        lib().oc_free(C.cast(p, C.c_void_p))
    return pi, pj, pf


def pair_links(pi, pj, x, y, z, c: Cfg) -> np.ndarray:
    pi = np.ascontiguousarray(pi, dtype=np.int64)
    pj = np.ascontiguousarray(pj, dtype=np.int64)
    xs = [_f32(a) for a in (x, y, z)]
    out = np.zeros(pi.shape[0], np.uint8)
    st = lib().oc_pair_links(pi.shape[0], _ptr(pi, C.c_int64), _ptr(pj, C.c_int64),
                             *[_ptr(a, C.c_float) for a in xs], C.byref(c), _ptr(out, C.c_uint8))
    if st:
        raise RuntimeError(st)
    return out.astype(bool)


def fof(x, y, z, c: Cfg, gid=None, brute=False):
    """FoF labels (Fig. 1): min gid per connected component of {d <= b}.  Returns
    (labels[n] uint32, n_groups)."""
    xs = [_f32(a) for a in (x, y, z)]
    n = xs[0].shape[0]
    g = None if gid is None else np.ascontiguousarray(np.asarray(gid, dtype=np.uint32))
    lab = np.zeros(n, np.uint32)
    ng = lib().oc_fof(n, *[_ptr(a, C.c_float) for a in xs], None if g is None else _ptr(g, C.c_uint32),
                      C.byref(c), int(brute), _ptr(lab, C.c_uint32))
    if ng < 0:
        raise RuntimeError(f"oc_fof status {-ng}")
    return lab, int(ng)


def tight_eval_f32(xh, yh, zh, pairs, c: Cfg, gid=None):
    """Pinned fp32 L_tight (Eq. 3): (active count, fp64 loss, dense fp32 gradient [n,3])."""
    pi, pj, pf = [np.ascontiguousarray(a) for a in pairs]
    xs = [_f32(a) for a in (xh, yh, zh)]
    n = xs[0].shape[0]
    g = None if gid is None else np.ascontiguousarray(np.asarray(gid, dtype=np.uint32))
    act, loss = C.c_int64(), C.c_double()
    grad = np.zeros((n, 3), np.float32)
    st = lib().oc_tight_eval_f32(n, *[_ptr(a, C.c_float) for a in xs], None if g is None else _ptr(g, C.c_uint32),
                                 pi.shape[0], _ptr(pi.astype(np.int64), C.c_int64),
                                 _ptr(pj.astype(np.int64), C.c_int64), _ptr(pf.astype(np.uint8), C.c_uint8),
                                 C.byref(c), C.byref(act), C.byref(loss), _ptr(grad, C.c_float))
    if st:
        raise RuntimeError(st)
    return act.value, loss.value, grad


def loss_eq1_f64(P, pairs, b, L=1.0, periodic=True) -> float:
    """Eq. (1) in fp64."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    pi, pj, pf = [np.ascontiguousarray(a) for a in pairs]
    pi = pi.astype(np.int64); pj = pj.astype(np.int64); pf = pf.astype(np.uint8)
    return lib().oc_loss_eq1_f64(_ptr(P, C.c_double), pi.shape[0], _ptr(pi, C.c_int64), _ptr(pj, C.c_int64),
                                 _ptr(pf, C.c_uint8), b, L, int(periodic))


def tight_f64(P, pairs, b, eps_q, L=1.0, periodic=True, grad=False):
    """Eq. (3) in fp64, with the analytic gradient if grad=True."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    pi, pj, pf = [np.ascontiguousarray(a) for a in pairs]
    pi = pi.astype(np.int64); pj = pj.astype(np.int64); pf = pf.astype(np.uint8)
    g = np.zeros_like(P) if grad else None
    v = lib().oc_tight_f64(_ptr(P, C.c_double), pi.shape[0], _ptr(pi, C.c_int64), _ptr(pj, C.c_int64),
                           _ptr(pf, C.c_uint8), b, eps_q, L, int(periodic),
                           None if g is None else _ptr(g, C.c_double))
    return (v, g) if grad else v


def correct(x, y, z, xh, yh, zh, pairs, c: Cfg, gid=None, trace=False):
    """Alg. 1 lines 4-10: PGD-Adam on L_tight with projection onto B(xi').
    Returns (xo, yo, zo, info dict[, (trace_active, trace_loss, trace_violated)])."""
    arrs = [_f32(a) for a in (x, y, z, xh, yh, zh)]
    n = arrs[0].shape[0]
    pi, pj, pf = [np.ascontiguousarray(a) for a in pairs]
    pi = pi.astype(np.int64); pj = pj.astype(np.int64); pf = pf.astype(np.uint8)
    g = None if gid is None else np.ascontiguousarray(np.asarray(gid, dtype=np.uint32))
    xo, yo, zo = (np.zeros(n, np.float32) for _ in range(3))
    info = CorrInfo()
    ta = np.zeros(c.t_max + 1, np.int64) if trace else None
    tl = np.zeros(c.t_max + 1, np.float64) if trace else None
    tv = np.zeros(c.t_max + 1, np.int64) if trace else None
    st = lib().oc_correct(n, *[_ptr(a, C.c_float) for a in arrs], None if g is None else _ptr(g, C.c_uint32),
                          pi.shape[0], _ptr(pi, C.c_int64), _ptr(pj, C.c_int64), _ptr(pf, C.c_uint8),
                          C.byref(c), _ptr(xo, C.c_float), _ptr(yo, C.c_float), _ptr(zo, C.c_float),
                          C.byref(info), None if ta is None else _ptr(ta, C.c_int64),
                          None if tl is None else _ptr(tl, C.c_double), None if tv is None else _ptr(tv, C.c_int64))
    if st:
        raise RuntimeError(f"oc_correct status {st}")
    d = {k: getattr(info, k) for k, _ in CorrInfo._fields_ if k != "pad"}
    d["converged"] = bool(d["converged"])
    if trace:
        k = d["iterations"] + 1
        return xo, yo, zo, d, (ta[:k], tl[:k], tv[:k])
    return xo, yo, zo, d


# ------------------------------------------------------------------------------------------
def mcc_counts(orig_linked, linked):
    """TP/TN/FP/FN over vulnerable pairs (§IV-A): FP = unlinked in the original but
    linked after; FN = linked in the original but broken after."""
    o = np.asarray(orig_linked, bool)
    l = np.asarray(linked, bool)
    tp = int(np.count_nonzero(o & l)); tn = int(np.count_nonzero(~o & ~l))
    fp = int(np.count_nonzero(~o & l)); fn = int(np.count_nonzero(o & ~l))
    return tp, tn, fp, fn


def mcc(tp: int, tn: int, fp: int, fn: int) -> float:
    """MCC = (TP*TN - FP*FN) / sqrt((TP+FP)(TP+FN)(TN+FP)(TN+FN)).  Degenerate
    denominators (R21): 1 if FP = FN = 0, else 0.  Numerator exact (Python int)."""
    a, b, c_, d = tp + fp, tp + fn, tn + fp, tn + fn
    if a == 0 or b == 0 or c_ == 0 or d == 0:
        return 1.0 if fp == 0 and fn == 0 else 0.0
    return float(tp * tn - fp * fn) / math.sqrt(float(a * b * c_ * d))


def halo_catalog(labels, min_size: int = 20) -> np.ndarray:
    """Component sizes N_i >= min_size, descending (halo threshold 20)."""
    _, counts = np.unique(np.asarray(labels), return_counts=True)
    s = np.sort(counts[counts >= min_size])[::-1]
    return s.astype(np.int64)


def hmf(sizes, vol: float, n_bins: int = 50, lo: float | None = None, hi: float | None = None,
        particle_mass: float = 1.0):
    """dn/dlog10 M (§II-B-2): masses M_i = m_p N_i in n_bins equal-width log10 bins over
    [lo, hi] (default [min, max] of this catalogue, R22), counts / (V * bin width).
    Returns (edges[n_bins+1], density[n_bins])."""
    m = np.asarray(sizes, dtype=np.float64) * particle_mass
    if m.size == 0:
        return np.zeros(0), np.zeros(0)
    lm = np.log10(m)
    lo = float(lm.min()) if lo is None else lo
    hi = float(lm.max()) if hi is None else hi
    if hi <= lo:
        hi = lo + 1.0
    width = (hi - lo) / n_bins
    edges = lo + width * np.arange(n_bins + 1)
    k = np.floor((lm - lo) / width).astype(np.int64)
    k = np.where(lm == hi, n_bins - 1, k)
    ok = (k >= 0) & (k < n_bins)
    counts = np.bincount(k[ok], minlength=n_bins).astype(np.float64)
    return edges, counts / (vol * width)


def iteration_budget(xi: float, n_tight: int, eps_loss: float) -> int:
    """T <= ceil(12 xi^2 |V_tight| / eps_L)  (§III-E)."""
    return int(math.ceil(12.0 * xi * xi * n_tight / eps_loss))


def edit_step(c: Cfg) -> float:
    """Quantiser lattice step s = xi_f 2^(1-m) (R30)."""
    return math.ldexp(float(np.float32(c.xi)), 1 - c.m)


def edit_encode(x, y, z, xh0, yh0, zh0, xc, yc, zc, c: Cfg):
    """Alg. 1 lines 11-13, §III-B P:446 (R29, R30, R32): returns (flags
    u8[ceil(3n/8)], q int64[n_edits]) for Delta = corrected - decompressed; x, y, z = P."""
    o = [_f32(a) for a in (x, y, z)]
    h = [_f32(a) for a in (xh0, yh0, zh0)]
    p = [_f32(a) for a in (xc, yc, zc)]
    n = h[0].size
    flags = np.zeros((3 * n + 7) // 8, np.uint8)
    cap = 3 * n
    q = np.zeros(max(cap, 1), np.int64)
    ne = C.c_int64(0)
    st = lib().oc_edit_encode(n, *[_ptr(a, C.c_float) for a in o + h + p], C.byref(c), _ptr(flags, C.c_uint8),
                              _ptr(q, C.c_int64), cap, C.byref(ne))
    if st:
        raise ValueError(f"oc_edit_encode status {st}")
    return flags, q[:ne.value].copy()


def edit_decode(xh0, yh0, zh0, flags, q, c: Cfg):
    """Reconstruction, §III-B P:456 (R31): x_hat0 + scatter(dequantise(q), flags)."""
    h = [_f32(a) for a in (xh0, yh0, zh0)]
    n = h[0].size
    flags = np.ascontiguousarray(flags, np.uint8)
    q = np.ascontiguousarray(q, np.int64)
    qq = q if q.size else np.zeros(1, np.int64)
    out = [np.empty(n, np.float32) for _ in range(3)]
    st = lib().oc_edit_decode(n, *[_ptr(a, C.c_float) for a in h], _ptr(flags, C.c_uint8),
                              _ptr(qq, C.c_int64), q.size, C.byref(c), *[_ptr(a, C.c_float) for a in out])
    if st:
        raise ValueError(f"oc_edit_decode status {st}")
    return tuple(out)


def edit_pack(q, m: int) -> np.ndarray:
    """(m+2)-bit two's-complement fields, LSB-first in 32-bit words (Alg. 1 l.13, R33)."""
    q = np.ascontiguousarray(q, np.int64)
    nw = lib().oc_edit_packed_words(q.size, m)
    w = np.zeros(max(nw, 1), np.uint32)
    qq = q if q.size else np.zeros(1, np.int64)
    st = lib().oc_edit_pack(_ptr(qq, C.c_int64), q.size, m, _ptr(w, C.c_uint32))
    if st:
        raise ValueError(f"oc_edit_pack status {st}")
    return w[:nw]


def edit_unpack(words, n_edits: int, m: int) -> np.ndarray:
    w = np.ascontiguousarray(words, np.uint32)
    ww = w if w.size else np.zeros(1, np.uint32)
    q = np.zeros(max(n_edits, 1), np.int64)
    st = lib().oc_edit_unpack(_ptr(ww, C.c_uint32), n_edits, m, _ptr(q, C.c_int64))
    if st:
        raise ValueError(f"oc_edit_unpack status {st}")
    return q[:n_edits]


@dataclass
class PipelineResult:
    pairs: tuple
    xo: np.ndarray
    yo: np.ndarray
    zo: np.ndarray
    info: dict
    labels_orig: np.ndarray
    labels_corr: np.ndarray
    groups_orig: int
    groups_corr: int
    mcc_before: tuple
    mcc_after: tuple


def pipeline(x, y, z, xh, yh, zh, c: Cfg, gid=None) -> PipelineResult:
    """S1-S7 end to end: pairs, correction, FoF on original and corrected, MCC before/after."""
    pairs = find_pairs(x, y, z, xh, yh, zh, c, gid)
    xo, yo, zo, info = correct(x, y, z, xh, yh, zh, pairs, c, gid)
    lo, go = fof(x, y, z, c, gid)
    lc, gc = fof(xo, yo, zo, c, gid)
    ol = (pairs[2] & 1).astype(bool)
    before = mcc_counts(ol, (pairs[2] & 2).astype(bool))
    after = mcc_counts(ol, pair_links(pairs[0], pairs[1], xo, yo, zo, c))
    return PipelineResult(pairs, xo, yo, zo, info, lo, lc, go, gc, before, after)
