"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no distances, thresholds, pairs, losses or
updates).  It only draws particle positions and the "decompressed" positions a base
compressor would return, with the shapes of the paper's datasets (PAPER.md `tab:datasets`
P:29-48):

* ``clumped``   -- G1: Gaussian halos with a truncated power-law mass function plus a
                   uniform background in a periodic box (HACC-shaped: C1, C4, C5).
* ``lattice``   -- quasi-uniform jittered cubic lattice (FPM-shaped meshfree cloud: C2).
* ``fcc``       -- jittered FCC crystal with vacancies (EXAALT-shaped: C3).
* ``quantise``  -- the seeded error-bounded base compressor of north_star ("seeded uniform
                   error-bounded quantiser at eps"), subtractive-dither form (R23)
                   or the plain step-2xi form (variant Q0).

Everything is torch so the same code runs on the host (parity tests, oracle inputs) and on
a GPU (full-size bench inputs, which would take minutes to draw with numpy).  Streams are
deterministic per (seed, device type); host and device streams differ, which is fine since
every consumer receives the drawn tensors, never re-draws them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

__all__ = ["Workload", "CONFIGS", "clumped", "lattice", "fcc", "quantise", "make", "halo_sizes"]


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=torch.device(device).type)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return g


def _wrap_f32(p64: torch.Tensor, L: float) -> torch.Tensor:
    """fp64 positions -> fp32 in [0, L) (periodic wrap, then guard the fp32 round-up to L)."""
    p64 = torch.remainder(p64, L)
    p32 = p64.to(torch.float32)
    top = torch.nextafter(torch.tensor(L, dtype=torch.float32, device=p32.device),
                          torch.tensor(0.0, dtype=torch.float32, device=p32.device))
    return torch.where(p32 >= L, top, p32)


def halo_sizes(n_halo: int, seed: int, slope: float = 1.9, m_min: int = 20, m_max: int = 10**6):
    """I.i.d. halo sizes from dn/dM ∝ M^-slope on [m_min, m_max] until their sum reaches
    n_halo; the last halo is trimmed so the total is exact."""
    rng = np.random.Generator(np.random.Philox(seed))
    a = 1.0 - slope
    lo, hi = m_min ** a, (m_max + 1) ** a
    sizes = []
    total = 0
    while total < n_halo:
        u = rng.random(4096)
        m = np.floor((lo + u * (hi - lo)) ** (1.0 / a)).astype(np.int64)
        m = np.clip(m, m_min, m_max)
        for s in m:
            if total >= n_halo:
                break
            s = int(min(s, n_halo - total))
            sizes.append(s)
            total += s
    return np.asarray(sizes, dtype=np.int64)


def clumped(n: int, L: float, seed: int, device="cpu", f_halo: float = 0.2, slope: float = 1.9,
            m_min: int = 20, m_max: int | None = None, shuffle: bool = True):
    """G1 clumped generator: a fraction f_halo of particles in Gaussian halos of rms radius
    r200/2 with r200 = (3M / (4*pi*200*nbar))^(1/3), centres uniform; the rest uniform.
    Returns (x, y, z) fp32 tensors in [0, L)."""
    dev = torch.device(device)
    g = _gen(seed, dev)
    nbar = n / L ** 3
    if m_max is None:
        m_max = int(max(m_min, min(n // 50, 10**6)))
    n_h = int(round(f_halo * n)) if n >= m_min else 0
    sizes = halo_sizes(n_h, seed + 17, slope, m_min, m_max) if n_h > 0 else np.zeros(0, np.int64)
    n_halos = len(sizes)
    sizes_t = torch.as_tensor(sizes, device=dev)
    centres = torch.rand((n_halos, 3), generator=g, device=dev, dtype=torch.float64) * L
    r200 = (3.0 * sizes_t.to(torch.float64) / (4.0 * math.pi * 200.0 * nbar)) ** (1.0 / 3.0)
    sigma = 0.5 * r200
    hid = torch.repeat_interleave(torch.arange(n_halos, device=dev), sizes_t)
    off = torch.randn((n_h, 3), generator=g, device=dev, dtype=torch.float64)
    ph = centres[hid] + off * sigma[hid, None]
    pb = torch.rand((n - n_h, 3), generator=g, device=dev, dtype=torch.float64) * L
    p = torch.cat([ph, pb], 0)
    del ph, pb, off, hid
    if shuffle and n > 1:
        p = p[torch.randperm(n, generator=g, device=dev)]
    p32 = _wrap_f32(p, L)
    return p32[:, 0].contiguous(), p32[:, 1].contiguous(), p32[:, 2].contiguous()


def lattice(n: int, L: float, seed: int, device="cpu", jitter: float = 0.15, shuffle: bool = True):
    """FPM-shaped quasi-uniform cloud: a cubic lattice of ceil(n^(1/3))^3 sites, the first n
    kept, each jittered by N(0, (jitter*a)^2) per axis."""
    dev = torch.device(device)
    g = _gen(seed, dev)
    k = int(math.ceil(round(n ** (1.0 / 3.0), 9)))
    while k ** 3 < n:
        k += 1
    a = L / k
    idx = torch.arange(n, device=dev, dtype=torch.int64)
    ijk = torch.stack([idx % k, (idx // k) % k, idx // (k * k)], 1).to(torch.float64)
    p = (ijk + 0.5) * a + torch.randn((n, 3), generator=g, device=dev, dtype=torch.float64) * (jitter * a)
    if shuffle and n > 1:
        p = p[torch.randperm(n, generator=g, device=dev)]
    p32 = _wrap_f32(p, L)
    return p32[:, 0].contiguous(), p32[:, 1].contiguous(), p32[:, 2].contiguous()


def fcc(cells: int, n_vac: int, L: float, seed: int, device="cpu", jitter: float = 0.05,
        shuffle: bool = True):
    """EXAALT-shaped crystal: cells^3 FCC unit cells (4 sites each) of side a = L/cells,
    n_vac seeded vacancies removed, thermal jitter N(0, (jitter*a)^2) per axis
    (SURVEY.md §8(d) C3)."""
    dev = torch.device(device)
    g = _gen(seed, dev)
    a = L / cells
    c = torch.arange(cells, device=dev, dtype=torch.float64)
    cz, cy, cx = torch.meshgrid(c, c, c, indexing="ij")
    base = torch.stack([cx.reshape(-1), cy.reshape(-1), cz.reshape(-1)], 1)
    basis = torch.tensor([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]],
                         device=dev, dtype=torch.float64)
    sites = (base[:, None, :] + basis[None, :, :]).reshape(-1, 3) * a
    keep = torch.randperm(sites.shape[0], generator=g, device=dev)[: sites.shape[0] - n_vac]
    keep, _ = torch.sort(keep)
    p = sites[keep]
    p = p + torch.randn(p.shape, generator=g, device=dev, dtype=torch.float64) * (jitter * a)
    if shuffle and p.shape[0] > 1:
        p = p[torch.randperm(p.shape[0], generator=g, device=dev)]
    p32 = _wrap_f32(p, L)
    return p32[:, 0].contiguous(), p32[:, 1].contiguous(), p32[:, 2].contiguous()


def quantise(x: torch.Tensor, xi: float, seed: int, dither: bool = True) -> torch.Tensor:
    """Seeded error-bounded base compressor for one coordinate array (fp32 in, fp32 out).

    dither=True  (R23): u = xi*(2U-1), xh = rnd_half_even((x+u)/(2 xi))*2 xi - u
                 in fp64, so the error is uniform on [-xi, xi] with no forced coincidences.
    dither=False (variant Q0): xh = rnd_half_even(x/(2 xi))*2 xi.
    Then rounded to fp32; any coordinate whose fp32 error exceeds xi_f = fl32(xi) is moved
    one ulp toward x until |xh - x| <= xi_f holds exactly (the bound every consumer checks)."""
    dev = x.device
    xi_f = float(np.float32(xi))
    x64 = x.to(torch.float64)
    if dither:
        g = _gen(seed, dev)
        u = (torch.rand(x.shape, generator=g, device=dev, dtype=torch.float64) * 2.0 - 1.0) * xi_f
        xh64 = torch.round((x64 + u) / (2.0 * xi_f)) * (2.0 * xi_f) - u
    else:
        xh64 = torch.round(x64 / (2.0 * xi_f)) * (2.0 * xi_f)
    xh = xh64.to(torch.float32)
    for _ in range(4):
        bad = (xh.to(torch.float64) - x64).abs() > xi_f
        if not bool(bad.any()):
            break
        xh = torch.where(bad, torch.nextafter(xh, x), xh)
    return xh


@dataclass
class Workload:
    name: str
    kind: str                 # clumped | lattice | fcc
    n: int
    L: float
    xi_rel: float
    eta: float = 0.2
    b: float | None = None    # explicit linking length (C3), else eta * (L^3/N)^(1/3)
    seed: int = 1
    extra: dict = field(default_factory=dict)

    @property
    def xi(self) -> float:
        """Absolute bound xi = xi_rel * L (global-range reading, R6)."""
        return self.xi_rel * self.L

    @property
    def linking_length(self) -> float:
        if self.b is not None:
            return self.b
        return self.eta * (self.L ** 3 / self.n) ** (1.0 / 3.0)

    def describe(self) -> dict:
        return {"workload": self.name, "kind": self.kind, "n": self.n, "box": self.L,
                "xi_rel": self.xi_rel, "b": self.linking_length, "seed": self.seed}


# BASELINE.json configs[0..4].
CONFIGS = {
    "C1": Workload("C1", "clumped", 65_536, 1.0, 1e-3, seed=1),
    "C2": Workload("C2", "lattice", 196_066, 1.0, 1e-3, seed=2),
    "C3": Workload("C3", "fcc", 2_869_440, 1.0, 1e-4, b=0.80 / 90.0, seed=3,
                   extra={"cells": 90, "n_vac": 46_560}),
    # C4 at SURVEY §8(d)'s xi_rel = 1e-6 (the paper's HACC error bound); the bench also
    # reports 1.2e-4 (density-matched heavy case) and 1e-5 via --xi-rel
    "C4": Workload("C4", "clumped", 280_953_867, 256.0, 1e-6, seed=4),
    "C5": Workload("C5", "clumped", 1_073_734_015, 256.0, 1e-6, seed=5),
}


def make(w: Workload, device="cpu", dither: bool = True):
    """Draw (x, y, z, xh, yh, zh) for a workload: originals then decompressed."""
    if w.kind == "clumped":
        x, y, z = clumped(w.n, w.L, w.seed, device)
    elif w.kind == "lattice":
        x, y, z = lattice(w.n, w.L, w.seed, device)
    elif w.kind == "fcc":
        x, y, z = fcc(w.extra["cells"], w.extra["n_vac"], w.L, w.seed, device)
    else:
        raise ValueError(w.kind)
    s = w.seed + 1000
    xh = quantise(x, w.xi, s * 3 + 0, dither)
    yh = quantise(y, w.xi, s * 3 + 1, dither)
    zh = quantise(z, w.xi, s * 3 + 2, dither)
    return x, y, z, xh, yh, zh
