"""Synthetic benchmark inputs for the BASELINE.json configurations.

* ``gen_psf`` restates the reference's named kernels (harness.py:147-167):
  truncated Gaussian ``exp(-(i^2+j^2)/(2 sigma^2))`` normalised to unit sum,
  plus the uniform ``box`` used by config 4 (``np.full((w,w), 1/w^2)``).
* ``gen_piecewise_image`` is the seeded piecewise-constant generator that
  BASELINE.json asks for; the reference has none (its only 2D generator is
  ``gen_image_2d``, harness.py:126-144).  The frozen choices:
  ``Generator(PCG64(seed))``; canvas ``T = n + 2m`` filled with 0.2;
  rectangles first (integer top-left uniform on ``[0, T)``, integer sides
  uniform on ``[ceil(T/16), floor(T/4)]``), then disks (centre uniform on
  ``[0, T)^2``, radius uniform on ``[T/32, T/8]``); each shape's intensity is
  ``U[0,1]`` drawn after its geometry; later shapes overwrite earlier ones;
  optional ramp ``0.1 (x + y) / 2`` on the normalised extended grid.
* ``blur_and_observe`` restates harness.py:170-198: valid convolution of the
  extended truth (no boundary model enters the data) plus
  ``PCG64(noise_seed).standard_normal`` noise rescaled to an exact NSR.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def gen_psf(kind: str, m: int, sigma: float | None = None) -> np.ndarray:
    """Named 2D PSFs of half-width ``m`` (harness.py:147-167)."""
    if m < 1:
        raise ValueError(f"psf half-width must be >= 1, got {m}")
    if kind == "gaussian":
        if sigma is None or sigma <= 0:
            raise ValueError("gaussian psf needs sigma > 0")
        idx = np.arange(-m, m + 1, dtype=float)
        g = np.exp(-(idx[:, None] ** 2 + idx[None, :] ** 2) / (2.0 * sigma * sigma))
        return g / g.sum()
    if kind == "box":
        w = 2 * m + 1
        return np.full((w, w), 1.0 / (w * w))
    raise ValueError(f"unknown psf kind {kind!r}")


def gen_piecewise_image(n: int, m: int, rects: int, disks: int, seed: int,
                        ramp: bool = False) -> np.ndarray:
    """Seeded piecewise-constant truth on the extended ``(n+2m)^2`` grid."""
    total = n + 2 * m
    rng = np.random.Generator(np.random.PCG64(seed))
    img = np.full((total, total), 0.2)
    lo, hi = max(1, math.ceil(total / 16)), max(1, total // 4)
    for _ in range(rects):
        r0, c0 = rng.integers(0, total, size=2)
        h, w = rng.integers(lo, hi + 1, size=2)
        img[r0:r0 + h, c0:c0 + w] = rng.uniform()
    for _ in range(disks):
        cy, cx = rng.uniform(0, total, size=2)
        rad = rng.uniform(total / 32, total / 8)
        val = rng.uniform()
        r0, r1 = max(0, int(cy - rad) - 1), min(total, int(cy + rad) + 2)
        c0, c1 = max(0, int(cx - rad) - 1), min(total, int(cx + rad) + 2)
        yy, xx = np.ogrid[r0:r1, c0:c1]
        sub = (yy - cy) ** 2 + (xx - cx) ** 2 <= rad * rad
        img[r0:r1, c0:c1][sub] = val
    if ramp:
        coord = np.arange(total) / max(1, total - 1)
        img = img + 0.1 * (coord[:, None] + coord[None, :]) / 2.0
    return img


def _separable_factors(h: np.ndarray):
    """``(g1, g2)`` with ``h ~= outer(g1, g2)`` to 1e-14, else ``None``."""
    g1, g2 = h.sum(axis=1), h.sum(axis=0)
    total = h.sum()
    approx = np.outer(g1, g2) / total
    if np.abs(approx - h).max() <= 1e-14 * np.abs(h).max():
        return g1 / total, g2
    return None


def _valid_convolve_device(ext: np.ndarray, h: np.ndarray, factors, device):
    """The valid convolution on a CUDA device through the library (``tvd_valid_convolve``):
    with ``factors`` (the separable pair of :func:`_separable_factors`) it runs the same
    shifted-slice sums in the same order and rounding as the host path below (bit-identical);
    otherwise a direct 2D convolution."""
    import ctypes

    import torch

    from . import _native as nat

    dev = torch.device(device)
    e = torch.from_numpy(np.ascontiguousarray(ext, dtype=float)).to(dev)
    k = h.shape[0]
    n = ext.shape[0] - k + 1
    out = torch.empty((n, n), dtype=torch.float64, device=dev)
    hc = np.ascontiguousarray(h, dtype=float)
    f1 = f2 = None
    if factors is not None:
        f1 = np.ascontiguousarray(factors[0], dtype=float)
        f2 = np.ascontiguousarray(factors[1], dtype=float)
    ctx = nat.context(dev)
    nat.check(nat.load().tvd_valid_convolve(
        ctx, e.data_ptr(), ext.shape[0], hc.ctypes.data, k,
        None if f1 is None else f1.ctypes.data, None if f2 is None else f2.ctypes.data,
        out.data_ptr()))
    return out.cpu().numpy()


def valid_convolve(ext: np.ndarray, h: np.ndarray, exact: bool = True,
                   device=None) -> np.ndarray:
    """``convolve2d(ext, h, 'valid')`` for a symmetric PSF.

    ``exact`` uses ``scipy.signal.convolve2d`` -- the very routine the
    reference's ``blur_and_observe`` calls (harness.py:186) -- so observations
    are bit-identical to the reference's; otherwise a separable shifted-slice
    sum (fast at 8192^2, equal to rounding).
    """
    if exact:
        try:
            from scipy.signal import convolve2d
            return convolve2d(ext, h, mode="valid")
        except ImportError:
            pass
    k = h.shape[0]
    n = ext.shape[0] - k + 1
    sep = _separable_factors(h)
    if device is not None:
        return _valid_convolve_device(ext, h, sep, device)
    if sep is not None:
        g1, g2 = sep
        rows = np.zeros((ext.shape[0], n))
        for b in range(k):
            rows += g2[k - 1 - b] * ext[:, b:b + n]
        out = np.zeros((n, n))
        for a in range(k):
            out += g1[k - 1 - a] * rows[a:a + n, :]
        return out
    out = np.zeros((n, n))
    hf = h[::-1, ::-1]
    for a in range(k):
        for b in range(k):
            out += hf[a, b] * ext[a:a + n, b:b + n]
    return out


def blur_and_observe(ext: np.ndarray, h: np.ndarray, n: int, nsr: float,
                     seed: int, exact: bool = True, device=None) -> np.ndarray:
    """Exact blur of the extended truth plus seeded noise at an exact NSR (harness.py:170-198)."""
    if nsr < 0:
        raise ValueError("noise-to-signal ratio must be >= 0")
    clean = valid_convolve(np.asarray(ext, dtype=float), h, exact, device)
    if clean.shape != (n, n):
        raise ValueError(f"extended input {ext.shape} does not crop to {(n, n)}")
    if nsr == 0:
        return clean
    rng = np.random.Generator(np.random.PCG64(seed))
    g = rng.standard_normal(clean.shape)
    return clean + g * (nsr * np.linalg.norm(clean.ravel()) / np.linalg.norm(g.ravel()))


@dataclass(frozen=True)
class ProblemSpec:
    """One BASELINE.json configuration."""

    name: str
    n: int
    psf: str
    m: int
    sigma: float | None
    bc: str            # 'anti_reflective' | 'reflective'
    nsr: float
    alpha: float
    beta: float
    fp_steps: int
    tol: float
    rects: int
    disks: int
    ramp: bool = False
    problems: int = 1


CONFIGS = {
    "c1": ProblemSpec("c1", 128, "gaussian", 4, 1.5, "anti_reflective", 0.01, 1e-3, 0.1, 10, 1e-4, 12, 6),
    "c2a": ProblemSpec("c2a", 512, "gaussian", 7, 2.5, "anti_reflective", 0.01, 5e-4, 0.1, 15, 1e-4, 40, 20),
    "c2b": ProblemSpec("c2b", 512, "gaussian", 7, 2.5, "reflective", 0.01, 5e-4, 0.1, 15, 1e-4, 40, 20),
    "c3": ProblemSpec("c3", 2048, "gaussian", 15, 4.0, "anti_reflective", 0.005, 2e-4, 0.05, 20, 1e-5, 200, 100, ramp=True),
    "c4": ProblemSpec("c4", 1024, "gaussian", 10, 3.0, "anti_reflective", 0.01, 1e-3, 0.1, 10, 1e-4, 80, 40, problems=64),
    "c5": ProblemSpec("c5", 8192, "gaussian", 31, 8.0, "anti_reflective", 0.01, 1e-4, 0.05, 8, 1e-4, 2000, 1000),
}


def make_problem(spec: ProblemSpec, index: int = 0, exact: bool | None = None, device=None):
    """``(psf, v, u_true)`` for problem ``index`` (seeds 2023+i / 7+i).

    Config 4 alternates Gaussian 21x21 (even i) and the 11x11 box (odd i).
    ``exact`` (default: n <= 2048) selects the reference's own convolve2d; otherwise
    ``device`` (a torch device) runs the separable shifted-slice sum there.
    """
    if spec.name == "c4" and index % 2 == 1:
        h, m = gen_psf("box", 5), 5
    else:
        h, m = gen_psf(spec.psf, spec.m, spec.sigma), spec.m
    if exact is None:
        exact = spec.n <= 2048
    ext = gen_piecewise_image(spec.n, m, spec.rects, spec.disks, 2023 + index, spec.ramp)
    v = blur_and_observe(ext, h, spec.n, spec.nsr, 7 + index, exact,
                         None if exact else device)
    return h, v, ext[m:m + spec.n, m:m + spec.n].copy()
