"""CPU restatement of the reference's PCG hot path (numpy + scipy.fft).

TEST INFRASTRUCTURE ONLY -- the checker for ``tests/`` and the timed CPU
baseline for ``bench.py``.  The product package never imports this module.

Every function below restates one piece of the reference package ``tvdeblur``
(``/root/reference/pkg/src/tvdeblur``, cited as ``<module>.py:<lines>``).  The
reference's arithmetic lives in third-party code that the reference does not
vendor and does not pin (``pkg/pyproject.toml:10-13`` lists bare ``numpy`` and
``scipy``): ``scipy.fft`` (pocketfft) for the DST-I / DCT and ``scipy.signal
.convolve2d`` for the exact blur.  Here the transforms are restated from their
published definitions on top of a plain complex/real FFT (``scipy.fft.fft`` /
``rfft``, which accept ``workers=`` so the CPU baseline can use every host
core), and the blur is restated as a direct shifted-slice sum.  The build
container has scipy 1.18.1 / numpy 2.3.5; ``tests/test_oracle_golden.py``
pins this module against outputs of the reference itself
(``tests/golden/``, produced by ``tests/golden/make_golden.py``).

Scope: 2D, blur BCs REFLECTIVE / ANTI_REFLECTIVE, diffusion BCs ZERO_NEUMANN /
ANTI_REFLECTIVE, NORMAL and REBLUR formulations, PCG and right-preconditioned
BiCGstab, preconditioner selectors NONE / DIAG / X / D_X / X_D (families R = DCT,
M = SINE_HAT, P = anti-reflective algebra) -- the rows of SURVEY.md section 8
including row f2.
"""

from __future__ import annotations

import math
import os

import numpy as np
from scipy import fft as _sfft

#: FFT worker threads (1 = the reference's own single-threaded behaviour,
#: ``transforms.py:56`` calls scipy.fft without ``workers=``).
WORKERS = 1


def set_workers(n: int | None) -> None:
    global WORKERS
    WORKERS = int(n) if n else (os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# transforms  (transforms.py:52-171)
# ---------------------------------------------------------------------------

def dst1(v: np.ndarray, axis: int = -1) -> np.ndarray:
    """Orthonormal DST-I ``S_N`` along ``axis`` (transforms.py:52-56).

    Published algorithm: odd extension of length ``2(N+1)``; its DFT is
    ``-2i * sum_j x_j sin(pi j k / (N+1))``.
    """
    x = np.moveaxis(np.asarray(v, dtype=float), axis, -1)
    n_int = x.shape[-1]
    period = n_int + 1
    ext = np.zeros(x.shape[:-1] + (2 * period,))
    ext[..., 1:period] = x
    ext[..., period + 1:] = -x[..., ::-1]
    spec = _sfft.rfft(ext, axis=-1, workers=WORKERS)
    out = spec[..., 1:period].imag * (-math.sqrt(0.5 / period))
    return np.moveaxis(out, -1, axis)


def _dct_weights(n: int) -> np.ndarray:
    w = np.full(n, math.sqrt(2.0 / n))
    w[0] = math.sqrt(1.0 / n)
    return w


def dct_analysis(v: np.ndarray, axis: int = -1) -> np.ndarray:
    """``C^T v`` = orthonormal DCT-II (transforms.py:59-69, ``inverse=True``).

    Published algorithm (Makhoul 1980): even samples forward, odd samples
    reversed, one length-n FFT, rotate by ``exp(-i pi k / 2n)``.
    """
    x = np.moveaxis(np.asarray(v, dtype=float), axis, -1)
    n = x.shape[-1]
    reordered = np.concatenate([x[..., 0::2], x[..., 1::2][..., ::-1]], axis=-1)
    spec = _sfft.fft(reordered, axis=-1, workers=WORKERS)
    k = np.arange(n)
    out = (np.exp(-1j * np.pi * k / (2 * n)) * spec).real * _dct_weights(n)
    return np.moveaxis(out, -1, axis)


def dct_synthesis(v: np.ndarray, axis: int = -1) -> np.ndarray:
    """``C v`` = orthonormal DCT-III (transforms.py:59-69, ``inverse=False``)."""
    y = np.moveaxis(np.asarray(v, dtype=float), axis, -1)
    n = y.shape[-1]
    k = np.arange(n)
    unscaled = y / _dct_weights(n)
    mirrored = np.zeros_like(unscaled)
    mirrored[..., 1:] = unscaled[..., :0:-1]
    spec = np.exp(1j * np.pi * k / (2 * n)) * (unscaled - 1j * mirrored)
    seq = _sfft.ifft(spec, axis=-1, workers=WORKERS).real
    half = (n + 1) // 2
    out = np.empty_like(seq)
    out[..., 0::2] = seq[..., :half]
    out[..., 1::2] = seq[..., half:][..., ::-1]
    return np.moveaxis(out, -1, axis)


def _interior(ndim: int, axis: int, sl: slice) -> tuple:
    idx = [slice(None)] * ndim
    idx[axis] = sl
    return tuple(idx)


def sinehat(v: np.ndarray, axis: int = -1) -> np.ndarray:
    """``Shat = diag(1, S_{n-2}, 1)`` (transforms.py:72-81)."""
    x = np.asarray(v, dtype=float)
    if x.shape[axis] < 3:
        raise ValueError("Shat_n requires length >= 3")
    out = x.copy()
    inner = _interior(x.ndim, axis, slice(1, -1))
    out[inner] = dst1(x[inner], axis=axis)
    return out


def _ar_cols(n: int) -> tuple[np.ndarray, np.ndarray]:
    """``S_{n-2} p`` and ``S_{n-2} J p`` with ``p_j = 1 - j/(n-1)`` (transforms.py:84-93)."""
    ramp = 1.0 - np.arange(1, n - 1, dtype=float) / (n - 1)
    return dst1(ramp), dst1(ramp[::-1])


def antireflective(v: np.ndarray, inverse: bool = False, transpose: bool = False,
                   axis: int = -1) -> np.ndarray:
    """AR transform ``T = Shat (I + U)`` and its inverse / transposes (transforms.py:96-140)."""
    x = np.moveaxis(np.asarray(v, dtype=float), axis, -1)
    n = x.shape[-1]
    if n < 3:
        raise ValueError("T_n requires length >= 3")
    ql, qr = _ar_cols(n)
    first, last, mid = x[..., :1], x[..., -1:], x[..., 1:-1]
    out = x.copy()
    if not transpose and not inverse:          # Shat (v + U v)
        out[..., 1:-1] = dst1(mid + first * ql + last * qr)
    elif not transpose:                        # (I - U) Shat v
        out[..., 1:-1] = dst1(mid) - (first * ql + last * qr)
    elif not inverse:                          # (I + U^T) Shat v
        s = dst1(mid)
        out[..., 1:-1] = s
        out[..., :1] += (s * ql).sum(axis=-1, keepdims=True)
        out[..., -1:] += (s * qr).sum(axis=-1, keepdims=True)
    else:                                      # Shat (I - U^T) v
        out[..., :1] -= (mid * ql).sum(axis=-1, keepdims=True)
        out[..., -1:] -= (mid * qr).sum(axis=-1, keepdims=True)
        out[..., 1:-1] = dst1(mid)
    return np.moveaxis(out, -1, axis)


def apply_1d(kind: str, v, inverse=False, transpose=False, axis=-1) -> np.ndarray:
    """Dispatcher (transforms.py:143-156); kinds 'dst1', 'dct', 'sine_hat', 'ar'."""
    if kind == "dst1":
        return dst1(v, axis)
    if kind == "sine_hat":
        return sinehat(v, axis)
    if kind == "dct":
        analysis = inverse != transpose
        return dct_analysis(v, axis) if analysis else dct_synthesis(v, axis)
    if kind == "ar":
        return antireflective(v, inverse, transpose, axis)
    raise ValueError(kind)


def tensor_2d(kind: str, g, inverse=False, transpose=False) -> np.ndarray:
    """``X G X^T``: axis 0 then axis 1 (transforms.py:159-171)."""
    g = np.asarray(g, dtype=float)
    return apply_1d(kind, apply_1d(kind, g, inverse, transpose, 0), inverse, transpose, 1)


# ---------------------------------------------------------------------------
# blur  (blur.py:45-50, 137-190, 197-326)
# ---------------------------------------------------------------------------

def _extend_axis0(u: np.ndarray, m: int, bc: str) -> np.ndarray:
    """Boundary extension by m along axis 0 from the scalar rules (blur.py:45-50)."""
    n = u.shape[0]
    out = np.empty((n + 2 * m,) + u.shape[1:])
    out[m:m + n] = u
    for j in range(1, m + 1):
        if bc == "reflective":           # u[-j] = u[j-1]
            lo, hi = u[j - 1], u[n - j]
        elif bc == "anti_reflective":    # u[-j] = 2 u[0] - u[j]
            lo, hi = 2.0 * u[0] - u[j], 2.0 * u[n - 1] - u[n - 1 - j]
        else:
            raise ValueError(bc)
        out[m - j] = lo
        out[m + n - 1 + j] = hi
    return out


def extend2(u: np.ndarray, m: int, bc: str) -> np.ndarray:
    """2D extension; corners compose the axis rules (blur.py:163-167)."""
    return _extend_axis0(_extend_axis0(u, m, bc).T, m, bc).T


def blur(u: np.ndarray, h: np.ndarray, bc: str) -> np.ndarray:
    """Exact ``H u``: extend, valid convolution, crop (blur.py:226-234)."""
    u = np.asarray(u, dtype=float)
    n = u.shape[0]
    m = (h.shape[0] - 1) // 2
    ext = extend2(u, m, bc)
    out = np.zeros((n, n))
    hf = h[::-1, ::-1]
    for a in range(2 * m + 1):
        for b in range(2 * m + 1):
            out += hf[a, b] * ext[a:a + n, b:b + n]
    return out


def _fold_axis0(w: np.ndarray, m: int, bc: str) -> np.ndarray:
    """Adjoint of the extension along axis 0 (blur.py:170-190)."""
    core = w[m:w.shape[0] - m].copy()
    lo, hi = w[:m], w[w.shape[0] - m:]
    if bc == "reflective":
        core[:m] += lo[::-1]
        core[-m:] += hi[::-1]
    elif bc == "anti_reflective":
        core[0] += 2.0 * lo.sum(axis=0)
        core[1:m + 1] -= lo[::-1]
        core[-1] += 2.0 * hi.sum(axis=0)
        core[-m - 1:-1] -= hi[::-1]
    else:
        raise ValueError(bc)
    return core


def blur_transpose(w: np.ndarray, h: np.ndarray, bc: str) -> np.ndarray:
    """Exact ``H^T w``: full convolution then fold (blur.py:236-247)."""
    w = np.asarray(w, dtype=float)
    n = w.shape[0]
    m = (h.shape[0] - 1) // 2
    full = np.zeros((n + 2 * m, n + 2 * m))
    for a in range(2 * m + 1):
        for b in range(2 * m + 1):
            full[a:a + n, b:b + n] += h[a, b] * w
    return _fold_axis0(_fold_axis0(full, m, bc).T, m, bc).T


def eigen_grid(bc: str, n: int) -> np.ndarray:
    """Symbol sample angles (blur.py:265-274)."""
    if bc == "reflective":
        return np.arange(n) * np.pi / n
    if bc == "anti_reflective":
        return np.concatenate([np.arange(n - 1) * np.pi / (n - 1), [0.0]])
    raise ValueError(bc)


def blur_eigenvalues(h: np.ndarray, bc: str, n: int) -> np.ndarray:
    """``lam[s,t] = sum_jk h[j,k] cos(j y_s) cos(k y_t)`` (blur.py:137-160, 276-291)."""
    m = (h.shape[0] - 1) // 2
    y = eigen_grid(bc, n)
    c = np.cos(np.multiply.outer(y, np.arange(-m, m + 1)))
    return c @ h @ c.T


def _fast_kind(bc: str) -> str:
    return "dct" if bc == "reflective" else "ar"


def blur_fast(u, lam, bc: str) -> np.ndarray:
    """Transform-diagonalised ``H u`` (blur.py:293-300)."""
    k = _fast_kind(bc)
    return tensor_2d(k, lam * tensor_2d(k, u, inverse=True))


def blur_transpose_fast(u, lam, bc: str) -> np.ndarray:
    """Transform-diagonalised ``H^T u`` (blur.py:302-314)."""
    k = _fast_kind(bc)
    return tensor_2d(k, lam * tensor_2d(k, u, transpose=True), inverse=True, transpose=True)


# ---------------------------------------------------------------------------
# total-variation diffusion  (tv.py:42-175, zero-Neumann ghosts)
# ---------------------------------------------------------------------------

def _ghost_pad(u: np.ndarray, bc: str) -> np.ndarray:
    """One ghost layer (tv.py:27-39): 'zn' copies the border (``symmetric``), 'ar' is the
    odd reflection ``u_{-1} = 2 u_0 - u_1`` (``reflect``, ``reflect_type='odd'``)."""
    u = np.asarray(u, dtype=float)
    if bc == "zn":
        return np.pad(u, 1, mode="edge")
    if bc == "ar":
        return np.pad(u, 1, mode="reflect", reflect_type="odd")
    raise ValueError(bc)


def diffusivity(u: np.ndarray, beta: float, spacing: float = 1.0, bc: str = "zn"):
    """Edge coefficients ``1/sqrt(|grad u|^2 + beta^2)`` (tv.py:42-71).

    Returns ``(a_h, a_v)`` of shapes ``n x (n+1)`` and ``(n+1) x n``.
    """
    g = _ghost_pad(u, bc)
    dx = (g[:, 1:] - g[:, :-1]) / spacing      # (n+2) x (n+1)
    dy = (g[1:, :] - g[:-1, :]) / spacing      # (n+1) x (n+2)
    cross_x = 0.25 * (dy[:-1, :-1] + dy[1:, :-1] + dy[:-1, 1:] + dy[1:, 1:])
    cross_y = 0.25 * (dx[:-1, :-1] + dx[:-1, 1:] + dx[1:, :-1] + dx[1:, 1:])
    bb = beta * beta
    a_h = 1.0 / np.sqrt(dx[1:-1, :] ** 2 + cross_x ** 2 + bb)
    a_v = 1.0 / np.sqrt(dy[:, 1:-1] ** 2 + cross_y ** 2 + bb)
    return a_h, a_v


def diffusion_apply(a_h, a_v, w, spacing: float = 1.0, bc: str = "zn") -> np.ndarray:
    """5-point flux form ``L w`` with zero-Neumann or AR ghosts (tv.py:96-108)."""
    g = _ghost_pad(w, bc)
    fx = a_h * (g[1:-1, 1:] - g[1:-1, :-1])
    fy = a_v * (g[1:, 1:-1] - g[:-1, 1:-1])
    return -(1.0 / (spacing * spacing)) * ((fx[:, 1:] - fx[:, :-1]) + (fy[1:, :] - fy[:-1, :]))


def diffusion_bands(a_h, a_v, spacing: float = 1.0, bc: str = "zn"):
    """Block bands of L (tv.py:138-175).

    Returns ``{(block_off, inner_off): array}`` with the reference's layout:
    (0,0) n x n, (0,+-1) n x (n-1), (+-1,0) (n-1) x n.  With AR ghosts the border
    cells lose twice their boundary edge and the first / last off-diagonals gain it
    (``w_{-1} = 2 w_0 - w_1``), so the +-1 bands differ at one end.
    """
    s = 1.0 / (spacing * spacing)
    diag = a_h[:, :-1] + a_h[:, 1:] + a_v[:-1, :] + a_v[1:, :]
    inner_up = -a_h[:, 1:-1]
    inner_lo = -a_h[:, 1:-1]
    block_up = -a_v[1:-1, :]
    block_lo = -a_v[1:-1, :]
    k = 1.0 if bc == "zn" else 2.0
    diag[:, 0] -= k * a_h[:, 0]
    diag[:, -1] -= k * a_h[:, -1]
    diag[0, :] -= k * a_v[0, :]
    diag[-1, :] -= k * a_v[-1, :]
    if bc == "ar":
        inner_up[:, 0] += a_h[:, 0]
        inner_lo[:, -1] += a_h[:, -1]
        block_up[0, :] += a_v[0, :]
        block_lo[-1, :] += a_v[-1, :]
    return {(0, 0): s * diag, (0, 1): s * inner_up, (0, -1): s * inner_lo,
            (1, 0): s * block_up, (-1, 0): s * block_lo}


# ---------------------------------------------------------------------------
# transform-algebra projections  (precond.py:82-199, 369-411, 419-573)
# ---------------------------------------------------------------------------

def _sine_band(band: np.ndarray, d: int, size: int) -> np.ndarray:
    """Band contribution to ``diag(S A S)`` for the size-``size`` sine algebra (precond.py:106-121).

    ``lam_t = (1/(N+1)) sum_i b_i [cos(d t th) - cos((2i+2+d) t th)]``, ``th = pi/(N+1)``;
    the second sum is a real FFT of the band scattered onto slots ``d+2+2i``.
    """
    d = abs(d)
    band = np.asarray(band, dtype=float)
    if size - d <= 0 or band.shape[-1] == 0:
        return np.zeros(band.shape[:-1] + (size,))
    period = size + 1
    slots = np.zeros(band.shape[:-1] + (2 * period,))
    slots[..., d + 2: d + 2 + 2 * (size - d): 2] = band
    far = _sfft.rfft(slots, axis=-1, workers=WORKERS)[..., 1:period].real
    t = np.arange(1, size + 1)
    near = band.sum(axis=-1, keepdims=True) * np.cos(d * t * np.pi / period)
    return (near - far) / period


def _cosine_band(band: np.ndarray, d: int, n: int) -> np.ndarray:
    """Band contribution to ``diag(C^T A C)`` (precond.py:82-103)."""
    d = abs(d)
    band = np.asarray(band, dtype=float)
    if n - d <= 0 or band.shape[-1] == 0:
        return np.zeros(band.shape[:-1] + (n,))
    slots = np.zeros(band.shape[:-1] + (2 * n,))
    slots[..., d + 1: d + 1 + 2 * (n - d): 2] = band
    far = _sfft.rfft(slots, axis=-1, workers=WORKERS)[..., :n].real
    t = np.arange(n)
    weight = np.where(t == 0, 1.0, 2.0) / n
    near = band.sum(axis=-1, keepdims=True) * np.cos(d * t * np.pi / n)
    return 0.5 * weight * (near + far)


def project_1d(family: str, bands: dict, n: int) -> np.ndarray:
    """Algebra eigenvalues of a banded matrix, batched (precond.py:168-199).

    family 'dct' (cosine algebra) or 'sine_hat' (bordered sine algebra).
    """
    shape = next(iter(bands.values())).shape[:-1]
    if family == "dct":
        out = np.zeros(shape + (n,))
        for d, b in bands.items():
            out = out + _cosine_band(b, d, n)
        return out
    if family == "sine_hat":
        out = np.zeros(shape + (n,))
        if 0 in bands:
            out[..., 0] = bands[0][..., 0]
            out[..., -1] = bands[0][..., -1]
        inner = np.zeros(shape + (n - 2,))
        for d, b in bands.items():
            sub = np.asarray(b, dtype=float)[..., 1: n - 1 - abs(d)]
            if sub.shape[-1] > 0:
                inner = inner + _sine_band(sub, d, n - 2)
        out[..., 1:-1] = inner
        return out
    if family == "ar":
        # anti-reflective algebra (precond.py:156-165, 186-196): sine projection of the
        # interior, its first-column representer z, border eigenvalue 2 sum(z) - z_0
        if n < 5:
            raise ValueError("anti-reflective projection requires n >= 5")
        inner = np.zeros(shape + (n - 2,))
        for d, b in bands.items():
            sub = np.asarray(b, dtype=float)[..., 1: n - 1 - abs(d)]
            if sub.shape[-1] > 0:
                inner = inner + _sine_band(sub, d, n - 2)
        z = _z_from_sine(inner)
        border = 2.0 * z.sum(axis=-1) - z[..., 0]
        out = np.zeros(shape + (n,))
        out[..., 0] = border
        out[..., 1:-1] = inner
        out[..., -1] = border
        return out
    raise ValueError(family)


def _z_from_sine(lam: np.ndarray) -> np.ndarray:
    """First-column representer of ``S diag(lam) S`` (precond.py:134-153): the first
    column is ``S (lam * s_1)`` and equals ``z`` minus itself shifted up by two, so
    ``z_k = col_k + z_{k+2}`` (suffix sums over each parity class)."""
    size = lam.shape[-1]
    t = np.arange(1, size + 1)
    first = np.sqrt(2.0 / (size + 1)) * np.sin(t * np.pi / (size + 1))
    col = dst1(lam * first)
    z = col.copy()
    for par in (size - 1, size - 2):
        if par >= 0:
            z[..., par::-2] = np.cumsum(col[..., par::-2], axis=-1)
    return z


def project_2d(family: str, blocks: dict, n: int) -> np.ndarray:
    """Two-level projection ``lam[s, t]`` (precond.py:369-395)."""
    per_offset: dict[int, dict[int, np.ndarray]] = {}
    for (do, di), b in blocks.items():
        per_offset.setdefault(do, {})[di] = b
    stage2 = {do: project_1d(family, inner, n).T for do, inner in per_offset.items()}
    return project_1d(family, stage2, n).T


FAMILY = {"R": "dct", "M": "sine_hat", "P": "ar"}


def scale_blocks(blocks: dict, s: np.ndarray) -> dict:
    """``s_i s_j L_ij`` on block bands (precond.py:501-513)."""
    out = {}
    for (do, di), b in blocks.items():
        r, c = b.shape
        r0, c0, r1, c1 = max(0, -do), max(0, -di), max(0, do), max(0, di)
        out[(do, di)] = b * s[r0:r0 + r, c0:c0 + c] * s[r1:r1 + r, c1:c1 + c]
    return out


class PreconditionerIndefinite(RuntimeError):
    def __init__(self, kind, alpha, smallest):
        super().__init__(f"preconditioner {kind!r} indefinite (min {smallest!r})")
        self.kind, self.alpha, self.min_eigenvalue = kind, alpha, smallest


def assemble(kind: str, lam_h: np.ndarray, blocks: dict, alpha: float):
    """Eigenvalues (+ optional ``d_sqrt``) of kinds R/D_R/R_D/M/D_M/M_D (precond.py:516-573).

    Returns ``(eigenvalues, inverse_eigenvalues, d_sqrt_or_None, n_clamped)``.
    """
    base = kind.replace("D_", "").replace("_D", "")
    fam = FAMILY[base]
    n = lam_h.shape[0]
    d = 1.0 + alpha * blocks[(0, 0)]
    if d.min() <= 0:
        raise PreconditionerIndefinite(kind, alpha, float(d.min()))
    d_sqrt = None
    if kind.endswith("_D"):
        s = d ** -0.5
        lam_d = project_2d(fam, {(0, 0): s}, n)
        lam = lam_h * lam_h * lam_d * lam_d + alpha * project_2d(fam, scale_blocks(blocks, s), n)
    else:
        lam = lam_h * lam_h + alpha * project_2d(fam, blocks, n)
        if kind.startswith("D_"):
            d_sqrt = np.sqrt(d)
    smallest = float(lam.min())
    if smallest <= 0.0:
        raise PreconditionerIndefinite(kind, alpha, smallest)
    floor = 1e-14 * float(lam.max())
    clamped = int(np.count_nonzero(lam < floor))
    return lam, 1.0 / np.maximum(lam, floor), d_sqrt, clamped


def precond_solve(family: str, lam_inv: np.ndarray, r: np.ndarray, d_sqrt=None) -> np.ndarray:
    """``M^{-1} r`` (precond.py:456-477)."""
    x = r if d_sqrt is None else r / d_sqrt
    z = tensor_2d(family, lam_inv * tensor_2d(family, x, inverse=True))
    return z if d_sqrt is None else z / d_sqrt


# ---------------------------------------------------------------------------
# PCG  (krylov.py:70-116)
# ---------------------------------------------------------------------------

class PcgIndefinite(RuntimeError):
    def __init__(self, iteration, curvature):
        super().__init__(f"nonpositive curvature {curvature!r} at iteration {iteration}")
        self.iteration, self.curvature = iteration, curvature


class PcgDivergence(RuntimeError):
    def __init__(self, iteration):
        super().__init__(f"non-finite values at iteration {iteration}")
        self.iteration = iteration


def pcg(apply_a, apply_minv, b, x0, tol: float, max_iterations: int,
        record_history: bool = False):
    """Textbook PCG with the reference's check order (krylov.py:82-116).

    Returns ``(x, iterations, history, converged)``.
    """
    minv = apply_minv or (lambda t: t)
    x = np.array(x0, dtype=float, copy=True)
    r = np.asarray(b, dtype=float) - apply_a(x)
    r0 = float(np.sqrt(np.dot(r.ravel(), r.ravel())))
    hist: list[float] = []
    if r0 == 0.0:
        return x, 0, np.array(hist), True
    z = minv(r)
    p = z.copy()
    rz = float(np.dot(r.ravel(), z.ravel()))
    for k in range(1, max_iterations + 1):
        q = apply_a(p)
        gamma = float(np.dot(p.ravel(), q.ravel()))
        if not np.isfinite(gamma):
            raise PcgDivergence(k)
        if gamma <= 0.0:
            raise PcgIndefinite(k, gamma)
        step = rz / gamma
        x += step * p
        r -= step * q
        rel = float(np.sqrt(np.dot(r.ravel(), r.ravel()))) / r0
        if not np.isfinite(rel):
            raise PcgDivergence(k)
        if record_history:
            hist.append(rel)
        if rel < tol:
            return x, k, np.array(hist), True
        z = minv(r)
        rz_next = float(np.dot(r.ravel(), z.ravel()))
        p = z + (rz_next / rz) * p
        rz = rz_next
    return x, max_iterations, np.array(hist), False


class SolverBreakdown(RuntimeError):
    def __init__(self, iteration, reason):
        super().__init__(f"pbicgstab breakdown at iteration {iteration}: {reason}")
        self.iteration, self.reason = iteration, reason


def pbicgstab(apply_a, apply_minv, b, x0, tol: float, max_iterations: int,
              record_history: bool = False):
    """Right-preconditioned BiCGstab with the reference's checks (krylov.py:119-174).

    Returns ``(x, iterations, history, converged)``.
    """
    minv = apply_minv or (lambda t: t)
    dot = lambda a, c: float(np.dot(a.ravel(), c.ravel()))  # noqa: E731
    b = np.asarray(b, dtype=float)
    x = np.array(x0, dtype=float, copy=True)
    r = b - apply_a(x)
    r0 = float(np.sqrt(dot(r, r)))
    hist: list[float] = []
    if r0 == 0.0:
        return x, 0, np.array(hist), True
    rs = r.copy()
    rho, alpha, omega = 1.0, 1.0, 1.0
    v = np.zeros_like(r)
    p = np.zeros_like(r)
    for k in range(1, max_iterations + 1):
        rho_next = dot(rs, r)
        if abs(rho_next) < 1e-30 * r0 * r0:
            raise SolverBreakdown(k, "rho vanished")
        beta = (rho_next / rho) * (alpha / omega)
        p = r + beta * (p - omega * v)
        p_hat = minv(p)
        v = apply_a(p_hat)
        denom = dot(rs, v)
        if abs(denom) < 1e-300:
            raise SolverBreakdown(k, "shadow angle vanished")
        alpha = rho_next / denom
        s = r - alpha * v
        rel = float(np.sqrt(dot(s, s))) / r0
        if not np.isfinite(rel):
            raise PcgDivergence(k)
        if rel < tol:
            x += alpha * p_hat
            if record_history:
                hist.append(rel)
            return x, k, np.array(hist), True
        s_hat = minv(s)
        t = apply_a(s_hat)
        tt = dot(t, t)
        if tt == 0.0:
            raise SolverBreakdown(k, "stabilizer direction vanished")
        omega = dot(t, s) / tt
        if abs(omega) < 1e-300:
            raise SolverBreakdown(k, "omega vanished")
        x += alpha * p_hat + omega * s_hat
        r = s - omega * t
        rel = float(np.sqrt(dot(r, r))) / r0
        if not np.isfinite(rel):
            raise PcgDivergence(k)
        if record_history:
            hist.append(rel)
        if rel < tol:
            return x, k, np.array(hist), True
        rho = rho_next
    return x, max_iterations, np.array(hist), False


# ---------------------------------------------------------------------------
# fixed-point driver  (pipeline.py:129-276)
# ---------------------------------------------------------------------------

def restore(v, h, bc: str, alpha: float, beta: float, selector: str = "x",
            fp_tol: float = 1e-300, fp_max: int = 10, tol: float = 1e-4,
            max_iterations: int = 2000, spacing: float = 1.0, fast: bool = True,
            pcg_hook=None, reblur: bool = False, bc_l: str = "zn"):
    """Lagged-diffusivity loop of ``pipeline.restore`` (pipeline.py:182-251).

    ``selector`` in {'none', 'diag', 'x', 'd_x', 'x_d'}.  ``pcg_hook``, if
    given, wraps each inner solve (used by bench.py to time only the PCG).
    Returns a dict with ``restored``, ``inner_iterations``, ``fp_steps``,
    ``gradient_norms``, ``fp_converged``, ``inner_converged``.
    """
    v = np.asarray(v, dtype=float)
    n = v.shape[0]
    lam_h = blur_eigenvalues(h, bc, n)
    if fast:
        fwd = lambda w: blur_fast(w, lam_h, bc)                       # noqa: E731
        back = fwd if bc == "reflective" else (lambda w: blur_transpose_fast(w, lam_h, bc))
    else:
        fwd = lambda w: blur(w, h, bc)                                # noqa: E731
        back = fwd if bc == "reflective" else (lambda w: blur_transpose(w, h, bc))
    if reblur:  # re-blurred normal equations: H applied twice (pipeline.py:173-174)
        back = fwd
    rhs = back(v)
    base = "R" if bc == "reflective" else ("P" if reblur else "M")
    fam = FAMILY[base]
    symmetric = not reblur and bc_l == "zn"  # pipeline.py:196-198
    solve = pcg_hook or (pcg if symmetric else pbicgstab)
    u = v.copy()
    counts, grads = [], []
    fp_converged, inner_ok = False, True
    for _ in range(fp_max):
        a_h, a_v = diffusivity(u, beta, spacing, bc_l)
        blocks = diffusion_bands(a_h, a_v, spacing, bc_l)

        def apply_a(w, a_h=a_h, a_v=a_v):
            return back(fwd(w)) + alpha * diffusion_apply(a_h, a_v, w, spacing, bc_l)

        grads.append(float(np.linalg.norm((apply_a(u) - rhs).ravel())))
        if selector == "x_d":
            d = 1.0 + alpha * blocks[(0, 0)]
            if d.min() <= 0:
                raise ValueError("nonpositive diagonal scaling")
            s = d ** -0.5
            _, lam_inv, _, _ = assemble(base + "_D", lam_h, blocks, alpha)
            x, its, _, ok = solve(lambda w: s * apply_a(s * w),
                                  lambda r: precond_solve(fam, lam_inv, r),
                                  s * rhs, u / s, tol, max_iterations)
            u_next = s * x
        else:
            if selector == "none":
                minv = None
            elif selector == "diag":
                d = 1.0 + alpha * blocks[(0, 0)]
                minv = lambda r, d=d: r / d                            # noqa: E731
            else:
                kind = base if selector == "x" else "D_" + base
                _, lam_inv, d_sqrt, _ = assemble(kind, lam_h, blocks, alpha)
                minv = lambda r, li=lam_inv, ds=d_sqrt: precond_solve(fam, li, r, ds)  # noqa: E731
            u_next, its, _, ok = solve(apply_a, minv, rhs, u, tol, max_iterations)
        counts.append(its)
        inner_ok = inner_ok and ok
        change = float(np.linalg.norm((u_next - u).ravel()))
        u = u_next
        scale = float(np.linalg.norm(u.ravel()))
        if scale > 0 and change / scale < fp_tol:
            fp_converged = True
            break
    return {"restored": u, "inner_iterations": counts, "fp_steps": len(counts),
            "gradient_norms": grads, "fp_converged": fp_converged,
            "inner_converged": inner_ok}
