"""Blur operators on the GPU (mirror of reference blur.py:29-326).

``StructuredBlurOperator(psf, bc, n)`` keeps the reference interface --
``apply`` / ``apply_transpose`` (exact pad/convolve/crop semantics),
``apply_fast`` / ``apply_transpose_fast``, ``reblur_apply``, ``eigenvalues``,
``eigenvalue_grid``, ``transform`` -- but every apply runs on the B200:

* rank-1 PSFs (all BASELINE.json kernels) factor as ``H = H1_0 (x) H1_1``;
  each 1D operator is a banded matrix with the boundary extension folded into
  its first/last rows, applied by the banded row/column kernels.  The
  normal operator ``H^T H`` is applied as ``G_0 p G_1`` with the Gram band
  ``G = H1^T H1`` (half-width 2m), one row pass plus one column pass.
* other quadrantally symmetric PSFs use the direct 2D path (explicit
  extension + valid convolution; full convolution + fold for ``H^T``).

The fast-path names are kept for API compatibility; on the GPU both names
run the exact operator (the reference's own transform path agrees with it to
1e-10, blur.py:293-314, pkg/tests/test_blur.py:180-189).

Only REFLECTIVE and ANTI_REFLECTIVE are in scope (the transform-
diagonalisable BCs).
"""

from __future__ import annotations

import ctypes
import warnings
from enum import Enum

import numpy as np
import torch

from . import _native as nat
from .transforms import TransformKind


class BoundaryCondition(Enum):
    ZERO_DIRICHLET = "zero"
    PERIODIC = "periodic"
    REFLECTIVE = "reflective"
    ANTI_REFLECTIVE = "anti_reflective"


class UnsupportedBoundaryConditionError(ValueError):
    """Raised when an operation needs a transform-diagonalizable extension."""


_BC_CODE = {BoundaryCondition.REFLECTIVE: nat.BC_REFLECTIVE,
            BoundaryCondition.ANTI_REFLECTIVE: nat.BC_ANTI_REFLECTIVE}


class SymmetricPsf:
    """Normalized quadrantally symmetric 2D kernel (blur.py:53-102 validation rules)."""

    def __init__(self, coefficients) -> None:
        h = np.asarray(coefficients, dtype=float)
        if h.ndim not in (1, 2):
            raise ValueError("PSF must be 1D or 2D")
        if h.ndim == 1:
            raise NotImplementedError("1D signals are outside this build's scope (2D PCG path)")
        if h.shape[0] != h.shape[1]:
            raise ValueError(f"2D PSF must be square, got {h.shape}")
        if h.shape[0] % 2 != 1:
            raise ValueError(f"PSF needs odd length (2m+1), got {h.shape}")
        if not np.all(np.isfinite(h)):
            raise ValueError("PSF coefficients must be finite")
        scale = np.max(np.abs(h)) or 1.0
        symmetric = (np.allclose(h, h[::-1, :], rtol=0.0, atol=1e-13 * scale)
                     and np.allclose(h, h[:, ::-1], rtol=0.0, atol=1e-13 * scale))
        if not symmetric:
            raise ValueError("PSF must be symmetric (quadrantally symmetric in 2D)")
        total = h.sum()
        if total <= 0:
            raise ValueError("PSF must have positive sum")
        if abs(total - 1.0) > 1e-12:
            warnings.warn(f"PSF sum {total!r} differs from 1; renormalizing", stacklevel=2)
            h = h / total
        self.coefficients = np.ascontiguousarray(h)
        self.coefficients.setflags(write=False)

    @property
    def ndim(self) -> int:
        return self.coefficients.ndim

    @property
    def half_width(self) -> int:
        return (self.coefficients.shape[0] - 1) // 2

    def __repr__(self) -> str:
        return f"SymmetricPsf(ndim={self.ndim}, half_width={self.half_width})"


class StructuredBlurOperator:
    """GPU blur under a reflective or anti-reflective extension (blur.py:197-326)."""

    def __init__(self, psf: SymmetricPsf, bc: BoundaryCondition, n: int,
                 device: torch.device | None = None) -> None:
        if not isinstance(psf, SymmetricPsf):
            psf = SymmetricPsf(psf)
        if psf.half_width >= n:
            raise ValueError(f"PSF half-width {psf.half_width} must be below size {n}")
        if bc not in _BC_CODE:
            raise UnsupportedBoundaryConditionError(
                f"boundary condition {bc.value!r} is outside this build's scope")
        self.psf = psf
        self.bc = bc
        self.n = int(n)
        self.ndim = 2
        self.device = device or nat.default_device()
        self._eig_host: np.ndarray | None = None
        self._eig_dev: torch.Tensor | None = None
        lib = nat.load()
        ctx = nat.context(self.device)
        h = psf.coefficients
        out = ctypes.c_void_p()
        sep = ctypes.c_int()
        nat.check(lib.tvd_blur_create(ctx, self.n, h.ctypes.data, h.shape[0], _BC_CODE[bc],
                                      ctypes.byref(out), ctypes.byref(sep)))
        self._handle = out.value
        self.separable = bool(sep.value)
        self._lib = lib

    def __del__(self) -> None:
        h = getattr(self, "_handle", None)
        if h:
            try:
                self._lib.tvd_blur_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._handle = None

    @property
    def handle(self) -> int:
        return self._handle

    # -- applies ---------------------------------------------------------
    def _run(self, u, which: int):
        t, was_np = self._check_shape(u)
        out = torch.empty_like(t)
        nat.context(self.device)
        if which == 2:
            nat.check(self._lib.tvd_blur_normal_apply(self._handle, t.data_ptr(), out.data_ptr()))
        else:
            nat.check(self._lib.tvd_blur_apply(self._handle, t.data_ptr(), out.data_ptr(), which))
        return nat.to_host_like(out, was_np)

    def apply(self, u):
        """Exact ``H u`` (blur.py:226-234)."""
        return self._run(u, 0)

    def apply_transpose(self, u):
        """Exact ``H^T u`` (blur.py:236-247)."""
        return self._run(u, 1)

    def normal_apply(self, u):
        """``H^T H u`` (``H H u`` for reflective, pipeline.py:167-179) in one fused pass pair."""
        return self._run(u, 2)

    reblur_apply = apply

    def apply_fast(self, u):
        """Transform-domain ``H u``: analysis, eigenvalue scaling, synthesis (blur.py:293-300).
        Equal to :meth:`apply` up to rounding; the solvers use the exact band form."""
        from .transforms import tensor_apply_2d

        t, was_np = self._check_shape(u)
        kind = self.transform
        mid = self.eigenvalues_device() * tensor_apply_2d(kind, t, inverse=True)
        return nat.to_host_like(tensor_apply_2d(kind, mid), was_np)

    def apply_transpose_fast(self, u):
        """Transform-domain ``H^T u = X^-T (lam .* X^T u)`` (blur.py:302-314): the
        anti-reflective ``T`` is not orthogonal, so this runs its transposed forms."""
        from .transforms import tensor_apply_2d

        t, was_np = self._check_shape(u)
        kind = self.transform
        mid = self.eigenvalues_device() * tensor_apply_2d(kind, t, transpose=True)
        return nat.to_host_like(tensor_apply_2d(kind, mid, inverse=True, transpose=True), was_np)

    # -- eigen structure -------------------------------------------------
    @property
    def transform(self) -> TransformKind:
        if self.bc is BoundaryCondition.REFLECTIVE:
            return TransformKind.DCT
        return TransformKind.ANTI_REFLECTIVE

    def eigenvalue_grid(self) -> np.ndarray:
        """Symbol sample angles (blur.py:265-274)."""
        n = self.n
        if self.bc is BoundaryCondition.REFLECTIVE:
            return np.arange(n) * np.pi / n
        return np.concatenate([np.arange(n - 1) * np.pi / (n - 1), [0.0]])

    def eigenvalues_device(self) -> torch.Tensor:
        """``lam[s,t]`` on the device (computed once, blur.py:276-291)."""
        if self._eig_dev is None:
            lam = torch.empty((self.n, self.n), dtype=torch.float64, device=self.device)
            nat.context(self.device)
            nat.check(self._lib.tvd_blur_eigenvalues(self._handle, lam.data_ptr()))
            self._eig_dev = lam
        return self._eig_dev

    def eigenvalues(self) -> np.ndarray:
        if self._eig_host is None:
            lam = self.eigenvalues_device().cpu().numpy()
            lam.setflags(write=False)
            self._eig_host = lam
        return self._eig_host

    def _check_shape(self, u):
        t, was_np = nat.to_device(u, self.device)
        if tuple(t.shape) != (self.n, self.n):
            raise ValueError(f"expected shape {(self.n, self.n)}, got {tuple(t.shape)}")
        return t, was_np
