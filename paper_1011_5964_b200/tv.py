"""Lagged-diffusivity operator on the GPU (mirror of reference tv.py:27-187).

``DiffusionOperator(u, beta, bc, spacing)`` computes the edge diffusivities
``a = 1/sqrt(|grad u|^2 + beta^2)`` (tv.py:42-71) with one stencil kernel and
applies the 5-point flux-form operator (tv.py:96-108).  Both kernels follow
the reference's floating-point operation order with explicit round-to-
nearest intrinsics, so ``a_h``, ``a_v``, ``L w`` and the block bands are
bit-identical to numpy's.

Ghost rules (tv.py:27-39): zero Neumann (the symmetric PCG systems) and
anti-reflective (odd reflection ``2 u_0 - u_1``), which makes ``L``
nonsymmetric -- its (0,+1)/(0,-1) and (+1,0)/(-1,0) bands differ at one end --
and routes the solve to BiCGstab (pipeline.py:196-198).
"""

from __future__ import annotations

from enum import Enum

import numpy as np
import torch

from . import _native as nat


class DiffusionBc(Enum):
    ZERO_NEUMANN = "zero_neumann"
    ANTI_REFLECTIVE = "anti_reflective"


_DBC = {DiffusionBc.ZERO_NEUMANN: nat.DBC_ZERO_NEUMANN,
        DiffusionBc.ANTI_REFLECTIVE: nat.DBC_ANTI_REFLECTIVE}


def _check_bc(bc: DiffusionBc) -> int:
    if bc not in _DBC:
        raise ValueError(f"unknown diffusion boundary condition {bc!r}")
    return _DBC[bc]


def diffusion_coefficients(u, beta: float, bc: DiffusionBc = DiffusionBc.ZERO_NEUMANN,
                           spacing: float = 1.0):
    """``(horizontal n x (n+1), vertical (n+1) x n)`` coefficients (tv.py:42-71)."""
    op = DiffusionOperator(u, beta, bc, spacing)
    if op.was_numpy:
        return op.a_h, op.a_v
    return op.a_h_device, op.a_v_device


class DiffusionOperator:
    """Device-resident lagged-diffusivity operator (tv.py:74-187)."""

    def __init__(self, u, beta: float, bc: DiffusionBc = DiffusionBc.ZERO_NEUMANN,
                 spacing: float = 1.0, device: torch.device | None = None) -> None:
        if beta <= 0:
            raise ValueError(f"beta must be positive, got {beta}")
        if spacing <= 0:
            raise ValueError(f"spacing must be positive, got {spacing}")
        self.bc_code = _check_bc(bc)
        t, was_np = nat.to_device(u, device)
        if t.ndim != 2 or t.shape[0] != t.shape[1]:
            raise ValueError(f"expected a square grid, got shape {tuple(t.shape)}")
        self.bc = bc
        self.beta = float(beta)
        self.spacing = float(spacing)
        self.ndim = 2
        self.n = n = int(t.shape[0])
        self.device = t.device
        self.was_numpy = was_np
        self.a_h_device = torch.empty((n, n + 1), dtype=torch.float64, device=t.device)
        self.a_v_device = torch.empty((n + 1, n), dtype=torch.float64, device=t.device)
        ctx = nat.context(t.device)
        nat.check(nat.load().tvd_diffusivity_bc(ctx, n, self.beta, self.spacing, self.bc_code,
                                                t.data_ptr(), self.a_h_device.data_ptr(),
                                                self.a_v_device.data_ptr()))
        self._bands: tuple[torch.Tensor, ...] | None = None

    @property
    def symmetric(self) -> bool:
        return self.bc is DiffusionBc.ZERO_NEUMANN

    @property
    def a_h(self) -> np.ndarray:
        return self.a_h_device.cpu().numpy()

    @property
    def a_v(self) -> np.ndarray:
        return self.a_v_device.cpu().numpy()

    def apply(self, w):
        """``L w`` (tv.py:96-108)."""
        t, was_np = nat.to_device(w, self.device)
        if tuple(t.shape) != (self.n, self.n):
            raise ValueError(f"expected shape {(self.n, self.n)}, got {tuple(t.shape)}")
        out = torch.empty_like(t)
        ctx = nat.context(self.device)
        nat.check(nat.load().tvd_diffusion_apply_bc(ctx, self.n, self.spacing, self.bc_code,
                                                    self.a_h_device.data_ptr(),
                                                    self.a_v_device.data_ptr(), t.data_ptr(),
                                                    out.data_ptr()))
        return nat.to_host_like(out, was_np)

    def bands_device(self) -> tuple[torch.Tensor, ...]:
        """``(diag n x n, inner_up, inner_lo n x (n-1), block_up, block_lo (n-1) x n)`` on the
        device (tv.py:138-175); up == lo for zero-Neumann ghosts."""
        if self._bands is None:
            n = self.n
            e = torch.empty
            kw = {"dtype": torch.float64, "device": self.device}
            diag = e((n, n), **kw)
            inner_up, inner_lo = e((n, max(n - 1, 1)), **kw), e((n, max(n - 1, 1)), **kw)
            block_up, block_lo = e((max(n - 1, 1), n), **kw), e((max(n - 1, 1), n), **kw)
            ctx = nat.context(self.device)
            nat.check(nat.load().tvd_diffusion_bands_bc(
                ctx, n, self.spacing, self.bc_code, self.a_h_device.data_ptr(),
                self.a_v_device.data_ptr(), diag.data_ptr(), inner_up.data_ptr(),
                inner_lo.data_ptr(), block_up.data_ptr(), block_lo.data_ptr()))
            self._bands = (diag, inner_up[:, : n - 1], inner_lo[:, : n - 1], block_up[: n - 1],
                           block_lo[: n - 1])
        return self._bands

    def diagonal_device(self) -> torch.Tensor:
        return self.bands_device()[0]

    def diagonal(self) -> np.ndarray:
        """Main diagonal incl. ghost substitution (tv.py:110-114)."""
        return self.diagonal_device().cpu().numpy()

    def block_banded(self) -> dict[tuple[int, int], np.ndarray]:
        """5-point stencil as block bands (tv.py:138-175)."""
        diag, iu, il, bu, bl = (b.cpu().numpy() for b in self.bands_device())
        return {(0, 0): diag, (0, 1): iu, (0, -1): il, (1, 0): bu, (-1, 0): bl}
