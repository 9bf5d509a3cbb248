"""Lagged-diffusivity fixed-point driver on the GPU (mirror of reference pipeline.py:29-276).

``restore(v, psf, config, u_true)`` accepts the reference's
``RestorationConfig`` unchanged and returns the same ``RestorationReport``.
Everything between the initial host->device copy of ``v`` and the final copy
of the restored image stays resident in HBM: per FP step the diffusivity
kernel, the device preconditioner assembly and the device PCG
(``tvd_pcg_solve``) run back to back on the current torch stream.

Systems: the NORMAL formulation with zero-Neumann diffusion (symmetric, solved by the
device PCG) for reflective (R family) and anti-reflective (M family) blur -- the BASELINE
hot path -- and, as the reference does (pipeline.py:196-198), the REBLUR formulation and the
anti-reflective diffusion BC (nonsymmetric, solved by the device BiCGstab with the P family,
SURVEY.md 8f #2); selectors NONE / DIAG / X / D_X / X_D.  Preconditioners are assembled with
their positivity checks left on the device and resolved after each solve
(``FactoredPreconditioner.check``), so an FP step synchronises the host only where the
reference's report needs a scalar (gradient norm, FP change).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native as nat
from .blur import BoundaryCondition, StructuredBlurOperator, SymmetricPsf
from .krylov import DiagonalInverse, KrylovConfig, SolveOutcome, pbicgstab, pcg
from .precond import assemble_preconditioner
from .tv import DiffusionBc, DiffusionOperator


class Formulation(Enum):
    NORMAL = "normal"
    REBLUR = "reblur"


class PrecondSelector(Enum):
    NONE = "none"
    DIAG = "diag"
    X = "x"
    D_X = "d_x"
    X_D = "x_d"


_BASE_KIND = {
    (BoundaryCondition.REFLECTIVE, Formulation.NORMAL): "R",
    (BoundaryCondition.ANTI_REFLECTIVE, Formulation.NORMAL): "M",
    (BoundaryCondition.ANTI_REFLECTIVE, Formulation.REBLUR): "P",
}


class ConfigurationError(ValueError):
    """Invalid restoration configuration, detected before any compute (pipeline.py:56-57)."""


class InvalidScalingError(ValueError):
    """Diagonal scaling is not positive (pipeline.py:60-61)."""


@dataclass(frozen=True)
class RestorationConfig:
    bc_h: BoundaryCondition
    alpha: float
    beta: float
    bc_l: DiffusionBc = DiffusionBc.ZERO_NEUMANN
    formulation: Formulation = Formulation.NORMAL
    preconditioner: PrecondSelector = PrecondSelector.NONE
    fp_tol: float = 1e-3
    fp_max: int = 100
    inner: KrylovConfig = field(default_factory=KrylovConfig)
    use_fast_blur: bool = True
    spacing: float = 1.0

    def validate(self) -> None:
        """Same invariants as pipeline.py:78-96."""
        if self.alpha <= 0 or self.beta <= 0:
            raise ConfigurationError("alpha and beta must be positive")
        if self.spacing <= 0:
            raise ConfigurationError("spacing must be positive")
        if self.fp_tol <= 0 or self.fp_max < 1:
            raise ConfigurationError("fp_tol must be positive and fp_max >= 1")
        if self.formulation is Formulation.REBLUR and \
                self.bc_h is not BoundaryCondition.ANTI_REFLECTIVE:
            raise ConfigurationError("the re-blurred formulation requires anti-reflective blur BCs")
        if self.preconditioner in (PrecondSelector.X, PrecondSelector.D_X, PrecondSelector.X_D):
            if (self.bc_h, self.formulation) not in _BASE_KIND:
                raise ConfigurationError(
                    "transform-algebra preconditioners need reflective or "
                    "anti-reflective blur boundary conditions")

    def base_kind(self) -> str | None:
        return _BASE_KIND.get((self.bc_h, self.formulation))

    def resolved_kind(self) -> str | None:
        base = self.base_kind()
        if base is None:
            return None
        return {PrecondSelector.NONE: "I", PrecondSelector.DIAG: "D", PrecondSelector.X: base,
                PrecondSelector.D_X: f"D_{base}", PrecondSelector.X_D: f"{base}_D"}[self.preconditioner]


@dataclass
class RestorationReport:
    restored: object
    fp_steps: int
    inner_iterations: list[int]
    avg_inner: float
    fp_converged: bool
    inner_converged: bool
    gradient_norms: list[float]
    final_gradient_norm: float
    rre: float | None
    wall_time: float
    pcg_time: float = 0.0      # seconds inside the device PCG solves (CUDA events)


class NormalSystem:
    """``A w = H^T H w + alpha L w`` (pipeline.py:209-210), optionally ``s .* A(s .* w)``.

    Calling it applies the operator with one fused device pass pair; handing
    it to :func:`~.krylov.pcg` selects the device-resident PCG.
    """

    def __init__(self, h_op: StructuredBlurOperator, l_op: DiffusionOperator, alpha: float,
                 s: torch.Tensor | None = None, reblur: bool = False) -> None:
        self.h_op, self.l_op, self.alpha, self.s = h_op, l_op, float(alpha), s
        self.reblur = bool(reblur)
        self.device = h_op.device
        self.n = h_op.n

    @property
    def symmetric(self) -> bool:
        """PCG applies (pipeline.py:196-198); otherwise BiCGstab."""
        return not self.reblur and self.l_op.symmetric

    def c_struct(self) -> nat.TvdSystem:
        return nat.TvdSystem(self.h_op.handle, self.alpha, self.l_op.spacing,
                             self.l_op.a_h_device.data_ptr(), self.l_op.a_v_device.data_ptr(),
                             nat.ptr(self.s), self.l_op.bc_code, int(self.reblur))

    def __call__(self, w):
        t, was_np = nat.to_device(w, self.device)
        if tuple(t.shape) != (self.n, self.n):
            raise ValueError(f"expected shape {(self.n, self.n)}, got {tuple(t.shape)}")
        out = torch.empty_like(t)
        csys = self.c_struct()
        ctx = nat.context(self.device)
        nat.check(nat.load().tvd_system_apply(ctx, ctypes.byref(csys), t.data_ptr(),
                                              out.data_ptr()))
        return nat.to_host_like(out, was_np)


@dataclass
class ScaledSystem:
    """Diagonally scaled system bundle (pipeline.py:129-142)."""

    d: torch.Tensor | None
    d_inv_sqrt: torch.Tensor
    apply: NormalSystem
    rhs: torch.Tensor

    def scale_iterate(self, u: torch.Tensor) -> torch.Tensor:
        return _binary(u, self.d_inv_sqrt, 1)

    def unscale(self, u_tilde: torch.Tensor) -> torch.Tensor:
        return _binary(self.d_inv_sqrt, u_tilde, 0)


def _binary(x: torch.Tensor, y: torch.Tensor, op: int) -> torch.Tensor:
    out = torch.empty_like(x)
    ctx = nat.context(x.device)
    nat.check(nat.load().tvd_vec_binary(ctx, x.numel(), op, x.data_ptr(), y.data_ptr(),
                                        out.data_ptr()))
    return out


def _norm(x: torch.Tensor) -> float:
    out = ctypes.c_double()
    ctx = nat.context(x.device)
    nat.check(nat.load().tvd_vec_dot(ctx, x.numel(), x.data_ptr(), x.data_ptr(), ctypes.byref(out)))
    return math.sqrt(out.value)


def _sub(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(x)
    ctx = nat.context(x.device)
    nat.check(nat.load().tvd_vec_axpby(ctx, x.numel(), 1.0, x.data_ptr(), -1.0, y.data_ptr(),
                                       out.data_ptr()))
    return out


def _scaling(l_op: DiffusionOperator, alpha: float, want: str):
    """``d = 1 + alpha diag L`` and ``s = d^{-1/2}`` (pipeline.py:145-158)."""
    diag = l_op.diagonal_device()
    d = torch.empty_like(diag)
    s = torch.empty_like(diag) if want == "s" else None
    mn = ctypes.c_double()
    ctx = nat.context(diag.device)
    rc = nat.load().tvd_scaling(ctx, diag.numel(), float(alpha), diag.data_ptr(), d.data_ptr(),
                                None, nat.ptr(s), ctypes.byref(mn))
    if rc == nat.TVD_ERR_SCALING:
        if want == "s":
            raise InvalidScalingError(
                f"diagonal scaling has nonpositive entries (min {mn.value!r})")
        raise InvalidScalingError("diagonal preconditioner has nonpositive entries")
    nat.check(rc)
    return d, s


def scale_system(system: NormalSystem, rhs, l_op: DiffusionOperator, alpha: float) -> ScaledSystem:
    """Symmetric diagonal scaling by ``D = I + alpha diag L`` (pipeline.py:145-164)."""
    if alpha <= 0:
        raise ConfigurationError(f"alpha must be positive, got {alpha}")
    d, s = _scaling(l_op, alpha, "s")
    rt = nat.to_device(rhs, system.device)[0]
    scaled = NormalSystem(system.h_op, system.l_op, system.alpha, s=s, reblur=system.reblur)
    return ScaledSystem(d=d, d_inv_sqrt=s, apply=scaled, rhs=_binary(s, rt, 0))


def _timed_solve(solver, apply_a, apply_minv, b, x0, cfg, acc: list[float],
                 precond=None) -> SolveOutcome:
    """One inner solve, timed with CUDA events.  ``precond``: a preconditioner assembled with
    deferred checks -- resolved after the solve (which synchronises anyway), and first when
    the solve raises, since the reference fails at assembly (precond.py:437-441, 558-560)
    before it would ever reach the solver."""
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record()
    try:
        out = solver(apply_a, apply_minv, b, x0, cfg)
    except Exception:
        if precond is not None:
            precond.check()
        raise
    if precond is not None:
        precond.check()
    stop.record()
    stop.synchronize()
    acc[0] += start.elapsed_time(stop) / 1e3
    return out


def restore(v, psf: SymmetricPsf, config: RestorationConfig, u_true=None) -> RestorationReport:
    """Run the fixed-point restoration of observed data ``v`` (pipeline.py:182-276)."""
    config.validate()
    vt, was_np = nat.to_device(v)
    if not bool(torch.isfinite(vt).all()):
        raise ConfigurationError("observed data must be finite")
    torch.cuda.synchronize(vt.device)
    started = time.perf_counter()
    if not isinstance(psf, SymmetricPsf):
        psf = SymmetricPsf(psf)
    n = vt.shape[0]
    h_op = StructuredBlurOperator(psf, config.bc_h, n, device=vt.device)
    reblur = config.formulation is Formulation.REBLUR
    # back operator (pipeline.py:166-179): H for the re-blurred and the (symmetric) reflective
    # systems, H^T otherwise
    back = h_op.apply if (reblur or config.bc_h is BoundaryCondition.REFLECTIVE) \
        else h_op.apply_transpose
    alpha = config.alpha
    rhs = back(vt)
    u = vt.clone()
    inner_iterations: list[int] = []
    gradient_norms: list[float] = []
    fp_converged = False
    inner_converged = True
    steps = 0
    pcg_time = [0.0]
    for _ in range(config.fp_max):
        l_op = DiffusionOperator(u, config.beta, config.bc_l, config.spacing, device=vt.device)
        system = NormalSystem(h_op, l_op, alpha, reblur=reblur)
        solver = pcg if system.symmetric else pbicgstab  # pipeline.py:196-198
        gradient_norms.append(_norm(_sub(system(u), rhs)))
        selector = config.preconditioner
        if selector is PrecondSelector.X_D:
            bundle = scale_system(system, rhs, l_op, alpha)
            precond = assemble_preconditioner(f"{config.base_kind()}_D", h_op, l_op, alpha,
                                              defer_checks=True)
            outcome = _timed_solve(solver, bundle.apply, precond.apply_inverse, bundle.rhs,
                                   bundle.scale_iterate(u), config.inner, pcg_time, precond)
            u_next = bundle.unscale(outcome.solution)
        else:
            precond = None
            if selector is PrecondSelector.NONE:
                apply_minv = None
            elif selector is PrecondSelector.DIAG:
                d, _ = _scaling(l_op, alpha, "d")
                apply_minv = DiagonalInverse(d)
            else:
                kind = config.base_kind() if selector is PrecondSelector.X \
                    else f"D_{config.base_kind()}"
                precond = assemble_preconditioner(kind, h_op, l_op, alpha, defer_checks=True)
                apply_minv = precond.apply_inverse
            outcome = _timed_solve(solver, system, apply_minv, rhs, u, config.inner, pcg_time,
                                   precond)
            u_next = outcome.solution
        steps += 1
        inner_iterations.append(outcome.iterations)
        inner_converged = inner_converged and outcome.converged
        change = _norm(_sub(u_next, u))
        u = u_next
        scale = _norm(u)
        if scale > 0 and change / scale < config.fp_tol:
            fp_converged = True
            break
    # el_residual (tv.py:190-204): H* (H u - v) + alpha L(u) u, H* = H for the re-blurred form
    residual = _sub(h_op.apply(u), vt)
    l_fin = DiffusionOperator(u, config.beta, config.bc_l, config.spacing, device=vt.device)
    grad = h_op.reblur_apply(residual) if reblur else h_op.apply_transpose(residual)
    lu = l_fin.apply(u)
    ctx = nat.context(vt.device)
    g_out = torch.empty_like(grad)
    nat.check(nat.load().tvd_vec_axpby(ctx, grad.numel(), 1.0, grad.data_ptr(), alpha,
                                       lu.data_ptr(), g_out.data_ptr()))
    final_gradient = _norm(g_out)
    rre = None
    if u_true is not None:
        ut = nat.to_device(u_true, vt.device)[0]
        rre = _norm(_sub(u, ut)) / _norm(ut)
    restored = nat.to_host_like(u, was_np)
    torch.cuda.synchronize(vt.device)
    return RestorationReport(
        restored=restored, fp_steps=steps, inner_iterations=inner_iterations,
        avg_inner=float(np.mean(inner_iterations)) if inner_iterations else 0.0,
        fp_converged=fp_converged, inner_converged=inner_converged,
        gradient_norms=gradient_norms, final_gradient_norm=final_gradient, rre=rre,
        wall_time=time.perf_counter() - started, pcg_time=pcg_time[0])
