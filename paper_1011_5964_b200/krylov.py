"""PCG and right-preconditioned BiCGstab with the reference's recurrences (krylov.py:23-174).

``pcg(apply_a, apply_minv, b, x0, config)`` keeps the reference's callable
contract.  Two execution paths, both on the GPU:

* **fused** -- when ``apply_a`` is a :class:`~.pipeline.NormalSystem` and
  ``apply_minv`` is ``None``, a :class:`DiagonalInverse` or a
  ``FactoredPreconditioner.apply_inverse``: the whole loop runs device-side
  through ``tvd_pcg_solve`` (matvec with fused ``p.q``, fused ``x/r`` update
  with ``r.r``, preconditioner passes with fused ``r.z``, deterministic
  reductions, host checks only every few iterations).
* **generic** -- any other callables on CUDA tensors; the recurrence runs in
  Python with the library's device vector kernels (``tvd_vec_*``).

Both stop when ``||r_k|| / ||r_0|| < tol`` (checked after the x/r update),
report non-convergence through ``converged=False`` and raise the reference's
exception types with the same fields.  ``pbicgstab`` (the nonsymmetric re-blurred /
anti-reflective-L systems, pipeline.py:196-198) has the same two paths
(``tvd_bicgstab_solve`` / generic).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat


class SolverBreakdownError(RuntimeError):
    """A recurrence scalar vanished (krylov.py:23-28)."""

    def __init__(self, method: str, iteration: int, what: str) -> None:
        super().__init__(f"{method} breakdown at iteration {iteration}: {what}")
        self.iteration = iteration


class SolverDivergenceError(RuntimeError):
    """A non-finite quantity appeared (krylov.py:31-36)."""

    def __init__(self, method: str, iteration: int) -> None:
        super().__init__(f"{method} produced non-finite values at iteration {iteration}")
        self.iteration = iteration


class IndefiniteOperatorError(RuntimeError):
    """Nonpositive curvature (krylov.py:39-46)."""

    def __init__(self, iteration: int, curvature: float) -> None:
        super().__init__(f"pcg met nonpositive curvature {curvature!r} at iteration {iteration}")
        self.iteration = iteration


@dataclass(frozen=True)
class KrylovConfig:
    tol: float = 1e-6
    max_iterations: int = 1000
    record_history: bool = False

    def __post_init__(self) -> None:
        if self.tol <= 0:
            raise ValueError(f"tol must be positive, got {self.tol}")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")


@dataclass
class SolveOutcome:
    solution: object
    iterations: int
    residual_history: np.ndarray
    converged: bool


class DiagonalInverse:
    """``apply_minv`` for the DIAG selector: ``w / d`` (pipeline.py:228-236)."""

    def __init__(self, d: torch.Tensor) -> None:
        self.d = d

    def __call__(self, w):
        t, was_np = nat.to_device(w, self.d.device)
        out = torch.empty_like(t)
        ctx = nat.context(t.device)
        nat.check(nat.load().tvd_vec_binary(ctx, t.numel(), 1, t.data_ptr(), self.d.data_ptr(),
                                            out.data_ptr()))
        return nat.to_host_like(out, was_np)


def _dot(x: torch.Tensor, y: torch.Tensor) -> float:
    out = ctypes.c_double()
    ctx = nat.context(x.device)
    nat.check(nat.load().tvd_vec_dot(ctx, x.numel(), x.data_ptr(), y.data_ptr(), ctypes.byref(out)))
    return out.value


def _axpby(a: float, x: torch.Tensor, b: float, y: torch.Tensor, out: torch.Tensor | None = None):
    out = torch.empty_like(x) if out is None else out
    ctx = nat.context(x.device)
    nat.check(nat.load().tvd_vec_axpby(ctx, x.numel(), a, x.data_ptr(), b, y.data_ptr(),
                                       out.data_ptr()))
    return out


def _as_tensor(v, like: torch.Tensor) -> torch.Tensor:
    t, _ = nat.to_device(v, like.device)
    return t.reshape(like.shape)


def _fused_precond(apply_minv):
    """``(kind, family, inv_eig, d)`` when ``apply_minv`` has a device-fused form."""
    from .precond import FactoredPreconditioner

    if apply_minv is None:
        return nat.PRE_NONE, 0, None, None
    if isinstance(apply_minv, DiagonalInverse):
        return nat.PRE_DIAG, 0, None, apply_minv.d
    owner = getattr(apply_minv, "__self__", None)
    if isinstance(owner, FactoredPreconditioner) and \
            getattr(apply_minv, "__func__", None) is FactoredPreconditioner.apply_inverse:
        return (nat.PRE_TRANSFORM, owner.family_code, owner.inverse_eigenvalues_device,
                owner.d_sqrt_device)
    return None


def pcg(apply_a, apply_minv, b, x0, config: KrylovConfig = KrylovConfig()) -> SolveOutcome:
    """Preconditioned conjugate gradient for SPD operators (krylov.py:82-116)."""
    from .pipeline import NormalSystem

    fused = _fused_precond(apply_minv) if isinstance(apply_a, NormalSystem) else None
    if fused is not None:
        return _pcg_fused(apply_a, fused, b, x0, config)
    return _pcg_generic(apply_a, apply_minv, b, x0, config)


def _pcg_fused(system, pre, b, x0, config: KrylovConfig) -> SolveOutcome:
    dev = system.device
    bt, was_np = nat.to_device(b, dev)
    xt = nat.to_device(x0, dev)[0].clone()
    kind, family, inv, d = pre
    cpre = nat.TvdPrecond(kind, family, nat.ptr(inv), nat.ptr(d))
    hist = (torch.empty(config.max_iterations, dtype=torch.float64, device=dev)
            if config.record_history else None)
    it, conv, err_it, err_val = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    ctx = nat.context(dev)
    csys = system.c_struct()
    rc = nat.load().tvd_pcg_solve(ctx, ctypes.byref(csys), ctypes.byref(cpre), bt.data_ptr(),
                                  xt.data_ptr(), xt.data_ptr(), float(config.tol),
                                  int(config.max_iterations), nat.ptr(hist), ctypes.byref(it),
                                  ctypes.byref(conv), ctypes.byref(err_it), ctypes.byref(err_val))
    if rc == nat.TVD_ERR_DIVERGED:
        raise SolverDivergenceError("pcg", err_it.value)
    if rc == nat.TVD_ERR_INDEFINITE:
        raise IndefiniteOperatorError(err_it.value, err_val.value)
    nat.check(rc)
    k = it.value
    history = hist[:k].cpu().numpy() if hist is not None else np.array([])
    return SolveOutcome(nat.to_host_like(xt, was_np), k, history, bool(conv.value))


def _pcg_generic(apply_a, apply_minv, b, x0, config: KrylovConfig) -> SolveOutcome:
    bt, was_np = nat.to_device(b)
    x = nat.to_device(x0, bt.device)[0].clone()
    minv = apply_minv or (lambda t: t)
    r = _axpby(1.0, bt, -1.0, _as_tensor(apply_a(x), bt))
    r0 = math.sqrt(_dot(r, r))
    history: list[float] = []
    if r0 == 0.0:
        return SolveOutcome(nat.to_host_like(x, was_np), 0, np.array(history), True)
    z = _as_tensor(minv(r), bt)
    p = z.clone()
    rz = _dot(r, z)
    for k in range(1, config.max_iterations + 1):
        q = _as_tensor(apply_a(p), bt)
        curvature = _dot(p, q)
        if not math.isfinite(curvature):
            raise SolverDivergenceError("pcg", k)
        if curvature <= 0.0:
            raise IndefiniteOperatorError(k, curvature)
        step = rz / curvature
        _axpby(1.0, x, step, p, out=x)
        r = _axpby(1.0, r, -step, q)
        rel = math.sqrt(_dot(r, r)) / r0
        if not math.isfinite(rel):
            raise SolverDivergenceError("pcg", k)
        if config.record_history:
            history.append(rel)
        if rel < config.tol:
            return SolveOutcome(nat.to_host_like(x, was_np), k, np.array(history), True)
        z = _as_tensor(minv(r), bt)
        rz_next = _dot(r, z)
        p = _axpby(1.0, z, rz_next / rz, p)
        rz = rz_next
    return SolveOutcome(nat.to_host_like(x, was_np), config.max_iterations, np.array(history), False)


def pbicgstab(apply_a, apply_minv, b, x0, config: KrylovConfig = KrylovConfig()) -> SolveOutcome:
    """Right-preconditioned BiCGstab for general invertible operators (krylov.py:119-174).

    Fused device loop (``tvd_bicgstab_solve``) for a :class:`~.pipeline.NormalSystem` with a
    device-fused preconditioner, otherwise the reference recurrence over the library's
    device vector kernels.  Raises :class:`SolverBreakdownError` /
    :class:`SolverDivergenceError` as the reference does.
    """
    from .pipeline import NormalSystem

    fused = _fused_precond(apply_minv) if isinstance(apply_a, NormalSystem) else None
    if fused is not None:
        return _bicg_fused(apply_a, fused, b, x0, config)
    return _bicg_generic(apply_a, apply_minv, b, x0, config)


_BREAKDOWN = {1: "rho vanished", 2: "shadow angle vanished", 3: "stabilizer direction vanished",
              4: "omega vanished"}


def _bicg_fused(system, pre, b, x0, config: KrylovConfig) -> SolveOutcome:
    dev = system.device
    bt, was_np = nat.to_device(b, dev)
    xt = nat.to_device(x0, dev)[0].clone()
    kind, family, inv, d = pre
    cpre = nat.TvdPrecond(kind, family, nat.ptr(inv), nat.ptr(d))
    hist = (torch.empty(config.max_iterations, dtype=torch.float64, device=dev)
            if config.record_history else None)
    it, conv, err_it, err_val = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    ctx = nat.context(dev)
    csys = system.c_struct()
    rc = nat.load().tvd_bicgstab_solve(ctx, ctypes.byref(csys), ctypes.byref(cpre), bt.data_ptr(),
                                       xt.data_ptr(), xt.data_ptr(), float(config.tol),
                                       int(config.max_iterations), nat.ptr(hist),
                                       ctypes.byref(it), ctypes.byref(conv), ctypes.byref(err_it),
                                       ctypes.byref(err_val))
    if rc == nat.TVD_ERR_DIVERGED:
        raise SolverDivergenceError("pbicgstab", err_it.value)
    if rc == nat.TVD_ERR_BREAKDOWN:
        raise SolverBreakdownError("pbicgstab", err_it.value, _BREAKDOWN.get(int(err_val.value), ""))
    nat.check(rc)
    k = it.value
    history = hist[:k].cpu().numpy() if hist is not None else np.array([])
    return SolveOutcome(nat.to_host_like(xt, was_np), k, history, bool(conv.value))


def _bicg_generic(apply_a, apply_minv, b, x0, config: KrylovConfig) -> SolveOutcome:
    bt, was_np = nat.to_device(b)
    x = nat.to_device(x0, bt.device)[0].clone()
    minv = apply_minv or (lambda t: t)
    r = _axpby(1.0, bt, -1.0, _as_tensor(apply_a(x), bt))
    r0 = math.sqrt(_dot(r, r))
    history: list[float] = []
    if r0 == 0.0:
        return SolveOutcome(nat.to_host_like(x, was_np), 0, np.array(history), True)
    rs = r.clone()
    rho = alpha = omega = 1.0
    v = torch.zeros_like(r)
    p = torch.zeros_like(r)
    for k in range(1, config.max_iterations + 1):
        rho_next = _dot(rs, r)
        if abs(rho_next) < 1e-30 * r0 * r0:
            raise SolverBreakdownError("pbicgstab", k, "rho vanished")
        beta = (rho_next / rho) * (alpha / omega)
        p = _axpby(1.0, r, beta, _axpby(1.0, p, -omega, v))
        p_hat = _as_tensor(minv(p), bt)
        v = _as_tensor(apply_a(p_hat), bt)
        denom = _dot(rs, v)
        if abs(denom) < 1e-300:
            raise SolverBreakdownError("pbicgstab", k, "shadow angle vanished")
        alpha = rho_next / denom
        s = _axpby(1.0, r, -alpha, v)
        rel = math.sqrt(_dot(s, s)) / r0
        if not math.isfinite(rel):
            raise SolverDivergenceError("pbicgstab", k)
        if rel < config.tol:
            _axpby(1.0, x, alpha, p_hat, out=x)
            if config.record_history:
                history.append(rel)
            return SolveOutcome(nat.to_host_like(x, was_np), k, np.array(history), True)
        s_hat = _as_tensor(minv(s), bt)
        t = _as_tensor(apply_a(s_hat), bt)
        tt = _dot(t, t)
        if tt == 0.0:
            raise SolverBreakdownError("pbicgstab", k, "stabilizer direction vanished")
        omega = _dot(t, s) / tt
        if abs(omega) < 1e-300:
            raise SolverBreakdownError("pbicgstab", k, "omega vanished")
        _axpby(1.0, x, 1.0, _axpby(alpha, p_hat, omega, s_hat), out=x)
        r = _axpby(1.0, s, -omega, t)
        rel = math.sqrt(_dot(r, r)) / r0
        if not math.isfinite(rel):
            raise SolverDivergenceError("pbicgstab", k)
        if config.record_history:
            history.append(rel)
        if rel < config.tol:
            return SolveOutcome(nat.to_host_like(x, was_np), k, np.array(history), True)
        rho = rho_next
    return SolveOutcome(nat.to_host_like(x, was_np), config.max_iterations, np.array(history), False)
