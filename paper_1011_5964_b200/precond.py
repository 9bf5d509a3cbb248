"""Transform-algebra preconditioners on the GPU (mirror of reference precond.py:47-573).

``assemble_preconditioner(kind, h_op, l_op, alpha)`` builds the kinds
R / D_R / R_D (cosine algebra, reflective blur) and M / D_M / M_D (bordered
sine algebra, anti-reflective blur) entirely on the device: the two-level
projection of the diffusion block bands (precond.py:369-395) runs as two
batched band-FFT passes (``k_band`` in csrc/tvd_lines.cu), the blur
eigenvalues come from the device symbol grid, and the positivity check /
``1e-14 max`` clamp of ``FactoredPreconditioner.__post_init__``
(precond.py:437-450) is done on device min/max reductions.

``FactoredPreconditioner.apply_inverse`` is one row pass, one fused
column "sandwich" pass (transform -> eigenvalue scaling -> transform) and one
row pass.  The P family (anti-reflective algebra, the re-blurred BiCGstab systems)
uses the same passes with ``T = Shat (I + U)``'s rank-2 border corrections fused in, and
its projection adds the AR border eigenvalues to the sine projection
(precond.py:156-165, 302-352).
"""

from __future__ import annotations

import ctypes
import logging

import numpy as np
import torch

from . import _native as nat
from .transforms import TransformKind

logger = logging.getLogger(__name__)

_FAMILIES = {"R": TransformKind.DCT, "M": TransformKind.SINE_HAT,
             "P": TransformKind.ANTI_REFLECTIVE}
_FAMILY_CODE = {TransformKind.DCT: nat.T_DCT, TransformKind.SINE_HAT: nat.T_SINE_HAT,
                TransformKind.ANTI_REFLECTIVE: nat.T_ANTI_REFLECTIVE}

PRECONDITIONER_KINDS = ("R", "D_R", "R_D", "M", "D_M", "M_D", "P", "D_P", "P_D")


class IndefinitePreconditionerError(RuntimeError):
    """A factored preconditioner came out with a nonpositive eigenvalue (precond.py:60-70)."""

    def __init__(self, kind: str, alpha: float, min_eigenvalue: float) -> None:
        super().__init__(
            f"preconditioner {kind!r} is indefinite at alpha={alpha!r} "
            f"(smallest eigenvalue {min_eigenvalue!r})")
        self.kind = kind
        self.alpha = alpha
        self.min_eigenvalue = min_eigenvalue


class FactoredPreconditioner:
    """Transform + eigenvalues (+ diagonal wrap) held on the device (precond.py:419-490)."""

    def __init__(self, kind: str, transform: TransformKind, eigenvalues, alpha: float,
                 d_sqrt=None, *, inverse_eigenvalues=None, clamped: int | None = None,
                 scaling=None, device: torch.device | None = None,
                 pending: torch.Tensor | None = None) -> None:
        if transform not in _FAMILY_CODE:
            raise NotImplementedError(f"{transform.value} preconditioners are outside this build's scope")
        self.kind = kind
        self.transform = transform
        self.alpha = float(alpha)
        lam, _ = nat.to_device(eigenvalues, device)
        self.device = lam.device
        self._lam = lam
        self._d_sqrt = None if d_sqrt is None else nat.to_device(d_sqrt, self.device)[0]
        #: X_D kinds: the diagonal scaling ``s = (1 + alpha diag L)^{-1/2}`` of the system
        self.scaling = scaling
        if inverse_eigenvalues is None:
            smallest = float(lam.min())
            if smallest <= 0.0:
                raise IndefinitePreconditionerError(kind, alpha, smallest)
            floor = 1e-14 * float(lam.max())
            clamped = int((lam < floor).sum())
            inverse_eigenvalues = 1.0 / torch.clamp(lam, min=floor)
        self._inv = inverse_eigenvalues
        #: deferred device-side checks (tvd_precond_assemble_async), resolved by check()
        self._pending = pending
        self._clamped = int(clamped or 0)
        if pending is None and clamped:
            logger.warning("preconditioner %s: clamped %d eigenvalue(s) below %.3e",
                           kind, clamped, 1e-14 * float(lam.max()))

    def check(self) -> None:
        """Resolve the construction checks of a deferred assembly (precond.py:437-450,
        558-560): raise :class:`IndefinitePreconditionerError` for a nonpositive scaling
        diagonal or eigenvalue, log the clamp warning.  Reads four device doubles (one
        synchronisation); a no-op for an eagerly checked preconditioner."""
        if self._pending is None:
            return
        min_d, mn, mx, cnt = (float(x) for x in self._pending.cpu())
        self._pending = None
        if not min_d > 0.0:
            raise IndefinitePreconditionerError(self.kind, self.alpha, min_d)
        if not mn > 0.0:
            raise IndefinitePreconditionerError(self.kind, self.alpha, mn)
        self._clamped = int(cnt)
        if self._clamped:
            logger.warning("preconditioner %s: clamped %d eigenvalue(s) below %.3e",
                           self.kind, self._clamped, 1e-14 * mx)

    @property
    def clamped(self) -> int:
        self.check()
        return self._clamped

    @property
    def ndim(self) -> int:
        return 2

    @property
    def eigenvalues(self) -> np.ndarray:
        return self._lam.cpu().numpy()

    @property
    def eigenvalues_device(self) -> torch.Tensor:
        return self._lam

    @property
    def inverse_eigenvalues_device(self) -> torch.Tensor:
        return self._inv

    @property
    def d_sqrt(self):
        return None if self._d_sqrt is None else self._d_sqrt.cpu().numpy()

    @property
    def d_sqrt_device(self):
        return self._d_sqrt

    @property
    def family_code(self) -> int:
        return _FAMILY_CODE[self.transform]

    def _run(self, b, inverse: bool):
        t, was_np = nat.to_device(b, self.device)
        n = self._lam.shape[0]
        if tuple(t.shape) != (n, n):
            raise ValueError(f"expected shape {(n, n)}, got {tuple(t.shape)}")
        out = torch.empty_like(t)
        ctx = nat.context(self.device)
        lib = nat.load()
        fn = lib.tvd_precond_apply_inverse if inverse else lib.tvd_precond_apply
        nat.check(fn(ctx, self.family_code, n, (self._inv if inverse else self._lam).data_ptr(),
                     nat.ptr(self._d_sqrt), t.data_ptr(), out.data_ptr()))
        return nat.to_host_like(out, was_np)

    def apply(self, b):
        """Multiply by the preconditioner matrix (precond.py:463-469)."""
        return self._run(b, False)

    def apply_inverse(self, b):
        """Solve ``M y = b`` (precond.py:471-477)."""
        return self._run(b, True)


def assemble_preconditioner(kind: str, h_op, l_op, alpha: float, *,
                            defer_checks: bool = False) -> FactoredPreconditioner:
    """Build one factored preconditioner on the device (precond.py:516-573).

    ``defer_checks``: leave the positivity checks and the clamp count on the device (no host
    synchronisation; ``tvd_precond_assemble_async``); the returned preconditioner raises /
    warns from :meth:`FactoredPreconditioner.check`, which the caller runs after its solve
    (``restore`` does).  The eigenvalues are identical either way."""
    from .blur import BoundaryCondition

    if kind not in PRECONDITIONER_KINDS:
        raise ValueError(f"unknown preconditioner kind {kind!r}")
    if alpha <= 0:
        raise ValueError(f"alpha must be positive, got {alpha}")
    base = kind.replace("D_", "").replace("_D", "")
    transform = _FAMILIES[base]
    expected_bc = (BoundaryCondition.REFLECTIVE if base == "R"
                   else BoundaryCondition.ANTI_REFLECTIVE)
    if h_op.bc is not expected_bc:
        raise ValueError(
            f"preconditioner {kind!r} requires a blur operator with "
            f"{expected_bc.value!r} boundary conditions, got {h_op.bc.value!r}")
    if kind.endswith("_D"):
        variant = nat.VARIANT_X_D
    elif kind.startswith("D_"):
        variant = nat.VARIANT_D_X
    else:
        variant = nat.VARIANT_X
    n = h_op.n
    dev = h_op.device
    lam_h = h_op.eigenvalues_device()
    # the projections read interior bands only, where up == low even for AR ghosts
    diag, inner, _, block, _ = l_op.bands_device()
    eig = torch.empty((n, n), dtype=torch.float64, device=dev)
    inv = torch.empty_like(eig)
    dvec = torch.empty_like(eig) if variant != nat.VARIANT_X else None
    mn, mx, cl = ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
    ctx = nat.context(dev)
    inner_c = inner.contiguous()
    block_c = block.contiguous()
    if defer_checks:
        chk = torch.empty(4, dtype=torch.float64, device=dev)
        nat.check(nat.load().tvd_precond_assemble_async(
            ctx, _FAMILY_CODE[transform], variant, n, float(alpha), lam_h.data_ptr(),
            diag.data_ptr(), inner_c.data_ptr(), block_c.data_ptr(), eig.data_ptr(),
            inv.data_ptr(), nat.ptr(dvec), chk.data_ptr()))
        if variant == nat.VARIANT_X_D:
            return FactoredPreconditioner(kind, transform, eig, alpha, inverse_eigenvalues=inv,
                                          scaling=dvec, device=dev, pending=chk)
        return FactoredPreconditioner(kind, transform, eig, alpha, d_sqrt=dvec,
                                      inverse_eigenvalues=inv, device=dev, pending=chk)
    rc = nat.load().tvd_precond_assemble(
        ctx, _FAMILY_CODE[transform], variant, n, float(alpha), lam_h.data_ptr(),
        diag.data_ptr(), inner_c.data_ptr(), block_c.data_ptr(), eig.data_ptr(), inv.data_ptr(),
        nat.ptr(dvec), ctypes.byref(mn), ctypes.byref(mx), ctypes.byref(cl))
    if rc == nat.TVD_ERR_PRECOND:
        raise IndefinitePreconditionerError(kind, alpha, mn.value)
    nat.check(rc)
    if variant == nat.VARIANT_X_D:
        return FactoredPreconditioner(kind, transform, eig, alpha, inverse_eigenvalues=inv,
                                      clamped=int(cl.value), scaling=dvec, device=dev)
    return FactoredPreconditioner(kind, transform, eig, alpha, d_sqrt=dvec,
                                  inverse_eigenvalues=inv, clamped=int(cl.value), device=dev)
