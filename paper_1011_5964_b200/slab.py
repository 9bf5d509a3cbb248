"""Row-slab decomposition of one large inner solve across ranks.

The reference solves one image on one CPU (krylov.py:82-116).  For an 8192^2 problem this
build splits the image into row slabs, one per GPU: rank ``rho`` of ``P`` owns the global
rows ``[rho R, rho R + R)``, ``R = n / P``, of every ``n x n`` array.  The kernels of one PCG
iteration run in the native library (``tvd_slab_phase``, ``csrc/tvd_slab.cuh``); between the
phases this module runs the collectives:

* **halo exchange** of ``t = p G_1^T`` (``khalo`` rows) and of ``p`` (one row, the ``L``
  stencil) with the two neighbouring slabs -- the column band pass ``G_0 t`` and ``L p`` are
  local otherwise;
* **all-to-all** twice inside the preconditioner: the row DST writes its output transposed,
  so block ``j`` of the send buffer already holds the columns of rank ``j``; after the
  exchange every column is a line of ``P`` contiguous segments (one TMA bulk copy each) for
  the column "sandwich" pass (DST, ``lambda^-1``, DST), and the second exchange brings the
  rows back for the last row DST;
* **allgather** of one double per dot product (``p.q``, ``r.r``, ``r.z``); every rank sums the
  ``P`` contributions in rank order, so every rank computes bit-identical scalars and takes
  the same branch (stop test, exceptions) without a broadcast.

The same schedule runs over three communicators: :class:`TorchComm` (``torch.distributed``,
NCCL over NVLink on the GPU box, gloo in the CPU tests), and :class:`LoopbackComm`, which
drives ``P`` slabs of one process on one device with local copies (single-GPU parity tests of
the slab kernels; nothing waits on another kernel).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .krylov import IndefiniteOperatorError, KrylovConfig, SolveOutcome, SolverDivergenceError

# phases and buffers (include/tvdeblur_b200.h TVD_SLAB_*)
MATVEC_ROWS, MATVEC_COLS, RESIDUAL, START, GAMMA_UPDATE, REL = 0, 1, 2, 3, 4, 5
PREC_ROWS, PREC_COLS, PREC_FINAL, RZ0, BETA_P = 6, 7, 8, 9, 10
BUF_X, BUF_R, BUF_Z, BUF_Q, BUF_P_EXT, BUF_T_EXT = 0, 1, 2, 3, 4, 5
BUF_SEND, BUF_RECV, BUF_CONTRIB, BUF_GATHER = 6, 7, 8, 9


@dataclass(frozen=True)
class SlabLayout:
    """Host-side geometry of one rank's slab (shared by every communicator)."""

    n: int
    nranks: int
    rank: int
    khalo: int
    exchanges: bool = True  # the preconditioner needs the two all-to-alls

    @property
    def rows(self) -> int:
        return self.n // self.nranks

    @property
    def row_lo(self) -> int:
        return self.rank * self.rows

    def ext_shape(self, halo: int) -> tuple[int, int]:
        return (self.rows + 2 * halo, self.n)

    def halo_plan(self, halo: int):
        """``[(peer, send_rows, recv_rows)]`` of an extended buffer with ``halo`` rows per side:
        my first interior rows become the bottom halo of rank - 1, my last ones the top halo
        of rank + 1 (no neighbour beyond the image border)."""
        R, h = self.rows, halo
        plan = []
        if self.rank > 0:
            plan.append((self.rank - 1, slice(h, 2 * h), slice(0, h)))
        if self.rank < self.nranks - 1:
            plan.append((self.rank + 1, slice(R, R + h), slice(R + h, R + 2 * h)))
        return plan

    def block(self, j: int) -> slice:
        """Flat range of all-to-all block ``j`` (``R x R`` doubles) of the send / recv buffers."""
        bs = self.rows * self.rows
        return slice(j * bs, (j + 1) * bs)


class _DeviceArray:
    """``__cuda_array_interface__`` over a library-owned device buffer."""

    def __init__(self, ptr: int, count: int) -> None:
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3, "strides": None}


@dataclass
class SlabOperands:
    """One rank's share of an FP step's operators: diffusivities of its rows (``a_h``
    ``R x (n+1)``, ``a_v`` ``(R+1) x n``), its rows of the transposed inverse eigenvalues
    (``inv_t`` = columns ``[lo, lo+R)`` of ``lambda^-1``, the layout of the preconditioner's
    column pass), ``d`` = ``sqrt(1 + alpha diag L)`` rows for D_X kinds, the native
    preconditioner kind / family codes, the global eigenvalue range and clamp count."""

    a_h: torch.Tensor
    a_v: torch.Tensor
    inv_t: torch.Tensor | None
    d: torch.Tensor | None
    kind: int
    family: int
    min_eig: float = float("nan")
    max_eig: float = float("nan")
    clamped: int = 0


class Slab:
    """One rank's slab solver (``tvd_slab``): buffers, phases and status."""

    def __init__(self, system, precond, nranks: int, rank: int) -> None:
        """``system``: a full-size :class:`~.pipeline.NormalSystem` (its diffusivities are
        sliced here); ``precond``: ``None``, a :class:`~.krylov.DiagonalInverse` or a
        ``FactoredPreconditioner.apply_inverse`` of the full problem."""
        from .krylov import _fused_precond

        n = system.n
        if n % nranks:
            raise ValueError(f"n = {n} is not divisible by {nranks} ranks")
        R = n // nranks
        lo = rank * R
        lop = system.l_op
        fused = _fused_precond(precond)
        if fused is None:
            raise ValueError("slab solves take None, a DiagonalInverse or "
                             "FactoredPreconditioner.apply_inverse")
        kind, family, inv, d = fused
        if system.s is not None or system.reblur:
            raise ValueError("slab solves support the X / D_X systems H^T H + alpha L")
        ops = SlabOperands(lop.a_h_device[lo:lo + R].contiguous(),
                           lop.a_v_device[lo:lo + R + 1].contiguous(),
                           None if inv is None else inv.t()[lo:lo + R].contiguous(),
                           None if d is None else d[lo:lo + R].contiguous(), kind, family)
        self._init(system.h_op, system.alpha, lop.spacing, lop.bc_code, ops, nranks, rank)

    @classmethod
    def from_operands(cls, h_op, alpha: float, ops: "SlabOperands", nranks: int, rank: int,
                      spacing: float = 1.0) -> "Slab":
        """A slab from this rank's own operands (:func:`slab_operators`) -- no full-size
        system or preconditioner exists anywhere."""
        self = cls.__new__(cls)
        self._init(h_op, alpha, spacing, 0, ops, nranks, rank)
        return self

    def _init(self, h_op, alpha, spacing, bc_code, ops: "SlabOperands", nranks, rank) -> None:
        n = h_op.n
        self.device = h_op.device
        self.n, self.nranks, self.rank = n, nranks, rank
        # slab operands (kept alive for the handle's lifetime)
        self._a_h, self._a_v, self._inv_t, self._d = ops.a_h, ops.a_v, ops.inv_t, ops.d
        self._csys = nat.TvdSystem(h_op.handle, float(alpha), float(spacing),
                                   self._a_h.data_ptr(), self._a_v.data_ptr(), None, bc_code, 0)
        self._cpre = nat.TvdPrecond(ops.kind, ops.family, nat.ptr(self._inv_t), nat.ptr(self._d))
        self._h_op = h_op  # the blur handle must outlive the slab
        lib = nat.load()
        ctx = nat.context(self.device)
        out = ctypes.c_void_p()
        nat.check(lib.tvd_slab_create(ctx, ctypes.byref(self._csys), ctypes.byref(self._cpre),
                                      nranks, rank, ctypes.byref(out)))
        self.handle = out.value
        info = (ctypes.c_int * 8)()
        nat.check(lib.tvd_slab_info(self.handle, info))
        self.layout = SlabLayout(n, nranks, rank, info[3], bool(info[7]))
        self._bufs: dict[int, torch.Tensor] = {}

    def __del__(self) -> None:
        h = getattr(self, "handle", None)
        if h:
            try:
                nat.load().tvd_slab_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.handle = None

    def buf(self, which: int) -> torch.Tensor:
        t = self._bufs.get(which)
        if t is None:
            p, cnt = ctypes.c_void_p(), ctypes.c_longlong()
            nat.check(nat.load().tvd_slab_buffer(self.handle, which, ctypes.byref(p),
                                                 ctypes.byref(cnt)))
            t = torch.as_tensor(_DeviceArray(p.value, cnt.value), device=self.device)
            self._bufs[which] = t
        return t

    def start(self, b: torch.Tensor, x0: torch.Tensor, config: KrylovConfig, history) -> None:
        self._b = b  # the library keeps the pointer for the whole solve
        nat.context(self.device)
        nat.check(nat.load().tvd_slab_start(self.handle, b.data_ptr(), x0.data_ptr(),
                                            float(config.tol), int(config.max_iterations),
                                            nat.ptr(history)))

    def phase(self, ph: int) -> None:
        nat.check(nat.load().tvd_slab_phase(self.handle, ph))

    def status(self) -> tuple[int, int, int, int, float]:
        """``(rc, done, iterations, converged, err_iteration, err_value)`` (synchronises)."""
        done, it, conv, eit = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        ev = ctypes.c_double()
        rc = nat.load().tvd_slab_status(self.handle, ctypes.byref(done), ctypes.byref(it),
                                        ctypes.byref(conv), ctypes.byref(eit), ctypes.byref(ev))
        return rc, done.value, it.value, conv.value, eit.value, ev.value


# ------------------------------------------------------------------ communicators
class TorchComm:
    """Collectives of one rank over ``torch.distributed`` (NCCL on GPUs, gloo on CPUs)."""

    def __init__(self, group=None) -> None:
        import torch.distributed as dist

        self.dist = dist
        self.group = group

    def halo(self, slabs) -> None:
        dist = self.dist
        (s,) = slabs
        lay = s.layout
        ops = []
        for which, h in ((BUF_T_EXT, lay.khalo), (BUF_P_EXT, 1)):
            ext = s.buf(which).view(lay.ext_shape(h))
            for peer, snd, rcv in lay.halo_plan(h):
                ops.append(dist.P2POp(dist.isend, ext[snd], peer, self.group))
                ops.append(dist.P2POp(dist.irecv, ext[rcv], peer, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def all_to_all(self, slabs) -> None:
        (s,) = slabs
        self.dist.all_to_all_single(s.buf(BUF_RECV), s.buf(BUF_SEND), group=self.group)

    def allgather(self, slabs) -> None:
        (s,) = slabs
        src, dst = s.buf(BUF_CONTRIB), s.buf(BUF_GATHER)
        if dst.is_cuda:
            self.dist.all_gather_into_tensor(dst, src, group=self.group)
        else:  # gloo has no all_gather_into_tensor
            parts = list(dst.split(1))
            self.dist.all_gather(parts, src, group=self.group)

    # -- tensor collectives of the FP-step setup (slab_operators) --------------------
    def halo_rows(self, exts, layouts, h: int = 1) -> None:
        dist = self.dist
        ((ext,), (lay,)) = (exts, layouts)
        ops = []
        for peer, snd, rcv in lay.halo_plan(h):
            ops.append(dist.P2POp(dist.isend, ext[snd], peer, self.group))
            ops.append(dist.P2POp(dist.irecv, ext[rcv], peer, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def all_to_all_blocks(self, sends):
        (send,) = sends
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send, group=self.group)
        return [recv]

    def allreduce_min_max(self, pairs):
        ((mn, mx),) = pairs
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
        t = torch.tensor([-mn, mx], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return -float(t[0]), float(t[1])


class LoopbackComm:
    """The same collectives over ``P`` slabs held by one process (local copies, in order)."""

    def halo(self, slabs) -> None:
        for s in slabs:
            lay = s.layout
            for which, h in ((BUF_T_EXT, lay.khalo), (BUF_P_EXT, 1)):
                mine = s.buf(which).view(lay.ext_shape(h))
                for peer, _, rcv in lay.halo_plan(h):
                    other = slabs[peer]
                    theirs = other.buf(which).view(other.layout.ext_shape(h))
                    snd = next(sl for p2, sl, _ in other.layout.halo_plan(h) if p2 == s.layout.rank)
                    mine[rcv].copy_(theirs[snd])

    def all_to_all(self, slabs) -> None:
        sends = [s.buf(BUF_SEND) for s in slabs]
        for s in slabs:
            recv, lay = s.buf(BUF_RECV), s.layout
            for i, snd in enumerate(sends):
                recv[lay.block(i)].copy_(snd[lay.block(lay.rank)])

    def allgather(self, slabs) -> None:
        vals = torch.cat([s.buf(BUF_CONTRIB)[:1] for s in slabs])
        for s in slabs:
            s.buf(BUF_GATHER)[: len(slabs)].copy_(vals)

    def halo_rows(self, exts, layouts, h: int = 1) -> None:
        for ext, lay in zip(exts, layouts):
            for peer, _, rcv in lay.halo_plan(h):
                snd = next(sl for p2, sl, _ in layouts[peer].halo_plan(h) if p2 == lay.rank)
                ext[rcv].copy_(exts[peer][snd])

    def all_to_all_blocks(self, sends):
        return [torch.stack([s[r] for s in sends]) for r in range(len(sends))]

    def allreduce_min_max(self, pairs):
        return min(p[0] for p in pairs), max(p[1] for p in pairs)


# ------------------------------------------------------------------ the schedule
def _run(slabs, ph: int) -> None:
    for s in slabs:
        s.phase(ph)


def _precond(slabs, comm) -> None:
    _run(slabs, PREC_ROWS)
    if slabs[0].layout.exchanges:
        comm.all_to_all(slabs)
        _run(slabs, PREC_COLS)
        comm.all_to_all(slabs)
        _run(slabs, PREC_FINAL)


def _matvec(slabs, comm) -> None:
    _run(slabs, MATVEC_ROWS)
    comm.halo(slabs)
    _run(slabs, MATVEC_COLS)


def iteration(slabs, comm) -> None:
    """One PCG iteration (krylov.py:99-116) of every local slab."""
    _matvec(slabs, comm)
    comm.allgather(slabs)
    _run(slabs, GAMMA_UPDATE)
    comm.allgather(slabs)
    _run(slabs, REL)
    _precond(slabs, comm)
    comm.allgather(slabs)
    _run(slabs, BETA_P)


def _capture(slabs, comm, iters: int):
    """A CUDA graph of ``iters`` iterations (kernels through the library on the capture
    stream, the communicator's copies / NCCL collectives captured by torch)."""
    dev = slabs[0].device
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        nat.context(dev)  # bind the native context to the capture stream
        for _ in range(iters):
            iteration(slabs, comm)
    nat.context(dev)  # and back to the current stream
    return g


def slab_pcg(slabs, comm, b_slabs, x0_slabs, config: KrylovConfig = KrylovConfig(),
             chunk: int = 4, graph: bool | None = None) -> list[SolveOutcome]:
    """Device-resident PCG over row slabs; same recurrence, stop test and exceptions as
    :func:`~.krylov.pcg`.  ``slabs`` are this process's :class:`Slab` objects (one per rank
    under ``torch.distributed``; all ``P`` under :class:`LoopbackComm`).  ``graph`` (default:
    CUDA slabs) replays ``chunk`` iterations -- phases and collectives -- as one CUDA graph
    between the host's stop checks instead of ~20 Python-issued calls per iteration."""
    hists = []
    for s, b, x0 in zip(slabs, b_slabs, x0_slabs):
        h = (torch.empty(config.max_iterations, dtype=torch.float64, device=s.device)
             if config.record_history else None)
        hists.append(h)
        s.start(b, x0, config, h)
    _matvec(slabs, comm)
    _run(slabs, RESIDUAL)
    comm.allgather(slabs)
    _run(slabs, START)
    _precond(slabs, comm)
    comm.allgather(slabs)
    _run(slabs, RZ0)
    if graph is None:
        graph = all(getattr(s, "device", torch.device("cpu")).type == "cuda" for s in slabs) \
            and getattr(comm, "graph_safe", True)
    g = _capture(slabs, comm, chunk) if graph else None
    done_it, reps = 0, 1
    while True:
        for _ in range(reps):
            if g is not None:
                g.replay()
            else:
                for _ in range(chunk):
                    iteration(slabs, comm)
        done_it += reps * chunk
        sts = [s.status() for s in slabs]
        if sts[0][1] or done_it >= config.max_iterations + chunk:
            break
        reps = min(reps * 2, 4)
    outs = []
    for s, st, h in zip(slabs, sts, hists):
        rc, done, it, conv, eit, ev = st
        if rc == nat.TVD_ERR_DIVERGED:
            raise SolverDivergenceError("pcg", eit)
        if rc == nat.TVD_ERR_INDEFINITE:
            raise IndefiniteOperatorError(eit, ev)
        nat.check(rc)
        hist = h[:it].cpu().numpy() if h is not None else np.array([])
        outs.append(SolveOutcome(s.buf(BUF_X).view(s.layout.rows, s.n).clone(), it, hist,
                                 bool(conv)))
    return outs


# ------------------------------------------------------------------ the FP-step setup
def slab_operators(h_op, u_slabs, layouts, comm, beta: float, alpha: float, kind: str = "M",
                   spacing: float = 1.0) -> list[SlabOperands]:
    """Each rank's operators of one FP step from its own rows of ``u`` -- no
    rank holds or recomputes the full image:

    * a one-row halo of ``u`` from each neighbour (``comm.halo_rows``), then the diffusivity
      of the rank's rows (``tvd_diffusivity_rows``, tv.py:42-71) and their block bands
      (``tvd_diffusion_bands_rows``, tv.py:138-175);
    * ``level2_project`` (precond.py:369-395) split at its transpose: the axis-1 band
      projections of the rank's rows (``tvd_band_project_lines``), ONE all-to-all of the
      ``R x R`` blocks of both level-1 results, the axis-0 projections of the rank's columns
      with the eigenvalue epilogue ``lambda_H^2 + alpha proj`` -- which leaves exactly the
      rank's rows of ``lambda^T``, the layout of the slab preconditioner's column pass;
    * the global min / max (``comm.allreduce_min_max``) for the positivity check and the
      ``1e-14 max`` clamp (precond.py:437-450), and ``d = 1 + alpha diag L > 0``
      (precond.py:558-560); D_X kinds get ``sqrt(d)`` of their rows.

    Every line is computed by the same kernels in the same order as the single-GPU assembly,
    so the operands are bit-identical to slices of ``assemble_preconditioner`` /
    ``DiffusionOperator`` (tests/test_gpu_slab.py).  ``u_slabs`` / ``layouts`` are this
    process's slabs (one under :class:`TorchComm`, all ``P`` under :class:`LoopbackComm`).
    Kinds: M, D_M (anti-reflective blur), R, D_R (reflective); zero-Neumann diffusion.
    """
    from .precond import IndefinitePreconditionerError

    base = kind.replace("D_", "")
    if base not in ("M", "R") or kind.endswith("_D"):
        raise ValueError(f"slab setup supports the kinds M, D_M, R, D_R, got {kind!r}")
    fam = nat.T_SINE_HAT if base == "M" else nat.T_DCT
    lay0 = layouts[0]
    n, P, R = lay0.n, lay0.nranks, lay0.rows
    dev = u_slabs[0].device
    lib = nat.load()
    ctx = nat.context(dev)
    dbl = dict(dtype=torch.float64, device=dev)
    exts = []
    for u, lay in zip(u_slabs, layouts):
        ext = torch.zeros((R + 2, n), **dbl)
        ext[1:R + 1].copy_(u)
        exts.append(ext)
    comm.halo_rows(exts, layouts)
    parts, sends0, sends1 = [], [], []
    min_d = float("inf")
    for ext, lay in zip(exts, layouts):
        lo = lay.row_lo
        a_h, a_v = torch.empty((R, n + 1), **dbl), torch.empty((R + 1, n), **dbl)
        nat.check(lib.tvd_diffusivity_rows(ctx, n, float(beta), float(spacing), ext.data_ptr(),
                                           lo - 1, R + 2, lo, lo + R, a_h.data_ptr(),
                                           a_v.data_ptr()))
        diag, inner, block = (torch.empty((R, n), **dbl), torch.empty((R, n - 1), **dbl),
                              torch.empty((R, n), **dbl))
        nat.check(lib.tvd_diffusion_bands_rows(ctx, n, float(spacing), a_h.data_ptr(),
                                               a_v.data_ptr(), lo, lo + R, diag.data_ptr(),
                                               inner.data_ptr(), block.data_ptr()))
        lam0, lam1 = torch.empty((R, n), **dbl), torch.zeros((R, n), **dbl)
        nat.check(lib.tvd_band_project_lines(ctx, fam, n, R, diag.data_ptr(), inner.data_ptr(),
                                             n - 1, 2.0, 0, None, 0.0, lam0.data_ptr(), None))
        nb = R if lay.rank < P - 1 else R - 1  # block rows i <= n - 2
        nat.check(lib.tvd_band_project_lines(ctx, fam, n, nb, block.data_ptr(), None, n, 0.0, 0,
                                             None, 0.0, lam1.data_ptr(), None))
        d = diag.mul(float(alpha)).add_(1.0)  # 1 + alpha diag L, numpy's two roundings
        min_d = min(min_d, float(d.min()))
        parts.append((a_h, a_v, d))
        sends0.append(lam0.view(R, P, R).permute(1, 0, 2).contiguous())
        sends1.append(lam1.view(R, P, R).permute(1, 0, 2).contiguous())
    recv0, recv1 = comm.all_to_all_blocks(sends0), comm.all_to_all_blocks(sends1)
    lamh_t = h_op.eigenvalues_device().t()
    eigs, lo_hi = [], []
    for lay, r0, r1 in zip(layouts, recv0, recv1):
        lo = lay.row_lo
        # line c = column lo + c of the level-1 results, element i = global row i
        lines0 = r0.permute(2, 0, 1).reshape(R, n).contiguous()
        lines1 = r1.permute(2, 0, 1).reshape(R, n).contiguous()
        lh = lamh_t[lo:lo + R].contiguous()
        eig_t = torch.empty((R, n), **dbl)
        mm = (ctypes.c_double * 2)()
        nat.check(lib.tvd_band_project_lines(ctx, fam, n, R, lines0.data_ptr(), lines1.data_ptr(),
                                             n, 2.0, 1, lh.data_ptr(), float(alpha),
                                             eig_t.data_ptr(), mm))
        eigs.append(eig_t)
        lo_hi.append((mm[0], mm[1]))
    min_d = comm.allreduce_min_max([(min_d, 0.0)] * len(layouts))[0]
    if not min_d > 0.0:
        raise IndefinitePreconditionerError(kind, alpha, min_d)
    mn, mx = comm.allreduce_min_max(lo_hi)
    if not mn > 0.0:
        raise IndefinitePreconditionerError(kind, alpha, mn)
    floor = 1e-14 * mx
    out = []
    for (a_h, a_v, d), eig_t in zip(parts, eigs):
        inv_t = 1.0 / torch.clamp(eig_t, min=floor)
        out.append(SlabOperands(a_h, a_v, inv_t, d.sqrt() if kind.startswith("D_") else None,
                                nat.PRE_TRANSFORM, fam, mn, mx, int((eig_t < floor).sum())))
    return out


def split_rows(a: torch.Tensor, nranks: int, rank: int) -> torch.Tensor:
    """Rank ``rank``'s slab of an ``n x n`` array (contiguous copy)."""
    R = a.shape[0] // nranks
    return a[rank * R:(rank + 1) * R].contiguous()
