"""Test double of one rank's native slab solver (``tvd_slab``, csrc/tvd_slab.cuh) in numpy.

Test infrastructure only: it lets the multi-rank schedule of ``paper_1011_5964_b200.slab``
run under ``torch.distributed`` / gloo on CPU (the CUDA phases cannot run without a GPU).
Each phase reads and writes only this rank's buffers -- slab rows, halo rows, all-to-all
blocks, one contribution per dot product -- with the same layouts as the native phases, so
a wrong halo, block order or segment map in the schedule / communicators shows up as a
mismatch against the full-array oracle PCG (oracle/tvd_oracle.py pcg, krylov.py:82-116).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from oracle import tvd_oracle as O
from paper_1011_5964_b200 import slab as SL


def ar_blur_matrix(g: np.ndarray, n: int) -> np.ndarray:
    """Dense 1D blur with anti-reflective padding x_{-j} = 2 x_0 - x_j (blur.py:45-50)."""
    m = (len(g) - 1) // 2
    H = np.zeros((n, n))
    for i in range(n):
        for k in range(-m, m + 1):
            j = i + k
            c = g[k + m]
            if j < 0:
                H[i, 0] += 2 * c
                H[i, -j] -= c
            elif j >= n:
                H[i, n - 1] += 2 * c
                H[i, 2 * (n - 1) - j] -= c
            else:
                H[i, j] += c
    return H


def sinehat_matrix(n: int) -> np.ndarray:
    return O.sinehat(np.eye(n), axis=0)


class MirrorSlab:
    """One rank of the slab PCG with numpy phases (same buffers and state machine)."""

    def __init__(self, G0, G1, alpha, a_h, a_v, inv_eig, d_sqrt, nranks, rank, khalo,
                 transform=True):
        n = G0.shape[0]
        self.n, self.device = n, torch.device("cpu")
        self.layout = SL.SlabLayout(n, nranks, rank, khalo, transform)
        R, lo = self.layout.rows, self.layout.row_lo
        bw = max(abs(i - j) for i, j in zip(*np.nonzero(G0)))
        assert bw <= khalo, (bw, khalo)
        self.G0, self.G1, self.alpha = G0, G1, alpha
        self.a_h, self.a_v = a_h[lo:lo + R], a_v[lo:lo + R + 1]
        self.inv_t = None if inv_eig is None else np.ascontiguousarray(inv_eig.T[lo:lo + R])
        self.d = None if d_sqrt is None else d_sqrt[lo:lo + R]
        self.S = sinehat_matrix(n)
        shapes = {SL.BUF_X: R * n, SL.BUF_R: R * n, SL.BUF_Z: R * n, SL.BUF_Q: R * n,
                  SL.BUF_P_EXT: (R + 2) * n, SL.BUF_T_EXT: (R + 2 * khalo) * n,
                  SL.BUF_SEND: R * n, SL.BUF_RECV: R * n, SL.BUF_CONTRIB: 1,
                  SL.BUF_GATHER: nranks}
        self._np = {k: np.full(v, np.nan) for k, v in shapes.items()}
        self._t = {k: torch.from_numpy(a) for k, a in self._np.items()}
        self.st = {}

    # buffers as (rows, n) numpy views
    def buf(self, which):
        return self._t[which]

    def _a(self, which, rows=None):
        a = self._np[which]
        return a if rows is None else a.reshape(rows, self.n)

    def start(self, b, x0, config, history):
        R = self.layout.rows
        self.b = b.numpy().reshape(R, self.n)
        self.tol, self.max_it, self.hist = config.tol, config.max_iterations, history
        self._a(SL.BUF_X, R)[:] = x0.numpy().reshape(R, self.n)
        self._a(SL.BUF_P_EXT, R + 2)[1:R + 1] = x0.numpy().reshape(R, self.n)
        self.loop = False
        self.st = dict(done=0, k=0, iters=0, converged=0, status=0, err_iter=0, err_val=0.0)

    def _skip(self):
        return self.st["done"] != 0

    def _segmented(self, which):
        """Lines of the all-to-all receive buffer: line l, element e at block e // R."""
        R, n = self.layout.rows, self.n
        blocks = self._a(which).reshape(n // R, R, R)  # [block][line][within]
        return np.concatenate(list(blocks), axis=1)  # (R lines, n)

    def phase(self, ph):  # noqa: C901 -- one branch per phase, like slab_phase
        lay, n = self.layout, self.n
        R, lo, K = lay.rows, lay.row_lo, lay.khalo
        st = self.st
        P_ext = self._a(SL.BUF_P_EXT, R + 2)
        p = P_ext[1:R + 1]
        x, r, z, q = (self._a(w, R) for w in (SL.BUF_X, SL.BUF_R, SL.BUF_Z, SL.BUF_Q))
        gsum = lambda: float(sum(self._np[SL.BUF_GATHER][: lay.nranks]))  # noqa: E731
        contrib = self._np[SL.BUF_CONTRIB]
        if ph == SL.MATVEC_ROWS:
            if self.loop and self._skip():
                return
            self._a(SL.BUF_T_EXT, R + 2 * K)[K:K + R] = p @ self.G1.T
        elif ph == SL.MATVEC_COLS:
            if self.loop and self._skip():
                return
            T = self._a(SL.BUF_T_EXT, R + 2 * K)
            k0, k1 = max(0, lo - K), min(n, lo + R + K)
            q[:] = self.G0[lo:lo + R, k0:k1] @ T[k0 - (lo - K):k1 - (lo - K)]
            W = P_ext.copy()
            if lay.rank == 0:
                W[0] = W[1]
            if lay.rank == lay.nranks - 1:
                W[R + 1] = W[R]
            Wc = W[1:R + 1]
            Wl = np.concatenate([Wc[:, :1], Wc[:, :-1]], axis=1)
            Wr = np.concatenate([Wc[:, 1:], Wc[:, -1:]], axis=1)
            fl = self.a_h[:, :n] * (Wc - Wl)
            fr = self.a_h[:, 1:] * (Wr - Wc)
            fu = self.a_v[:R] * (Wc - W[0:R])
            fd = self.a_v[1:] * (W[2:R + 2] - Wc)
            q += self.alpha * (-((fr - fl) + (fd - fu)))
            contrib[0] = float(np.sum(p * q))
        elif ph == SL.RESIDUAL:
            r[:] = self.b - q
            contrib[0] = float(np.sum(r * r))
        elif ph == SL.START:
            st.update(r0=math.sqrt(gsum()), k=1, done=0, iters=0, converged=0, status=0)
            if st["r0"] == 0.0:
                st.update(done=1, converged=1)
        elif ph == SL.GAMMA_UPDATE:
            if self._skip():
                return
            g = gsum()
            if not math.isfinite(g):
                st.update(status=2, err_iter=st["k"], done=1)
                return
            if g <= 0:
                st.update(status=3, err_iter=st["k"], err_val=g, done=1)
                return
            step = st["rz"] / g
            x += step * p
            r -= step * q
            contrib[0] = float(np.sum(r * r))
        elif ph == SL.REL:
            if self._skip():
                return
            rel = math.sqrt(gsum()) / st["r0"]
            if not math.isfinite(rel):
                st.update(status=2, err_iter=st["k"], done=1)
                return
            if self.hist is not None:
                self.hist[st["k"] - 1] = rel
            if rel < self.tol:
                st.update(iters=st["k"], converged=1, done=1)
        elif ph in (SL.PREC_ROWS, SL.PREC_COLS, SL.PREC_FINAL):
            if self._skip():
                return
            if not lay.exchanges:
                z[:] = r if self.d is None else r / self.d
                contrib[0] = float(np.sum(r * z))
                return
            send = self._a(SL.BUF_SEND)
            if ph == SL.PREC_ROWS:
                y = (r if self.d is None else r / self.d) @ self.S.T
                send[:] = y.T.ravel()
            elif ph == SL.PREC_COLS:
                lines = self._segmented(SL.BUF_RECV)
                y = ((lines @ self.S.T) * self.inv_t) @ self.S.T
                send[:] = y.T.ravel()
            else:
                y = self._segmented(SL.BUF_RECV) @ self.S.T
                z[:] = y if self.d is None else y / self.d
                contrib[0] = float(np.sum(z * r))
        elif ph == SL.RZ0:
            if self._skip():
                return
            st["rz"] = gsum()
            p[:] = z
            self.loop = True
        elif ph == SL.BETA_P:
            if self._skip():
                return
            rz = gsum()
            beta = rz / st["rz"]
            st["rz"] = rz
            st["k"] += 1
            if st["k"] > self.max_it:
                st.update(iters=self.max_it, converged=0, done=1)
                return
            p[:] = z + beta * p
        else:
            raise ValueError(ph)

    def status(self):
        s = self.st
        rc = s["status"] if s["done"] else 0
        return rc, s["done"], s["iters"], s["converged"], s["err_iter"], s["err_val"]


def build_case(n=32, m=2, sigma=1.0, alpha=1e-2, beta=0.1, seed=3):
    """Full-size operators of a small AR problem + the oracle's inverse eigenvalues."""
    from paper_1011_5964_b200.harness import gen_psf

    h = gen_psf("gaussian", m, sigma)
    g = h.sum(axis=1)
    rng = np.random.default_rng(seed)
    u = rng.uniform(size=(n, n))
    v = O.blur(u, h, "anti_reflective") + 1e-3 * rng.standard_normal((n, n))
    H1 = ar_blur_matrix(g / g.sum(), n)
    G = H1.T @ H1
    a_h, a_v = O.diffusivity(v, beta)
    lam_h = O.blur_eigenvalues(h, "anti_reflective", n)
    _, lam_inv, d_sqrt, _ = O.assemble("D_M", lam_h, O.diffusion_bands(a_h, a_v), alpha)
    rhs = O.blur_transpose(v, h, "anti_reflective")
    return dict(h=h, v=v, G=G, H1=H1, a_h=a_h, a_v=a_v, lam_inv=lam_inv, d_sqrt=d_sqrt,
                rhs=rhs, alpha=alpha)
