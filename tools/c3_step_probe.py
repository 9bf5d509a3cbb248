"""Replay single config-c3 FP steps of the reference from its own iterates (parity evidence).

    PYTHONPATH=/root/reference/pkg/src python tools/c3_step_probe.py TRACEDIR K [K ...]

``TRACEDIR`` holds ``tools/c3_ref_trace.py``'s output (the reference's ``u_k`` per FP step,
its residual histories).  For every FP step ``k`` the reference's own ``krylov.pcg``
(``krylov.py:82-116``) is run from ``u_k`` on two operator variants of the reference:

* ``fast``  -- the reference's default system (``pipeline.py:167-179,209-210``): ``H`` =
  ``apply_fast``, ``H^T`` = ``apply_transpose_fast`` (the AR transform transpose path,
  ``blur.py:302-314``) for both the rhs and the matvec;
* ``exact`` -- the same with the reference's exact adjoint ``apply_transpose``
  (``blur.py:236-247``: full convolution + fold) for the rhs and the matvec: the operator
  whose symmetric rounding the GPU's exact ``H^T`` follows.

It also splits the initial residual ``r0 = rhs - A u_k`` of the fast system into the part
the exact system shares and the rest (the fast transpose's rounding), and reports how much
of that rest lies in the border rows / columns 0 and n-1.  Output: ``TRACEDIR/step_K.json``.
"""
import json
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

from tvdeblur.blur import BoundaryCondition, StructuredBlurOperator, SymmetricPsf  # noqa: E402
from tvdeblur.krylov import KrylovConfig, pcg  # noqa: E402
from tvdeblur.precond import assemble_preconditioner  # noqa: E402
from tvdeblur.tv import DiffusionOperator  # noqa: E402

from paper_1011_5964_b200 import harness as bh  # noqa: E402

d = pathlib.Path(sys.argv[1])
spec = bh.CONFIGS["c3"]
v = np.load(d / "v.npy")
psf = SymmetricPsf(np.load(d / "psf.npy"))
n = v.shape[0]
hop = StructuredBlurOperator(psf, BoundaryCondition.ANTI_REFLECTIVE, n)
rhs_fast = hop.apply_transpose_fast(v)
rhs_exact = hop.apply_transpose(v)
trace = json.loads((d / "trace.json").read_text())


def border_share(e):
    mask = np.zeros(e.shape, bool)
    mask[[0, -1], :] = True
    mask[:, [0, -1]] = True
    tot = float(np.sum(e * e))
    return float(np.sum(e[mask] ** 2) / tot) if tot > 0 else 0.0


for k in map(int, sys.argv[2:]):
    u = np.load(d / f"u_{k}.npy")
    lop = DiffusionOperator(u, spec.beta)
    pre = assemble_preconditioner("M", hop, lop, spec.alpha)
    a = spec.alpha

    def a_fast(w):
        return hop.apply_transpose_fast(hop.apply_fast(w)) + a * lop.apply(w)

    def a_exact(w):
        return hop.apply_transpose(hop.apply_fast(w)) + a * lop.apply(w)

    r0f = rhs_fast - a_fast(u)
    r0e = rhs_exact - a_exact(u)
    noise = r0f - r0e
    out = {"k": k, "ref_trace_count": trace["counts"][k], "ref_trace_hist": trace["hist"][k],
           "r0_fast": float(np.linalg.norm(r0f)), "r0_exact": float(np.linalg.norm(r0e)),
           "rhs_norm": float(np.linalg.norm(rhs_fast)),
           "r0_noise_rel": float(np.linalg.norm(noise) / np.linalg.norm(r0e)),
           "r0_noise_border_share": border_share(noise)}
    cfg = KrylovConfig(spec.tol, 2000, True)
    for name, op, rhs in (("fast", a_fast, rhs_fast), ("exact", a_exact, rhs_exact)):
        t0 = time.perf_counter()
        res = pcg(op, pre.apply_inverse, rhs, u, cfg)
        out[name] = {"count": int(res.iterations),
                     "hist": [float(h) for h in res.residual_history],
                     "seconds": time.perf_counter() - t0}
        np.save(d / f"x_{name}_{k}.npy", res.solution)
        print(k, name, res.iterations, res.residual_history[-3:], flush=True)
    (d / f"step_{k}.json").write_text(json.dumps(out))
    print(json.dumps({kk: vv for kk, vv in out.items() if "hist" not in kk and kk not in ("fast", "exact")}), flush=True)
