"""Config-c3 single FP step with mixed device / host operators (parity diagnostics).

    python tools/c3_mixed_step.py DIR K

From the reference's iterate ``u_K`` (``tools/c3_ref_trace.py``), runs the oracle's
restatement of the reference PCG loop (``oracle/tvd_oracle.py`` ``pcg`` = krylov.py:82-116:
numpy updates, BLAS dots) with each combination of
  A    : device ``NormalSystem`` (exact H^T, banded Gram passes) | host oracle fast path
         (the reference's apply_transpose_fast(apply_fast(.)) + alpha L)
  M^-1 : device DST engine | host scipy.fft restatement,
both preconditioners from the reference's own eigenvalues ``lam_K.npy``, and reports the
count and residual history of each.  Output ``gpurun_out/c3_mixed_K.json``.
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from oracle import tvd_oracle as O  # noqa: E402
from paper_1011_5964_b200.harness import CONFIGS  # noqa: E402

O.set_workers(16)
d = pathlib.Path(sys.argv[1])
k = int(sys.argv[2])
spec = CONFIGS["c3"]
dev = torch.device("cuda", 0)
v = np.load(d / "v.npy")
h = np.load(d / "psf.npy")
rhs_ref = np.load(d / "rhs.npy")
u = np.load(d / f"u_{k}.npy")
lam = np.load(d / f"lam_{k}.npy")
n = v.shape[0]
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), tvd.BoundaryCondition.ANTI_REFLECTIVE, n,
                                 device=dev)
lop = tvd.DiffusionOperator(torch.from_numpy(u).to(dev), spec.beta, device=dev)
system = tvd.NormalSystem(hop, lop, spec.alpha)
pre = tvd.FactoredPreconditioner("M", tvd.TransformKind.SINE_HAT, lam, spec.alpha, device=dev)
lam_inv = 1.0 / np.maximum(lam, 1e-14 * lam.max())
lam_h = O.blur_eigenvalues(h, "anti_reflective", n)
a_h, a_v = O.diffusivity(u, spec.beta)


def a_dev(w):
    return system(w)


def a_host(w):
    hw = O.blur_fast(w, lam_h, "anti_reflective")
    return O.blur_transpose_fast(hw, lam_h, "anti_reflective") + spec.alpha * O.diffusion_apply(a_h, a_v, w)


def m_dev(r):
    return pre.apply_inverse(r)


def m_host(r):
    return O.precond_solve("sine_hat", lam_inv, r)


out = {}
for an, af in (("A_dev", a_dev), ("A_host", a_host)):
    for mn, mf in (("M_dev", m_dev), ("M_host", m_host)):
        for bn, b in (("b_ref", rhs_ref),):
            x, its, hist, ok = O.pcg(af, mf, b, u, spec.tol, 2000, True)
            out[f"{an}+{mn}"] = {"count": int(its), "hist": [float(t) for t in hist]}
            print(k, an, mn, its, hist[-3:], flush=True)
pathlib.Path("gpurun_out").mkdir(exist_ok=True)
pathlib.Path(f"gpurun_out/c3_mixed_{k}.json").write_text(json.dumps(out))
