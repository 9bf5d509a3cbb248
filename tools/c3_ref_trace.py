"""Trace the REFERENCE's config-c3 restore (build container only; parity evidence).

    PYTHONPATH=/root/reference/pkg/src python tools/c3_ref_trace.py OUTDIR [FP_STEPS] [--exact]
        [--exact-dots]

Runs ``tvdeblur.pipeline.restore`` (reference ``pipeline.py:182-276``) unchanged on the c3
fixture of ``tests/golden/make_golden.py`` and, through a wrapper around the module-level
``pcg`` it calls (``pipeline.py:198``), records for every FP step the starting iterate
``u_k`` (``OUTDIR/u_{k}.npy``), the reference's residual history
(``krylov.py:105-109``) and the solution.  ``tools/c3_step_probe.py`` then replays single FP
steps from these iterates with other operator variants and with the GPU.  ``--exact`` runs the
reference with ``use_fast_blur=False`` (``pipeline.py:75,167-179``): its exact pad / convolve /
crop ``H`` and full-convolve + fold ``H^T`` (``blur.py:226-247``) in place of the transform
path.  ``--exact-dots`` replaces the reference's BLAS ``_dot`` / ``_norm`` (krylov.py:70-75)
by exactly rounded dot products (tools/c3_dot_probe.py ``exact_dot``): the reference's
recurrence with reductions free of summation-order error.
"""
import json
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

from tvdeblur import harness as rh  # noqa: E402
from tvdeblur import krylov as rk  # noqa: E402
from tvdeblur import pipeline as rpipe  # noqa: E402
from tvdeblur.blur import BoundaryCondition  # noqa: E402
from tvdeblur.krylov import KrylovConfig  # noqa: E402
from tvdeblur.pipeline import PrecondSelector, RestorationConfig, restore  # noqa: E402

from paper_1011_5964_b200 import harness as bh  # noqa: E402

out = pathlib.Path(sys.argv[1])
out.mkdir(parents=True, exist_ok=True)
spec = bh.CONFIGS["c3"]
exact = "--exact" in sys.argv
exact_dots = "--exact-dots" in sys.argv
argv = [a for a in sys.argv if a not in ("--exact", "--exact-dots")]
if exact_dots:
    import math

    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))
    from c3_dot_probe_lib import exact_dot

    rk._dot = exact_dot
    rk._norm = lambda x: math.sqrt(exact_dot(x, x))
fp = int(argv[2]) if len(argv) > 2 else spec.fp_steps
psf = rh.gen_psf("gaussian", spec.m, spec.sigma)
ext = bh.gen_piecewise_image(spec.n, spec.m, spec.rects, spec.disks, 2023, spec.ramp)
v = rh.blur_and_observe(ext, psf, spec.n, spec.nsr, 7)
np.save(out / "v.npy", v)
np.save(out / "psf.npy", psf.coefficients)
log = {"counts": [], "hist": [], "r0": [], "seconds": []}
real_pcg = rk.pcg


def traced(apply_a, apply_minv, b, x0, config):
    k = len(log["counts"])
    np.save(out / f"u_{k}.npy", np.asarray(x0))
    if k == 0:
        np.save(out / "rhs.npy", np.asarray(b))
    t0 = time.perf_counter()
    res = real_pcg(apply_a, apply_minv, b, x0,
                   KrylovConfig(config.tol, config.max_iterations, True))
    log["seconds"].append(time.perf_counter() - t0)
    log["counts"].append(int(res.iterations))
    log["hist"].append([float(h) for h in res.residual_history])
    (out / "trace.json").write_text(json.dumps(log))
    print(f"FP {k}: {res.iterations} its, last rel {res.residual_history[-3:]}", flush=True)
    return res


rpipe.pcg = traced
cfg = RestorationConfig(bc_h=BoundaryCondition.ANTI_REFLECTIVE, alpha=spec.alpha, beta=spec.beta,
                        preconditioner=PrecondSelector.X, fp_tol=1e-300, fp_max=fp,
                        inner=KrylovConfig(tol=spec.tol, max_iterations=2000),
                        use_fast_blur=not exact)
rep = restore(v, psf, cfg, u_true=ext[spec.m:spec.m + spec.n, spec.m:spec.m + spec.n])
np.save(out / f"u_{fp}.npy", rep.restored)
log["gradient_norms"] = [float(g) for g in rep.gradient_norms]
(out / "trace.json").write_text(json.dumps(log))
print("counts", rep.inner_iterations)
