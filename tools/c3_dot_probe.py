"""Reference c3 FP step from its own iterate with exactly rounded dot products (parity evidence).

    PYTHONPATH=/root/reference/pkg/src python tools/c3_dot_probe.py TRACEDIR K [K ...]

Runs the reference's own ``krylov.pcg`` (``krylov.py:82-116``) and operators from ``u_K``
twice: as shipped (``_dot`` / ``_norm`` = BLAS ``ddot``, ``krylov.py:70-75``, whose summation
order and error depend on the BLAS thread count) and with both replaced by exactly rounded
dot products (``math.fsum`` of the exact products, via a Dekker split).  Output
``TRACEDIR/dot_K.json``.
"""
import json
import math
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))

from tvdeblur import krylov as rk  # noqa: E402
from tvdeblur.blur import BoundaryCondition, StructuredBlurOperator, SymmetricPsf  # noqa: E402
from tvdeblur.krylov import KrylovConfig, pcg  # noqa: E402
from tvdeblur.precond import assemble_preconditioner  # noqa: E402
from tvdeblur.tv import DiffusionOperator  # noqa: E402

from paper_1011_5964_b200 import harness as bh  # noqa: E402


from c3_dot_probe_lib import exact_dot  # noqa: E402



d = pathlib.Path(sys.argv[1])
spec = bh.CONFIGS["c3"]
psf = SymmetricPsf(np.load(d / "psf.npy"))
v = np.load(d / "v.npy")
n = v.shape[0]
hop = StructuredBlurOperator(psf, BoundaryCondition.ANTI_REFLECTIVE, n)
rhs = hop.apply_transpose_fast(v)
blas_dot, blas_norm = rk._dot, rk._norm


def exact_norm(x) -> float:
    return math.sqrt(exact_dot(x, x))
for k in map(int, sys.argv[2:]):
    u = np.load(d / f"u_{k}.npy")
    lop = DiffusionOperator(u, spec.beta)
    pre = assemble_preconditioner("M", hop, lop, spec.alpha)

    def a_fast(w):
        return hop.apply_transpose_fast(hop.apply_fast(w)) + spec.alpha * lop.apply(w)

    out = {"k": k}
    for name, dot, nrm in (("blas_dot", blas_dot, blas_norm),
                           ("exact_dot", exact_dot, exact_norm)):
        rk._dot, rk._norm = dot, nrm
        res = pcg(a_fast, pre.apply_inverse, rhs, u, KrylovConfig(spec.tol, 2000, True))
        out[name] = {"count": int(res.iterations), "hist": [float(h) for h in res.residual_history]}
        print(k, name, res.iterations, res.residual_history[-3:], flush=True)
    rk._dot, rk._norm = blas_dot, blas_norm
    (d / f"dot_{k}.json").write_text(json.dumps(out))
