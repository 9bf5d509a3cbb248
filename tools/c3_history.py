"""Per-FP-step PCG residual histories of config c3 on the GPU (parity diagnostics)."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200 import krylov  # noqa: E402
from paper_1011_5964_b200.harness import CONFIGS, make_problem  # noqa: E402

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
h, v, ut = make_problem(spec)
hist = []
orig = krylov._pcg_fused


def spy(system, pre, b, x0, config):
    out = orig(system, pre, b, x0, krylov.KrylovConfig(config.tol, config.max_iterations, True))
    hist.append([float(x) for x in out.residual_history[-4:]])
    return out


krylov._pcg_fused = spy
cfg = tvd.RestorationConfig(bc_h=tvd.BoundaryCondition(spec.bc), alpha=spec.alpha, beta=spec.beta,
                            preconditioner=tvd.PrecondSelector.X, fp_tol=1e-300,
                            fp_max=spec.fp_steps,
                            inner=tvd.KrylovConfig(tol=spec.tol, max_iterations=2000))
rep = tvd.restore(v, tvd.SymmetricPsf(h), cfg, u_true=ut)
print(json.dumps({"counts": rep.inner_iterations, "tail": hist, "rre": rep.rre}))
np.save("gpurun_out/c3_restored.npy", np.asarray(rep.restored))
