"""Config-c3 restore (20 FP steps, 2048^2) on the device under rounding-different but equally
valid operator paths -- the device's own run-to-run spread, next to the reference's
(tests/golden/c3_parity.json).  Variants: default; generic mixed-radix DST engine
(generic_fft); CUDA-core band passes (band_slide); general 2D blur (general_blur); eager
solves (solver_graph 0, bit-identical to the default).  Output gpurun_out/c3_variants.json:
per-FP counts, the restored image's norm, sub-sample and 64-projection sketch."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200 import _native as nat  # noqa: E402
from paper_1011_5964_b200.harness import CONFIGS, make_problem  # noqa: E402
from sketch import sketch_torch  # noqa: E402

spec = CONFIGS["c3"]
h, v, u_true = make_problem(spec)
dev = torch.device("cuda", 0)
cfg = tvd.RestorationConfig(bc_h=tvd.BoundaryCondition.ANTI_REFLECTIVE, alpha=spec.alpha,
                            beta=spec.beta, preconditioner=tvd.PrecondSelector.X, fp_tol=1e-300,
                            fp_max=spec.fp_steps,
                            inner=tvd.KrylovConfig(tol=spec.tol, max_iterations=2000))
out = {}
for name, opt, val in (("default", None, 0), ("generic_fft", "generic_fft", 1),
                       ("band_slide", "band_slide", 1), ("general_blur", "general_blur", 1),
                       ("eager", "solver_graph", 0)):
    if opt:
        saved = nat.get_option(opt, dev)
        nat.set_option(opt, val, dev)
    rep = tvd.restore(torch.from_numpy(v).to(dev), tvd.SymmetricPsf(h), cfg, u_true=u_true)
    if opt:
        nat.set_option(opt, saved, dev)
    r = rep.restored
    out[name] = {"counts": rep.inner_iterations, "norm": float(torch.linalg.norm(r)),
                 "rre": rep.rre, "sketch": sketch_torch(r, 64).tolist(),
                 "sub": r[::16, ::16].cpu().numpy().tolist()}
    print(name, rep.inner_iterations, flush=True)
ref = np.array(out["default"]["sub"])
for name, o in out.items():
    o["sub_rel_vs_default"] = float(np.linalg.norm(np.array(o["sub"]) - ref) / np.linalg.norm(ref))
pathlib.Path("gpurun_out").mkdir(exist_ok=True)
pathlib.Path("gpurun_out/c3_variants.json").write_text(json.dumps(out))
