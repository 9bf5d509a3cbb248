"""CUDA-event timing of the hot-path operators at n (default 2048, config-3 PSF): the fused
normal-equation matvec (band passes + L) and the M^-1 solve.  Profiling aid."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200 import precond as P, transforms as T  # noqa: E402
from paper_1011_5964_b200.harness import gen_psf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
m = int(sys.argv[2]) if len(sys.argv) > 2 else 15
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
u = torch.from_numpy(rng.uniform(size=(n, n))).cuda()
lam = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).cuda()
pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, lam, 1e-3)
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", m, m / 3.75)),
                                 tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
lop = tvd.DiffusionOperator(u, 0.05)
sysm = tvd.NormalSystem(hop, lop, 2e-4)
out = {}
for name, f in (("matvec", lambda: sysm(w)), ("minv", lambda: pre.apply_inverse(w))):
    for _ in range(3):
        r = f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        r = f()
    e1.record()
    torch.cuda.synchronize()
    out[name + "_us"] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    out[name + "_norm"] = float(r.norm())
print(json.dumps(out))
