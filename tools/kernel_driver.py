"""Minimal driver for ncu: runs the hot-path passes at n=2048 a few times."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200 import transforms as T, precond as P
from paper_1011_5964_b200.harness import gen_psf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
lam = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).cuda()
pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, lam, 1e-3)
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 15, 4.0)),
                                 tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
lop = tvd.DiffusionOperator(w, 0.05)
sys_ = tvd.NormalSystem(hop, lop, 2e-4)
for _ in range(reps):
    z = pre.apply_inverse(w)
    q = sys_(w)
torch.cuda.synchronize()
print("ok", float(z.norm()), float(q.norm()))
