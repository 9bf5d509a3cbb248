import sys, time, pathlib
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200 import transforms as T, precond as P
from paper_1011_5964_b200.harness import gen_psf
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(0)
w = torch.randn(n, n, dtype=torch.float64, device="cuda")
lam = torch.rand(n, n, dtype=torch.float64, device="cuda") + 0.5
pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, lam, 1e-3)
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 31, 8.0)), tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
lop = tvd.DiffusionOperator(w, 0.05)
sys_ = tvd.NormalSystem(hop, lop, 2e-4)
for name, f in (("minv", lambda: pre.apply_inverse(w)), ("matvec", lambda: sys_(w))):
    f(); torch.cuda.synchronize()
    t = time.time(); f(); torch.cuda.synchronize()
    print(name, f"{(time.time() - t) * 1e3:.1f} ms", flush=True)
# identity check: lambda = 1 -> M^-1 = S S = I (orthonormal, self-inverse DST-I)
one = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, torch.ones(n, n, dtype=torch.float64, device="cuda"), 1e-3)
z = one.apply_inverse(w)
print("identity rel err", float((z - w).norm() / w.norm()), flush=True)
# per-FP-step assembly at this size (band FFTs of length 2(n - 1))
import time as _t
hop2 = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 31, 8.0)), tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
lop2 = tvd.DiffusionOperator(w * 0.01, 0.05)
torch.cuda.synchronize(); t0 = _t.time()
pa = tvd.assemble_preconditioner("M", hop2, lop2, 2e-4)
torch.cuda.synchronize(); print("assembly", f"{(_t.time() - t0) * 1e3:.1f} ms", flush=True)
torch.cuda.synchronize(); t0 = _t.time()
pa = tvd.assemble_preconditioner("M", hop2, lop2, 2e-4)
torch.cuda.synchronize(); print("assembly (warm)", f"{(_t.time() - t0) * 1e3:.1f} ms", flush=True)
