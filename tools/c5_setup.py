import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200 import _native as nat
from paper_1011_5964_b200.harness import gen_psf
n = 8192
u = torch.rand(n, n, dtype=torch.float64, device="cuda")
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 31, 8.0)), tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    lop = tvd.DiffusionOperator(u, 0.05)
    torch.cuda.synchronize(); t1 = time.time()
    pre = tvd.assemble_preconditioner("M", hop, lop, 1e-4)
    torch.cuda.synchronize(); t2 = time.time()
    print(f"diffusivity {1e3*(t1-t0):.1f} ms  assemble {1e3*(t2-t1):.1f} ms", flush=True)
nat.profile(True)
pre = tvd.assemble_preconditioner("M", hop, lop, 1e-4)
torch.cuda.synchronize()
print(nat.profile_read())
