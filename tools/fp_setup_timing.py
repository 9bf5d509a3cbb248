"""CUDA-event timing of the per-FP-step setup at n (diffusivity, bands, assembly).  Profiling aid."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200 import _native as nat  # noqa: E402
from paper_1011_5964_b200.harness import gen_psf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
m = int(sys.argv[2]) if len(sys.argv) > 2 else 15
u = torch.rand(n, n, dtype=torch.float64, device="cuda")
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", m, m / 3.75)),
                                 tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
for _ in range(2):
    lop = tvd.DiffusionOperator(u, 0.05)
    pre = tvd.assemble_preconditioner("M", hop, lop, 2e-4)
torch.cuda.synchronize()
nat.profile(True)
lop = tvd.DiffusionOperator(u, 0.05)
pre = tvd.assemble_preconditioner("M", hop, lop, 2e-4)
torch.cuda.synchronize()
print(json.dumps({k: [round(t * 1e3, 1), c] for k, (t, c) in nat.profile_read().items()}))
