"""A/B of the 2048^2 (or argv[1]) preconditioner assembly under a library option: time per
assembly and bit-identity of the eigenvalues.  python tools/ab_assembly.py OPTION v1,v2 [n]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200 import _native as nat
from paper_1011_5964_b200.harness import gen_psf
name, vals = sys.argv[1], [int(v) for v in sys.argv[2].split(",")]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
rng = np.random.default_rng(0)
u = torch.from_numpy(rng.uniform(size=(n, n))).cuda()
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 15, 4.0)),
                                 tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
lop = tvd.DiffusionOperator(u, 0.05)
ref = None
for v in vals:
    nat.set_option(name, v)
    for _ in range(3): pre = tvd.assemble_preconditioner("M", hop, lop, 2e-4, defer_checks=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): pre = tvd.assemble_preconditioner("M", hop, lop, 2e-4, defer_checks=True)
    e1.record(); torch.cuda.synchronize()
    lam = pre.eigenvalues_device.clone()
    ref = lam if ref is None else ref
    print(name, v, round(e0.elapsed_time(e1) / 10 * 1e3, 1), "us  identical:", bool(torch.equal(lam, ref)))
