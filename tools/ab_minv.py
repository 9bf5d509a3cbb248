"""A/B of one 2048^2 M^-1 application under a library option, with bit-identity check.
    python tools/ab_minv.py OPTION v1,v2,...   (profiling aid)"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1011_5964_b200 import _native as nat
from paper_1011_5964_b200 import precond as P, transforms as T
name, vals = sys.argv[1], [int(v) for v in sys.argv[2].split(",")]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
lam = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).cuda()
pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, lam, 1e-3)
ref = None
for v in vals:
    nat.set_option(name, v)
    for _ in range(3): z = pre.apply_inverse(w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): z = pre.apply_inverse(w)
    e1.record(); torch.cuda.synchronize()
    ref = z.clone() if ref is None else ref
    print(name, v, round(e0.elapsed_time(e1) / 20 * 1e3, 1), "us  identical:", bool(torch.equal(z, ref)))
