"""A/B timing of the 2048^2 normal-equation matvec (band passes + L) under library options,
with a bit-identity check against the first setting.  Profiling aid.

    python tools/op_ab.py OPTION v1,v2,...
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200 import _native as nat  # noqa: E402
from paper_1011_5964_b200.harness import gen_psf  # noqa: E402

name = sys.argv[1]
vals = [int(v) for v in sys.argv[2].split(",")]
n = 2048
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
u = torch.from_numpy(rng.uniform(size=(n, n))).cuda()
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 15, 4.0)),
                                 tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
lop = tvd.DiffusionOperator(u, 0.05)
sysm = tvd.NormalSystem(hop, lop, 2e-4)
out, ref = {}, None
saved = nat.get_option(name)
for v in vals:
    nat.set_option(name, v)
    for _ in range(3):
        r = sysm(w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        r = sysm(w)
    e1.record()
    torch.cuda.synchronize()
    ref = r.clone() if ref is None else ref
    out[v] = {"matvec_us": round(e0.elapsed_time(e1) / 50 * 1e3, 1),
              "identical": bool(torch.equal(r, ref))}
nat.set_option(name, saved)
print(json.dumps({name: out}))
