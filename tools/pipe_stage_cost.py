"""Cost split of the 2048^2 M^-1 solve (three DST pipeline passes) by DFT stage: times the solve
with the engine's first k stages only (option pfa_stages = 0: pack / unpack and the passes'
streams alone, 1: + the q = 89 stage, 2: + the q = 23 stage = the full transform).  The
truncated transforms' outputs are meaningless; only the timing is.  Profiling aid."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1011_5964_b200 import _native as nat  # noqa: E402
from paper_1011_5964_b200 import precond as P, transforms as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
lam = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).cuda()
pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, lam, 1e-3)
out = {}
for stages in (0, 1, 2, 3):
    nat.set_option("pfa_stages", stages)
    for _ in range(3):
        pre.apply_inverse(w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        pre.apply_inverse(w)
    e1.record()
    torch.cuda.synchronize()
    out[stages] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
nat.set_option("pfa_stages", 3)
print(json.dumps({"minv_us_by_stages": out}))
