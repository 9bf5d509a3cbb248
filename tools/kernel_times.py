"""Per-kernel device times (torch.profiler / CUPTI) of the 2048^2 M^-1 solve at each PFA stage
count and of the normal-equation matvec.  Profiling aid: kernel names carry the pass mode
(k_dst_pipe<..., PM, ...>: bit 0 sandwich, bit 1 transposed output)."""
import collections
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200 import _native as nat  # noqa: E402
from paper_1011_5964_b200 import precond as P, transforms as T  # noqa: E402
from paper_1011_5964_b200.harness import gen_psf  # noqa: E402

n = 2048
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
u = torch.from_numpy(rng.uniform(size=(n, n))).cuda()
lam = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).cuda()
pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, lam, 1e-3)
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 15, 4.0)),
                                 tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
sysm = tvd.NormalSystem(hop, tvd.DiffusionOperator(u, 0.05), 2e-4)


def times(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    acc = collections.defaultdict(list)
    for e in prof.events():
        if e.device_type.name == "CUDA" and "memcpy" not in e.name.lower():
            acc[e.name].append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time)
    return {k[:110]: round(sum(v) / len(v), 1) for k, v in acc.items() if len(v) >= reps}


out = {}
for stages in (0, 3):
    nat.set_option("pfa_stages", stages)
    out[f"minv_stages{stages}"] = times(lambda: pre.apply_inverse(w))
nat.set_option("pfa_stages", 3)
out["matvec"] = times(lambda: sysm(w))
print(json.dumps(out, indent=1))
