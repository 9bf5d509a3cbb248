"""Split one c3-style e2e step (diffusivity, preconditioner assembly, PCG) into its phases:
CUDA-event device time and host wall time per phase, averaged over a few steps.  Profiling aid:
``python tools/e2e_breakdown.py [config]``."""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200.harness import CONFIGS, make_problem  # noqa: E402

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dev = torch.device("cuda", 0)
n = spec.n
bc = tvd.BoundaryCondition(spec.bc)
kind = "M" if bc is tvd.BoundaryCondition.ANTI_REFLECTIVE else "R"
h, v, _ = make_problem(spec)
cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=2000)
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), bc, n, device=dev)
v_dev = torch.from_numpy(v).to(dev)
rhs = (hop.apply if bc is tvd.BoundaryCondition.REFLECTIVE else hop.apply_transpose)(v_dev)
u = v_dev.clone()
for _ in range(2):
    lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
    pre = tvd.assemble_preconditioner(kind, hop, lop, spec.alpha)
    u = tvd.pcg(tvd.NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, u, cfg).solution


def one(acc):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    wall = []
    ev[0].record()
    t0 = time.perf_counter()
    lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
    ev[1].record()
    t1 = time.perf_counter()
    pre = tvd.assemble_preconditioner(kind, hop, lop, spec.alpha)
    ev[2].record()
    t2 = time.perf_counter()
    res = tvd.pcg(tvd.NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, u, cfg)
    ev[3].record()
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    wall = [t1 - t0, t2 - t1, t3 - t2]
    for k, name in enumerate(("diffusivity", "assembly", "pcg")):
        a = acc.setdefault(name, [0.0, 0.0])
        a[0] += ev[k].elapsed_time(ev[k + 1])
        a[1] += 1e3 * wall[k]
    acc.setdefault("iters", [0, 0])[0] += res.iterations


for _ in range(3):
    one({})
acc = {}
K = 5
for _ in range(K):
    one(acc)
out = {k: {"device_ms": round(a[0] / K, 3), "host_ms": round(a[1] / K, 3)}
       for k, a in acc.items() if k != "iters"}
out["pcg_iters"] = acc["iters"][0] / K
print(json.dumps(out))
