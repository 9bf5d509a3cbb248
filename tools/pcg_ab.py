"""A/B of one inner PCG solve (FP state 2 as in bench.py; default config c3) under a library
option: iterations/s over repeated solves and bit-identity of the solutions.  Profiling aid.

    python tools/pcg_ab.py OPTION v1,v2,... [CONFIG]
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200 import _native as nat  # noqa: E402
from paper_1011_5964_b200.harness import CONFIGS, make_problem  # noqa: E402

name = sys.argv[1]
vals = [int(v) for v in sys.argv[2].split(",")]
spec = CONFIGS[sys.argv[3] if len(sys.argv) > 3 else "c3"]
dev = torch.device("cuda", 0)
h, v, _ = make_problem(spec)
bc = tvd.BoundaryCondition(spec.bc)
kind = "M" if bc is tvd.BoundaryCondition.ANTI_REFLECTIVE else "R"
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), bc, spec.n, device=dev)
v = torch.from_numpy(v).to(dev)
rhs = hop.apply(v) if kind == "R" else hop.apply_transpose(v)
cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=2000)
u = v.clone()
for _ in range(2):
    lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
    pre = tvd.assemble_preconditioner(kind, hop, lop, spec.alpha)
    u = tvd.pcg(tvd.NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, u, cfg).solution
lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
pre = tvd.assemble_preconditioner(kind, hop, lop, spec.alpha)
system = tvd.NormalSystem(hop, lop, spec.alpha)
saved = nat.get_option(name)
out, ref = {}, None
for val in vals:
    nat.set_option(name, val)
    for _ in range(3):
        res = tvd.pcg(system, pre.apply_inverse, rhs, u, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = 0
    e0.record()
    for _ in range(10 if spec.n >= 2048 else 50):
        res = tvd.pcg(system, pre.apply_inverse, rhs, u, cfg)
        its += res.iterations
    e1.record()
    torch.cuda.synchronize()
    sol = res.solution
    ref = sol.clone() if ref is None else ref
    out[val] = {"it_per_s": round(its / (e0.elapsed_time(e1) / 1e3), 1), "iters": res.iterations,
                "identical": bool(torch.equal(sol, ref))}
nat.set_option(name, saved)
print(json.dumps({name: out}))
