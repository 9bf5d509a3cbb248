"""Kernel durations and inter-kernel gaps inside one c3 PCG solve as it runs in production
(graph replay + PDL), from CUPTI timestamps (torch.profiler).  Profiling aid."""
import collections, json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200.harness import CONFIGS, make_problem

spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dev = torch.device("cuda", 0)
h, v, _ = make_problem(spec)
hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), tvd.BoundaryCondition(spec.bc), spec.n, device=dev)
v = torch.from_numpy(v).to(dev)
rhs = hop.apply_transpose(v)
cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=2000)
u = v.clone()
for _ in range(2):
    lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
    pre = tvd.assemble_preconditioner("M", hop, lop, spec.alpha)
    u = tvd.pcg(tvd.NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, u, cfg).solution
lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
pre = tvd.assemble_preconditioner("M", hop, lop, spec.alpha)
system = tvd.NormalSystem(hop, lop, spec.alpha)
for _ in range(3):
    res = tvd.pcg(system, pre.apply_inverse, rhs, u, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = tvd.pcg(system, pre.apply_inverse, rhs, u, cfg)
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_time > 0 and "Memcpy" not in e.name and "Memset" not in e.name),
            key=lambda e: e.time_range.start)
import re
def cat(name):
    m = re.search(r"(k_\w+)", name)
    k = m.group(1) if m else name[:30]
    m2 = re.search(r"k_dst_pipe<.*?(\d+), (?:true|false), \d+>", name)
    return k + ("/" + m2.group(1) if m2 else "")
dur = collections.defaultdict(list)
gaps = []
for a, b in zip(ev, ev[1:] + [None]):
    dur[cat(a.name)].append(a.device_time)
    if b is not None: gaps.append(b.time_range.start - a.time_range.end)
span = ev[-1].time_range.end - ev[0].time_range.start
print("iterations", res.iterations, "span_us", round(span, 1), "sum kernels", round(sum(e.device_time for e in ev), 1),
      "positive gaps", round(sum(g for g in gaps if g > 0), 1))
for k, x in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
    big = [d for d in x if d >= 5.0]
    print(f"{k:28s} n={len(x):3d} total {sum(x):8.1f} us   launches >= 5 us: {len(big):3d} avg {sum(big)/max(1,len(big)):7.1f}")
