"""Time the 2048^2 M-preconditioner solve (three DST pipeline passes) per TVD_PIPE_VARIANT
(tvd_pfa.cu pipe_variant) in fresh processes, and check each against the default variant.
Profiling aid: python tools/pipe_variants.py 2048 -1 14 15 16"""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, pathlib
sys.path.insert(0, "%s")
import numpy as np, torch
from paper_1011_5964_b200 import precond as P, transforms as T
n = %d
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
lam = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).cuda()
pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, lam, 1e-3)
for _ in range(3):
    z = pre.apply_inverse(w)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    z = pre.apply_inverse(w)
e1.record(); torch.cuda.synchronize()
np.save("/tmp/pv_%%s.npy" %% "%s", z[::7, ::7].cpu().numpy())
print(json.dumps({"ms": e0.elapsed_time(e1) / 20}))
'''

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1])
import numpy as np  # noqa: E402
base = None
for v in sys.argv[2:]:
    # a token is a TVD_PIPE_VARIANT id or a comma list of NAME=value environment settings
    if "=" in v:
        env = dict(os.environ, **dict(kv.split("=", 1) for kv in v.split(",")))
        v = v.replace("=", "").replace(",", "_")
    else:
        env = dict(os.environ, TVD_PIPE_VARIANT=v)
    out = subprocess.run([sys.executable, "-c", CHILD % (root, n, v)], env=env,
                         capture_output=True, text=True)
    if out.returncode:
        print(v, "FAILED", out.stderr[-800:])
        continue
    ms = json.loads(out.stdout.strip().splitlines()[-1])["ms"]
    z = np.load(f"/tmp/pv_{v}.npy")
    if base is None:
        base = z
    err = float(np.abs(z - base).max() / np.abs(base).max())
    print(f"variant {v:>3}: {ms * 1e3:8.1f} us per M^-1 (3 passes)   max rel diff vs first {err:.1e}",
          flush=True)
