"""Per-phase cycle split of the DST pipeline kernel (needs a -DTVD_PIPE_TIMING build).

One M-preconditioner application at n = 2048 (three pipeline launches); prints the
mean cycles per batch of each phase as seen by thread 0 of every CTA.  Profiling aid.
"""
import ctypes
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200 import _native
from paper_1011_5964_b200 import precond as P
from paper_1011_5964_b200 import transforms as T

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
lib = _native.load()
fn = lib.tvd_debug_pipe_phases
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
fn.restype = ctypes.c_int
rng = np.random.default_rng(0)
w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
lam = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).cuda()
pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, lam, 1e-3)
z = pre.apply_inverse(w)
torch.cuda.synchronize()
st_fn = lib.tvd_debug_stage_times
st_fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
st_fn.restype = ctypes.c_int
st_buf = (ctypes.c_ulonglong * 128)()
buf = (ctypes.c_ulonglong * 8)()
st_fn(st_buf, 1)
if fn(buf, 1) != 0:
    raise SystemExit("library built without -DTVD_PIPE_TIMING")
for _ in range(3):
    z = pre.apply_inverse(w)
torch.cuda.synchronize()
fn(buf, 1)
st_fn(st_buf, 1)
ctas = buf[7]
names = ["wait+zero", "pack", "stages", "mid(+stages)", "unpack"]
tot = sum(buf[i] for i in range(5))
batches = 3 * 3 * (n // 2)  # 3 applications x 3 launches x n/2 batches
print(f"CTAs flushed {ctas}; cycles per batch (thread 0 view), total {tot / batches:.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:14s} {buf[i] / batches:9.0f}  ({buf[i] / tot:.1%})")
print(f"  warp-0 DMMA loop per batch: stage q=89 {buf[5] / batches:.0f}, other {buf[6] / batches:.0f}")
transforms = 3 * 4 * (n // 2)  # 4 transforms per application (the sandwich pass has two)
for si, nm in enumerate(["q=89 stage", "other stage"]):
    print(f"{nm}: cycles per batch-transform by warp [setup, DMMA loop, epilogue, barrier]")
    for w in range(16):
        v = [st_buf[(si * 16 + w) * 4 + k] / transforms for k in range(4)]
        if sum(v) > 0:
            print(f"  warp {w:2d}: " + "  ".join(f"{x:7.0f}" for x in v))
