"""One small pass over every hand-written kernel family, for compute-sanitizer.

    compute-sanitizer --tool {memcheck|racecheck|synccheck} python tools/sanitize_run.py

Covers: the DST pipeline (2047 = 89 x 23 half layout with the column-owner stages, 1023 =
31 x 11 x 3, 511 = 73 x 7, 127), the generic mixed-radix engine (DCT / R family), the DMMA
band passes and the CUDA-core sliding-window passes, the diffusivity / L / band kernels,
the device assembly (k_band), the fused PCG loop (finalizers in the last CTA, graph replay,
PDL on), device BiCGstab with AR-ghost diffusion and the P family, the general 2D blur,
the valid convolution, and the row-slab phases over LoopbackComm.  The prime-core Rader
engine runs at its only size (8192, one M^-1 application) unless --no-rader.
"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200 import _native as nat  # noqa: E402
from paper_1011_5964_b200 import slab as SL  # noqa: E402
from paper_1011_5964_b200.harness import gen_psf, valid_convolve  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(3)
AR, RE = tvd.BoundaryCondition.ANTI_REFLECTIVE, tvd.BoundaryCondition.REFLECTIVE


def system(n, m, bc, kind, bc_l=tvd.DiffusionBc.ZERO_NEUMANN, reblur=False):
    u = torch.from_numpy(np.cumsum(rng.standard_normal((n, n)), axis=1) * 0.05).to(dev)
    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", m, m / 2.0)), bc, n,
                                     device=dev)
    lop = tvd.DiffusionOperator(u, 0.1, bc_l, device=dev)
    pre = tvd.assemble_preconditioner(kind, hop, lop, 1e-3)
    return hop, lop, tvd.NormalSystem(hop, lop, 1e-3, reblur=reblur), pre, u


def step(name):
    torch.cuda.synchronize()
    print("ok", name, flush=True)


cfg = tvd.KrylovConfig(tol=1e-30, max_iterations=6)
for n, m, kind in ((2048, 15, "M"), (1024, 10, "M"), (512, 7, "M"), (128, 4, "M"),
                   (512, 7, "R"), (256, 7, "D_M"), (256, 7, "M_D")):
    hop, lop, sysm, pre, u = system(n, m, RE if kind.startswith("R") else AR, kind)
    b = hop.apply_transpose(u)
    tvd.pcg(sysm, pre.apply_inverse, b, u, cfg)
    tvd.pcg(sysm, pre.apply_inverse, b, u, cfg)  # repeated system: captured graph replay
    step(f"pcg n={n} kind={kind}")
with nat.option("pdl", 1):
    hop, lop, sysm, pre, u = system(512, 7, AR, "M")
    tvd.pcg(sysm, pre.apply_inverse, hop.apply_transpose(u), u, cfg)
    step("pcg with PDL")
with nat.option("band_slide", 1):
    hop, lop, sysm, pre, u = system(512, 7, AR, "M")
    tvd.pcg(sysm, pre.apply_inverse, hop.apply_transpose(u), u, cfg)
    step("pcg on the CUDA-core band passes")
with nat.option("split_x", 1):
    hop, lop, sysm, pre, u = system(512, 7, AR, "M")
    tvd.pcg(sysm, pre.apply_inverse, hop.apply_transpose(u), u, cfg)
    step("pcg with the split x update")
hop, lop, sysm, pre, u = system(128, 4, AR, "P", tvd.DiffusionBc.ANTI_REFLECTIVE, reblur=True)
tvd.pbicgstab(sysm, pre.apply_inverse, hop.apply(u), u, tvd.KrylovConfig(1e-30, 4))
step("bicgstab P family / AR ghosts")
with nat.option("general_blur", 1):
    hg = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 4, 2.0)), AR, 96,
                                    device=dev)
w = torch.from_numpy(rng.standard_normal((96, 96))).to(dev)
hg.apply(w), hg.apply_transpose(w)
step("general 2D blur")
ext = rng.standard_normal((140, 140))
valid_convolve(ext, gen_psf("gaussian", 6, 3.0), exact=False, device=dev)
step("valid convolution")
hop, lop, sysm, pre, u = system(512, 7, AR, "M")
b = hop.apply_transpose(u)
slabs = [SL.Slab(sysm, pre.apply_inverse, 4, r) for r in range(4)]
SL.slab_pcg(slabs, SL.LoopbackComm(), [SL.split_rows(b, 4, r) for r in range(4)],
            [SL.split_rows(u, 4, r) for r in range(4)], cfg, graph=False)
step("slab phases P=4")
if "--no-rader" not in sys.argv:
    n = 8192
    lam = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).to(dev)
    pre = tvd.FactoredPreconditioner("M", tvd.TransformKind.SINE_HAT, lam, 1e-3, device=dev)
    pre.apply_inverse(torch.from_numpy(rng.standard_normal((n, n))).to(dev))
    step("Rader M^-1 at 8192")
print("sanitize_run done")
