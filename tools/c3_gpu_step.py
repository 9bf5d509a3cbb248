"""GPU side of the config-c3 single-FP-step replay (parity evidence; see tools/c3_step_probe.py).

    python tools/c3_gpu_step.py DIR K [K ...]

``DIR`` holds the reference's iterates ``u_K.npy``, its observation ``v.npy``, PSF ``psf.npy``
and its rhs ``rhs.npy`` (= ``apply_transpose_fast(v)``) from ``tools/c3_ref_trace.py``.  For
each ``K`` the device PCG (``tvd_pcg_solve``) runs FP step ``K`` from the reference's own
``u_K`` with (a) the device's exact ``H^T v`` as rhs (the production path) and (b) the
reference's fast-transpose rhs, recording the residual histories.  Output:
``gpurun_out/c3_gpu_step.json``.
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_5964_b200 as tvd  # noqa: E402
from paper_1011_5964_b200.harness import CONFIGS  # noqa: E402

d = pathlib.Path(sys.argv[1])
spec = CONFIGS["c3"]
dev = torch.device("cuda", 0)
v = torch.from_numpy(np.load(d / "v.npy")).to(dev)
psf = tvd.SymmetricPsf(np.load(d / "psf.npy"))
n = v.shape[0]
hop = tvd.StructuredBlurOperator(psf, tvd.BoundaryCondition.ANTI_REFLECTIVE, n, device=dev)
rhs_dev = hop.apply_transpose(v)
rhs_ref = torch.from_numpy(np.load(d / "rhs.npy")).to(dev)
out = {"rhs_rel_diff": float(torch.linalg.norm(rhs_dev - rhs_ref) / torch.linalg.norm(rhs_ref))}
cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=2000, record_history=True)
for k in map(int, sys.argv[2:]):
    u = torch.from_numpy(np.load(d / f"u_{k}.npy")).to(dev)
    lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
    pre = tvd.assemble_preconditioner("M", hop, lop, spec.alpha)
    system = tvd.NormalSystem(hop, lop, spec.alpha)
    res = {}
    variants = [("device_rhs", rhs_dev, pre), ("ref_rhs", rhs_ref, pre)]
    lam_path = d / f"lam_{k}.npy"
    if lam_path.exists():  # the reference's own assembled eigenvalues (precond.py:516-573)
        lam_ref = torch.from_numpy(np.load(lam_path)).to(dev)
        lam_dev = pre.eigenvalues_device
        res["lam_rel_max"] = float(((lam_dev - lam_ref).abs() / lam_ref.abs()).max())
        res["lam_rel_l2"] = float(torch.linalg.norm(lam_dev - lam_ref) / torch.linalg.norm(lam_ref))
        pre_ref = tvd.FactoredPreconditioner("M", tvd.TransformKind.SINE_HAT, lam_ref,
                                             spec.alpha, device=dev)
        variants.append(("ref_lam", rhs_dev, pre_ref))
    for name, rhs, pc in variants:
        r0 = float(torch.linalg.norm(rhs - system(u)))
        o = tvd.pcg(system, pc.apply_inverse, rhs, u, cfg)
        res[name] = {"count": o.iterations, "r0": r0,
                     "hist": [float(h) for h in o.residual_history]}
        print(k, name, o.iterations, o.residual_history[-3:], flush=True)
    # the same solve through other device paths: the generic (host-driven) PCG loop, the
    # generic mixed-radix DST engine, and the general (non-separable) 2D blur
    from paper_1011_5964_b200 import _native as nat
    extra = [("generic_loop", lambda: tvd.pcg(lambda w: system(w), lambda r: pre.apply_inverse(r),
                                              rhs_dev, u, cfg))]
    def generic_fft():
        nat.set_generic_fft(True, dev)
        try:
            return tvd.pcg(system, pre.apply_inverse, rhs_dev, u, cfg)
        finally:
            nat.set_generic_fft(False, dev)
    extra.append(("generic_fft", generic_fft))
    def general_blur():
        with nat.option("general_blur", 1):
            hop_g = tvd.StructuredBlurOperator(psf, tvd.BoundaryCondition.ANTI_REFLECTIVE, n,
                                               device=dev)
        sys_g = tvd.NormalSystem(hop_g, lop, spec.alpha)
        return tvd.pcg(sys_g, pre.apply_inverse, hop_g.apply_transpose(v), u, cfg)
    extra.append(("general_blur", general_blur))
    for name, fn in extra:
        o = fn()
        res[name] = {"count": o.iterations, "r0": r0,
                     "hist": [float(h) for h in o.residual_history]}
        np.save(pathlib.Path("gpurun_out") / f"c3_x_{name}_{k}.npy",
                o.solution.cpu().numpy()[::16, ::16])
        print(k, name, o.iterations, o.residual_history[-3:], flush=True)
    out[str(k)] = res
pathlib.Path("gpurun_out").mkdir(exist_ok=True)
pathlib.Path("gpurun_out/c3_gpu_step.json").write_text(json.dumps(out))
