"""Generate golden vectors by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

The reference package ``tvdeblur`` is pure Python and imports in the build
container; it does not exist on the GPU box, so its outputs are frozen here as
``.npz`` fixtures.  Inputs are seeded (numpy ``default_rng`` / PCG64) and the
restore fixtures use the build's BASELINE generator
(``paper_1011_5964_b200.harness``) with the reference's own ``gen_psf`` /
``blur_and_observe`` so the observation is exactly what the reference sees.

Files written:
* ``ops_n{N}.npz``     -- per-op outputs (H, H^T exact and fast, eigenvalues,
  diffusivity, L w, diagonal, block bands, 2D transforms, preconditioner
  eigenvalues and M^{-1} r for R/D_R/R_D/M/D_M/M_D) at small N.
* ``restore_*.npz``    -- full ``restore`` reports (per-FP inner iteration
  counts, restored image, gradient norms) for config 1 (AR + M/M_D/D_M,
  reflective + R) and config 2a/2b (512^2).
* ``restore_c3_head.npz`` (``--big``) -- the 2048^2 headline config, first
  FP steps only (counts + image checksums; the image itself is 32 MB).
* ``restore_c4_{gauss,box}.npz`` (``--c4``) -- config 4's two problem types at 1024^2
  (problem 0: Gaussian 21x21 sigma 3; problem 1: box 11x11), full 10-FP restores: counts,
  gradient norms, RRE, a 1/64 subsample and a 64-projection sketch of the whole image
  (``tests/sketch.py``).
* ``c5_ops.npz`` (``--c5``) -- config 5 at 8192^2 (Gaussian 63x63 sigma 8, m = 31): the
  reference's exact ``apply`` / ``apply_transpose``, diffusivity, the assembled kind-M
  eigenvalues and ``apply_inverse`` of a seeded field, and the first FP step's PCG count and
  iterate, each as a subsample + sketch (the arrays are 512 MB).
* ``f2_ops_n{N}.npz`` / ``restore_c1_reblur_*.npz`` (``--f2``) -- row f2:
  anti-reflective-BC diffusion, the AR transform T and its inverse / transposes, the
  re-blurred matvec, P-family eigenvalues and solves, right-preconditioned BiCGstab, and
  full restores of the AR+Reblur+ZN / AR+Reblur+AR configurations.
"""

from __future__ import annotations

import argparse
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import tvdeblur  # noqa: E402
from tvdeblur import harness as rh  # noqa: E402
from tvdeblur import precond as rp  # noqa: E402
from tvdeblur import transforms as rt  # noqa: E402
from tvdeblur.blur import BoundaryCondition, StructuredBlurOperator, SymmetricPsf  # noqa: E402
from tvdeblur.krylov import KrylovConfig, pbicgstab  # noqa: E402
from tvdeblur.pipeline import Formulation, PrecondSelector, RestorationConfig, restore  # noqa: E402
from tvdeblur.tv import DiffusionBc, DiffusionOperator  # noqa: E402

from paper_1011_5964_b200 import harness as bh  # noqa: E402

sys.path.insert(0, str(HERE.parent))
from sketch import sketch  # noqa: E402

BCS = {"anti_reflective": BoundaryCondition.ANTI_REFLECTIVE,
       "reflective": BoundaryCondition.REFLECTIVE}


def disk_psf(m: int) -> np.ndarray:
    """Quadrantally symmetric, NOT separable (exercises the general 2D path)."""
    i = np.arange(-m, m + 1)
    h = ((i[:, None] ** 2 + i[None, :] ** 2) <= m * m + 0.5).astype(float)
    h *= 1.0 + 0.1 * np.cos(i[:, None] * 0.7) * np.cos(i[None, :] * 0.7)
    return h / h.sum()


def ops_fixture(n: int, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    out: dict[str, np.ndarray] = {}
    u = rng.standard_normal((n, n))
    w = rng.standard_normal((n, n))
    out["u"], out["w"] = u, w
    psfs = {"gauss": rh.gen_psf("gaussian", 3, 1.3).coefficients, "disk": disk_psf(3)}
    for pname, h in psfs.items():
        out[f"psf_{pname}"] = h
        for bname, bc in BCS.items():
            op = StructuredBlurOperator(SymmetricPsf(h), bc, n)
            key = f"{pname}_{bname}"
            out[f"H_{key}"] = op.apply(u)
            out[f"HT_{key}"] = op.apply_transpose(u)
            out[f"Hfast_{key}"] = op.apply_fast(u)
            out[f"HTfast_{key}"] = op.apply_transpose_fast(u)
            out[f"eig_{key}"] = op.eigenvalues()
    beta, alpha = 0.1, 1e-3
    lop = DiffusionOperator(u, beta)
    out["a_h"], out["a_v"] = lop.a_h, lop.a_v
    out["Lw"] = lop.apply(w)
    out["diagL"] = lop.diagonal()
    for (do, di), band in lop.block_banded().items():
        out[f"band_{do}_{di}"] = band
    for kind in ("dst1", "sine_hat", "dct"):
        tk = rt.TransformKind(kind)
        out[f"T2_{kind}"] = rt.tensor_apply_2d(tk, w)
        out[f"T2inv_{kind}"] = rt.tensor_apply_2d(tk, w, inverse=True)
    # 1D transforms on every length 3..n (odd and even periods)
    for length in range(3, 12):
        x = rng.standard_normal((4, length))
        out[f"T1in_{length}"] = x
        out[f"T1_dst1_{length}"] = rt.dst1_apply(x)
        out[f"T1_sine_hat_{length}"] = rt.sinehat_apply(x)
        out[f"T1_dct_{length}"] = rt.dct_apply(x)
        out[f"T1inv_dct_{length}"] = rt.dct_apply(x, inverse=True)
    gauss = SymmetricPsf(psfs["gauss"])
    for bname, fam in (("anti_reflective", "M"), ("reflective", "R")):
        op = StructuredBlurOperator(gauss, BCS[bname], n)
        for kind in (fam, "D_" + fam, fam + "_D"):
            pre = rp.assemble_preconditioner(kind, op, lop, alpha)
            out[f"lam_{kind}"] = pre.eigenvalues
            out[f"minv_{kind}"] = pre.apply_inverse(w)
    out["alpha"], out["beta"] = np.array(alpha), np.array(beta)
    return out


def f2_ops_fixture(n: int, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    out: dict[str, np.ndarray] = {}
    u = rng.standard_normal((n, n)).cumsum(axis=1) * 0.1
    w = rng.standard_normal((n, n))
    out["u"], out["w"] = u, w
    beta, alpha = 0.1, 1e-3
    out["alpha"], out["beta"] = np.array(alpha), np.array(beta)
    h = rh.gen_psf("gaussian", 3, 1.3).coefficients
    out["psf"] = h
    lops = {"zn": DiffusionOperator(u, beta), "ar": DiffusionOperator(u, beta, DiffusionBc.ANTI_REFLECTIVE)}
    lar = lops["ar"]
    out["a_h_ar"], out["a_v_ar"] = lar.a_h, lar.a_v
    out["Lw_ar"] = lar.apply(w)
    out["diagL_ar"] = lar.diagonal()
    for (do, di), band in lar.block_banded().items():
        out[f"band_ar_{do}_{di}"] = band
    ark = rt.TransformKind.ANTI_REFLECTIVE
    for inv in (False, True):
        for tr in (False, True):
            out[f"AR2_{int(inv)}{int(tr)}"] = rt.tensor_apply_2d(ark, w, inverse=inv, transpose=tr)
    op = StructuredBlurOperator(SymmetricPsf(h), BoundaryCondition.ANTI_REFLECTIVE, n)
    out["HHw"] = op.apply(op.apply(w))
    for bcl, lop in lops.items():
        out[f"reblur_Aw_{bcl}"] = op.apply(op.apply(w)) + alpha * lop.apply(w)
        for kind in ("P", "D_P", "P_D"):
            pre = rp.assemble_preconditioner(kind, op, lop, alpha)
            out[f"lam_{kind}_{bcl}"] = pre.eigenvalues
            out[f"minv_{kind}_{bcl}"] = pre.apply_inverse(w)
    pre_p = rp.assemble_preconditioner("P", op, lar, alpha)

    def apply_a(x):
        return op.apply(op.apply(x)) + alpha * lar.apply(x)

    b = op.apply(w)
    out["bicg_b"] = b
    for name, minv in (("none", None), ("P", pre_p.apply_inverse)):
        res = pbicgstab(apply_a, minv, b, u,
                        KrylovConfig(tol=1e-8, max_iterations=400, record_history=True))
        out[f"bicg_{name}_x"] = res.solution
        out[f"bicg_{name}_its"] = np.array(res.iterations)
        out[f"bicg_{name}_hist"] = np.asarray(res.residual_history)
    return out


def restore_fixture(spec: bh.ProblemSpec, selector: str, bc: str | None = None,
                    fp_steps: int | None = None, keep_image: bool = True,
                    fast: bool = True, bc_l: str = "zn", reblur: bool = False) -> dict:
    m = spec.m
    psf = rh.gen_psf("gaussian", m, spec.sigma)
    ext = bh.gen_piecewise_image(spec.n, m, spec.rects, spec.disks, 2023, spec.ramp)
    v = rh.blur_and_observe(ext, psf, spec.n, spec.nsr, 7)
    u_true = ext[m:m + spec.n, m:m + spec.n]
    bc = bc or spec.bc
    cfg = RestorationConfig(
        bc_h=BCS[bc], alpha=spec.alpha, beta=spec.beta,
        preconditioner=PrecondSelector(selector), fp_tol=1e-300,
        bc_l=DiffusionBc.ANTI_REFLECTIVE if bc_l == "ar" else DiffusionBc.ZERO_NEUMANN,
        formulation=Formulation.REBLUR if reblur else Formulation.NORMAL,
        fp_max=fp_steps or spec.fp_steps,
        inner=KrylovConfig(tol=spec.tol, max_iterations=2000), use_fast_blur=fast)
    t0 = time.perf_counter()
    rep = restore(v, psf, cfg, u_true=u_true)
    dt = time.perf_counter() - t0
    print(f"  {spec.name} {bc} {selector}: counts={rep.inner_iterations} "
          f"rre={rep.rre:.4f} ({dt:.1f}s)", flush=True)
    out = {"psf": psf.coefficients, "inner_iterations": np.array(rep.inner_iterations),
           "gradient_norms": np.array(rep.gradient_norms), "rre": np.array(rep.rre),
           "alpha": np.array(spec.alpha), "beta": np.array(spec.beta),
           "tol": np.array(spec.tol), "fp_max": np.array(cfg.fp_max),
           "restored_norm": np.array(np.linalg.norm(rep.restored)),
           "restored_sum": np.array(rep.restored.sum()),
           "restored_sub": rep.restored[::16, ::16].copy(),
           "final_gradient_norm": np.array(rep.final_gradient_norm),
           "seconds": np.array(dt)}
    if keep_image:
        out["v"], out["restored"] = v, rep.restored
    else:
        out["v_norm"] = np.array(np.linalg.norm(v))
    return out


def c4_fixture(index: int) -> dict:
    """Config 4's problem ``index`` (even: Gaussian, odd: box) restored by the reference."""
    spec = bh.CONFIGS["c4"]
    h, v, u_true = bh.make_problem(spec, index=index)
    cfg = RestorationConfig(bc_h=BoundaryCondition.ANTI_REFLECTIVE, alpha=spec.alpha,
                            beta=spec.beta, preconditioner=PrecondSelector.X, fp_tol=1e-300,
                            fp_max=spec.fp_steps,
                            inner=KrylovConfig(tol=spec.tol, max_iterations=2000))
    t0 = time.perf_counter()
    rep = restore(v, SymmetricPsf(h), cfg, u_true=u_true)
    dt = time.perf_counter() - t0
    print(f"  c4[{index}]: counts={rep.inner_iterations} rre={rep.rre:.4f} ({dt:.1f}s)",
          flush=True)
    r = rep.restored
    return {"index": np.array(index), "psf": h, "v_norm": np.array(np.linalg.norm(v)),
            "inner_iterations": np.array(rep.inner_iterations),
            "gradient_norms": np.array(rep.gradient_norms), "rre": np.array(rep.rre),
            "final_gradient_norm": np.array(rep.final_gradient_norm),
            "restored_norm": np.array(np.linalg.norm(r)), "restored_sum": np.array(r.sum()),
            "restored_sub": r[::8, ::8].copy(), "restored_sketch": sketch(r, 64),
            "seconds": np.array(dt)}


def _big(out: dict, key: str, a: np.ndarray, k: int = 16) -> None:
    """A 512 MB array as norm + subsample (prime stride) + border rows + sketch."""
    out[f"{key}_norm"] = np.array(np.linalg.norm(a))
    out[f"{key}_sub"] = a[::61, ::61].copy()
    out[f"{key}_rows"] = a[[0, 1, 2, 30, 31, 32, -33, -32, -31, -3, -2, -1], ::7].copy()
    out[f"{key}_cols"] = a[::7, [0, 1, 2, 30, 31, 32, -33, -32, -31, -3, -2, -1]].copy()
    out[f"{key}_sketch"] = sketch(a, k)
    print(f"  c5 {key}: norm {float(out[key + '_norm']):.6e}", flush=True)


def c5_fixture() -> dict:
    """Config 5 (8192^2) per-op outputs of the reference plus its first FP step."""
    spec = bh.CONFIGS["c5"]
    h, v, _ = bh.make_problem(spec, exact=False)
    psf = SymmetricPsf(h)
    n = spec.n
    op = StructuredBlurOperator(psf, BoundaryCondition.ANTI_REFLECTIVE, n)
    out: dict[str, np.ndarray] = {"psf": h, "alpha": np.array(spec.alpha),
                                  "beta": np.array(spec.beta)}
    _big(out, "v", v)
    t0 = time.perf_counter()
    _big(out, "H_v", op.apply(v))
    _big(out, "HT_v", op.apply_transpose(v))
    print(f"  c5 exact blur {time.perf_counter() - t0:.0f}s", flush=True)
    lop = DiffusionOperator(v, spec.beta)
    _big(out, "a_h", lop.a_h)
    _big(out, "a_v", lop.a_v)
    t0 = time.perf_counter()
    pre = rp.assemble_preconditioner("M", op, lop, spec.alpha)
    print(f"  c5 assembly {time.perf_counter() - t0:.0f}s", flush=True)
    _big(out, "lam_M", pre.eigenvalues)
    w = np.random.default_rng(8192).standard_normal((n, n))
    _big(out, "minv_w", pre.apply_inverse(w))
    del w
    # first FP step of restore (pipeline.py:194-244): rhs = H^T_fast v, u0 = v, kind M
    from tvdeblur.krylov import pcg

    rhs = op.apply_transpose_fast(v)

    def apply_a(x):
        return op.apply_transpose_fast(op.apply_fast(x)) + spec.alpha * lop.apply(x)

    t0 = time.perf_counter()
    res = pcg(apply_a, pre.apply_inverse, rhs, v,
              KrylovConfig(tol=spec.tol, max_iterations=2000, record_history=True))
    print(f"  c5 FP step 1: {res.iterations} its ({time.perf_counter() - t0:.0f}s)", flush=True)
    out["fp1_iterations"] = np.array(res.iterations)
    out["fp1_history"] = np.asarray(res.residual_history)
    _big(out, "fp1_u", res.solution)
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run the 2048^2 head")
    ap.add_argument("--big-steps", type=int, default=3)
    ap.add_argument("--only-exact", action="store_true")
    ap.add_argument("--f2", action="store_true", help="only the row-f2 fixtures")
    ap.add_argument("--c4", action="store_true", help="only the config-4 restores")
    ap.add_argument("--exact-dots", action="store_true",
                    help="only the rounding-sensitive config-1 restores (selector I, re-blurred "
                         "none / diag) with the reference's dot products exactly rounded")
    ap.add_argument("--c5", action="store_true", help="only the config-5 (8192^2) ops")
    args = ap.parse_args()
    print("reference tvdeblur from", tvdeblur.__file__)
    if args.exact_dots:
        # the reference's own krylov.py with _dot / _norm (krylov.py:70-75) replaced by exactly
        # rounded dot products: the restores whose counts move with the BLAS summation order
        import math

        from tvdeblur import krylov as rk
        sys.path.insert(0, str(HERE.parents[1] / "tools"))
        from c3_dot_probe_lib import exact_dot

        rk._dot = exact_dot
        rk._norm = lambda x: math.sqrt(exact_dot(x, x))
        c1 = bh.CONFIGS["c1"]
        np.savez_compressed(HERE / "restore_c1_I_xdot.npz", **restore_fixture(c1, "none"))
        for bcl in ("zn", "ar"):
            for sel in ("none", "diag"):
                np.savez_compressed(HERE / f"restore_c1_reblur_{bcl}_{sel}_xdot.npz",
                                    **restore_fixture(c1, sel, bc_l=bcl, reblur=True, fp_steps=4))
        return
    if args.c4:
        for i, tag in ((0, "gauss"), (1, "box")):
            np.savez_compressed(HERE / f"restore_c4_{tag}.npz", **c4_fixture(i))
        return
    if args.c5:
        np.savez_compressed(HERE / "c5_ops.npz", **c5_fixture())
        return
    if args.f2:
        for n, seed in ((32, 21), (33, 22)):
            np.savez_compressed(HERE / f"f2_ops_n{n}.npz", **f2_ops_fixture(n, seed))
            print("wrote f2 ops", n)
        c1 = bh.CONFIGS["c1"]
        for bcl in ("zn", "ar"):
            for sel in ("none", "diag", "x", "d_x", "x_d"):
                np.savez_compressed(HERE / f"restore_c1_reblur_{bcl}_{sel}.npz",
                                    **restore_fixture(c1, sel, bc_l=bcl, reblur=True,
                                                      fp_steps=4))
        return
    if "--only-exact" in sys.argv:
        np.savez_compressed(HERE / "restore_c1_I_exact.npz",
                            **restore_fixture(bh.CONFIGS["c1"], "none", fast=False))
        return
    for n, seed in ((32, 11), (33, 12), (16, 13)):
        np.savez_compressed(HERE / f"ops_n{n}.npz", **ops_fixture(n, seed))
        print("wrote ops", n)
    c1 = bh.CONFIGS["c1"]
    for sel, bc, tag in (("x", None, "c1_M"), ("x_d", None, "c1_M_D"),
                         ("d_x", None, "c1_D_M"), ("x", "reflective", "c1_R"),
                         ("x_d", "reflective", "c1_R_D"), ("none", None, "c1_I")):
        np.savez_compressed(HERE / f"restore_{tag}.npz", **restore_fixture(c1, sel, bc))
    # the reference's exact (pad/convolve/crop) operator path, use_fast_blur=False
    np.savez_compressed(HERE / "restore_c1_I_exact.npz",
                        **restore_fixture(c1, "none", fast=False))
    for key in ("c2a", "c2b"):
        np.savez_compressed(HERE / f"restore_{key}.npz",
                            **restore_fixture(bh.CONFIGS[key], "x"))
    if args.big:
        np.savez_compressed(
            HERE / "restore_c3_head.npz",
            **restore_fixture(bh.CONFIGS["c3"], "x", fp_steps=args.big_steps,
                              keep_image=False))


if __name__ == "__main__":
    main()
