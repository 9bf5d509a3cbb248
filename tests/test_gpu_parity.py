"""GPU parity: every hot-path operator through the C ABI vs the reference's own outputs.

Goldens (``tests/golden/*.npz``) were produced by running the reference package
itself (``tests/golden/make_golden.py``); the oracle restatement covers sizes
the goldens do not.  Tolerances follow BASELINE.json's north_star: per-op
1e-12 relative (bit-identical where the arithmetic allows), restored image
1e-8 relative L2, identical per-FP-step PCG iteration counts.
"""

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import tvd_oracle as O

import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200 import blur as B
from paper_1011_5964_b200 import krylov as K
from paper_1011_5964_b200 import precond as P
from paper_1011_5964_b200 import transforms as T
from paper_1011_5964_b200 import tv as TV
from paper_1011_5964_b200.harness import CONFIGS

pytestmark = pytest.mark.gpu

OPS = ["ops_n16.npz", "ops_n32.npz", "ops_n33.npz"]
BCS = {"anti_reflective": B.BoundaryCondition.ANTI_REFLECTIVE,
       "reflective": B.BoundaryCondition.REFLECTIVE}


# ----------------------------------------------------------------- transforms
@pytest.mark.parametrize("name", OPS)
def test_transforms_2d_match_reference(golden, name):
    g = golden(name)
    for kind in ("dst1", "sine_hat", "dct"):
        tk = T.TransformKind(kind)
        assert rel_err(T.tensor_apply_2d(tk, g["w"]), g[f"T2_{kind}"]) < 1e-13
        assert rel_err(T.tensor_apply_2d(tk, g["w"], inverse=True), g[f"T2inv_{kind}"]) < 1e-13


def test_transforms_1d_every_short_length(golden):
    g = golden("ops_n16.npz")
    for length in range(3, 12):
        x = g[f"T1in_{length}"]
        assert rel_err(T.dst1_apply(x), g[f"T1_dst1_{length}"]) < 1e-13, length
        assert rel_err(T.sinehat_apply(x), g[f"T1_sine_hat_{length}"]) < 1e-13, length
        assert rel_err(T.dct_apply(x), g[f"T1_dct_{length}"]) < 1e-13, length
        assert rel_err(T.dct_apply(x, inverse=True), g[f"T1inv_dct_{length}"]) < 1e-13, length


@pytest.mark.parametrize("n", [127, 128, 511, 512, 1023, 1024, 2048])
def test_transforms_2d_vs_oracle(n, rng):
    w = rng.standard_normal((n, n))
    for kind in ("dst1", "sine_hat", "dct"):
        tk = T.TransformKind(kind)
        assert rel_err(T.tensor_apply_2d(tk, w), O.tensor_2d(kind, w)) < 1e-12, (n, kind)
        assert rel_err(T.tensor_apply_2d(tk, w, inverse=True),
                       O.tensor_2d(kind, w, inverse=True)) < 1e-12, (n, kind)


@pytest.mark.parametrize("n", [5, 17, 45, 128, 512, 1024, 2048])
def test_prime_factor_engine_matches_generic_engine(n, rng):
    """The odd-symmetric PFA DST engine and the generic mixed-radix engine agree."""
    from paper_1011_5964_b200 import _native as nat
    w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    d = torch.from_numpy(rng.uniform(0.5, 2.0, (n, n))).cuda()
    outs = []
    for generic in (False, True):
        nat.set_generic_fft(generic)
        try:
            outs.append([T.tensor_apply_2d(T.TransformKind.SINE_HAT, w),
                         T.tensor_apply_2d(T.TransformKind.DST1, w),
                         P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT, d, 1e-3,
                                                  d_sqrt=d).apply_inverse(w)])
        finally:
            nat.set_generic_fft(False)
    for a, b in zip(*outs):
        assert float((a - b).norm() / b.norm()) < 1e-13


def test_transform_known_answers():
    # S_2 (1,1) = (sqrt2, 0) and C e1 = n^-1/2 (pkg/tests/test_transforms.py:31-48)
    np.testing.assert_allclose(T.dst1_apply(np.array([[1.0, 1.0]])), [[np.sqrt(2.0), 0.0]],
                               atol=1e-14)
    e1 = np.zeros((1, 12))
    e1[0, 0] = 1.0
    np.testing.assert_allclose(T.dct_apply(e1), np.full((1, 12), np.sqrt(1 / 12)), atol=1e-14)
    assert np.all(T.dst1_apply(np.zeros((2, 7))) == 0.0)


@pytest.mark.parametrize("n", [2048])
def test_full_size_transform_round_trips(n, rng):
    """Size-independent properties at the headline size: Shat is an involution,
    DCT synthesis inverts analysis."""
    w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    sh = T.tensor_apply_2d(T.TransformKind.SINE_HAT, T.tensor_apply_2d(T.TransformKind.SINE_HAT, w))
    assert float((sh - w).norm() / w.norm()) < 1e-13
    dc = T.tensor_apply_2d(T.TransformKind.DCT, T.tensor_apply_2d(T.TransformKind.DCT, w, inverse=True))
    assert float((dc - w).norm() / w.norm()) < 1e-13


# ---------------------------------------------------------------------- blur
@pytest.mark.parametrize("name", OPS)
@pytest.mark.parametrize("pname", ["gauss", "disk"])
@pytest.mark.parametrize("bname", list(BCS))
def test_blur_exact_vs_reference(golden, name, pname, bname):
    g = golden(name)
    n = g["u"].shape[0]
    op = B.StructuredBlurOperator(B.SymmetricPsf(g[f"psf_{pname}"]), BCS[bname], n)
    assert op.separable == (pname == "gauss")
    key = f"{pname}_{bname}"
    assert rel_err(op.apply(g["u"]), g[f"H_{key}"]) < 1e-12
    assert rel_err(op.apply_transpose(g["u"]), g[f"HT_{key}"]) < 1e-12
    np.testing.assert_allclose(op.eigenvalues(), g[f"eig_{key}"], rtol=0, atol=1e-13)
    # normal operator == back(H(u)) of pipeline.py:167-179
    hu = g[f"H_{key}"]
    back = O.blur(hu, g[f"psf_{pname}"], bname) if bname == "reflective" else \
        O.blur_transpose(hu, g[f"psf_{pname}"], bname)
    assert rel_err(op.normal_apply(g["u"]), back) < 1e-12


@pytest.mark.parametrize("n,m,bname", [(512, 7, "anti_reflective"), (512, 7, "reflective"),
                                       (300, 15, "anti_reflective"), (1024, 10, "anti_reflective")])
def test_blur_vs_oracle_midsize(n, m, bname, rng):
    from paper_1011_5964_b200.harness import gen_psf
    h = gen_psf("gaussian", m, m / 2.0)
    u = rng.standard_normal((n, n))
    op = B.StructuredBlurOperator(B.SymmetricPsf(h), BCS[bname], n)
    assert rel_err(op.apply(u), O.blur(u, h, bname)) < 1e-12
    assert rel_err(op.apply_transpose(u), O.blur_transpose(u, h, bname)) < 1e-12


@pytest.mark.parametrize("n,m,bname", [(256, 7, "anti_reflective"), (512, 15, "reflective"),
                                       (1024, 10, "anti_reflective"), (768, 31, "anti_reflective"),
                                       (1024, -5, "anti_reflective")])
def test_normal_system_vs_oracle_midsize(n, m, bname, rng):
    """Fused H^T H + alpha L matvec (tensor-core band passes at these sizes), plain and X_D-scaled.
    m < 0: the config-4 box PSF (11 x 11 uniform, half-width |m|)."""
    from paper_1011_5964_b200.harness import gen_psf
    from paper_1011_5964_b200.pipeline import NormalSystem
    h = gen_psf("box", -m) if m < 0 else gen_psf("gaussian", m, m / 2.0)
    u = np.cumsum(rng.standard_normal((n, n)), axis=1) * 0.05
    w = rng.standard_normal((n, n))
    alpha, beta = 2e-3, 0.05
    hop = B.StructuredBlurOperator(B.SymmetricPsf(h), BCS[bname], n)
    lop = TV.DiffusionOperator(u, beta)
    back = O.blur_transpose if bname == "anti_reflective" else O.blur
    want = back(O.blur(w, h, bname), h, bname) + alpha * O.diffusion_apply(lop.a_h, lop.a_v, w)
    assert rel_err(NormalSystem(hop, lop, alpha)(w), want) < 1e-12
    s = rng.uniform(0.5, 1.5, (n, n))
    st = torch.from_numpy(s).cuda()
    want_s = s * (back(O.blur(s * w, h, bname), h, bname)
                  + alpha * O.diffusion_apply(lop.a_h, lop.a_v, s * w))
    assert rel_err(NormalSystem(hop, lop, alpha, s=st)(w), want_s) < 1e-12


@pytest.mark.parametrize("n", [2048])
def test_full_size_blur_adjointness_and_linearity(n, rng):
    from paper_1011_5964_b200.harness import gen_psf
    h = gen_psf("gaussian", 15, 4.0)
    op = B.StructuredBlurOperator(B.SymmetricPsf(h), B.BoundaryCondition.ANTI_REFLECTIVE, n)
    x = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    y = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    lhs = float((op.apply(x) * y).sum())
    rhs = float((x * op.apply_transpose(y)).sum())
    assert abs(lhs - rhs) <= 1e-11 * abs(lhs)
    lin = op.apply(2.0 * x - 3.0 * y) - (2.0 * op.apply(x) - 3.0 * op.apply(y))
    assert float(lin.norm() / op.apply(x).norm()) < 1e-13
    nrm = op.normal_apply(x) - op.apply_transpose(op.apply(x))
    assert float(nrm.norm() / op.normal_apply(x).norm()) < 1e-12


# ----------------------------------------------------------------- diffusion
@pytest.mark.parametrize("name", OPS)
def test_diffusion_bit_identical(golden, name):
    g = golden(name)
    lop = TV.DiffusionOperator(g["u"], float(g["beta"]))
    np.testing.assert_array_equal(lop.a_h, g["a_h"])
    np.testing.assert_array_equal(lop.a_v, g["a_v"])
    np.testing.assert_array_equal(lop.apply(g["w"]), g["Lw"])
    np.testing.assert_array_equal(lop.diagonal(), g["diagL"])
    bands = lop.block_banded()
    for (do, di), band in bands.items():
        np.testing.assert_array_equal(band, g[f"band_{do}_{di}"])


def test_diffusion_known_answers():
    a_h, a_v = TV.diffusion_coefficients(np.full((5, 5), 3.0), 0.5)
    np.testing.assert_allclose(a_h, 2.0)
    np.testing.assert_allclose(a_v, 2.0)
    lop = TV.DiffusionOperator(np.random.default_rng(0).standard_normal((6, 6)), 0.1)
    np.testing.assert_allclose(lop.apply(np.full((6, 6), 4.0)), 0.0, atol=1e-12)


@pytest.mark.parametrize("n", [2048])
def test_full_size_diffusion_bit_identical(n, rng):
    u = rng.standard_normal((n, n)).cumsum(axis=0) * 0.01
    w = rng.standard_normal((n, n))
    lop = TV.DiffusionOperator(u, 0.05)
    a_h, a_v = O.diffusivity(u, 0.05)
    np.testing.assert_array_equal(lop.a_h, a_h)
    np.testing.assert_array_equal(lop.a_v, a_v)
    np.testing.assert_array_equal(lop.apply(w), O.diffusion_apply(a_h, a_v, w))


# ------------------------------------------------------------ preconditioner
@pytest.mark.parametrize("name", OPS)
def test_preconditioner_eigenvalues_and_inverse(golden, name):
    g = golden(name)
    n = g["u"].shape[0]
    alpha = float(g["alpha"])
    lop = TV.DiffusionOperator(g["u"], float(g["beta"]))
    psf = B.SymmetricPsf(g["psf_gauss"])
    for bname, fam in (("anti_reflective", "M"), ("reflective", "R")):
        hop = B.StructuredBlurOperator(psf, BCS[bname], n)
        for kind in (fam, "D_" + fam, fam + "_D"):
            pre = P.assemble_preconditioner(kind, hop, lop, alpha)
            assert rel_err(pre.eigenvalues, g[f"lam_{kind}"]) < 1e-12, kind
            assert rel_err(pre.apply_inverse(g["w"]), g[f"minv_{kind}"]) < 1e-12, kind
            back = pre.apply(pre.apply_inverse(g["w"]))
            assert rel_err(back, g["w"]) < 1e-9, kind


@pytest.mark.parametrize("n,kind", [(512, "M"), (512, "R"), (512, "M_D"), (1024, "D_M"),
                                    (2048, "M")])
def test_preconditioner_vs_oracle_large(n, kind, rng):
    from paper_1011_5964_b200.harness import gen_psf
    h = gen_psf("gaussian", 7, 2.5)
    u = rng.standard_normal((n, n)).cumsum(axis=1) * 0.05
    alpha = 5e-4
    bname = "reflective" if "R" in kind else "anti_reflective"
    hop = B.StructuredBlurOperator(B.SymmetricPsf(h), BCS[bname], n)
    lop = TV.DiffusionOperator(u, 0.1)
    pre = P.assemble_preconditioner(kind, hop, lop, alpha)
    a_h, a_v = O.diffusivity(u, 0.1)
    blocks = O.diffusion_bands(a_h, a_v)
    lam_h = O.blur_eigenvalues(h, bname, n)
    lam, lam_inv, d_sqrt, _ = O.assemble(kind, lam_h, blocks, alpha)
    assert rel_err(pre.eigenvalues, lam) < 1e-12
    r = rng.standard_normal((n, n))
    fam = O.FAMILY[kind.replace("D_", "").replace("_D", "")]
    assert rel_err(pre.apply_inverse(r), O.precond_solve(fam, lam_inv, r, d_sqrt)) < 1e-12


def test_prime_core_preconditioner_8192(rng):
    """Config-5 size: odd core L = 8191 is prime -> Rader engine.  Round trip (lambda = 1 gives
    S S = I) and the M^-1 r solve vs the oracle with random positive eigenvalues."""
    n = 8192
    w = rng.standard_normal((n, n))
    wt = torch.from_numpy(w).cuda()
    one = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT,
                                   torch.ones(n, n, dtype=torch.float64, device="cuda"), 1e-3)
    z = one.apply_inverse(wt)
    assert float((z - wt).norm() / wt.norm()) < 1e-13
    lam = rng.uniform(0.5, 2.0, (n, n))
    pre = P.FactoredPreconditioner("M", T.TransformKind.SINE_HAT,
                                   torch.from_numpy(lam).cuda(), 1e-3)
    got = pre.apply_inverse(wt).cpu().numpy()
    assert rel_err(got, O.precond_solve("sine_hat", 1.0 / lam, w)) < 1e-12


def test_preconditioner_rejects_wrong_bc(golden):
    g = golden("ops_n16.npz")
    lop = TV.DiffusionOperator(g["u"], 0.1)
    hop = B.StructuredBlurOperator(B.SymmetricPsf(g["psf_gauss"]), B.BoundaryCondition.REFLECTIVE, 16)
    with pytest.raises(ValueError):
        P.assemble_preconditioner("M", hop, lop, 1e-3)
    with pytest.raises(ValueError):
        P.assemble_preconditioner("Q", hop, lop, 1e-3)


# ----------------------------------------------------------------------- PCG
def _dev(a):
    return torch.from_numpy(np.asarray(a, dtype=float)).cuda()


def test_pcg_generic_reference_cases(rng):
    b = rng.standard_normal(6)
    out = K.pcg(lambda x: x.clone(), None, _dev(b), _dev(np.zeros(6)))
    assert out.converged and out.iterations == 1
    d = np.arange(1.0, 11.0)
    bb = rng.standard_normal(10)
    dd = _dev(d)
    out = K.pcg(lambda x: dd * x, lambda r: r / dd, _dev(bb), _dev(np.zeros(10)))
    assert out.converged and out.iterations == 1
    np.testing.assert_allclose(out.solution.cpu().numpy(), bb / d, atol=1e-12)
    m = rng.standard_normal((8, 8))
    a = m @ m.T + 8 * np.eye(8)
    ad = _dev(a)
    bv = rng.standard_normal(8)
    out = K.pcg(lambda x: ad @ x, None, _dev(bv), _dev(np.zeros(8)),
                K.KrylovConfig(tol=1e-12, max_iterations=100))
    np.testing.assert_allclose(out.solution.cpu().numpy(), np.linalg.solve(a, bv), atol=1e-8)
    with pytest.raises(K.IndefiniteOperatorError) as err:
        K.pcg(lambda x: -x, None, _dev(rng.standard_normal(5)), _dev(np.zeros(5)))
    assert err.value.iteration == 1
    with pytest.raises(K.SolverDivergenceError):
        K.pcg(lambda x: torch.full_like(x, float("nan")), None, _dev(rng.standard_normal(4)),
              _dev(np.zeros(4)))
    out = K.pcg(lambda x: x.clone(), None, _dev(np.zeros(4)), _dev(np.zeros(4)))
    assert out.converged and out.iterations == 0


def _system(g, bname, n):
    from paper_1011_5964_b200.pipeline import NormalSystem
    hop = B.StructuredBlurOperator(B.SymmetricPsf(g["psf_gauss"]), BCS[bname], n)
    lop = TV.DiffusionOperator(g["u"], float(g["beta"]))
    return hop, lop, NormalSystem(hop, lop, float(g["alpha"]))


@pytest.mark.parametrize("name", OPS)
@pytest.mark.parametrize("kind", ["M", "D_M", "none"])
def test_fused_pcg_matches_oracle_iteration_by_iteration(golden, name, kind):
    g = golden(name)
    n = g["u"].shape[0]
    hop, lop, system = _system(g, "anti_reflective", n)
    rhs = hop.apply_transpose(g["w"])
    cfg = K.KrylovConfig(tol=1e-9, max_iterations=400, record_history=True)
    if kind == "none":
        minv_gpu, minv_cpu = None, None
    else:
        pre = P.assemble_preconditioner(kind, hop, lop, float(g["alpha"]))
        minv_gpu = pre.apply_inverse
        lam_inv = pre.inverse_eigenvalues_device.cpu().numpy()
        dsq = pre.d_sqrt
        minv_cpu = lambda r: O.precond_solve("sine_hat", lam_inv, r, dsq)  # noqa: E731
    out = K.pcg(system, minv_gpu, rhs, g["u"], cfg)
    h = g["psf_gauss"]

    def apply_a(w):
        return O.blur_transpose(O.blur(w, h, "anti_reflective"), h, "anti_reflective") + \
            float(g["alpha"]) * O.diffusion_apply(lop.a_h, lop.a_v, w)

    x, its, hist, ok = O.pcg(apply_a, minv_cpu, rhs, g["u"], 1e-9, 400, True)
    assert out.converged and ok
    # 240 unpreconditioned steps to 1e-9: rounding may move the stop by one step
    assert abs(out.iterations - its) <= (1 if kind == "none" else 0)
    # unpreconditioned CG loses orthogonality over ~150 steps, so rounding-level
    # differences grow along the history; the early history must agree tightly
    head = 10 if kind == "none" else len(hist)
    np.testing.assert_allclose(out.residual_history[:head], hist[:head], rtol=1e-6)
    assert rel_err(out.solution, x) < (1e-6 if kind == "none" else 1e-8)


def test_fused_pcg_errors_and_limits(golden):
    g = golden("ops_n16.npz")
    hop, lop, system = _system(g, "anti_reflective", 16)
    rhs = hop.apply_transpose(g["w"])
    out = K.pcg(system, None, rhs, g["u"], K.KrylovConfig(tol=1e-14, max_iterations=3))
    assert not out.converged and out.iterations == 3
    out = K.pcg(system, None, np.zeros((16, 16)), np.zeros((16, 16)))
    assert out.converged and out.iterations == 0
    from paper_1011_5964_b200.pipeline import NormalSystem
    neg = NormalSystem(hop, lop, -50.0)  # alpha < 0 with a large L -> indefinite
    with pytest.raises(K.IndefiniteOperatorError):
        K.pcg(neg, None, rhs, np.zeros((16, 16)), K.KrylovConfig(tol=1e-12, max_iterations=200))


# ------------------------------------------------------------------- restore
RESTORES = [("restore_c1_M.npz", "x", "anti_reflective"),
            ("restore_c1_M_D.npz", "x_d", "anti_reflective"),
            ("restore_c1_D_M.npz", "d_x", "anti_reflective"),
            ("restore_c1_R.npz", "x", "reflective"),
            ("restore_c1_R_D.npz", "x_d", "reflective"),
            ("restore_c2a.npz", "x", "anti_reflective"),
            ("restore_c2b.npz", "x", "reflective")]


@pytest.mark.parametrize("name,selector,bname", RESTORES)
def test_restore_matches_reference(golden, name, selector, bname):
    g = golden(name)
    cfg = tvd.RestorationConfig(
        bc_h=BCS[bname], alpha=float(g["alpha"]), beta=float(g["beta"]),
        preconditioner=tvd.PrecondSelector(selector), fp_tol=1e-300, fp_max=int(g["fp_max"]),
        inner=K.KrylovConfig(tol=float(g["tol"]), max_iterations=2000))
    rep = tvd.restore(g["v"], B.SymmetricPsf(g["psf"]), cfg)
    assert rep.inner_iterations == [int(k) for k in g["inner_iterations"]]
    assert rel_err(rep.restored, g["restored"]) < 1e-8
    np.testing.assert_allclose(rep.gradient_norms, g["gradient_norms"], rtol=1e-6)
    assert abs(rep.final_gradient_norm - float(g["final_gradient_norm"])) <= \
        1e-6 * float(g["final_gradient_norm"])


@pytest.mark.parametrize("name", ["restore_c1_I.npz", "restore_c1_I_exact.npz"])
def test_restore_unpreconditioned(golden, name):
    """Selector I (no preconditioner, ~55 CG steps per FP step): the reference's two
    operator paths (fast transforms vs exact pad/convolve/crop) already disagree by
    +-1 iteration at several FP steps with images 1.1e-9 apart, so rounding decides
    the last step (the CPU restatement lands 2 steps off at one FP step with the image
    1.5e-9 away).  Gate: image inside 1e-8 (the north_star's image gate), counts
    within 2 per step."""
    g = golden(name)
    cfg = tvd.RestorationConfig(
        bc_h=BCS["anti_reflective"], alpha=float(g["alpha"]), beta=float(g["beta"]),
        preconditioner=tvd.PrecondSelector.NONE, fp_tol=1e-300, fp_max=int(g["fp_max"]),
        inner=K.KrylovConfig(tol=float(g["tol"]), max_iterations=2000))
    rep = tvd.restore(g["v"], B.SymmetricPsf(g["psf"]), cfg)
    ref = [int(k) for k in g["inner_iterations"]]
    assert all(abs(a - b) <= 2 for a, b in zip(rep.inner_iterations, ref))
    assert rel_err(rep.restored, g["restored"]) < 1e-8


def test_headline_c3_restore_matches_reference():
    """Config 3 (2048^2 AR, 20 FP steps, tol 1e-5) end to end against the reference's own
    CPU runs (tests/golden/c3_parity.json, made by tests/golden/make_c3_parity.py and
    add_c3_run.py from five 0.5-4 h runs of the reference on identical inputs).

    Counts: at tol 1e-5 the stopping iteration is not a property of the algorithm.  The
    reference disagrees with ITSELF by up to 3 iterations per FP step between runs that
    differ only in the BLAS thread count of its dot products (krylov.py:70-75) or in its
    fast vs exact H^T (blur.py:236-247 vs 302-314).  The committed residual histories show
    why: near the stop the relative residual sits within a few percent of tol and then bumps
    up for two iterations (e.g. FP step 9 of the exact-dot run: 1.0326e-5 at iteration 30,
    2.3e-5 at 31, stop at 32), so rounding decides whether the solve ends before or after
    the bump; single-step replays from the reference's own iterates give the device's count
    exactly once the reference's dots are rounded exactly (same file).
    The gate is the reference's own envelope: each device count within [min, max] of the
    reference runs widened by one, and by one more iteration on the low side at the steps
    where a committed reference history came within 6 % of tol before its own stop (a
    near-tie: stopping there is the same solve up to rounding).  The image is gated over
    every pixel (sketch) and on the subsample against each reference run at 1e-8 -- the
    runs agree with each other to ~1e-10.
    """
    import json

    from sketch import sketch

    from paper_1011_5964_b200.harness import make_problem
    ev = json.loads((__import__("pathlib").Path(__file__).parent / "golden" /
                     "c3_parity.json").read_text())
    spec = CONFIGS["c3"]
    h, v, u_true = make_problem(spec)
    assert abs(np.linalg.norm(v) - ev["v_norm"]) <= 1e-14 * ev["v_norm"]
    cfg = tvd.RestorationConfig(
        bc_h=BCS["anti_reflective"], alpha=spec.alpha, beta=spec.beta,
        preconditioner=tvd.PrecondSelector.X, fp_tol=1e-300, fp_max=spec.fp_steps,
        inner=K.KrylovConfig(tol=spec.tol, max_iterations=2000))
    rep = tvd.restore(v, B.SymmetricPsf(h), cfg, u_true=u_true)
    runs = list(ev["reference_runs"].values())
    lo = [min(r["counts"][k] for r in runs) for k in range(spec.fp_steps)]
    hi = [max(r["counts"][k] for r in runs) for k in range(spec.fp_steps)]
    got = rep.inner_iterations
    tol = ev["tol"]

    def near_tie(k):
        tails = [r.get("hist_tail") or r.get("last_residuals") for r in runs]
        return any(t is not None and min(t[k][:-1]) <= 1.06 * tol for t in tails)

    bad = [(k, got[k], lo[k], hi[k]) for k in range(spec.fp_steps)
           if not lo[k] - 1 - (1 if near_tie(k) else 0) <= got[k] <= hi[k] + 1]
    assert not bad, (bad, list(got))
    r = np.asarray(rep.restored)
    s = sketch(r, 64)
    for name, run in ev["reference_runs"].items():
        img = run["image"]
        assert abs(np.linalg.norm(r) - img["norm"]) <= 1e-8 * img["norm"], name
        if "sketch" in img:  # every pixel (the round-1 golden holds the subsample only)
            est = np.linalg.norm(s - np.asarray(img["sketch"])) / 8.0 / img["norm"]
            assert est < 1e-8, (name, est)
        sub = np.asarray(img["sub"])
        stride = r.shape[0] // sub.shape[0]
        assert rel_err(r[::stride, ::stride], sub) < 1e-8, name
        assert abs(rep.rre - run["rre"]) < 1e-8, name


# ------------------------------------------------------------------ row f2
F2_OPS = ["f2_ops_n32.npz", "f2_ops_n33.npz"]


@pytest.mark.parametrize("name", F2_OPS)
def test_f2_ar_diffusion_bit_identical(golden, name):
    g = golden(name)
    lop = TV.DiffusionOperator(g["u"], float(g["beta"]), TV.DiffusionBc.ANTI_REFLECTIVE)
    assert np.array_equal(lop.a_h, g["a_h_ar"]) and np.array_equal(lop.a_v, g["a_v_ar"])
    assert np.array_equal(lop.apply(g["w"]), g["Lw_ar"])
    for (do, di), b in lop.block_banded().items():
        assert np.array_equal(b, g[f"band_ar_{do}_{di}"]), (do, di)


@pytest.mark.parametrize("name", F2_OPS)
def test_f2_reblur_matvec(golden, name):
    from paper_1011_5964_b200.pipeline import NormalSystem
    g = golden(name)
    n = g["u"].shape[0]
    hop = B.StructuredBlurOperator(B.SymmetricPsf(g["psf"]), B.BoundaryCondition.ANTI_REFLECTIVE, n)
    for bcl, bc in (("zn", TV.DiffusionBc.ZERO_NEUMANN), ("ar", TV.DiffusionBc.ANTI_REFLECTIVE)):
        lop = TV.DiffusionOperator(g["u"], float(g["beta"]), bc)
        sysr = NormalSystem(hop, lop, float(g["alpha"]), reblur=True)
        assert rel_err(sysr(g["w"]), g[f"reblur_Aw_{bcl}"]) < 1e-12


@pytest.mark.parametrize("n,m", [(256, 7), (512, 15)])
def test_f2_reblur_ar_matvec_tensor_core_sizes(n, m, rng):
    """Re-blurred H H + alpha L_AR at sizes that run the DMMA band passes, vs the oracle."""
    from paper_1011_5964_b200.harness import gen_psf
    from paper_1011_5964_b200.pipeline import NormalSystem
    h = gen_psf("gaussian", m, m / 2.0)
    u = np.cumsum(rng.standard_normal((n, n)), axis=1) * 0.05
    w = rng.standard_normal((n, n))
    alpha, beta = 2e-3, 0.05
    hop = B.StructuredBlurOperator(B.SymmetricPsf(h), B.BoundaryCondition.ANTI_REFLECTIVE, n)
    lop = TV.DiffusionOperator(u, beta, TV.DiffusionBc.ANTI_REFLECTIVE)
    ah, av = O.diffusivity(u, beta, bc="ar")
    want = O.blur(O.blur(w, h, "anti_reflective"), h, "anti_reflective") + \
        alpha * O.diffusion_apply(ah, av, w, bc="ar")
    assert rel_err(NormalSystem(hop, lop, alpha, reblur=True)(w), want) < 1e-12


@pytest.mark.parametrize("name", F2_OPS)
def test_f2_bicgstab_device_loop(golden, name):
    """Fused device BiCGstab (tvd_bicgstab_solve) vs the generic path and the oracle on the
    re-blurred + anti-reflective-L system with the diagonal preconditioner."""
    from paper_1011_5964_b200.pipeline import NormalSystem
    g = golden(name)
    n, alpha, beta = g["u"].shape[0], float(g["alpha"]), float(g["beta"])
    hop = B.StructuredBlurOperator(B.SymmetricPsf(g["psf"]), B.BoundaryCondition.ANTI_REFLECTIVE, n)
    lop = TV.DiffusionOperator(g["u"], beta, TV.DiffusionBc.ANTI_REFLECTIVE)
    system = NormalSystem(hop, lop, alpha, reblur=True)
    assert not system.symmetric
    b = hop.apply(g["w"])
    d = 1.0 + alpha * lop.diagonal()
    minv = K.DiagonalInverse(torch.from_numpy(d).cuda())
    cfg = K.KrylovConfig(tol=1e-6, max_iterations=400, record_history=True)
    fused = K.pbicgstab(system, minv, b, g["u"], cfg)
    generic = K.pbicgstab(lambda w: system(w), minv, b, g["u"], cfg)
    ah, av = O.diffusivity(g["u"], beta, bc="ar")
    h = g["psf"]

    def apply_a(x):
        return O.blur(O.blur(x, h, "anti_reflective"), h, "anti_reflective") + \
            alpha * O.diffusion_apply(ah, av, x, bc="ar")

    x, its, hist, ok = O.pbicgstab(apply_a, lambda r: r / d, b, g["u"], 1e-6, 400, True)
    assert fused.converged and generic.converged and ok
    assert abs(fused.iterations - its) <= 1 and abs(generic.iterations - its) <= 1
    head = min(8, len(hist))
    np.testing.assert_allclose(fused.residual_history[:head], hist[:head], rtol=1e-7)
    np.testing.assert_allclose(generic.residual_history[:head], hist[:head], rtol=1e-7)
    assert rel_err(fused.solution, x) < 1e-5 and rel_err(generic.solution, x) < 1e-5
    # zero residual: zero iterations, converged (krylov.py:127-128)
    exact = K.pbicgstab(system, minv, system(g["u"]), g["u"], cfg)
    assert exact.iterations == 0 and exact.converged


@pytest.mark.parametrize("name", F2_OPS)
def test_f2_ar_transform_2d(golden, name):
    g = golden(name)
    for inv in (0, 1):
        got = T.tensor_apply_2d(T.TransformKind.ANTI_REFLECTIVE, g["w"], inverse=bool(inv))
        assert rel_err(got, g[f"AR2_{inv}0"]) < 1e-13


@pytest.mark.parametrize("name", F2_OPS)
def test_ar_transform_transposes(golden, name):
    """T^T (x) T^T and T^-T (x) T^-T against the reference's tensor_apply_2d
    (transforms.py:130-139, 159-171), and the 1D forms along either axis against the dense
    matrices of the defining formula."""
    g = golden(name)
    ark = T.TransformKind.ANTI_REFLECTIVE
    for inv in (0, 1):
        got = T.tensor_apply_2d(ark, g["w"], inverse=bool(inv), transpose=True)
        assert rel_err(got, g[f"AR2_{inv}1"]) < 1e-13
    w = g["w"]
    n = w.shape[0]
    for inv in (False, True):
        m = T.dense_matrix(ark, n, inverse=inv)
        for tr in (False, True):
            mm = m.T if tr else m
            assert rel_err(T.ar_apply(w, inverse=inv, transpose=tr, axis=0), mm @ w) < 1e-12
            assert rel_err(T.ar_apply(w, inverse=inv, transpose=tr, axis=1), w @ mm.T) < 1e-12
            assert rel_err(T.apply_1d(ark, w[3], inverse=inv, transpose=tr), mm @ w[3]) < 1e-12
    # round trips: T^-1 T = I and T^-T T^T = I
    for tr in (False, True):
        back = T.ar_apply(T.ar_apply(w, transpose=tr), inverse=True, transpose=tr)
        assert rel_err(back, w) < 1e-12


@pytest.mark.parametrize("name", ["ops_n16.npz", "ops_n32.npz", "ops_n33.npz"])
def test_blur_transform_domain_paths(golden, name):
    """apply_fast / apply_transpose_fast (blur.py:293-314): analysis, eigenvalue scaling,
    synthesis on the device against the reference's own fast paths, both BCs; for the
    anti-reflective adjoint this is X^-T (lam .* X^T u) with the non-orthogonal T."""
    g = golden(name)
    n = g["u"].shape[0]
    for psf_name in ("gauss", "disk"):
        for bc in ("reflective", "anti_reflective"):
            hop = B.StructuredBlurOperator(B.SymmetricPsf(g[f"psf_{psf_name}"]), BCS[bc], n)
            key = f"{psf_name}_{bc}"
            assert rel_err(hop.apply_fast(g["u"]), g[f"Hfast_{key}"]) < 1e-12
            assert rel_err(hop.apply_transpose_fast(g["u"]), g[f"HTfast_{key}"]) < 1e-12


@pytest.mark.parametrize("name", F2_OPS)
def test_f2_p_family_assembly_and_solve(golden, name):
    g = golden(name)
    n = g["u"].shape[0]
    hop = B.StructuredBlurOperator(B.SymmetricPsf(g["psf"]), B.BoundaryCondition.ANTI_REFLECTIVE, n)
    for bcl, bc in (("zn", TV.DiffusionBc.ZERO_NEUMANN), ("ar", TV.DiffusionBc.ANTI_REFLECTIVE)):
        lop = TV.DiffusionOperator(g["u"], float(g["beta"]), bc)
        for kind in ("P", "D_P", "P_D"):
            pre = P.assemble_preconditioner(kind, hop, lop, float(g["alpha"]))
            assert rel_err(pre.eigenvalues, g[f"lam_{kind}_{bcl}"]) < 1e-12, (kind, bcl)
            assert rel_err(pre.apply_inverse(g["w"]), g[f"minv_{kind}_{bcl}"]) < 1e-12, (kind, bcl)


@pytest.mark.parametrize("n", [128, 512, 1024, 2048])
def test_f2_p_family_vs_oracle_config_sizes(n, rng):
    """P-family M^-1 r (fused AR corrections in the pipelined row passes) vs the oracle at the
    config sizes (odd cores 127, 511, 1023, 2047)."""
    lam = rng.uniform(0.5, 2.0, (n, n))
    w = rng.standard_normal((n, n))
    pre = P.FactoredPreconditioner("P", T.TransformKind.ANTI_REFLECTIVE,
                                   torch.from_numpy(lam).cuda(), 1e-3)
    got = pre.apply_inverse(torch.from_numpy(w).cuda()).cpu().numpy()
    assert rel_err(got, O.precond_solve("ar", 1.0 / lam, w)) < 1e-12


REBLUR = [(bcl, sel) for bcl in ("zn", "ar") for sel in ("none", "diag", "x", "d_x", "x_d")]


@pytest.mark.parametrize("bcl,sel", REBLUR)
def test_f2_reblur_restore_matches_reference(golden, bcl, sel):
    """AR+Reblur+ZN / AR+Reblur+AR (harness.py:56-59) through restore: BiCGstab per FP step with
    the P family (x, d_x, x_d), the diagonal or no preconditioner.  Identical per-FP-step
    counts; image 1e-8 (P family) / 1e-7 (none, diag: rounding-sensitive BiCGstab histories)."""
    g = golden(f"restore_c1_reblur_{bcl}_{sel}.npz")
    cfg = tvd.RestorationConfig(
        bc_h=B.BoundaryCondition.ANTI_REFLECTIVE, alpha=float(g["alpha"]), beta=float(g["beta"]),
        bc_l=TV.DiffusionBc.ANTI_REFLECTIVE if bcl == "ar" else TV.DiffusionBc.ZERO_NEUMANN,
        formulation=tvd.Formulation.REBLUR, preconditioner=tvd.PrecondSelector(sel),
        fp_tol=1e-300, fp_max=int(g["fp_max"]),
        inner=K.KrylovConfig(tol=float(g["tol"]), max_iterations=2000))
    rep = tvd.restore(g["v"], B.SymmetricPsf(g["psf"]), cfg)
    assert rep.inner_iterations == [int(k) for k in g["inner_iterations"]]
    tol = 1e-8 if sel in ("x", "d_x", "x_d") else 1e-7
    assert rel_err(rep.restored, g["restored"]) < tol
    np.testing.assert_allclose(rep.gradient_norms, g["gradient_norms"], rtol=1e-6)
    assert abs(rep.final_gradient_norm - float(g["final_gradient_norm"])) <= \
        1e-6 * float(g["final_gradient_norm"])


def test_prime_core_assembly_rader_matches_generic_8192():
    """Config-5 preconditioner assembly: the band projections of length L = 8191 (prime) run
    on the Rader engine (launch_band_rader); the generic mixed-radix engine (option
    band_generic) computes the same eigenvalues in O(L) per point -- they agree to rounding."""
    from paper_1011_5964_b200 import _native as nat
    n = 8192
    g = torch.Generator(device="cpu").manual_seed(5)
    u = torch.rand(n // 64, n // 64, generator=g, dtype=torch.float64)
    u = torch.nn.functional.interpolate(u[None, None], size=(n, n), mode="bilinear")[0, 0].cuda()
    hop = B.StructuredBlurOperator(B.SymmetricPsf(O_gauss(31, 8.0)),
                                   B.BoundaryCondition.ANTI_REFLECTIVE, n)
    lop = TV.DiffusionOperator(u, 0.05)
    fast = P.assemble_preconditioner("D_M", hop, lop, 1e-4).eigenvalues_device.clone()
    with nat.option("band_generic", 1):
        slow = P.assemble_preconditioner("D_M", hop, lop, 1e-4).eigenvalues_device
    assert float((fast - slow).norm() / slow.norm()) < 1e-12


def O_gauss(m, sigma):
    from paper_1011_5964_b200.harness import gen_psf
    return gen_psf("gaussian", m, sigma)


# ------------------------------------------------- observation pipeline
def test_valid_convolve_device_matches_host(rng):
    """tvd_valid_convolve: separable PSFs bit-identical to the harness's shifted-slice sums;
    a non-separable PSF (direct 2D path) within rounding of scipy's convolve2d (the routine
    the reference's blur_and_observe calls, harness.py:186)."""
    from scipy.signal import convolve2d
    from paper_1011_5964_b200.harness import gen_psf, valid_convolve
    ext = rng.uniform(size=(300, 300))
    for h in (gen_psf("gaussian", 10, 3.0), gen_psf("box", 5)):
        dev = valid_convolve(ext, h, exact=False, device="cuda")
        host = valid_convolve(ext, h, exact=False)
        assert np.array_equal(dev, host)
        assert rel_err(dev, convolve2d(ext, h, mode="valid")) < 1e-14
    h = rng.uniform(size=(9, 9))
    h = (h + h[::-1, ::-1]) / 2  # symmetric, not rank 1
    dev = valid_convolve(ext, h, exact=False, device="cuda")
    assert rel_err(dev, convolve2d(ext, h, mode="valid")) < 1e-13


def test_observation_at_config5_scale_on_device():
    """8192^2 observation (config 5: 63 x 63 Gaussian over the 8254^2 extended truth) on the
    GPU: spot rows against the host shifted-slice sums."""
    from paper_1011_5964_b200.harness import gen_psf, valid_convolve
    g = np.random.default_rng(1)
    ext = g.uniform(size=(8254, 8254))
    h = gen_psf("gaussian", 31, 8.0)
    dev = valid_convolve(ext, h, exact=False, device="cuda")
    assert dev.shape == (8192, 8192)
    for r0, c0 in ((0, 0), (4000, 7000), (8064, 8064)):  # 128 x 128 blocks need 190 x 190
        host = valid_convolve(ext[r0:r0 + 190, c0:c0 + 190], h, exact=False)
        assert np.array_equal(dev[r0:r0 + 128, c0:c0 + 128], host)


# ------------------------------------------------------------ sweeps
def test_sweep_matches_reference_files(tmp_path):
    """The reference's own 2D sweep (tests/golden/make_sweep_golden.py: R / AR+Sine+ZN /
    AR+Reblur+ZN x alpha 1e-3, 1e-2 x preconditioners x, d_x at n = 48) against the same
    spec on the device path: identical cells, FP step counts and file set; average inner
    counts within one iteration, RRE within 1e-8, restored PGM bytes within one grey level."""
    import pathlib
    from paper_1011_5964_b200 import sweep as SW
    ref = pathlib.Path(__file__).resolve().parent / "golden" / "sweep_ref"
    spec = SW.BenchmarkSpec(ns=(48,), alphas=(1e-3, 1e-2), betas=(0.1,),
                            configurations=("R", "AR+Sine+ZN", "AR+Reblur+ZN"),
                            preconditioners=("x", "d_x"), fp_max=40)
    res = SW.run_sweep(spec, out_dir=tmp_path)
    assert sorted(p.name for p in res.files) == sorted(p.name for p in ref.iterdir())
    hdr, rows = SW.read_csv(tmp_path / "iterations.csv")
    rhdr, rrows = SW.read_csv(ref / "iterations.csv")
    assert hdr == rhdr and len(rows) == len(rrows)
    for a, b in zip(rows, rrows):
        assert a[:5] == b[:5], (a, b)  # label, alpha, beta, n, fp_steps
        assert abs(float(a[5]) - float(b[5])) <= 1.0, (a, b)
        assert abs(float(a[6]) - float(b[6])) <= 1e-8 * float(b[6]), (a, b)
    for f in ref.glob("*.pgm"):
        mine, theirs = SW.read_pgm(tmp_path / f.name), SW.read_pgm(f)
        assert mine.shape == theirs.shape
        assert int(np.abs(mine.astype(int) - theirs.astype(int)).max()) <= 1, f.name


# ------------------------------------------------- size-independent properties at full size
def test_full_size_operator_symmetry_and_linearity_2048():
    """Config-3 size: the device normal-equation matvec A = H^T H + alpha L and the M^-1 solve
    are symmetric (x . A y = y . A x) and positive (x . A x > 0), and A is linear -- checked
    through the C ABI at 2048^2 where the oracle would take minutes."""
    n = 2048
    g = torch.Generator(device="cpu").manual_seed(11)
    u = torch.rand(n, n, generator=g, dtype=torch.float64).cuda()
    x = torch.randn(n, n, generator=g, dtype=torch.float64).cuda()
    y = torch.randn(n, n, generator=g, dtype=torch.float64).cuda()
    hop = B.StructuredBlurOperator(B.SymmetricPsf(O_gauss(15, 4.0)),
                                   B.BoundaryCondition.ANTI_REFLECTIVE, n)
    lop = TV.DiffusionOperator(u, 0.05)
    sysm = tvd.NormalSystem(hop, lop, 2e-4)
    pre = P.assemble_preconditioner("M", hop, lop, 2e-4)
    ax, ay = sysm(x), sysm(y)
    sxy, syx = float((x * ay).sum()), float((y * ax).sum())
    assert abs(sxy - syx) <= 1e-12 * max(abs(sxy), float(x.norm() * ay.norm()) * 1e-3)
    assert float((x * ax).sum()) > 0
    lin = sysm(2.0 * x - 3.0 * y)
    assert float((lin - (2.0 * ax - 3.0 * ay)).norm() / lin.norm()) < 1e-13
    mx, my = pre.apply_inverse(x), pre.apply_inverse(y)
    mxy, myx = float((x * my).sum()), float((y * mx).sum())
    assert abs(mxy - myx) <= 1e-12 * float(x.norm() * my.norm())
    assert float((x * mx).sum()) > 0


def test_solver_graph_cache_follows_the_blur(rng):
    """Two solves in a row at 2048^2 (where the fused PCG replays a captured CUDA graph) with
    blurs of the same width but different taps, the first blur freed before the second is
    built (so its host address and device tables are likely reused): each fused solve must
    equal the generic-path solve of its own system, i.e. no stale graph replays the old taps."""
    import gc

    from paper_1011_5964_b200.harness import gen_psf
    from paper_1011_5964_b200.pipeline import NormalSystem

    n = 2048
    u = np.cumsum(rng.standard_normal((n, n)), axis=1) * 0.01
    b = rng.standard_normal((n, n))
    lop = TV.DiffusionOperator(u, 0.1)
    cfg = K.KrylovConfig(tol=1e-6, max_iterations=60)
    seen = []
    for sigma in (2.0, 3.5, 2.0):
        hop = B.StructuredBlurOperator(B.SymmetricPsf(gen_psf("gaussian", 7, sigma)),
                                       B.BoundaryCondition.ANTI_REFLECTIVE, n)
        system = NormalSystem(hop, lop, 1e-3)
        pre = P.assemble_preconditioner("M", hop, lop, 1e-3)
        fused = K.pcg(system, pre.apply_inverse, b, np.zeros((n, n)), cfg)
        generic = K.pcg(lambda w, s=system: s(w), lambda r, p=pre: p.apply_inverse(r), b,
                        np.zeros((n, n)), cfg)
        assert fused.converged and fused.iterations == generic.iterations, sigma
        assert rel_err(fused.solution, generic.solution) < 1e-10, sigma
        seen.append(fused.solution)
        del hop, system, pre, fused, generic
        gc.collect()
    assert rel_err(seen[0], seen[1]) > 1e-3
    assert rel_err(seen[0], seen[2]) < 1e-14


# ------------------------------------------------- numerical edge cases of the reference's tests
def test_indefinite_preconditioner_reports_kind_and_alpha():
    """reference pkg/tests/test_precond.py:348-354 (precond.py:437-441), on device arrays."""
    lam = np.ones((16, 16))
    lam[3, 5] = -0.5
    with pytest.raises(P.IndefinitePreconditionerError) as err:
        P.FactoredPreconditioner("R", T.TransformKind.DCT, lam, alpha=0.25,
                                 device=torch.device("cuda"))
    assert err.value.kind == "R" and err.value.alpha == 0.25
    assert err.value.min_eigenvalue == -0.5
    assert "R" in str(err.value) and "0.25" in str(err.value)


def test_clamping_logs_warning(caplog):
    """reference pkg/tests/test_precond.py:357-364 (precond.py:442-450): eigenvalues below
    1e-14 max are clamped with a logged warning and the inverse stays finite."""
    import logging

    lam = np.ones((16, 16)) * 2.0
    lam[0, 0] = 1.0
    lam[7, 9] = 1e-20
    with caplog.at_level(logging.WARNING, logger="paper_1011_5964_b200.precond"):
        fp = P.FactoredPreconditioner("R", T.TransformKind.DCT, lam, alpha=1e-3,
                                      device=torch.device("cuda"))
    assert any("clamped 1 eigenvalue" in rec.message for rec in caplog.records)
    assert fp.clamped == 1
    inv = fp.inverse_eigenvalues_device.cpu().numpy()
    assert inv[7, 9] == 1.0 / (1e-14 * 2.0)
    assert np.all(np.isfinite(fp.apply_inverse(np.ones((16, 16)))))


def test_device_assembly_clamps_like_the_reference(caplog):
    """The device assembly's positivity check and clamp (tvd_precond_assemble) on a system
    whose projected eigenvalues fall below 1e-14 max: a box PSF whose symbol nearly vanishes
    on the DCT grid and a vanishing alpha.  Clamp count and the clamped inverse agree with the
    oracle's restatement of precond.py:437-450, and the warning is logged."""
    import logging

    n = 48
    h = np.full((3, 3), 1.0 / 9.0)  # symbol (1 + 2 cos y) / 3 ~ 0 at y = 2 pi / 3 (j = 32)
    u = np.random.default_rng(5).standard_normal((n, n))
    hop = B.StructuredBlurOperator(B.SymmetricPsf(h), B.BoundaryCondition.REFLECTIVE, n)
    lop = TV.DiffusionOperator(u, 0.1)
    alpha = 1e-300
    with caplog.at_level(logging.WARNING, logger="paper_1011_5964_b200.precond"):
        pre = P.assemble_preconditioner("R", hop, lop, alpha)
    lam_h = O.blur_eigenvalues(h, "reflective", n)
    lam, lam_inv, _, _ = O.assemble("R", lam_h, O.diffusion_bands(lop.a_h, lop.a_v), alpha)
    expect = int(np.count_nonzero(lam < 1e-14 * lam.max()))
    assert expect > 0 and pre.clamped == expect
    assert any("clamped" in rec.message for rec in caplog.records)
    assert rel_err(pre.inverse_eigenvalues_device.cpu().numpy(), lam_inv) < 1e-12


def test_assembly_rejects_nonpositive_scaling_diagonal():
    """precond.py:558-560: d = 1 + alpha diag L <= 0 (anti-reflective diffusion has negative
    border diagonal entries, reference test_pipeline.py:88-97) raises
    IndefinitePreconditionerError(kind, alpha, min d) for every kind."""
    from paper_1011_5964_b200.tv import DiffusionBc

    n = 16
    u = np.random.default_rng(20230814).standard_normal((n, n)) * 5.0
    lop = TV.DiffusionOperator(u, 0.01, DiffusionBc.ANTI_REFLECTIVE)
    dmin = float(lop.diagonal().min())
    assert dmin < 0
    alpha = 2.0 / abs(dmin)
    hop = B.StructuredBlurOperator(B.SymmetricPsf(np.full((3, 3), 1 / 9.0)),
                                   B.BoundaryCondition.ANTI_REFLECTIVE, n)
    for kind in ("M", "D_M", "M_D", "P", "D_P", "P_D"):
        with pytest.raises(P.IndefinitePreconditionerError) as err:
            P.assemble_preconditioner(kind, hop, lop, alpha)
        assert err.value.kind == kind and err.value.alpha == alpha
        assert err.value.min_eigenvalue == pytest.approx(1.0 + alpha * dmin, rel=1e-12)


def test_scaling_errors_match_the_reference():
    """pipeline.py:154-158 (scale_system) and :229-233 (the DIAG selector): a nonpositive
    scaling diagonal raises InvalidScalingError, through the API and through restore."""
    from paper_1011_5964_b200.pipeline import NormalSystem, scale_system
    from paper_1011_5964_b200.tv import DiffusionBc

    n = 16
    u = np.random.default_rng(20230814).standard_normal((n, n)) * 5.0
    lop = TV.DiffusionOperator(u, 0.01, DiffusionBc.ANTI_REFLECTIVE)
    alpha = 2.0 / abs(float(lop.diagonal().min()))
    hop = B.StructuredBlurOperator(B.SymmetricPsf(np.full((3, 3), 1 / 9.0)),
                                   B.BoundaryCondition.ANTI_REFLECTIVE, n)
    with pytest.raises(tvd.InvalidScalingError):
        scale_system(NormalSystem(hop, lop, alpha), np.ones((n, n)), lop, alpha)
    for sel in (tvd.PrecondSelector.DIAG, tvd.PrecondSelector.X_D):
        cfg = tvd.RestorationConfig(
            bc_h=B.BoundaryCondition.ANTI_REFLECTIVE, alpha=alpha, beta=0.01,
            bc_l=DiffusionBc.ANTI_REFLECTIVE, formulation=tvd.Formulation.REBLUR,
            preconditioner=sel, fp_tol=1e-3, fp_max=2,
            inner=K.KrylovConfig(tol=1e-6, max_iterations=50))
        with pytest.raises(tvd.InvalidScalingError):
            tvd.restore(u, B.SymmetricPsf(np.full((3, 3), 1 / 9.0)), cfg)


# ------------------------------------------------- config 4 (1024^2 batch problems) vs the reference
@pytest.mark.parametrize("name", ["restore_c4_gauss.npz", "restore_c4_box.npz"])
def test_c4_restore_matches_reference(golden, name):
    """Config 4's two problem types (Gaussian 21x21 sigma 3 / box 11x11, 1024^2 AR, 10 FP
    steps, tol 1e-4) restored on the device against the reference's own restore
    (tests/golden/make_golden.py --c4): identical per-FP-step PCG counts, gradient norms,
    and the restored image within 1e-8 on a 1/64 subsample AND over every pixel through a
    64-projection sketch (tests/sketch.py, a Johnson-Lindenstrauss estimate of the full-image
    relative L2 difference)."""
    from sketch import sketch_rel_err

    from paper_1011_5964_b200.harness import make_problem

    g = golden(name)
    spec = CONFIGS["c4"]
    h, v, u_true = make_problem(spec, index=int(g["index"]))
    assert np.array_equal(h, g["psf"])
    assert abs(np.linalg.norm(v) - float(g["v_norm"])) <= 1e-14 * float(g["v_norm"])
    cfg = tvd.RestorationConfig(
        bc_h=BCS["anti_reflective"], alpha=spec.alpha, beta=spec.beta,
        preconditioner=tvd.PrecondSelector.X, fp_tol=1e-300, fp_max=spec.fp_steps,
        inner=K.KrylovConfig(tol=spec.tol, max_iterations=2000))
    rep = tvd.restore(v, B.SymmetricPsf(h), cfg, u_true=u_true)
    assert rep.inner_iterations == [int(k) for k in g["inner_iterations"]]
    np.testing.assert_allclose(rep.gradient_norms, g["gradient_norms"], rtol=1e-6)
    r = np.asarray(rep.restored)
    assert rel_err(r[::8, ::8], g["restored_sub"]) < 1e-8
    assert abs(np.linalg.norm(r) - float(g["restored_norm"])) <= 1e-8 * float(g["restored_norm"])
    assert sketch_rel_err(r, g["restored_sketch"], float(g["restored_norm"])) < 1e-8
    assert abs(rep.rre - float(g["rre"])) < 1e-8


# ------------------------------------------------- config 5 (8192^2) vs the reference
def _big_check(g, key, t, tol):
    """``t`` (device tensor) against the reference's 512 MB array ``key`` frozen as norm,
    prime-stride subsample, border rows / columns and a 16-projection sketch."""
    from sketch import sketch_torch

    ref_norm = float(g[f"{key}_norm"])
    assert abs(float(torch.linalg.norm(t)) - ref_norm) <= tol * ref_norm, key
    a = t.cpu().numpy() if t.numel() <= (1 << 27) else None
    sub = t[::61, ::61].cpu().numpy()
    assert rel_err(sub, g[f"{key}_sub"]) < tol, key
    rows = t[[0, 1, 2, 30, 31, 32, -33, -32, -31, -3, -2, -1], ::7].cpu().numpy()
    cols = t[::7, [0, 1, 2, 30, 31, 32, -33, -32, -31, -3, -2, -1]].cpu().numpy()
    assert rel_err(rows, g[f"{key}_rows"]) < tol, key
    assert rel_err(cols, g[f"{key}_cols"]) < tol, key
    sk = g[f"{key}_sketch"]
    est = np.linalg.norm(sketch_torch(t, len(sk)) - sk) / np.sqrt(len(sk)) / ref_norm
    assert est < tol, (key, est)
    del a


def test_c5_ops_and_first_fp_step_match_reference(golden):
    """Config 5 (8192^2 AR, Gaussian 63 x 63 sigma 8, m = 31) against the reference's own
    outputs (tests/golden/make_golden.py --c5, ~1 h of CPU): the observation, exact H v and
    H^T v, the diffusivities, the assembled kind-M eigenvalues (Rader band projections at the
    prime core 8191), M^-1 of a seeded field, and the first FP step's PCG solve (count within
    one, iterate within 1e-8).  Every array is gated over all of its 67M entries through a
    sketch plus subsample / border rows (tests/sketch.py)."""
    from paper_1011_5964_b200.harness import make_problem

    g = golden("c5_ops.npz")
    spec = CONFIGS["c5"]
    n = spec.n
    dev = torch.device("cuda")
    h, v, _ = make_problem(spec, exact=False, device=dev)
    assert np.array_equal(h, g["psf"])
    vd = torch.from_numpy(v).to(dev)
    del v
    _big_check(g, "v", vd, 1e-14)
    hop = B.StructuredBlurOperator(B.SymmetricPsf(h), B.BoundaryCondition.ANTI_REFLECTIVE, n,
                                   device=dev)
    _big_check(g, "H_v", hop.apply(vd), 1e-12)
    rhs = hop.apply_transpose(vd)
    _big_check(g, "HT_v", rhs, 1e-12)
    lop = TV.DiffusionOperator(vd, spec.beta, device=dev)
    _big_check(g, "a_h", lop.a_h_device, 1e-14)
    _big_check(g, "a_v", lop.a_v_device, 1e-14)
    pre = P.assemble_preconditioner("M", hop, lop, spec.alpha)
    _big_check(g, "lam_M", pre.eigenvalues_device, 1e-12)
    w = torch.from_numpy(np.random.default_rng(8192).standard_normal((n, n))).to(dev)
    _big_check(g, "minv_w", pre.apply_inverse(w), 1e-12)
    del w
    from paper_1011_5964_b200.pipeline import NormalSystem
    out = K.pcg(NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, vd,
                K.KrylovConfig(tol=spec.tol, max_iterations=2000, record_history=True))
    assert abs(out.iterations - int(g["fp1_iterations"])) <= 1
    _big_check(g, "fp1_u", out.solution, 1e-8)


# ---------------------- rounding-sensitive restores vs the reference with exactly rounded dots
@pytest.mark.parametrize("name", ["restore_c1_I_xdot.npz", "restore_c1_reblur_zn_none_xdot.npz",
                                  "restore_c1_reblur_zn_diag_xdot.npz",
                                  "restore_c1_reblur_ar_none_xdot.npz",
                                  "restore_c1_reblur_ar_diag_xdot.npz"])
def test_rounding_sensitive_restores_match_reference_with_exact_dots(golden, name):
    """The restores whose stopping iterations move with the stock reference's BLAS summation
    order (unpreconditioned CG, BiCGstab with the diagonal or no preconditioner), against the
    reference's own krylov.py with _dot / _norm exactly rounded (make_golden.py --exact-dots).
    The stock and the exact-dot reference runs differ from EACH OTHER by a count at two FP
    steps of c1-I and by up to 1.1e-8 in the re-blurred images, so the gates are the
    reference's own spread: re-blurred counts identical to the exact-dot run, c1-I counts
    within one of either reference run, images within max(1e-8, 2 x the two reference runs'
    distance)."""
    g = golden(name)
    reblur = "reblur" in name
    bcl = "ar" if "_ar_" in name else "zn"
    sel = "none" if ("_none" in name or "_I_" in name) else "diag"
    cfg = tvd.RestorationConfig(
        bc_h=B.BoundaryCondition.ANTI_REFLECTIVE, alpha=float(g["alpha"]), beta=float(g["beta"]),
        bc_l=TV.DiffusionBc.ANTI_REFLECTIVE if bcl == "ar" else TV.DiffusionBc.ZERO_NEUMANN,
        formulation=tvd.Formulation.REBLUR if reblur else tvd.Formulation.NORMAL,
        preconditioner=tvd.PrecondSelector(sel), fp_tol=1e-300, fp_max=int(g["fp_max"]),
        inner=K.KrylovConfig(tol=float(g["tol"]), max_iterations=2000))
    rep = tvd.restore(g["v"], B.SymmetricPsf(g["psf"]), cfg)
    stock = golden(name.replace("_xdot", ""))
    runs = [[int(k) for k in r["inner_iterations"]] for r in (g, stock)]
    if reblur:
        assert rep.inner_iterations == runs[0]
    else:
        assert all(min(a, b) - 1 <= c <= max(a, b) + 1
                   for c, a, b in zip(rep.inner_iterations, *runs)), (rep.inner_iterations, runs)
    spread = rel_err(stock["restored"], g["restored"])
    assert rel_err(rep.restored, g["restored"]) < max(1e-8, 2.0 * spread)


@pytest.mark.parametrize("n,kind", [(2048, "M"), (1024, "D_M"), (1024, "M_D"), (512, "M_D"),
                                    (128, "M")])
def test_assembly_band_projections_pfa_match_generic(n, kind):
    """The sine-family band projections of the assembly on the prime-factor engine's tensor-core
    stages run as a general DFT (k_band_pfa; at 2048 / 1024 the column-owner k_band_pfa_co with
    the row-wise level 2 and the fused transpose + eigenvalue epilogue, both epilogue forms)
    against the generic mixed-radix engine (option band_generic) and the oracle's restatement
    of precond.py:369-395: eigenvalues within 1e-12."""
    from paper_1011_5964_b200 import _native as nat
    from paper_1011_5964_b200.harness import gen_psf

    g = torch.Generator(device="cpu").manual_seed(n)
    u = torch.rand(n // 16, n // 16, generator=g, dtype=torch.float64)
    u = torch.nn.functional.interpolate(u[None, None], size=(n, n), mode="bilinear")[0, 0].cuda()
    h = gen_psf("gaussian", 7, 3.0)
    hop = B.StructuredBlurOperator(B.SymmetricPsf(h), B.BoundaryCondition.ANTI_REFLECTIVE, n)
    lop = TV.DiffusionOperator(u, 0.05)
    fast = P.assemble_preconditioner(kind, hop, lop, 1e-3).eigenvalues_device.clone()
    with nat.option("band_generic", 1):
        slow = P.assemble_preconditioner(kind, hop, lop, 1e-3).eigenvalues_device
    assert float((fast - slow).norm() / slow.norm()) < 1e-12
    if n <= 512:
        lam_h = O.blur_eigenvalues(h, "anti_reflective", n)
        s = lop.diagonal() if kind != "M" else None
        want = O.assemble(kind, lam_h, O.diffusion_bands(lop.a_h, lop.a_v), 1e-3)[0]
        assert rel_err(fast.cpu().numpy(), want) < 1e-12
        del s
