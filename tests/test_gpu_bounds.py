"""Out-of-bounds and input-mutation checks of the hand-written kernels through the C ABI.

compute-sanitizer is closed on the GPU pool (profiles/r02/sanitizer/), so the bounds are
checked with the library's own instruments: (1) every scratch slot of a fresh context
allocated under the option ``guard_slots`` carries 4 KB guard bands on both sides, verified
by ``tvd_ctx_check_guards`` after a workload touching every kernel family; (2) the caller's
output buffers are carved out of larger tensors whose surrounding guard bands must keep
their sentinel, and the inputs must come back bit-identical (the reference never mutates
its inputs).  Sizes cover every DST engine: the 89 x 23 / 31 x 11 x 3 / 73 x 7
/ 127 pipelines, the generic engine (DCT), and the Rader engine at 8192.
"""
import ctypes
import threading

import numpy as np
import pytest
import torch

import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200 import _native as nat
from paper_1011_5964_b200.harness import gen_psf

pytestmark = pytest.mark.gpu
G = 1024  # guard doubles on each side
SENTINEL = -7.25e300


def _guarded(n_elems, fill=None):
    big = torch.full((n_elems + 2 * G,), SENTINEL, dtype=torch.float64, device="cuda")
    if fill is not None:
        big[G:G + n_elems] = fill.reshape(-1)
    return big


def _view(big, shape):
    return big[G:G + int(np.prod(shape))].view(*shape)


def _intact(big):
    return bool((big[:G] == SENTINEL).all()) and bool((big[-G:] == SENTINEL).all())


@pytest.mark.parametrize("n,m,bc", [(2048, 15, "anti_reflective"), (1024, 10, "anti_reflective"),
                                    (512, 7, "anti_reflective"), (128, 4, "anti_reflective"),
                                    (512, 7, "reflective"), (8192, 31, "anti_reflective")])
def test_abi_writes_stay_inside_caller_buffers(n, m, bc):
    lib = nat.load()
    ctx = nat.context()
    rng = np.random.default_rng(n + m)
    u = torch.from_numpy(np.cumsum(rng.standard_normal((n, n)), axis=1) * 0.05).cuda()
    w = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    bcv = tvd.BoundaryCondition(bc)
    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", m, m / 2.0)), bcv, n)
    lop = tvd.DiffusionOperator(u, 0.1)
    kind = "M" if bc == "anti_reflective" else "R"
    pre = tvd.assemble_preconditioner(kind, hop, lop, 1e-3)
    system = tvd.NormalSystem(hop, lop, 1e-3)
    win = _guarded(n * n, w)
    w_in = _view(win, (n, n))
    w_copy = w_in.clone()
    calls = {
        "blur": lambda o: lib.tvd_blur_apply(hop.handle, w_in.data_ptr(), o, 0),
        "blur_t": lambda o: lib.tvd_blur_apply(hop.handle, w_in.data_ptr(), o, 1),
        "system": lambda o: lib.tvd_system_apply(ctx, ctypes.byref(system.c_struct()),
                                                 w_in.data_ptr(), o),
        "minv": lambda o: lib.tvd_precond_apply_inverse(
            ctx, pre.family_code, n, pre.inverse_eigenvalues_device.data_ptr(), None,
            w_in.data_ptr(), o),
        "transform": lambda o: lib.tvd_transform_2d(ctx, pre.family_code, n, w_in.data_ptr(),
                                                    o, 1),
    }
    if n == 8192:  # the 512 MB cases: the preconditioner engines only
        calls = {k: calls[k] for k in ("minv", "transform")}
    for name, call in calls.items():
        out = _guarded(n * n)
        nat.check(call(_view(out, (n, n)).data_ptr()))
        torch.cuda.synchronize()
        assert _intact(out), name
        assert torch.equal(w_in, w_copy), f"{name} mutated its input"
        assert _intact(win), name
    if n <= 2048:  # the fused PCG: solution and history buffers
        b = hop.apply_transpose(w)
        xg, hg = _guarded(n * n), _guarded(40)
        it, conv, ei, ev = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
        cpre = nat.TvdPrecond(nat.PRE_TRANSFORM, pre.family_code,
                              pre.inverse_eigenvalues_device.data_ptr(), None)
        nat.check(lib.tvd_pcg_solve(ctx, ctypes.byref(system.c_struct()), ctypes.byref(cpre),
                                    b.data_ptr(), u.data_ptr(), _view(xg, (n, n)).data_ptr(),
                                    1e-30, 40, _view(hg, (40,)).data_ptr(), ctypes.byref(it),
                                    ctypes.byref(conv), ctypes.byref(ei), ctypes.byref(ev)))
        torch.cuda.synchronize()
        assert it.value == 40 and _intact(xg) and _intact(hg)


def test_scratch_guard_bands_after_every_kernel_family():
    """A fresh context (own thread) with guarded scratch runs PCG at every pipeline size,
    the DCT family, D_X / X_D kinds, BiCGstab with the P family and AR ghosts, the slab
    phases, and the 8192 Rader M^-1; no guard byte may change."""
    result = {}

    def work():
        from paper_1011_5964_b200 import slab as SL

        torch.cuda.set_device(0)
        nat.set_option("guard_slots", 1)
        try:
            rng = np.random.default_rng(9)
            cfg = tvd.KrylovConfig(tol=1e-30, max_iterations=6)
            for n, m, bc, kind in ((2048, 15, "anti_reflective", "M"),
                                   (1024, 10, "anti_reflective", "D_M"),
                                   (512, 7, "anti_reflective", "M_D"),
                                   (128, 4, "anti_reflective", "M"),
                                   (512, 7, "reflective", "R")):
                u = torch.from_numpy(np.cumsum(rng.standard_normal((n, n)), 1) * 0.05).cuda()
                hop = tvd.StructuredBlurOperator(
                    tvd.SymmetricPsf(gen_psf("gaussian", m, m / 2.0)), tvd.BoundaryCondition(bc), n)
                lop = tvd.DiffusionOperator(u, 0.1)
                pre = tvd.assemble_preconditioner(kind, hop, lop, 1e-3)
                system = tvd.NormalSystem(hop, lop, 1e-3)
                b = hop.apply(u) if bc == "reflective" else hop.apply_transpose(u)
                for _ in range(2):
                    tvd.pcg(system, pre.apply_inverse, b, u, cfg)
            n = 128
            u = torch.from_numpy(np.cumsum(rng.standard_normal((n, n)), 1) * 0.05).cuda()
            hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 4, 2.0)),
                                             tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
            lop = tvd.DiffusionOperator(u, 0.1, tvd.DiffusionBc.ANTI_REFLECTIVE)
            pre = tvd.assemble_preconditioner("P", hop, lop, 1e-3)
            tvd.pbicgstab(tvd.NormalSystem(hop, lop, 1e-3, reblur=True), pre.apply_inverse,
                          hop.apply(u), u, tvd.KrylovConfig(1e-30, 4))
            n = 512
            u = torch.from_numpy(np.cumsum(rng.standard_normal((n, n)), 1) * 0.05).cuda()
            hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 7, 3.5)),
                                             tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
            lop = tvd.DiffusionOperator(u, 0.1)
            pre = tvd.assemble_preconditioner("M", hop, lop, 1e-3)
            system = tvd.NormalSystem(hop, lop, 1e-3)
            b = hop.apply_transpose(u)
            slabs = [SL.Slab(system, pre.apply_inverse, 4, r) for r in range(4)]
            SL.slab_pcg(slabs, SL.LoopbackComm(), [SL.split_rows(b, 4, r) for r in range(4)],
                        [SL.split_rows(u, 4, r) for r in range(4)], cfg, graph=False)
            lam = torch.from_numpy(rng.uniform(0.5, 2.0, (8192, 8192))).cuda()
            tvd.FactoredPreconditioner("M", tvd.TransformKind.SINE_HAT, lam, 1e-3).apply_inverse(
                torch.from_numpy(rng.standard_normal((8192, 8192))).cuda())
            result["guards"] = nat.check_guards()
        except Exception as exc:  # noqa: BLE001 - reported below
            result["error"] = exc
        finally:
            nat.set_option("guard_slots", 0)

    t = threading.Thread(target=work)
    t.start()
    t.join()
    if "error" in result:
        raise result["error"]
    bad, slots = result["guards"]
    assert slots >= 8, slots
    assert bad == 0, f"{bad} guard bytes overwritten"
