"""GPU parity of the row-slab decomposition (SURVEY.md 8e, config 5 path).

The slab kernels (row-window band passes, all-to-all-segmented DST passes, the PCG phases)
run through the C ABI for P slabs of one device, driven by the same schedule as the
multi-GPU run with :class:`~paper_1011_5964_b200.slab.LoopbackComm` standing in for NCCL
(local copies between the slabs' buffers, in stream order; no kernel waits on another).
Reference: the single-GPU fused PCG on the same system (itself pinned to the oracle and the
reference goldens in test_gpu_parity.py) and, at small n, the oracle PCG.  Gates: identical
iteration counts (the dot products are summed per slab, then over slabs: a different
rounding order, which the tolerances of BASELINE.json's north_star absorb -- counts +-1) and
the solution within 1e-10 relative.
"""

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import tvd_oracle as O

import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200 import slab as SL
from paper_1011_5964_b200.harness import CONFIGS, gen_psf, make_problem

pytestmark = pytest.mark.gpu


def _problem(n, m, sigma, alpha, beta, kind="M", seed=0):
    """A lagged-diffusivity state of a seeded piecewise-constant image blurred on the GPU."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    u = torch.rand(n // 64 + 1, n // 64 + 1, generator=g, dtype=torch.float64)
    u = torch.nn.functional.interpolate(u[None, None], size=(n, n), mode="nearest")[0, 0]
    u = u.cuda()
    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", m, sigma)),
                                     tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
    v = hop.apply(u)
    v = v + 0.01 * v.norm() / n * torch.randn(n, n, generator=g, dtype=torch.float64).cuda()
    lop = tvd.DiffusionOperator(v, beta)
    system = tvd.NormalSystem(hop, lop, alpha)
    pre = None if kind == "I" else tvd.assemble_preconditioner(kind, hop, lop, alpha)
    rhs = hop.apply_transpose(v)
    return system, pre, rhs, v


def _solve_both(system, pre, rhs, x0, nranks, tol, max_it=400):
    cfg = tvd.KrylovConfig(tol=tol, max_iterations=max_it, record_history=True)
    minv = None if pre is None else pre.apply_inverse
    ref = tvd.pcg(system, minv, rhs, x0, cfg)
    slabs = [SL.Slab(system, minv, nranks, r) for r in range(nranks)]
    outs = SL.slab_pcg(slabs, SL.LoopbackComm(),
                       [SL.split_rows(rhs, nranks, r) for r in range(nranks)],
                       [SL.split_rows(x0, nranks, r) for r in range(nranks)], cfg)
    x = torch.cat([o.solution for o in outs])
    its = {o.iterations for o in outs}
    assert len(its) == 1, its  # every slab took the same branch
    return ref, outs[0], x


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
@pytest.mark.parametrize("kind", ["M", "D_M", "I"])
def test_slab_pcg_matches_single_gpu_512(nranks, kind):
    spec = CONFIGS["c2a"]
    system, pre, rhs, v = _problem(512, spec.m, spec.sigma, spec.alpha, spec.beta, kind)
    ref, out, x = _solve_both(system, pre, rhs, v, nranks, spec.tol)
    assert ref.converged and out.converged
    if kind == "I":
        # unpreconditioned CG is rounding-sensitive near tol (the reference's own
        # two operator paths disagree by +-1 there): the gate is the image, counts within 2
        assert abs(out.iterations - ref.iterations) <= (0 if nranks == 1 else 2)
        assert rel_err(x.cpu().numpy(), ref.solution.cpu().numpy()) < 1e-8
        return
    assert abs(out.iterations - ref.iterations) <= (0 if nranks == 1 else 1)
    if out.iterations == ref.iterations:
        assert rel_err(out.residual_history, ref.residual_history) < 1e-9
    assert rel_err(x.cpu().numpy(), ref.solution.cpu().numpy()) < 1e-10


def test_slab_pcg_matches_oracle_c2a():
    """Config 2a through 4 slabs vs the oracle's PCG on the reference's own operators."""
    spec = CONFIGS["c2a"]
    h, v, _ = make_problem(spec)
    n = spec.n
    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), tvd.BoundaryCondition.ANTI_REFLECTIVE, n)
    lop = tvd.DiffusionOperator(v, spec.beta)
    pre = tvd.assemble_preconditioner("M", hop, lop, spec.alpha)
    system = tvd.NormalSystem(hop, lop, spec.alpha)
    vt = torch.from_numpy(v).cuda()
    rhs = hop.apply_transpose(vt)
    cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=400)
    slabs = [SL.Slab(system, pre.apply_inverse, 4, r) for r in range(4)]
    outs = SL.slab_pcg(slabs, SL.LoopbackComm(), [SL.split_rows(rhs, 4, r) for r in range(4)],
                       [SL.split_rows(vt, 4, r) for r in range(4)], cfg)
    x = torch.cat([o.solution for o in outs]).cpu().numpy()
    a_h, a_v = O.diffusivity(v, spec.beta)
    lam_h = O.blur_eigenvalues(h, "anti_reflective", n)
    _, lam_inv, _, _ = O.assemble("M", lam_h, O.diffusion_bands(a_h, a_v), spec.alpha)

    def apply_a(w):
        return O.blur_transpose(O.blur(w, h, "anti_reflective"), h, "anti_reflective") + \
            spec.alpha * O.diffusion_apply(a_h, a_v, w)

    xo, its, _, ok = O.pcg(apply_a, lambda r: O.precond_solve("sine_hat", lam_inv, r),
                           O.blur_transpose(v, h, "anti_reflective"), v, spec.tol, 400)
    assert ok and outs[0].converged
    assert abs(outs[0].iterations - its) <= 1
    assert rel_err(x, xo) < 1e-8


@pytest.mark.parametrize("nranks", [2, 8])
def test_slab_pcg_matches_single_gpu_2048(nranks):
    spec = CONFIGS["c3"]
    system, pre, rhs, v = _problem(2048, spec.m, spec.sigma, spec.alpha, spec.beta)
    ref, out, x = _solve_both(system, pre, rhs, v, nranks, spec.tol)
    assert ref.converged and out.converged
    assert abs(out.iterations - ref.iterations) <= 1
    assert rel_err(x.cpu().numpy(), ref.solution.cpu().numpy()) < 1e-10


def test_slab_pcg_rader_8192_eight_slabs():
    """Config 5 geometry: 8192^2, Gaussian 63x63 (band halo 64 rows), prime odd core 8191
    (Rader engine with segmented input + rectangular transposes), 8 slabs of 1024 rows."""
    spec = CONFIGS["c5"]
    system, pre, rhs, v = _problem(8192, spec.m, spec.sigma, spec.alpha, spec.beta)
    ref, out, x = _solve_both(system, pre, rhs, v, 8, spec.tol)
    assert ref.converged and out.converged
    assert abs(out.iterations - ref.iterations) <= 1
    assert float((x - ref.solution).norm() / ref.solution.norm()) < 1e-10


def test_slab_first_fp_step_8192_matches_reference(golden):
    """The config-5 problem itself (8192^2, seeded observation) over 8 row slabs against the
    REFERENCE's own first FP step (tests/golden/c5_ops.npz, make_golden.py --c5: rhs =
    H^T_fast v, u0 = v, kind M, tol 1e-4): count within one, iterate within 1e-8 over all
    67M pixels (sketch) and on the subsample."""
    from conftest import rel_err as _rel
    from sketch import sketch_torch

    g = golden("c5_ops.npz")
    spec = CONFIGS["c5"]
    n = spec.n
    dev = torch.device("cuda")
    h, v_np, _ = make_problem(spec, exact=False, device=dev)
    v = torch.from_numpy(v_np).to(dev)
    del v_np
    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), tvd.BoundaryCondition.ANTI_REFLECTIVE,
                                     n, device=dev)
    lop = tvd.DiffusionOperator(v, spec.beta, device=dev)
    pre = tvd.assemble_preconditioner("M", hop, lop, spec.alpha)
    system = tvd.NormalSystem(hop, lop, spec.alpha)
    rhs = hop.apply_transpose(v)
    P = 8
    slabs = [SL.Slab(system, pre.apply_inverse, P, r) for r in range(P)]
    outs = SL.slab_pcg(slabs, SL.LoopbackComm(), [SL.split_rows(rhs, P, r) for r in range(P)],
                       [SL.split_rows(v, P, r) for r in range(P)],
                       tvd.KrylovConfig(tol=spec.tol, max_iterations=2000))
    x = torch.cat([o.solution for o in outs], dim=0)
    assert outs[0].converged
    assert abs(outs[0].iterations - int(g["fp1_iterations"])) <= 1
    ref_norm = float(g["fp1_u_norm"])
    sk = g["fp1_u_sketch"]
    est = np.linalg.norm(sketch_torch(x, len(sk)) - sk) / np.sqrt(len(sk)) / ref_norm
    assert est < 1e-8, est
    assert _rel(x[::61, ::61].cpu().numpy(), g["fp1_u_sub"]) < 1e-8


def test_slab_rejects_bad_geometry():
    spec = CONFIGS["c2a"]
    system, pre, rhs, v = _problem(512, spec.m, spec.sigma, spec.alpha, spec.beta)
    with pytest.raises(ValueError):
        SL.Slab(system, pre.apply_inverse, 3, 0)  # 512 not divisible by 3
    with pytest.raises(tvd._native.NativeError):
        SL.Slab(system, pre.apply_inverse, 64, 0)  # 8-row slabs: below the band halo


def test_slab_pcg_over_nccl_single_rank():
    """The TorchComm collectives on the library's device buffers through a real NCCL process
    group (world size 1 on the one GPU of the test box: all-to-all and allgather run, the halo
    plan is empty), against the single-GPU PCG."""
    import os
    import socket

    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        spec = CONFIGS["c2a"]
        system, pre, rhs, v = _problem(512, spec.m, spec.sigma, spec.alpha, spec.beta)
        cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=400)
        ref = tvd.pcg(system, pre.apply_inverse, rhs, v, cfg)
        (out,) = SL.slab_pcg([SL.Slab(system, pre.apply_inverse, 1, 0)], SL.TorchComm(),
                             [rhs.contiguous()], [v.contiguous()], cfg)
        assert out.converged and out.iterations == ref.iterations
        assert rel_err(out.solution.cpu().numpy(), ref.solution.cpu().numpy()) < 1e-12
        # the distributed FP-step setup's NCCL tensor collectives (slab_operators)
        (ops,) = SL.slab_operators(system.h_op, [v.contiguous()], [SL.SlabLayout(512, 1, 0, 1)],
                                   SL.TorchComm(), spec.beta, spec.alpha, "M")
        assert torch.equal(ops.inv_t, pre.inverse_eigenvalues_device.t())
        assert torch.equal(ops.a_h, system.l_op.a_h_device)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 4])
def test_slab_pcg_graph_replay_matches_eager(nranks):
    """The slab iteration captured as a CUDA graph (phases + loopback copies) replays to the
    same iterates as the eager schedule, bit for bit."""
    spec = CONFIGS["c2a"]
    system, pre, rhs, v = _problem(512, spec.m, spec.sigma, spec.alpha, spec.beta)
    cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=400, record_history=True)
    outs = {}
    for graph in (False, True):
        slabs = [SL.Slab(system, pre.apply_inverse, nranks, r) for r in range(nranks)]
        outs[graph] = SL.slab_pcg(slabs, SL.LoopbackComm(),
                                  [SL.split_rows(rhs, nranks, r) for r in range(nranks)],
                                  [SL.split_rows(v, nranks, r) for r in range(nranks)], cfg,
                                  graph=graph)
    for a, b in zip(outs[False], outs[True]):
        assert a.iterations == b.iterations and a.converged and b.converged
        assert torch.equal(a.solution, b.solution)
        assert np.array_equal(a.residual_history, b.residual_history)


@pytest.mark.parametrize("n,P,kind", [(512, 4, "M"), (512, 2, "D_M"), (2048, 8, "M"),
                                      (512, 4, "R")])
def test_distributed_fp_setup_is_bit_identical(n, P, kind):
    """slab.slab_operators: each slab's diffusivity, its rows of lambda^-T (level-2
    projection split at one all-to-all) and d_sqrt, computed from its own rows of u plus a
    one-row halo, equal the slices of the single-GPU DiffusionOperator / assemble_preconditioner
    bit for bit; a PCG over the resulting slabs equals one over slabs cut from the full
    operators."""
    bc = tvd.BoundaryCondition.REFLECTIVE if kind.endswith("R") else \
        tvd.BoundaryCondition.ANTI_REFLECTIVE
    g = torch.Generator(device="cpu").manual_seed(n + P)
    u = torch.rand(n // 32, n // 32, generator=g, dtype=torch.float64)
    u = torch.nn.functional.interpolate(u[None, None], size=(n, n), mode="bilinear")[0, 0].cuda()
    u = u + 0.01 * torch.randn(n, n, generator=g, dtype=torch.float64).cuda()
    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(gen_psf("gaussian", 7, 3.0)), bc, n)
    beta, alpha = 0.05, 1e-3
    lop = tvd.DiffusionOperator(u, beta)
    pre = tvd.assemble_preconditioner(kind, hop, lop, alpha)
    layouts = [SL.SlabLayout(n, P, r, 1) for r in range(P)]
    ops = SL.slab_operators(hop, [SL.split_rows(u, P, r) for r in range(P)], layouts,
                            SL.LoopbackComm(), beta, alpha, kind)
    R = n // P
    inv_t = pre.inverse_eigenvalues_device.t()
    for r, o in enumerate(ops):
        lo = r * R
        assert torch.equal(o.a_h, lop.a_h_device[lo:lo + R]), r
        assert torch.equal(o.a_v, lop.a_v_device[lo:lo + R + 1]), r
        assert torch.equal(o.inv_t, inv_t[lo:lo + R]), r
        if kind.startswith("D_"):
            assert torch.equal(o.d, pre.d_sqrt_device[lo:lo + R]), r
    if kind.endswith("R"):
        return  # the slab solver itself runs the M family (config 5)
    system = tvd.NormalSystem(hop, lop, alpha)
    rhs = hop.apply_transpose(u)
    cfg = tvd.KrylovConfig(tol=1e-6, max_iterations=300)
    comm = SL.LoopbackComm()
    b_s = [SL.split_rows(rhs, P, r) for r in range(P)]
    x_s = [SL.split_rows(u, P, r) for r in range(P)]
    a = SL.slab_pcg([SL.Slab(system, pre.apply_inverse, P, r) for r in range(P)], comm, b_s, x_s,
                    cfg)
    b = SL.slab_pcg([SL.Slab.from_operands(hop, alpha, ops[r], P, r) for r in range(P)], comm,
                    b_s, x_s, cfg)
    assert [o.iterations for o in a] == [o.iterations for o in b]
    for oa, ob in zip(a, b):
        assert torch.equal(oa.solution, ob.solution)
