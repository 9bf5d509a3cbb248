"""CPU tests of the row-slab decomposition: slab geometry, the collectives of
``TorchComm`` (gloo, world_size 2) against ``LoopbackComm``, and the whole multi-rank PCG
schedule of ``paper_1011_5964_b200.slab`` driving numpy test doubles of the native phases
(tests/slab_mirror.py), checked against the oracle PCG on the full arrays."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tvd_oracle as O
from paper_1011_5964_b200 import slab as SL
from paper_1011_5964_b200.krylov import KrylovConfig
from slab_mirror import MirrorSlab, ar_blur_matrix, build_case


# ------------------------------------------------------------------ geometry
def test_layout_halo_plan_and_blocks():
    lay = SL.SlabLayout(n=64, nranks=4, rank=1, khalo=8)
    assert (lay.rows, lay.row_lo) == (16, 16)
    assert lay.ext_shape(8) == (32, 64)
    plan = lay.halo_plan(8)
    assert plan == [(0, slice(8, 16), slice(0, 8)), (2, slice(16, 24), slice(24, 32))]
    assert SL.SlabLayout(64, 4, 0, 8).halo_plan(1) == [(1, slice(16, 17), slice(17, 18))]
    assert SL.SlabLayout(64, 4, 3, 8).halo_plan(1) == [(2, slice(1, 2), slice(0, 1))]
    assert SL.SlabLayout(64, 1, 0, 8).halo_plan(8) == []
    assert lay.block(2) == slice(512, 768)


def test_ar_blur_matrix_matches_oracle_blur():
    from paper_1011_5964_b200.harness import gen_psf
    h = gen_psf("gaussian", 3, 1.2)
    g = h.sum(axis=1)
    H1 = ar_blur_matrix(g / g.sum(), 24)
    u = np.random.default_rng(0).uniform(size=(24, 24))
    np.testing.assert_allclose(H1 @ u @ H1.T, O.blur(u, h, "anti_reflective"), rtol=0, atol=1e-14)


# ------------------------------------------------------------------ schedule (loopback)
def _mirrors(case, nranks, transform=True, d=True, khalo=4):
    return [MirrorSlab(case["G"], case["G"], case["alpha"], case["a_h"], case["a_v"],
                       case["lam_inv"] if transform else None,
                       case["d_sqrt"] if d else None, nranks, r, khalo, transform)
            for r in range(nranks)]


def _oracle_pcg(case, tol, max_it, transform=True, d=True):
    h, alpha, a_h, a_v = case["h"], case["alpha"], case["a_h"], case["a_v"]

    def apply_a(w):
        return O.blur_transpose(O.blur(w, h, "anti_reflective"), h, "anti_reflective") + \
            alpha * O.diffusion_apply(a_h, a_v, w)

    ds = case["d_sqrt"] if d else None
    if transform:
        minv = lambda r: O.precond_solve("sine_hat", case["lam_inv"], r, ds)  # noqa: E731
    else:
        minv = (lambda r: r / ds) if d else None
    return O.pcg(apply_a, minv, case["rhs"], case["v"], tol, max_it, record_history=True)


def _split(a, nranks):
    return [torch.from_numpy(np.ascontiguousarray(x)) for x in np.split(a, nranks)]


@pytest.mark.parametrize("nranks", [1, 2, 4])
@pytest.mark.parametrize("mode", [(True, True), (True, False), (False, True), (False, False)])
def test_loopback_schedule_matches_oracle_pcg(nranks, mode):
    transform, d = mode
    case = build_case()
    cfg = KrylovConfig(tol=1e-8, max_iterations=200, record_history=True)
    outs = SL.slab_pcg(_mirrors(case, nranks, transform, d), SL.LoopbackComm(),
                       _split(case["rhs"], nranks), _split(case["v"], nranks), cfg)
    x = np.concatenate([o.solution.numpy() for o in outs])
    xo, its, hist, ok = _oracle_pcg(case, 1e-8, 200, transform, d)
    assert ok and all(o.converged for o in outs)
    assert {o.iterations for o in outs} == {its}
    np.testing.assert_allclose(outs[0].residual_history, hist, rtol=1e-9)
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)


def test_loopback_schedule_reports_nonconvergence():
    case = build_case()
    cfg = KrylovConfig(tol=1e-30, max_iterations=3)
    outs = SL.slab_pcg(_mirrors(case, 2), SL.LoopbackComm(), _split(case["rhs"], 2),
                       _split(case["v"], 2), cfg)
    assert [(o.iterations, o.converged) for o in outs] == [(3, False), (3, False)]


# ------------------------------------------------------------------ multi-rank (gloo)
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _FakeSlab:
    """Buffers only: deterministic contents per rank, to compare the two communicators."""

    def __init__(self, n, nranks, rank, khalo):
        self.n = n
        self.layout = SL.SlabLayout(n, nranks, rank, khalo)
        R = self.layout.rows
        g = torch.Generator().manual_seed(100 + rank)
        sizes = {SL.BUF_P_EXT: (R + 2) * n, SL.BUF_T_EXT: (R + 2 * khalo) * n,
                 SL.BUF_SEND: R * n, SL.BUF_RECV: R * n, SL.BUF_CONTRIB: 1,
                 SL.BUF_GATHER: nranks}
        self._b = {k: torch.rand(v, generator=g, dtype=torch.float64) for k, v in sizes.items()}

    def buf(self, which):
        return self._b[which]


def _comm_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, k = 32, 4
        # collectives: gloo vs loopback on identical buffers
        mine = _FakeSlab(n, world, rank, k)
        ref = [_FakeSlab(n, world, r, k) for r in range(world)]
        comm, loop = SL.TorchComm(), SL.LoopbackComm()
        comm.halo([mine])
        comm.all_to_all([mine])
        comm.allgather([mine])
        loop.halo(ref)
        loop.all_to_all(ref)
        loop.allgather(ref)
        same = all(torch.equal(mine.buf(w), ref[rank].buf(w))
                   for w in (SL.BUF_P_EXT, SL.BUF_T_EXT, SL.BUF_RECV, SL.BUF_GATHER))
        # the FP-step setup's collectives (slab_operators): u halo rows, the level-2 block
        # all-to-all, the eigenvalue min / max
        lays = [SL.SlabLayout(n, world, r, 1) for r in range(world)]
        R = n // world

        def ext_of(r):
            return torch.rand((R + 2, n), generator=torch.Generator().manual_seed(7 + r),
                              dtype=torch.float64)

        def send_of(r):
            return torch.rand((world, R, R), generator=torch.Generator().manual_seed(70 + r),
                              dtype=torch.float64)

        e_mine, e_ref = ext_of(rank), [ext_of(r) for r in range(world)]
        comm.halo_rows([e_mine], [lays[rank]])
        loop.halo_rows(e_ref, lays)
        (recv,) = comm.all_to_all_blocks([send_of(rank)])
        recv_ref = loop.all_to_all_blocks([send_of(r) for r in range(world)])[rank]
        mm = comm.allreduce_min_max([(0.5 + rank, 2.0 * rank)])
        same = same and torch.equal(e_mine, e_ref[rank]) and torch.equal(recv, recv_ref) and \
            mm == loop.allreduce_min_max([(0.5 + r, 2.0 * r) for r in range(world)])
        # the whole PCG schedule over gloo with the numpy phases
        case = build_case()
        cfg = KrylovConfig(tol=1e-8, max_iterations=200)
        (o,) = SL.slab_pcg(_mirrors(case, world)[rank:rank + 1], comm,
                           _split(case["rhs"], world)[rank:rank + 1],
                           _split(case["v"], world)[rank:rank + 1], cfg)
        out.put((rank, same, o.iterations, o.converged, o.solution.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_slab_collectives_and_schedule():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), "gloo collectives differ from the loopback reference"
    case = build_case()
    xo, its, _, ok = _oracle_pcg(case, 1e-8, 200)
    assert ok and all(r[3] for r in res) and {r[2] for r in res} == {its}
    x = np.concatenate([r[4] for r in res])
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
