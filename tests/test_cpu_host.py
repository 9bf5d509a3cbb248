"""CPU-only tests: C-ABI library surface, host-side logic, the multi-rank sharding
(gloo, world_size 2) and the no-CPU-fallback contract."""

import ctypes
import os
import pathlib
import re
import socket
import warnings

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1011_5964_b200 import _native as nat
from paper_1011_5964_b200 import harness as H
from paper_1011_5964_b200.blur import BoundaryCondition, StructuredBlurOperator, SymmetricPsf
from paper_1011_5964_b200.krylov import KrylovConfig
from paper_1011_5964_b200.pipeline import (ConfigurationError, Formulation, PrecondSelector,
                                           RestorationConfig, restore)
from paper_1011_5964_b200.sharding import reduce_run, shard_problems

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tvdeblur_b200.h"


# ------------------------------------------------------------------ C ABI
def _declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tvd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("tvd_ctx_create", "tvd_blur_apply", "tvd_diffusivity", "tvd_transform_2d",
                     "tvd_precond_assemble", "tvd_precond_apply_inverse", "tvd_pcg_solve"):
        assert required in names


def test_library_loads_and_exports_every_declared_symbol():
    lib = nat.load()
    declared = _declared_functions()
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(nat.EXPORTED), set(declared) ^ set(nat.EXPORTED)
    abi = int(re.search(r"#define TVD_ABI_VERSION (\d+)", HEADER.read_text()).group(1))
    assert lib.tvd_abi_version() == abi


def test_library_is_built_for_sm_100a():
    so = ROOT / "paper_1011_5964_b200" / "libtvdeblur_b200.so"
    import subprocess
    res = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    out = res.stdout + res.stderr
    assert "sm_100a" in out


def test_profile_categories_are_named():
    lib = nat.load()
    names = []
    while (nm := lib.tvd_profile_category(len(names))) is not None:
        names.append(nm.decode())
    assert {"trig_rows", "trig_cols", "band_rows", "band_cols", "vector"} <= set(names)


# -------------------------------------------------------- no CPU fallback
@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only contract")
def test_operators_fail_loudly_without_a_device():
    psf = SymmetricPsf(H.gen_psf("gaussian", 2, 1.0))
    with pytest.raises(RuntimeError, match="CUDA"):
        StructuredBlurOperator(psf, BoundaryCondition.ANTI_REFLECTIVE, 16)
    cfg = RestorationConfig(bc_h=BoundaryCondition.ANTI_REFLECTIVE, alpha=1e-3, beta=0.1)
    with pytest.raises(RuntimeError, match="CUDA"):
        restore(np.ones((16, 16)), psf, cfg)


# ------------------------------------------------------------ host logic
def test_config_invariants_match_reference():
    # pkg/tests/test_pipeline.py:25-42
    bad = RestorationConfig(bc_h=BoundaryCondition.REFLECTIVE, alpha=1e-3, beta=0.1,
                            formulation=Formulation.REBLUR)
    with pytest.raises(ConfigurationError):
        bad.validate()
    bad = RestorationConfig(bc_h=BoundaryCondition.PERIODIC, alpha=1e-3, beta=0.1,
                            preconditioner=PrecondSelector.X)
    with pytest.raises(ConfigurationError):
        bad.validate()
    with pytest.raises(ConfigurationError):
        RestorationConfig(bc_h=BoundaryCondition.REFLECTIVE, alpha=-1.0, beta=0.1).validate()
    with pytest.raises(ConfigurationError):
        RestorationConfig(bc_h=BoundaryCondition.REFLECTIVE, alpha=1.0, beta=0.1,
                          fp_tol=0.0).validate()
    with pytest.raises(ConfigurationError):  # raised before any compute, device or not
        restore(np.ones((16, 16)), SymmetricPsf(np.ones((1, 1))),
                RestorationConfig(bc_h=BoundaryCondition.REFLECTIVE, alpha=1e-3, beta=0.1,
                                  formulation=Formulation.REBLUR))


def test_resolved_kind_labels():
    cfg = RestorationConfig(bc_h=BoundaryCondition.ANTI_REFLECTIVE, alpha=1e-3, beta=0.1,
                            formulation=Formulation.REBLUR, preconditioner=PrecondSelector.D_X)
    assert cfg.resolved_kind() == "D_P"
    cfg = RestorationConfig(bc_h=BoundaryCondition.REFLECTIVE, alpha=1e-3, beta=0.1,
                            preconditioner=PrecondSelector.X_D)
    assert cfg.resolved_kind() == "R_D"
    cfg = RestorationConfig(bc_h=BoundaryCondition.ANTI_REFLECTIVE, alpha=1e-3, beta=0.1,
                            preconditioner=PrecondSelector.NONE)
    assert cfg.resolved_kind() == "I"


def test_krylov_config_validation():
    with pytest.raises(ValueError):
        KrylovConfig(tol=0.0)
    with pytest.raises(ValueError):
        KrylovConfig(max_iterations=0)


def test_symmetric_psf_validation():
    with pytest.raises(ValueError):
        SymmetricPsf(np.ones((3, 5)))
    with pytest.raises(ValueError):
        SymmetricPsf(np.ones((4, 4)))
    with pytest.raises(ValueError):
        SymmetricPsf(np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 0.0], [0.0, 0.0, 0.0]]))
    with pytest.raises(ValueError):
        SymmetricPsf(np.full((3, 3), np.nan))
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        psf = SymmetricPsf(np.ones((3, 3)))
    assert any("renormalizing" in str(x.message) for x in w)
    np.testing.assert_allclose(psf.coefficients.sum(), 1.0)
    assert psf.half_width == 1


# -------------------------------------------------------------- harness
def test_generator_is_deterministic_and_shaped():
    a = H.gen_piecewise_image(64, 4, 12, 6, seed=2023)
    b = H.gen_piecewise_image(64, 4, 12, 6, seed=2023)
    c = H.gen_piecewise_image(64, 4, 12, 6, seed=2024)
    assert a.shape == (72, 72)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, c)
    assert a.min() >= 0.0 and a.max() <= 1.0
    r = H.gen_piecewise_image(64, 4, 12, 6, seed=2023, ramp=True)
    np.testing.assert_allclose(r - a, 0.1 * (np.arange(72)[:, None] + np.arange(72)[None, :])
                               / 71 / 2.0)


def test_observation_has_exact_nsr_and_matches_reference_formula():
    h = H.gen_psf("gaussian", 3, 1.2)
    ext = H.gen_piecewise_image(40, 3, 5, 3, seed=1)
    clean = H.blur_and_observe(ext, h, 40, 0.0, 7)
    sep = H.blur_and_observe(ext, h, 40, 0.0, 7, exact=False)
    np.testing.assert_allclose(sep, clean, rtol=0, atol=1e-14)
    v = H.blur_and_observe(ext, h, 40, 0.01, 7)
    assert abs(np.linalg.norm(v - clean) / np.linalg.norm(clean) - 0.01) < 1e-12
    # separable fast path == direct 2D valid convolution
    direct = np.zeros((40, 40))
    for a in range(7):
        for b in range(7):
            direct += h[6 - a, 6 - b] * ext[a:a + 40, b:b + 40]
    np.testing.assert_allclose(clean, direct, rtol=0, atol=1e-14)


def test_gen_psf_matches_reference_definition():
    h = H.gen_psf("gaussian", 4, 1.5)
    i = np.arange(-4, 5)
    g = np.exp(-(i[:, None] ** 2 + i[None, :] ** 2) / (2 * 1.5 ** 2))
    np.testing.assert_allclose(h, g / g.sum(), rtol=1e-15)
    box = H.gen_psf("box", 5)
    assert box.shape == (11, 11) and np.allclose(box, 1 / 121)


# ------------------------------------------------------ multi-rank (gloo)
def test_shard_problems_partition_and_balance():
    for world in (1, 2, 4, 8):
        seen = []
        for rank in range(world):
            mine = shard_problems(64, world, rank)
            assert len(mine) == 64 // world
            assert sum(1 for i in mine if i % 2) == len(mine) // 2  # gaussian / box balance
            seen.extend(mine)
        assert sorted(seen) == list(range(64))
    with pytest.raises(ValueError):
        shard_problems(8, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard_problems(16, world, rank)
        elapsed = 1.0 + rank  # fake per-rank device times
        t, it, ln = reduce_run(elapsed, iterations=10 * len(mine), launches=7)
        out.put((rank, mine, t, it, ln))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert sorted(res[0][1] + res[1][1]) == list(range(16))
    for _, _, t, it, ln in res:
        assert t == 2.0          # max over ranks
        assert it == 160         # summed iterations
        assert ln == 14


# ------------------------------------------------------------ sweep file formats (row f4)
def test_sweep_file_formats_round_trip(tmp_path):
    """CSV / PGM writers keep the reference's formats (harness.py:452-489): the committed
    reference outputs read back, and re-written files are byte-identical."""
    from paper_1011_5964_b200 import sweep as SW
    ref = ROOT / "tests" / "golden" / "sweep_ref"
    hdr, rows = SW.read_csv(ref / "iterations.csv")
    assert tuple(hdr) == SW.TABLE_HEADER and len(rows) == 12
    SW.write_csv(tmp_path / "t.csv", hdr, rows)
    assert (tmp_path / "t.csv").read_bytes() == (ref / "iterations.csv").read_bytes()
    for f in sorted(ref.glob("*.pgm"))[:3]:
        img = SW.read_pgm(f)
        assert img.shape == (48, 48) and img.dtype == np.uint8
        SW.write_pgm(tmp_path / f.name, img.astype(float), 0.0, 255.0)
        assert (tmp_path / f.name).read_bytes() == f.read_bytes()
    with pytest.raises(ValueError):
        SW.BenchmarkSpec(configurations=("bogus",))
    assert SW.default_half_width(48) == 6
    img, (fr, fc) = SW.gen_image_2d(32, 4)
    assert img.shape == (40, 40) and (fr.start, fr.stop) == (4, 36)


def test_sweep_csv_matches_the_csv_module_and_sweep_files_parse(tmp_path):
    """The hand-written CSV writer agrees byte for byte with ``csv.writer`` (the reference's
    writer, harness.py:452-460) on floats, ints, numpy scalars, stars and fields that need
    quoting; sweep files (harness.py:512-568) parse to the same spec as keyword arguments."""
    import csv
    import io

    from paper_1011_5964_b200 import sweep as SW

    rows = [("R/x", 1e-3, 0.1, 48, 7, 12.25, 0.0123456789), ("AR+Sine+ZN/d_x", np.float64(2.5e-4),
            np.int64(3), 64, "*", "*", "*"), ('a,"b"', 1.0, -0.0, 0, 1e300, float("inf"), "x\ny")]
    SW.write_csv(tmp_path / "a.csv", SW.TABLE_HEADER, rows)
    buf = io.StringIO(newline="")
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(SW.TABLE_HEADER)
    for r in rows:
        w.writerow([repr(float(x)) if isinstance(x, (float, np.floating)) else
                    int(x) if isinstance(x, np.integer) else x for x in r])
    assert (tmp_path / "a.csv").read_text() == buf.getvalue()
    hdr, back = SW.read_csv(tmp_path / "a.csv")
    assert tuple(hdr) == SW.TABLE_HEADER and back[2][0] == 'a,"b"'
    (tmp_path / "s.cfg").write_text("# sweep\nn = 48, 64\nalpha = 1e-3,1e-2  # two\n"
                                    "config = R, AR+Sine+ZN\nprecond = x, d_x\nfp_max = 40\n"
                                    "save_restored = no\n")
    spec = SW.parse_sweep_config(tmp_path / "s.cfg")
    assert spec == SW.BenchmarkSpec(ns=(48, 64), alphas=(1e-3, 1e-2),
                                    configurations=("R", "AR+Sine+ZN"),
                                    preconditioners=("x", "d_x"), fp_max=40,
                                    save_restored=False)
    keys = list(SW.cell_keys(spec))
    assert len(keys) == 16 and keys[0] == ("R", 48, 0.1, 1e-3, "x") and \
        keys[-1] == ("AR+Sine+ZN", 64, 0.1, 1e-2, "d_x")
    (tmp_path / "bad.cfg").write_text("n 48\n")
    with pytest.raises(ValueError):
        SW.parse_sweep_config(tmp_path / "bad.cfg")
    with pytest.raises(ValueError):
        SW.BenchmarkSpec(dimension=1)
