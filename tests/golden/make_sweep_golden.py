"""Freeze a reference 2D sweep (row f4, harness.py:215-502) as fixtures (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sweep_golden.py

Runs the REAL reference ``tvdeblur.harness.run_sweep`` on a small 2D spec and copies its
output files (``iterations.csv``, ``rre_vs_alpha.csv``, the restored PGMs) into
``tests/golden/sweep_ref/``; ``tests/test_gpu_parity.py`` runs the same spec through
``paper_1011_5964_b200.sweep`` and compares.
"""
import pathlib
import shutil
import tempfile

from tvdeblur import harness as H

OUT = pathlib.Path(__file__).resolve().parent / "sweep_ref"

SPEC = dict(dimension=2, psf_kind="gaussian", ns=(48,), alphas=(1e-3, 1e-2), betas=(0.1,),
            configurations=("R", "AR+Sine+ZN", "AR+Reblur+ZN"),
            preconditioners=("x", "d_x"), fp_max=40)

if __name__ == "__main__":
    with tempfile.TemporaryDirectory() as td:
        res = H.run_sweep(H.BenchmarkSpec(**SPEC), out_dir=td)
        if OUT.exists():
            shutil.rmtree(OUT)
        OUT.mkdir()
        for f in res.files:
            shutil.copy(f, OUT / pathlib.Path(f).name)
    print(sorted(p.name for p in OUT.iterdir()))
