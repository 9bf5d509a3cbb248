"""Programmatic dependent launch (TVD_PDL=1, csrc/tvd_common.cuh) must not change a single bit.

The attribute is read once per process, so each arm runs in its own interpreter: a c2a-sized
solve (AR + M: DST pipeline, DMMA band passes, fused vector kernels, graph replay) and a
c2b-sized one (reflective + R: the generic mixed-radix engine), solutions compared bit for bit
and iteration counts equal.
"""
import hashlib
import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]

_SCRIPT = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_1011_5964_b200 as tvd
from paper_1011_5964_b200.harness import CONFIGS, make_problem

import torch
dev = torch.device("cuda", 0)
for name in ("c2a", "c2b"):
    spec = CONFIGS[name]
    h, v, _ = make_problem(spec)
    bc = tvd.BoundaryCondition(spec.bc)
    kind = "M" if bc is tvd.BoundaryCondition.ANTI_REFLECTIVE else "R"
    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), bc, spec.n, device=dev)
    v_dev = torch.from_numpy(v).to(dev)
    back = hop.apply if bc is tvd.BoundaryCondition.REFLECTIVE else hop.apply_transpose
    rhs = back(v_dev)
    lop = tvd.DiffusionOperator(v_dev, spec.beta, device=dev)
    pre = tvd.assemble_preconditioner(kind, hop, lop, spec.alpha)
    cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=300)
    for rep in range(2):  # the repeated system is captured into a graph and replayed
        out = tvd.pcg(tvd.NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, v_dev, cfg)
        sol = out.solution.cpu().numpy()
        print(name, rep, out.iterations, hashlib.sha256(sol.tobytes()).hexdigest())
"""


def _run(pdl: bool) -> str:
    env = dict(os.environ)
    env.pop("TVD_PDL", None)
    if pdl:
        env["TVD_PDL"] = "1"
    res = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=str(ROOT))], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return res.stdout


@pytest.mark.gpu
def test_pdl_bit_identical():
    plain, pdl = _run(False), _run(True)
    assert len(plain.strip().splitlines()) == 4, plain
    assert plain == pdl, (plain, pdl, hashlib.sha256(plain.encode()).hexdigest())
