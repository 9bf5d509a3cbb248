"""Programmatic dependent launch (option ``pdl``, csrc/tvd_common.cuh) must not change a bit.

A c2a-sized solve (AR + M: DST pipeline, DMMA band passes, fused vector kernels, graph
replay) and a c2b-sized one (reflective + R: the generic mixed-radix engine) run with the
attribute off and on (setting the option drops the captured solver graphs, so the second arm
re-captures with the attribute); solutions compared bit for bit, iteration counts equal.
"""
import hashlib

import pytest


def _solves() -> list[tuple]:
    import torch

    import paper_1011_5964_b200 as tvd
    from paper_1011_5964_b200.harness import CONFIGS, make_problem

    dev = torch.device("cuda", 0)
    out = []
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
            res = tvd.pcg(tvd.NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, v_dev,
                          cfg)
            sol = res.solution.cpu().numpy()
            out.append((name, rep, res.iterations, hashlib.sha256(sol.tobytes()).hexdigest()))
    return out


@pytest.mark.gpu
def test_pdl_bit_identical():
    from paper_1011_5964_b200 import _native as nat

    assert nat.get_option("pdl") == 1  # the default
    with nat.option("pdl", 0):
        assert nat.get_option("pdl") == 0
        plain = _solves()
    assert nat.get_option("pdl") == 1
    pdl = _solves()
    assert len(plain) == 4 and plain == pdl, (plain, pdl)
