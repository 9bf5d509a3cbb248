"""Add one finished reference c3 run to tests/golden/c3_parity.json (build container).

    python tests/golden/add_c3_run.py NAME TRACE_DIR "how it was run"

TRACE_DIR is the output of tools/c3_ref_trace.py (trace.json + u_20.npy): the UNMODIFIED
reference restore on the c3 inputs, optionally with ``--exact`` (use_fast_blur=False) or
``--exact-dots`` (its BLAS dots replaced by exactly rounded ones).  Stored per run: counts,
RRE, image norm / 16-stride subsample / 64-projection sketch, and for every FP step the last
six relative residuals of the reference's own history (krylov.py:105-109), which the device
test uses to recognise near-ties at the tolerance.  make_c3_parity.py rebuilds the whole file
from all traces; this script merges one run when the other traces are no longer on disk.
"""
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))
from sketch import sketch  # noqa: E402

from paper_1011_5964_b200.harness import CONFIGS, make_problem  # noqa: E402

name, d, how = sys.argv[1], pathlib.Path(sys.argv[2]), sys.argv[3]
spec = CONFIGS["c3"]
_, _, u_true = make_problem(spec)
tr = json.loads((d / "trace.json").read_text())
assert len(tr["counts"]) == spec.fp_steps, "unfinished run"
u = np.load(d / f"u_{spec.fp_steps}.npy")
path = HERE / "c3_parity.json"
ev = json.loads(path.read_text())
ev["reference_runs"][name] = {
    "how": how,
    "counts": tr["counts"],
    "rre": float(np.linalg.norm(u - u_true) / np.linalg.norm(u_true)),
    "image": {"norm": float(np.linalg.norm(u)), "sub": u[::16, ::16].tolist(),
              "sketch": sketch(u, 64).tolist()},
    "last_residuals": [hh[-4:] for hh in tr["hist"]],
    "hist_tail": [hh[-6:] for hh in tr["hist"]]}
path.write_text(json.dumps(ev, indent=1))
print(name, tr["counts"])
