"""Collect the config-c3 parity evidence into tests/golden/c3_parity.json (build container).

Inputs (all produced in this container from the unmodified reference, except the device
runs, which come back from the GPU box in gpurun_out/):

* reference restores on identical inputs (tools/c3_ref_trace.py; about 30 min each, the
  exact-operator run about 2 h):
    A  round-1 golden   tests/golden/restore_c3_head.npz (counts, norm, 1/256 subsample)
    B  OpenBLAS 8 threads      TRACE_B = /tmp/c3ref      (trace.json, u_20.npy)
    C  OpenBLAS 1 thread       TRACE_C = /tmp/c3ref1
    D  use_fast_blur=False     TRACE_D = /tmp/c3exact    (exact pad/convolve H, H^T)
* single FP-step replays from run B's iterates u_k:
    tools/c3_step_probe.py  -> step_K.json  (reference fast / exact H^T)
    tools/c3_dot_probe.py   -> dot_K.json   (reference with BLAS vs exactly rounded dots)
    tools/c3_gpu_step.py    -> gpurun_out/c3_gpu_step*.json (device fused PCG variants)
    tools/c3_mixed_step.py  -> gpurun_out/c3_mixed_6.json (oracle loop, device / host ops)
* device restores under rounding-different operator paths: tools/c3_variants.py ->
  gpurun_out/c3_variants.json.

    python tests/golden/make_c3_parity.py
"""
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE.parent))
from sketch import sketch  # noqa: E402

from paper_1011_5964_b200.harness import CONFIGS, make_problem  # noqa: E402

TRACES = {"B_blas_8_threads": "/tmp/c3ref", "C_blas_1_thread": "/tmp/c3ref1",
          "D_exact_operators": "/tmp/c3exact"}
spec = CONFIGS["c3"]
h, v, u_true = make_problem(spec)
out = {"config": "c3", "tol": spec.tol, "fp_steps": spec.fp_steps,
       "v_norm": float(np.linalg.norm(v)), "reference_runs": {}}
g = np.load(HERE / "restore_c3_head.npz")
out["reference_runs"]["A_round1_golden"] = {
    "counts": [int(k) for k in g["inner_iterations"]], "rre": float(g["rre"]),
    "image": {"norm": float(g["restored_norm"]), "sub": g["restored_sub"].tolist()}}
for name, d in TRACES.items():
    d = pathlib.Path(d)
    tr = json.loads((d / "trace.json").read_text())
    if len(tr["counts"]) < spec.fp_steps or not (d / f"u_{spec.fp_steps}.npy").exists():
        print("skipping unfinished", name)
        continue
    u = np.load(d / f"u_{spec.fp_steps}.npy")
    out["reference_runs"][name] = {
        "counts": tr["counts"],
        "rre": float(np.linalg.norm(u - u_true) / np.linalg.norm(u_true)),
        "image": {"norm": float(np.linalg.norm(u)), "sub": u[::16, ::16].tolist(),
                  "sketch": sketch(u, 64).tolist()},
        "last_residuals": [hh[-4:] for hh in tr["hist"]]}
# agreement of the reference runs' images with each other
imgs = {n: np.load(pathlib.Path(d) / f"u_{spec.fp_steps}.npy") for n, d in TRACES.items()
        if n in out["reference_runs"]}
names = sorted(imgs)
out["reference_image_spread"] = {
    f"{a} vs {b}": float(np.linalg.norm(imgs[a] - imgs[b]) / np.linalg.norm(imgs[b]))
    for i, a in enumerate(names) for b in names[i + 1:]}
# single-step replays
steps = {}
B = pathlib.Path(TRACES["B_blas_8_threads"])
for f in sorted(B.glob("step_*.json")):
    s = json.loads(f.read_text())
    k = str(s["k"])
    steps.setdefault(k, {})["reference_fast_HT"] = {"count": s["fast"]["count"],
                                                    "tail": s["fast"]["hist"][-4:]}
    steps[k]["reference_exact_HT"] = {"count": s["exact"]["count"], "tail": s["exact"]["hist"][-4:]}
    steps[k]["r0_fast_transpose_noise_rel"] = s["r0_noise_rel"]
    steps[k]["r0_noise_border_share"] = s["r0_noise_border_share"]
for f in sorted(B.glob("dot_*.json")):
    s = json.loads(f.read_text())
    k = str(s["k"])
    for name in ("blas_dot", "exact_dot"):
        steps.setdefault(k, {})[f"reference_{name}"] = {"count": s[name]["count"],
                                                        "tail": s[name]["hist"][-4:]}
G = ROOT / "gpurun_out"
for f in ("c3_gpu_step2.json", "c3_gpu_step3.json"):
    if (G / f).exists():
        s = json.loads((G / f).read_text())
        for k, res in s.items():
            if not isinstance(res, dict):
                continue
            for name, r in res.items():
                if isinstance(r, dict) and "count" in r:
                    steps.setdefault(k, {})[f"device_{name}"] = {"count": r["count"],
                                                                 "tail": r["hist"][-4:]}
if (G / "c3_mixed_6.json").exists():
    for name, r in json.loads((G / "c3_mixed_6.json").read_text()).items():
        steps.setdefault("6", {})[f"oracle_loop_{name}"] = {"count": r["count"],
                                                            "tail": r["hist"][-4:]}
out["single_step_replays_from_run_B"] = steps
if (G / "c3_variants.json").exists():
    out["device_variants"] = {n: {"counts": o["counts"], "sub_rel_vs_default": o["sub_rel_vs_default"]}
                              for n, o in json.loads((G / "c3_variants.json").read_text()).items()}
(HERE / "c3_parity.json").write_text(json.dumps(out, indent=1))
for n, r in out["reference_runs"].items():
    print(f"{n:22s} {r['counts']}")
print("image spread", out["reference_image_spread"])
