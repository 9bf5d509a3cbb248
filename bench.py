"""Benchmark: PCG iterations/s of the TV-deblurring inner solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

Workload (N=1): BASELINE.json configs[2] = "c3", the 2048^2 anti-reflective
fp64 headline case (Gaussian 31x31 sigma 4, alpha 2e-4, beta 0.05, PCG tol
1e-5, DST-I/Shat preconditioner M).  Synthetic seeded inputs from
``paper_1011_5964_b200.harness`` (the BASELINE generator; no dataset exists).

A *step* is one inner PCG solve of one FP step: the lagged-diffusivity state
after ``--state-fp`` FP steps is prepared untimed, then every step calls the
public ``pcg(system, precond.apply_inverse, rhs, u, cfg)`` on device-resident
inputs and runs to tol.  ``value`` = PCG iterations of all ranks / device
time (CUDA events, max over ranks).  Multi-GPU: one independent problem per
rank (batch sharding, no collective on the hot path) -> ``scaling: weak``.

``e2e``: the same metric through the public API from pinned HOST buffers:
per step H2D of (u, rhs), diffusivity, device preconditioner assembly, PCG,
D2H of the solution.

``--impl reference``: the reference algorithm's CPU path (the oracle port in
``oracle/tvd_oracle.py``; the reference package itself is Python that cannot
travel to the GPU box) with all host cores for its FFTs, each step a bounded
sample of PCG iterations of the same config; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import subprocess
import sys
import tempfile
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "PCG iters/sec at 2048^2 AR fp64 (config c3, DST-I/Shat preconditioner M)"
UNIT = "PCG iters/s"


def metric_for(spec) -> str:
    """The headline METRIC for c3; the same metric, named for its own problem, otherwise."""
    if spec.name == "c3":
        return METRIC
    ar = spec.bc == "anti_reflective"
    pre = "DST-I/Shat preconditioner M" if ar else "DCT preconditioner R"
    return f"PCG iters/sec at {spec.n}^2 {'AR' if ar else 'reflective'} fp64 (config {spec.name}, {pre})"


def bc_tag(spec) -> str:
    return "AR" if spec.bc == "anti_reflective" else "reflective"


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "fallback": True}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int) -> None:
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        self.out = os.fdopen(fd, "w")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.out, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        self.out.close()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx.append(float(f[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        finally:
            os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# -------------------------------------------------------------- reference
def workload(spec) -> str:
    """The one workload label both arms print (``config.workload``)."""
    kind = "M" if spec.bc == "anti_reflective" else "R"
    if spec.name == "c4":
        psf = "Gaussian 21x21 sigma 3 / box 11x11 alternating"
        return (f"{spec.name}: {spec.problems} x {spec.n}^2 AR fp64, {psf}, alpha {spec.alpha}, "
                f"beta {spec.beta}, tol {spec.tol}, preconditioner M")
    return (f"{spec.name}: {spec.n}^2 {bc_tag(spec)} fp64, Gaussian {2 * spec.m + 1}x"
            f"{2 * spec.m + 1} sigma {spec.sigma}, alpha {spec.alpha}, beta {spec.beta}, "
            f"tol {spec.tol}, preconditioner {kind}")


def bench_config(spec, state_fp: int) -> dict:
    """``config`` of the JSON line, identical in both arms for the same workload."""
    ws = 15 * 8 * spec.n ** 2 * spec.problems / 2 ** 20
    l2 = (f"inputs larger than L2 (~15 n^2 fp64 arrays = {ws:.0f} MiB working set vs 126 MB L2)"
          if ws > 126 else f"working set {ws:.0f} MiB fits in L2 (not flushed; small config)")
    return {"workload": workload(spec), "n": spec.n, "problems_per_gpu": 1,
            "state_fp": state_fp, "l2": l2}


def cpu_state(spec, h, v, state_fp: int, u_state=None):
    """Host operators of the oracle port (the reference's fast-operator path,
    pipeline.py:167-179,209-210) at the lagged-diffusivity state after ``state_fp`` FP steps
    from ``u = v`` (pipeline.py:200-244), each step a full PCG solve to tol."""
    from oracle import tvd_oracle as O

    bc = spec.bc
    lam_h = O.blur_eigenvalues(h, bc, spec.n)
    fam = "sine_hat" if bc == "anti_reflective" else "dct"
    kind = "M" if bc == "anti_reflective" else "R"

    def operators(u):
        a_h, a_v = O.diffusivity(u, spec.beta)
        _, lam_inv, _, _ = O.assemble(kind, lam_h, O.diffusion_bands(a_h, a_v), spec.alpha)

        def apply_a(w):
            hw = O.blur_fast(w, lam_h, bc)
            back = hw if bc == "reflective" else O.blur_transpose_fast(hw, lam_h, bc)
            return back + spec.alpha * O.diffusion_apply(a_h, a_v, w)

        return apply_a, (lambda r: O.precond_solve(fam, lam_inv, r))

    rhs = O.blur_transpose_fast(v, lam_h, bc) if bc == "anti_reflective" else O.blur_fast(v, lam_h, bc)
    u = v.copy() if u_state is None else np.asarray(u_state, dtype=float)
    for _ in range(state_fp if u_state is None else 0):
        apply_a, minv = operators(u)
        u = O.pcg(apply_a, minv, rhs, u, spec.tol, 2000)[0]
    apply_a, minv = operators(u)
    return apply_a, minv, rhs, u


def cpu_sample(apply_a, minv, rhs, u, iters: int) -> float:
    """Seconds for exactly ``iters`` PCG loop iterations (krylov.py:95-115: one matvec, one
    M^-1, three dots, three updates) of the oracle port.  The setup ``r = b - A x0``,
    ``z = M^-1 r`` runs untimed, as the GPU arm's per-iteration figure amortises it."""
    x = np.array(u, dtype=float, copy=True)
    r = rhs - apply_a(x)
    z = minv(r)
    p = z.copy()
    rz = float(np.dot(r.ravel(), z.ravel()))
    t0 = time.perf_counter()
    for _ in range(iters):
        q = apply_a(p)
        step = rz / float(np.dot(p.ravel(), q.ravel()))
        x += step * p
        r -= step * q
        math.sqrt(float(np.dot(r.ravel(), r.ravel())))
        z = minv(r)
        rz_next = float(np.dot(r.ravel(), z.ravel()))
        p = z + (rz_next / rz) * p
        rz = rz_next
    return time.perf_counter() - t0


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return None
    from oracle import tvd_oracle as O
    from paper_1011_5964_b200.harness import CONFIGS, make_problem

    cores = os.cpu_count() or 1
    O.set_workers(cores)
    spec = CONFIGS[args.config]
    h, v, _ = make_problem(spec)
    apply_a, minv, rhs, u = cpu_state(spec, h, v, args.state_fp)
    per_step = args.ref_iters
    for _ in range(args.warmup):
        cpu_sample(apply_a, minv, rhs, u, per_step)
    t = 0.0
    for _ in range(args.steps):
        t += cpu_sample(apply_a, minv, rhs, u, per_step)
    iters = per_step * args.steps
    value = iters / t
    sample = (f"{per_step} PCG loop iterations per step (setup untimed) of config {spec.name} "
              f"({spec.n}^2) at FP state {args.state_fp}, oracle restatement of the reference "
              f"(scipy.fft workers={cores}, numpy elementwise)")
    return {
        "impl": "reference", "metric": metric_for(spec), "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE piecewise-constant generator, PCG64 noise)",
        "config": bench_config(spec, args.state_fp),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "mpix_iter_per_s": value * spec.n ** 2 / 1e6,
    }


# --------------------------------------------------------------------- ours
def alg_bytes_per_launch(cat: str, n: int) -> float:
    """Algorithmic bytes one launch of a kernel category must move."""
    px = float(n) * n
    return {
        "band_rows": 32.0 * px,         # read z, p_old; write p_new, t (fused p = z + beta p)
        "band_cols": 40.0 * px,         # read t, p, a_h, a_v; write q  (+ p.q)
        "trig_cols": 24.0 * px,         # read t, inv_eig; write t'
        "trig_rows": 20.0 * px,         # avg of pass 1 (16 B/px) and pass 3 (24 B/px, reads r)
        "vector": 48.0 * px,            # x / r update (the p update is fused into band_rows)
    }.get(cat, 0.0)


def run_ours(args, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    import paper_1011_5964_b200 as tvd
    from paper_1011_5964_b200 import _native as nat
    from paper_1011_5964_b200.harness import CONFIGS, make_problem

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    spec = CONFIGS[args.config]
    n = spec.n
    bc = tvd.BoundaryCondition(spec.bc)
    h, v, _ = make_problem(spec, index=rank)
    kind = "M" if bc is tvd.BoundaryCondition.ANTI_REFLECTIVE else "R"
    cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=2000)

    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), bc, n, device=dev)
    v_dev = torch.from_numpy(v).to(dev)
    back = hop.apply if bc is tvd.BoundaryCondition.REFLECTIVE else hop.apply_transpose
    rhs = back(v_dev)
    u = v_dev.clone()
    for _ in range(args.state_fp):  # untimed: reach a representative lagged-diffusivity state
        lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
        pre = tvd.assemble_preconditioner(kind, hop, lop, spec.alpha)
        u = tvd.pcg(tvd.NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, u, cfg).solution
    lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
    pre = tvd.assemble_preconditioner(kind, hop, lop, spec.alpha)
    system = tvd.NormalSystem(hop, lop, spec.alpha)

    def step() -> int:
        return tvd.pcg(system, pre.apply_inverse, rhs, u, cfg).iterations

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = nat.launch_count(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    with ClockSampler(local) as clocks:
        e0.record()
        for _ in range(args.steps):
            iters += step()
        e1.record()
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = nat.launch_count(dev) - l0
    elapsed = e0.elapsed_time(e1) / 1e3
    stats = torch.tensor([elapsed, float(iters), float(launches)], dtype=torch.float64, device=dev)
    if world > 1:
        t_max = stats[:1].clone()
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        sums = stats[1:].clone()
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        elapsed, iters, launches = float(t_max[0]), float(sums[0]), float(sums[1])
    value = iters / elapsed

    # ---- live per-kernel timing (CUDA events on the launch stream) for the roofline
    nat.profile(True, dev)
    prof_iters = step()
    prof = nat.profile_read(dev)
    nat.profile(False, dev)
    cats = {k: v for k, v in prof.items() if alg_bytes_per_launch(k, n) > 0}
    dom = max(cats, key=lambda k: cats[k][0])
    ms_tot, cnt = cats[dom]
    achieved = alg_bytes_per_launch(dom, n) / (ms_tot / cnt / 1e3) / 1e9
    peaks = _peaks()
    hbm = float(peaks["hbm_gbs"])
    step_ms = sum(t for t, _ in prof.values())
    kernels = {k: {"ms_total": round(t, 4), "launches": c, "share": round(t / step_ms, 4),
                   "gbs": (round(alg_bytes_per_launch(k, n) / (t / c / 1e3) / 1e9, 1)
                           if alg_bytes_per_launch(k, n) else None)}
               for k, (t, c) in sorted(prof.items(), key=lambda kv: -kv[1][0])}

    # ---- e2e through the public API from pinned host buffers.  Every step copies its inputs
    # (u, rhs) host -> device and its solution device -> host inside the timed region; the
    # copies run on two copy streams, double-buffered, so step s + 1's upload and step s - 1's
    # download overlap step s's compute (as a streaming deployment would run it).
    u_host = u.cpu().pin_memory()
    rhs_host = rhs.cpu().pin_memory()
    outs_host = [torch.empty_like(u_host).pin_memory() for _ in range(2)]
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    dbuf = [(torch.empty_like(u), torch.empty_like(rhs)) for _ in range(2)]
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]

    def upload(k):
        with torch.cuda.stream(h2d):
            h2d.wait_event(comp_done[k % 2])  # step k - 2 has finished with this buffer
            dbuf[k % 2][0].copy_(u_host, non_blocking=True)
            dbuf[k % 2][1].copy_(rhs_host, non_blocking=True)
            h2d_done[k % 2].record(h2d)

    step_ev = []  # compute-stream event at the end of every step (per-step e2e times)

    def run_steps(nsteps: int) -> int:
        step_ev.clear()
        cur = torch.cuda.current_stream(dev)
        for e in comp_done + d2h_done:
            e.record(cur)
        h2d.wait_stream(cur)
        d2h.wait_stream(cur)
        its = 0
        upload(0)
        for k in range(nsteps):
            if k + 1 < nsteps:
                upload(k + 1)
            cur.wait_event(h2d_done[k % 2])
            cur.wait_event(d2h_done[k % 2])  # outs_host[k % 2] drained (its step k - 2)
            ud, rd = dbuf[k % 2]
            l_op = tvd.DiffusionOperator(ud, spec.beta, device=dev)
            # the assembly's checks stay on the device until the solve has synchronised
            p_op = tvd.assemble_preconditioner(kind, hop, l_op, spec.alpha, defer_checks=True)
            res = tvd.pcg(tvd.NormalSystem(hop, l_op, spec.alpha), p_op.apply_inverse, rd, ud,
                          cfg)
            p_op.check()
            comp_done[k % 2].record(cur)
            step_ev.append(torch.cuda.Event(enable_timing=True))
            step_ev[-1].record(cur)
            with torch.cuda.stream(d2h):
                d2h.wait_event(comp_done[k % 2])
                outs_host[k % 2].copy_(res.solution, non_blocking=True)
                res.solution.record_stream(d2h)  # not recycled before the copy has read it
                d2h_done[k % 2].record(d2h)
            its += res.iterations
        cur.wait_stream(h2d)
        cur.wait_stream(d2h)
        return its

    run_steps(4)  # steady state: after 2 warm-up steps the 3rd step ran 0.4-4.8 ms slow
    torch.cuda.synchronize()
    barrier()
    e2e_steps = max(2, min(args.steps, 10))
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    e2e_iters = run_steps(e2e_steps)
    s1.record()
    torch.cuda.synchronize()
    e2e_t = s0.elapsed_time(s1) / 1e3
    e2e_step_ms = [round(s0.elapsed_time(step_ev[0]), 2)] + [
        round(a.elapsed_time(b), 2) for a, b in zip(step_ev, step_ev[1:])]
    if world > 1:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ii = torch.tensor([float(e2e_iters)], dtype=torch.float64, device=dev)
        dist.all_reduce(ii, op=dist.ReduceOp.SUM)
        e2e_t, e2e_iters = float(tt[0]), float(ii[0])
    e2e_value = e2e_iters / e2e_t

    if rank != 0:
        return None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        from oracle import tvd_oracle as O
        cores = os.cpu_count() or 1
        O.set_workers(cores)
        # the same FP state as the timed GPU solves (the GPU's u after state_fp steps)
        apply_a, minv, crhs, cu = cpu_state(spec, h, v, args.state_fp, u.cpu().numpy())
        cpu_sample(apply_a, minv, crhs, cu, 1)  # warm (plans, page-in)
        t = cpu_sample(apply_a, minv, crhs, cu, args.cpu_iters)
        cpu = {"value": args.cpu_iters / t, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{args.cpu_iters} PCG loop iterations (setup untimed) of config "
                         f"{spec.name} ({n}^2) at FP state {args.state_fp}, oracle "
                         f"restatement (scipy.fft workers={cores}); {t:.1f} s"}
    clk = clocks.summary()
    alg_iter = 128.0 * n * n
    line = {
        "metric": metric_for(spec), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE piecewise-constant generator, PCG64 noise)",
        "config": bench_config(spec, args.state_fp),
        "pcg_iters_per_step": iters / (args.steps * world),
        "mpix_iter_per_s": value * n * n / 1e6,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic_per_launch(dom, spec.name, n),
                     "kernel": dom,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs"
                     if not peaks.get("fallback") else "fallback 6650 GB/s"},
        "pcg_roofline": {"alg_bytes_per_iter": alg_iter,
                         "achieved_gbs": alg_iter * value / world / 1e9,
                         "frac": alg_iter * value / world / 1e9 / hbm},
        "kernels": kernels, "profiled_iterations": prof_iters,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * n * n,
                "d2h_bytes_per_step": 8 * n * n, "steps": e2e_steps, "step_ms": e2e_step_ms,
                "includes": "H2D u,rhs; diffusivity; device assembly; PCG; D2H solution "
                            "(copies double-buffered on two copy streams, overlapping the "
                            "neighbouring steps' compute)"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    return line


def _time_region(step, args, world: int, local: int, dev):
    """Warm-up, then K timed steps bracketed by barrier + synchronize, CUDA events on the
    launching stream; returns (elapsed_s max over ranks, local work sum, launches, clocks)."""
    import torch
    import torch.distributed as dist

    from paper_1011_5964_b200 import _native as nat

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = nat.launch_count(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    work = 0
    with ClockSampler(local) as clocks:
        e0.record()
        for _ in range(args.steps):
            work += step()
        e1.record()
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = nat.launch_count(dev) - l0
    elapsed = e0.elapsed_time(e1) / 1e3
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t[0])
    return elapsed, work, launches, clocks.summary()


def _sum_over_ranks(vals, world: int, dev):
    import torch
    import torch.distributed as dist

    if world == 1:
        return [float(v) for v in vals]
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t]


def _profile_kernels(step, n, dev, config: str):
    """Per-category live CUDA-event timing of one step (tvd_ctx_profile) and the dominant
    HBM-streaming category's roofline entry."""
    from paper_1011_5964_b200 import _native as nat

    nat.profile(True, dev)
    work = step()
    prof = nat.profile_read(dev)
    nat.profile(False, dev)
    cats = {k: v for k, v in prof.items() if alg_bytes_per_launch(k, n) > 0}
    dom = max(cats, key=lambda k: cats[k][0])
    ms_tot, cnt = cats[dom]
    achieved = alg_bytes_per_launch(dom, n) / (ms_tot / cnt / 1e3) / 1e9
    step_ms = sum(t for t, _ in prof.values())
    kernels = {k: {"ms_total": round(t, 4), "launches": c, "share": round(t / step_ms, 4),
                   "gbs": (round(alg_bytes_per_launch(k, n) / (t / c / 1e3) / 1e9, 1)
                           if alg_bytes_per_launch(k, n) else None)}
               for k, (t, c) in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    peaks = _peaks()
    hbm = float(peaks["hbm_gbs"])
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic_per_launch(dom, config, n), "kernel": dom,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not peaks.get("fallback")
            else "fallback 6650 GB/s"}
    return roof, kernels, work, hbm


def run_slab(args, rank: int, world: int) -> None:
    """Config 5: one 8192^2 problem.  N = 1: the single-GPU fused PCG.  N > 1: row slabs of
    n / N rows per rank (slab.py): halo exchanges, two all-to-alls per preconditioner solve
    and one 8-byte allgather per dot product over NCCL; strong scaling (fixed total work)."""
    import torch
    import torch.distributed as dist

    import paper_1011_5964_b200 as tvd
    from paper_1011_5964_b200 import slab as SL
    from paper_1011_5964_b200.harness import CONFIGS, make_problem

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    spec = CONFIGS[args.config]
    n = spec.n
    bc = tvd.BoundaryCondition(spec.bc)
    # every rank generates the same seeded problem (the blur of the truth runs on its GPU)
    h, v_np, _ = make_problem(spec, exact=False, device=dev)
    cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=2000)
    hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), bc, n, device=dev)
    v = torch.from_numpy(v_np).to(dev)
    del v_np
    rhs = hop.apply_transpose(v)
    comm = SL.TorchComm() if world > 1 else None

    def operators(u_full):
        lop = tvd.DiffusionOperator(u_full, spec.beta, device=dev)
        pre = tvd.assemble_preconditioner("M", hop, lop, spec.alpha)
        return tvd.NormalSystem(hop, lop, spec.alpha), pre

    layout = SL.SlabLayout(n, world, rank, 1)

    def slab_of(u_slab):
        """This rank's slab solver for the FP state u: diffusivity and assembly of its own
        rows only (slab.slab_operators: a one-row u halo, one all-to-all, a min / max
        allreduce) -- no rank rebuilds the full image's operators."""
        (ops,) = SL.slab_operators(hop, [u_slab], [layout], comm, spec.beta, spec.alpha, "M")
        return SL.Slab.from_operands(hop, spec.alpha, ops, world, rank)

    if world == 1:
        u = v.clone()
        for _ in range(args.state_fp):  # untimed: a representative lagged-diffusivity state
            system, pre = operators(u)
            u = tvd.pcg(system, pre.apply_inverse, rhs, u, cfg).solution
        system, pre = operators(u)

        def step() -> int:
            return tvd.pcg(system, pre.apply_inverse, rhs, u, cfg).iterations
    else:
        b_s = SL.split_rows(rhs, world, rank)
        x_s = SL.split_rows(v, world, rank)
        for _ in range(args.state_fp):
            (o,) = SL.slab_pcg([slab_of(x_s)], comm, [b_s], [x_s], cfg)
            x_s = o.solution
        slab = slab_of(x_s)
        u = None

        def step() -> int:
            (o,) = SL.slab_pcg([slab], comm, [b_s], [x_s], cfg)
            return o.iterations

    elapsed, iters, launches, clk = _time_region(step, args, world, local, dev)
    (launches,) = _sum_over_ranks([launches], world, dev)
    value = iters / elapsed  # iterations of the one global problem (identical on every rank)
    roof, kernels, prof_iters, hbm = _profile_kernels(step, n, dev, spec.name if world == 1 else f"{spec.name}/slab{world}")
    if world > 1:  # per-rank kernels move 1/N of the bytes of a full-size launch
        R = n // world
        for k in kernels.values():
            if k["gbs"]:
                k["gbs"] = round(k["gbs"] * R / n, 1)
        roof["achieved"] *= R / n
        roof["frac"] = roof["achieved"] / hbm

    # e2e: this rank's slabs of (u, rhs) from pinned host memory, the FP-step setup of its
    # rows (u halo, diffusivity, assembly with one all-to-all), the slab solve, D2H of the
    # solution slab
    R = n // world
    u_host = (u if world == 1 else x_s).cpu().pin_memory()
    rhs_host = SL.split_rows(rhs, world, rank).cpu().pin_memory()
    out_host = torch.empty_like(u_host).pin_memory()

    def e2e_step() -> int:
        us = u_host.to(dev, non_blocking=True)
        rs = rhs_host.to(dev, non_blocking=True)
        if world == 1:
            sysm, p_op = operators(us)
            res = tvd.pcg(sysm, p_op.apply_inverse, rs, us, cfg)
            out_host.copy_(res.solution, non_blocking=True)
            return res.iterations
        (o,) = SL.slab_pcg([slab_of(us)], comm, [rs], [us], cfg)
        out_host.copy_(o.solution, non_blocking=True)
        return o.iterations

    e2e_step()
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    e2e_iters = sum(e2e_step() for _ in range(e2e_steps))
    s1.record()
    torch.cuda.synchronize()
    e2e_t = s0.elapsed_time(s1) / 1e3
    if world > 1:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt[0])
    if rank != 0:
        return None
    line = {
        "metric": f"PCG iters/sec at {n}^2 AR fp64 (config {spec.name}, one image, "
                  f"{'row slabs' if world > 1 else 'single GPU'})",
        "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE piecewise-constant generator, PCG64 noise)",
        "config": {**bench_config(spec, args.state_fp), "slab_rows": R,
                   "parallelism": f"row slabs x{world}"},
        "pcg_iters_per_step": iters / args.steps,
        "mpix_iter_per_s": value * n * n / 1e6,
        "roofline": roof,
        "pcg_roofline": {"alg_bytes_per_iter": 128.0 * n * n,
                         "achieved_gbs": 128.0 * n * n * value / world / 1e9,
                         "frac": 128.0 * n * n * value / world / 1e9 / hbm},
        "kernels": kernels, "profiled_iterations": prof_iters,
        "cpu_baseline": None,
        "e2e": {"value": e2e_iters / e2e_t, "unit": UNIT, "h2d_bytes_per_step": 16 * R * n,
                "d2h_bytes_per_step": 8 * R * n, "steps": e2e_steps,
                "includes": "H2D u,rhs slabs; u halo rows; slab diffusivity and assembly "
                            "(one all-to-all); slab PCG; D2H solution slab"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    return line


def run_batch(args, rank: int, world: int) -> None:
    """Config 4: 64 independent 1024^2 problems (Gaussian 21x21 / box 11x11 alternating),
    dealt to the ranks in Gaussian/box pairs (sharding.py); a step is one inner PCG solve of
    every problem of the rank, ``--streams`` host threads each driving its own stream over
    its share.  Strong scaling (fixed 64 problems); no collective on the hot path."""
    from concurrent.futures import ThreadPoolExecutor

    import torch

    import paper_1011_5964_b200 as tvd
    from paper_1011_5964_b200 import _native as nat
    from paper_1011_5964_b200.harness import CONFIGS, make_problem
    from paper_1011_5964_b200.sharding import shard_problems

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    spec = CONFIGS[args.config]
    n = spec.n
    bc = tvd.BoundaryCondition(spec.bc)
    mine = shard_problems(spec.problems, world, rank)
    cfg = tvd.KrylovConfig(tol=spec.tol, max_iterations=2000)
    probs = []
    for i in mine:  # untimed: a representative lagged-diffusivity state per problem
        h, v_np, _ = make_problem(spec, index=i)
        hop = tvd.StructuredBlurOperator(tvd.SymmetricPsf(h), bc, n, device=dev)
        v = torch.from_numpy(v_np).to(dev)
        rhs = hop.apply_transpose(v)
        u = v.clone()
        for _ in range(args.state_fp):
            lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
            pre = tvd.assemble_preconditioner("M", hop, lop, spec.alpha)
            u = tvd.pcg(tvd.NormalSystem(hop, lop, spec.alpha), pre.apply_inverse, rhs, u,
                        cfg).solution
        lop = tvd.DiffusionOperator(u, spec.beta, device=dev)
        pre = tvd.assemble_preconditioner("M", hop, lop, spec.alpha)
        probs.append((tvd.NormalSystem(hop, lop, spec.alpha), pre, rhs, u))
    nstreams = max(1, min(args.streams, len(probs)))
    streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    groups = [probs[k::nstreams] for k in range(nstreams)]
    # persistent workers: each keeps its thread-local native context (stream, plans, scratch)
    pool = ThreadPoolExecutor(max_workers=nstreams)

    def solve_group(k):
        torch.cuda.set_device(local)
        with torch.cuda.stream(streams[k]):
            return sum(tvd.pcg(s, p.apply_inverse, b, x0, cfg).iterations
                       for s, p, b, x0 in groups[k])

    def step() -> int:
        cur = torch.cuda.current_stream(dev)
        for st in streams:
            st.wait_stream(cur)
        its = sum(pool.map(solve_group, range(nstreams)))
        for st in streams:
            cur.wait_stream(st)
        return its

    def solve_all() -> int:  # main thread, one stream (launch counting, kernel profile)
        return sum(tvd.pcg(s, p.apply_inverse, b, x0, cfg).iterations for s, p, b, x0 in probs)

    elapsed, iters, _, clk = _time_region(step, args, world, local, dev)

    # e2e through the public API: every problem's (u, rhs) host -> device from pinned memory
    # and its solution device -> host, on the problem's worker stream; the streams overlap
    # one another's copies with their solves
    hosts = [(x0.cpu().pin_memory(), b.cpu().pin_memory(), torch.empty(x0.shape, dtype=x0.dtype, pin_memory=True))
             for _, _, b, x0 in probs]
    hgroups = [hosts[k::nstreams] for k in range(nstreams)]
    dbufs = [(torch.empty_like(probs[0][3]), torch.empty_like(probs[0][2]))
             for _ in range(nstreams)]

    def e2e_group(k):
        torch.cuda.set_device(local)
        ud, bd = dbufs[k]
        its = 0
        with torch.cuda.stream(streams[k]):
            for (s, p, _, _), (uh, bh, oh) in zip(groups[k], hgroups[k]):
                ud.copy_(uh, non_blocking=True)
                bd.copy_(bh, non_blocking=True)
                res = tvd.pcg(s, p.apply_inverse, bd, ud, cfg)
                oh.copy_(res.solution, non_blocking=True)
                its += res.iterations
        return its

    def e2e_step() -> int:
        cur = torch.cuda.current_stream(dev)
        for st in streams:
            st.wait_stream(cur)
        its = sum(pool.map(e2e_group, range(nstreams)))
        for st in streams:
            cur.wait_stream(st)
        return its

    e2e_args = argparse.Namespace(warmup=1, steps=max(1, min(args.steps, 3)))
    e2e_t, e2e_iters, _, _ = _time_region(e2e_step, e2e_args, world, local, dev)
    (e2e_iters,) = _sum_over_ranks([e2e_iters], world, dev)
    pool.shutdown()
    l0 = nat.launch_count(dev)
    solve_all()
    launches = (nat.launch_count(dev) - l0) * args.steps  # the contexts of the workers
    iters, launches = _sum_over_ranks([iters, launches], world, dev)
    value = iters / elapsed
    roof, kernels, prof_iters, hbm = _profile_kernels(solve_all, n, dev, spec.name)
    if rank != 0:
        return None
    line = {
        "metric": f"PCG iters/sec, batch of {spec.problems} x {n}^2 AR fp64 (config {spec.name})",
        "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE piecewise-constant generator, PCG64 noise)",
        "config": {**bench_config(spec, args.state_fp), "problems_per_gpu": len(mine),
                   "streams": nstreams, "parallelism": f"problem sharding x{world}"},
        "pcg_iters_per_step": iters / args.steps,
        "mpix_iter_per_s": value * n * n / 1e6,
        "roofline": roof,
        "pcg_roofline": {"alg_bytes_per_iter": 128.0 * n * n,
                         "achieved_gbs": 128.0 * n * n * value / world / 1e9,
                         "frac": 128.0 * n * n * value / world / 1e9 / hbm},
        "kernels": kernels, "profiled_iterations": prof_iters,
        "cpu_baseline": None,
        "e2e": {"value": e2e_iters / e2e_t, "unit": UNIT,
                "h2d_bytes_per_step": 16 * n * n * len(mine),
                "d2h_bytes_per_step": 8 * n * n * len(mine), "steps": e2e_args.steps,
                "path": "per problem: pinned H2D of (u, rhs), tvd.pcg, D2H of the solution, "
                        "on the problem's worker stream"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    return line


def traffic_per_launch(category: str, config: str, n: int):
    """DRAM bytes (read + write) per launch of the category's kernel for this workload, from
    the newest committed ``ncu --set full`` capture summarised in a ``profiles/**/traffic.json``
    (``{"config": ..., "n": ..., "kernels": {category: {"dram_bytes": ...}}}``; the round-1
    files without the keys are c3 / 2048 captures); None when no capture of this config and
    size exists."""
    import glob
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    paths = glob.glob(os.path.join(root, "**", "traffic.json"), recursive=True)
    # newest round first (profiles/rNN/...), deeper (later) captures of a round first
    paths.sort(key=lambda p: (os.path.relpath(p, root).split(os.sep)[0], p.count(os.sep)),
               reverse=True)
    for path in paths:
        try:
            doc = json.load(open(path))
        except (OSError, ValueError):
            continue
        if "kernels" in doc:
            cfg, size, table = doc.get("config"), doc.get("n"), doc["kernels"]
        else:
            cfg, size, table = "c3", 2048, doc
        if cfg != config or size != n:
            continue
        ent = table.get(category)
        if ent:
            return ent["dram_bytes"]
    return None


def launch_ranks(args) -> int:
    """``--gpus N`` without a torchrun environment: re-run this script under
    ``torch.distributed.run`` with N local ranks (127.0.0.1 rendezvous), NCCL's INFO log on
    stderr so the communicator's N ranks are visible.  Returns the launcher's exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def launch_check(rank: int, world: int):
    """``--launch-check``: the process group forms with ``world`` ranks (NCCL on GPUs, gloo
    on a CPU-only host) and every rank takes part in one all-reduce."""
    import torch
    import torch.distributed as dist

    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if world > 1:
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend)
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))) \
        if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t)
        dist.destroy_process_group()
    if rank == 0:
        return {"launch_check": True, "n_gpus": world, "backend": backend,
                "rank_sum": float(t[0])}
    return None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--state-fp", type=int, default=2)
    ap.add_argument("--cpu-iters", type=int, default=6)
    ap.add_argument("--ref-iters", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=4, help="c4: host threads / CUDA streams")
    ap.add_argument("--extra", default="auto",
                    help="extra workloads measured after the main one and attached under "
                         "'extra' (comma list of c4 / c5, 'none'); auto = c4 at N > 1")
    ap.add_argument("--launch-check", action="store_true",
                    help="only form the N-rank process group and all-reduce once")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.launch_check:
        line = launch_check(rank, world)
        if line:
            print(json.dumps(line), flush=True)
        return
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    runners = {"c5": run_slab, "c4": run_batch}
    try:
        line = runners.get(args.config, run_ours)(args, rank, world)
        extra = ([] if args.extra == "none" else
                 (["c4"] if world > 1 and args.config == "c3" else [])
                 if args.extra == "auto" else [e for e in args.extra.split(",") if e])
        for cfg in extra:
            sub = argparse.Namespace(**{**vars(args), "config": cfg, "no_cpu_baseline": True})
            out = runners.get(cfg, run_ours)(sub, rank, world)
            if line is not None and out is not None:
                line.setdefault("extra", {})[cfg] = {
                    k: out[k] for k in ("metric", "value", "unit", "scaling", "ms_per_step",
                                        "config", "pcg_iters_per_step", "roofline",
                                        "pcg_roofline", "e2e", "gpu_launches") if k in out}
        if line is not None:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
