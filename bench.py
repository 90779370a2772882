#!/usr/bin/env python
"""Benchmark of the B200 GADI hot path (contract: see DESIGN.md "Measurement").

Metric (BASELINE.json): GADI solve time in seconds to fp64 accuracy at
n ~ 1.3e8 -- cd3d 512^3 (n = 134,217,728), bf16 inner solves, u = u_r = fp64,
stopping at relres <= outer_tol (fp64-level backward error).  A step is one
complete ``gadi_solve`` (||A||_2 power iteration included, as in the
reference's gadi_solve) on inputs resident in HBM; ``e2e`` is the same solve
through the public API from host buffers (H2D of b, D2H of x inside the
timed region).  Lower is better.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Inner-solver arithmetic: the storage model (``--rounding storage``, default):
bf16 storage with fp32 compute, the paper's GPU design.
The reference package's per-operation bf16 emulation is the other mode
(``gadi_solve(..., rounding="reference")``, bitwise the reference wherever
the reference runs, tests/test_gpu_reference_fused.py); at this size its bf16
partial sums cannot resolve the H-system and the solve diverges -- the line
reports that run too (``reference_rounding_solve``).

N > 1: the grid is slab-partitioned along its slowest axis, one slab per GPU,
NCCL halo exchanges and rank-ordered scalar all-gathers (strong scaling: the
same n = 512^3 system at every N); the time is the max over ranks of the
device-timed solve.  ``--gpus N`` without torchrun re-launches this script
under ``torch.distributed.run`` with N ranks.

The fp64 comparison (north star: >= 2x over the same code in full fp64) runs
by default: the same code with u_s = fp64 (a) on the bf16 run's splitting
(precision alone), (b) at fp64's own best (alpha, inner_tol) from the GPU sweep
(profiles/fp64_sweep_r2.jsonl).

``--impl reference`` times the CPU oracle port (oracle/gadi_oracle.py, the
reference's algorithm restated in numpy; the reference itself is pure Python
and cannot hold n = 512^3) on bounded samples of the same workload on the
host cores and extrapolates to the solve's measured iteration counts; a
measured full CPU solve at 32^3 calibrates the extrapolation model.
"""

from __future__ import annotations

import os

# BLAS threads of numpy (the CPU baseline's np.dot / norms; elementwise numpy
# is single-threaded): the same setting in both arms, before numpy loads
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
# slab ranks on the peer transport spin on device flags: load every kernel at
# context creation (a lazily loaded kernel's first launch can wait for the
# device while a collective kernel spins)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import argparse  # noqa: E402
import json  # noqa: E402
import socket  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import tempfile  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GADI solve time (s) to fp64 accuracy, n~1.3e8; SpMV/inner HBM GB/s vs peak"
UNIT = "s"
# iteration counts of the benchmark workload measured on B200 (bench.py run,
# profiles/); the reference arm extrapolates its per-iteration CPU costs with
# them.  Updated from the last GPU measurement.
COUNTS_FILE = ROOT / "profiles" / "bench_counts.json"
# fp64's own best (alpha, inner_tol) at 512^3 from scripts/fp64_sweep.py
FP64_BEST = {"alpha": 0.0015, "inner_tol": 1e-2}  # 56 s, 699 outer (profiles/fp64_sweep_r2.jsonl)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--family", default="cd3d")
    ap.add_argument("--ng", type=int, default=512)
    ap.add_argument("--alpha", type=float, default=0.0125)
    ap.add_argument("--us", default="bf16")
    ap.add_argument("--outer-tol", type=float, default=1e-12)
    ap.add_argument("--inner-tol", type=float, default=1e-2)
    ap.add_argument("--outer-maxit", type=int, default=2000)
    ap.add_argument("--rounding", choices=["storage", "reference"], default="storage",
                    help="inner-solver arithmetic (gadi_solve rounding=): the storage model or the reference's "
                         "per-operation rounding in the fused passes")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-ng", type=int, default=128, help="grid of the bounded CPU sample")
    ap.add_argument("--fp64", type=int, default=1, help="time the fp64 comparison solves (north star >= 2x)")
    ap.add_argument("--ref-rounding", type=int, default=1,
                    help="also run the solve with the reference's per-operation rounding (reported, not timed "
                         "against the headline)")
    ap.add_argument("--report-dir", default=str(ROOT / "gpurun_out" / "bench_report"),
                    help="where the reference CLI's summary.csv / trace JSONL are written (report.py)")
    return ap.parse_args()


def workload(a):
    return {"workload": f"{a.family} {a.ng}^{3 if a.family == 'cd3d' else 2}, u_s={a.us} inner, u=u_r=fp64",
            "family": a.family, "n_g": a.ng, "n": a.ng ** 3 if a.family == "cd3d" else a.ng ** 2,
            "alpha": a.alpha, "omega": 1.0, "u_s": a.us, "u": "fp64", "u_r": "fp64",
            "outer_tol": a.outer_tol, "inner_tol": a.inner_tol, "strict_model": False,
            "rounding": a.rounding,
            "arithmetic": ("storage model: u_s storage, fp32 compute, fp64 dot accumulation (PAPER.md:1180-1199)"
                           if a.rounding == "storage" else "the reference's per-operation u_s rounding emulation"),
            "l2_policy": "inputs larger than L2 (fp64 vectors 1 GiB >> 126 MB L2)",
            "rhs": "b = A 1 generated in HBM (manufactured solution x* = 1)"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU sample
def cpu_threads():
    return int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))


def cpu_units(a, ng, us):
    """Per-unit CPU costs of the oracle (the reference's algorithm) on a
    cd3d(ng) problem: one H-CG iteration, one CGNR iteration (u_s emulated, or
    fp64), one outer pass (update + residual + monitor), one power iteration."""
    from oracle import gadi_oracle as O

    op = O.build(a.family, ng)
    n = op.n
    H, S, ST = O.splitting(op, a.alpha, us)
    rng = np.random.default_rng(0)
    r = O.q(rng.standard_normal(n) * 1e-3, us)
    b = O.rhs_ones(op)

    def per(fn, reps=1):
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return (time.perf_counter() - t0) / reps

    t_h = per(lambda: O.cg_spd(H, r, 0.0, 2, us, False)) / 2
    t_s = per(lambda: O.cg_normal_skew(S, ST, r, 0.0, 2, us, False)) / 2
    x = np.ones(n)
    t_o = per(lambda: (O.stencil_residual(op, x, b), b - O.stencil_apply(op, x), O.stencil_apply(op, x - 1.0)))
    t_n = per(lambda: O.stencil_apply(op, O.stencil_apply(op, x)))
    return {"n": n, "h_it": t_h, "s_it": t_s, "outer": t_o, "power_it": t_n}


def extrapolate(units, counts):
    scale = counts["n"] / units["n"]
    return scale * (counts["outer"] * units["outer"] + counts["inner_h"] * units["h_it"]
                    + counts["inner_s"] * units["s_it"] + counts["norm_iters"] * units["power_it"])


def cpu_sample(a, counts):
    """(extrapolated seconds, detail, units) of the bounded sample."""
    u = cpu_units(a, a.cpu_ng, a.us)
    est = extrapolate(u, counts)
    detail = (f"oracle port (numpy restatement of gadimp) on {a.family} {a.cpu_ng}^3 (n={u['n']}): "
              f"{u['h_it']:.3f} s/H-CG it, {u['s_it']:.3f} s/CGNR it, {u['outer']:.3f} s/outer pass, "
              f"{u['power_it']:.3f} s/power it (emulated {a.us} inner arithmetic, fp64 outer), scaled "
              f"x{counts['n'] / u['n']:.0f} per unknown and extrapolated to the B200 solve's {counts['outer']} outer "
              f"/ {counts['inner_h']} H / {counts['inner_s']} S / {counts['norm_iters']} power iterations; "
              f"{cpu_threads()} BLAS threads (elementwise numpy single-threaded)")
    return est, detail, u


def cpu_calibration(a):
    """A real, measured full CPU solve (oracle port, bench parameters) at
    32^3 for 20 outer steps vs the extrapolation model's prediction for it."""
    from oracle import gadi_oracle as O

    ng, steps = 32, 20
    op = O.build(a.family, ng)
    b = O.rhs_ones(op)
    out = {}
    for us in (a.us, "fp64"):
        t0 = time.perf_counter()
        rep = O.gadi_solve(op, b, a.alpha, u_s=us, outer_tol=a.outer_tol, outer_maxit=steps,
                           inner_tol=a.inner_tol, strict=False, exact=np.ones(op.n))
        wall = time.perf_counter() - t0
        c = {"n": op.n, "outer": len(rep.history), "inner_h": sum(h.inner_h for h in rep.history),
             "inner_s": sum(h.inner_s for h in rep.history), "norm_iters": 0}
        u = cpu_units(a, ng, us)
        # the measured run includes ||A||_2 (power iteration count not exposed by
        # the port: compare without it, i.e. measured minus one matrix_norm_2)
        t1 = time.perf_counter()
        O.matrix_norm_2(op)
        t_norm = time.perf_counter() - t1
        pred = extrapolate(u, c)
        out[us] = {"n_g": ng, "outer_steps": c["outer"], "inner_h": c["inner_h"], "inner_s": c["inner_s"],
                   "measured_s": round(wall - t_norm, 3), "predicted_s": round(pred, 3),
                   "measured_over_predicted": round((wall - t_norm) / pred, 3) if pred > 0 else None,
                   "status": rep.status}
    return out


def load_counts(a):
    if COUNTS_FILE.exists():
        c = json.loads(COUNTS_FILE.read_text())
        key = f"{a.family}_{a.ng}_{a.us}_{a.alpha}_{a.outer_tol}_{a.inner_tol}"
        if key in c:
            return c[key]
    return None


def save_counts(a, counts):
    c = json.loads(COUNTS_FILE.read_text()) if COUNTS_FILE.exists() else {}
    c[f"{a.family}_{a.ng}_{a.us}_{a.alpha}_{a.outer_tol}_{a.inner_tol}"] = counts
    COUNTS_FILE.parent.mkdir(parents=True, exist_ok=True)
    COUNTS_FILE.write_text(json.dumps(c, indent=1))


# ---------------------------------------------------------------- roofline
def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel):
    """Per-launch DRAM bytes of `kernel` from the committed ncu capture summary."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None
    d = json.loads(f.read_text())
    return d.get(kernel, {}).get("dram_bytes_per_launch")


def ssz(us):
    return {"bf16": 2, "fp16": 2, "fp32": 4, "fp64": 8}[us]


# ---------------------------------------------------------------- ours
class Timer:
    def __init__(self):
        self.ms = None

    def on_start(self, ctx):
        ctx.timer_start()

    def on_end(self, ctx):
        self.ms = ctx.timer_stop()


def run_ours(a, rank, world):
    import paper_2512_21164_b200 as g
    from paper_2512_21164_b200 import _lib, report

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    build = {"cd3d": g.build_cd_3d, "cdr2d": g.build_cdr_2d, "crd": g.build_complex_rd}[a.family]
    cfg = g.GadiConfig(alpha=a.alpha, u_s=a.us, outer_tol=a.outer_tol, inner_tol=a.inner_tol,
                       outer_maxit=a.outer_maxit, strict_model=False)
    comm = g.SlabComm.from_torch(device=dev) if world > 1 else None

    def solve(timer=None, problem=None, return_x=False, c=cfg, splitting=None, rounding=a.rounding):
        p = problem if problem is not None else build(a.ng)
        return g.gadi_solve(p, splitting, c, device=dev, return_x=return_x, hooks=timer, comm=comm,
                            rounding=rounding)

    for _ in range(a.warmup):
        solve()
    ctx = next(iter(g.device._CACHE.values()))
    dist_barrier(world)
    clocks = ClockSampler(dev)
    clocks.start()
    times, reps = [], []
    launches0 = ctx.kernel_launches()
    for _ in range(a.steps):
        t = Timer()
        rep = solve(t)
        times.append(t.ms / 1e3)
        reps.append(rep)
    launches = ctx.kernel_launches() - launches0
    clk = clocks.stop()
    dist_barrier(world)
    t_solve = dist_max(float(np.mean(times)), world)
    # per-kernel device timers: one more solve with an event pair around every
    # launch (this turns the inner loops' CUDA graphs off, so it is not timed)
    ctx.prof_enable(True)
    solve()
    prof = ctx.prof_read()
    ctx.prof_enable(False)

    rep = reps[-1]
    n = (a.ng ** 3 if a.family == "cd3d" else a.ng ** 2) * (2 if a.family == "crd" else 1)
    rep_n = ctx.n  # unknowns of this rank's slab (= n on one GPU)
    counts = {"n": n, "outer": rep.iterations,
              "inner_h": sum(h.inner_h_iterations for h in rep.history),
              "inner_s": sum(h.inner_s_iterations for h in rep.history),
              "norm_iters": rep.norm_iterations,
              "status": rep.status, "relres": rep.history[-1].relative_residual,
              "berr": rep.history[-1].backward_error, "ferr": rep.history[-1].forward_error}
    if rank == 0 and world == 1 and a.rounding == "storage":
        save_counts(a, counts)

    # roofline of the dominant kernel (H-CG pass B: reads p (haloed), z, r;
    # writes z, r -> 5 u_s values per unknown) and of the full H-CG iteration
    peak, peak_src = load_peaks()
    s = ssz(a.us)
    # Per-kernel averages over the launches that did work: the inner loops
    # enqueue a predicted number of iterations and the launches past
    # convergence exit at once, so the raw launch count overstates the work;
    # dividing each kernel's total device time (no-op launches included) by
    # the iterations actually run gives a conservative time per real launch.
    real = {"hcg_init": counts["outer"], "hcg_a": counts["inner_h"], "hcg_b": counts["inner_h"],
            "cgnr_init": counts["outer"], "cgnr_p1": counts["inner_s"], "cgnr_p2": counts["inner_s"],
            # the last iteration of every S-solve stops at P2's relres test
            "cgnr_p3": max(1, counts["inner_s"] - counts["outer"]), "outer": counts["outer"] + 1,
            "norm_b": counts["norm_iters"], "norm_a": counts["norm_iters"]}
    kt = {k: (ms / max(1, min(cnt, real.get(k, cnt))), cnt, ms) for k, (ms, cnt) in prof.items()}
    total_kernel_ms = sum(v[2] for v in kt.values())
    dom = max(kt, key=lambda k: kt[k][2])
    alg = {"hcg_a": 3 * s, "hcg_b": 5 * s, "cgnr_p1": 3 * s, "cgnr_p2": 5 * s, "cgnr_p3": 2 * s,
           "outer": 4 * 8 + s, "norm_a": 16, "norm_b": 16, "hcg_init": 8 + 2 * s, "cgnr_init": 4 * s}
    kernels = {}
    for k, (avg_ms, cnt, tot) in kt.items():
        bpl = alg.get(k, 0) * rep_n
        kernels[k] = {"launches": cnt, "active_launches": min(cnt, real.get(k, cnt)),
                      "avg_us": round(avg_ms * 1e3, 2), "share": round(tot / total_kernel_ms, 4),
                      "alg_bytes_per_launch": bpl,
                      "achieved_gbs": round(bpl / (avg_ms * 1e-3) / 1e9, 1) if bpl else None}
    d_avg = kt[dom][0]
    d_bytes = alg.get(dom, 0) * rep_n
    achieved = d_bytes / (d_avg * 1e-3) / 1e9
    roofline = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(dom), "peak_source": peak_src,
                "alg_bytes_per_unit": alg.get(dom, 0), "units_per_launch": rep_n}
    if "hcg_a" in kt and "hcg_b" in kt:
        it_us = (kt["hcg_a"][0] + kt["hcg_b"][0]) * 1e3
        roofline["hcg_iteration"] = {"us": round(it_us, 2), "alg_bytes": 8 * s * rep_n,
                                     "achieved": round(8 * s * rep_n / (it_us * 1e-6) / 1e9, 1),
                                     "frac": round(8 * s * rep_n / (it_us * 1e-6) / 1e9 / peak, 4)}

    # end to end through the public API from host buffers: b in (H2D), x out
    # (D2H) inside the timed region, one untimed warm-up, then K timed runs
    e2e = None
    if not a.no_e2e:
        p = build(a.ng)
        b_host = np.ascontiguousarray(p.b)  # materialise b on the host (input preparation, untimed)
        ev = []
        last = None
        for i in range(a.steps + 1):
            p = build(a.ng)
            p.b = b_host
            dist_barrier(world)
            t0 = time.perf_counter()
            last = solve(problem=p, return_x=True)
            dt = time.perf_counter() - t0
            assert last.x is not None and last.x.shape == (rep_n,)
            if i > 0:
                ev.append(dist_max(dt, world))
        e2e = {"value": round(float(np.mean(ev)), 4), "unit": UNIT, "runs": [round(v, 4) for v in ev],
               "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n + 48 * last.iterations * world,
               "status": last.status, "outer": last.iterations,
               "path": "gadi_solve(problem with host b) -> H2D of b, D2H of x per rank's slab"}
        if rank == 0:
            # the reference CLI's bench outputs (REF/cli.py:320-342) for this run
            out = Path(a.report_dir)
            out.mkdir(parents=True, exist_ok=True)
            report.append_summary(out / "summary.csv", p, cfg, last, float(np.mean(ev)), 0,
                                  gpu={"n_gpus": world, "device_time_s": t_solve,
                                       "achieved_gbs": roofline["achieved"], "roofline_frac": roofline["frac"]})
            report.write_trace(out / f"{p.label}_ng{a.ng}_{a.us}_trace.jsonl", last)

    # the north star's ">= 2x over the same code in full fp64"
    fp64 = None
    if a.fp64 and a.us != "fp64":
        fp64 = {}
        sp = g.make_hss_splitting(build(a.ng).A, a.alpha, a.us)
        runs = {"bf16_splitting": (g.GadiConfig(alpha=a.alpha, u_s="fp64", outer_tol=a.outer_tol,
                                                inner_tol=a.inner_tol, outer_maxit=a.outer_maxit,
                                                strict_model=False), sp),
                "own_best": (g.GadiConfig(alpha=FP64_BEST["alpha"], u_s="fp64", outer_tol=a.outer_tol,
                                          inner_tol=FP64_BEST["inner_tol"], outer_maxit=a.outer_maxit,
                                          strict_model=False), None)}
        # fp64 kernels loaded on a small grid (the full-size contexts are built
        # outside the device timer: hooks start after context creation)
        g.gadi_solve(build(min(a.ng, 64)), cfg=runs["own_best"][0], device=dev, return_x=False, rounding="storage",
                     comm=comm)
        for tag, (c64, spl) in runs.items():
            dist_barrier(world)
            t = Timer()
            r64 = solve(timer=t, c=c64, splitting=spl, rounding="storage")
            t64 = dist_max(t.ms / 1e3, world)
            fp64[tag] = {"value": round(t64, 4), "unit": UNIT, "alpha": c64.alpha, "inner_tol": c64.inner_tol,
                         "coef_fmt": spl.u_s.name if spl is not None else "fp64",
                         "status": r64.status, "outer": r64.iterations,
                         "inner_h": sum(h.inner_h_iterations for h in r64.history),
                         "inner_s": sum(h.inner_s_iterations for h in r64.history),
                         "relres": r64.history[-1].relative_residual, "berr": r64.history[-1].backward_error,
                         "speedup_of_bf16": round(t64 / t_solve, 3)}

    # the reference's own arithmetic at this size (reported: it diverges)
    ref_round = None
    if a.ref_rounding and a.rounding == "storage" and world == 1:
        t = Timer()
        rr = solve(timer=t, rounding="reference")
        ref_round = {"s": round(t.ms / 1e3, 3), "status": rr.status, "outer": rr.iterations,
                     "relres": [h.relative_residual for h in rr.history],
                     "inner_h": [h.inner_h_iterations for h in rr.history],
                     "note": "gadi_solve(rounding='reference'): the reference's per-operation bf16 emulation "
                             "(bitwise the reference at 32^3-128^3, tests/golden/headline_*.json)"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:  # the CPU baseline: rank 0 at N = 1 only
        est, detail, _ = cpu_sample(a, counts)
        cpu = {"value": round(est, 2), "unit": UNIT, "cores": cpu_threads(), "kind": "port", "sample": detail,
               "extrapolated": True}

    line = {"metric": METRIC, "value": round(t_solve, 4), "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(t_solve * 1e3, 2), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": a.us + " inner / fp64 outer",
            "data": "synthetic (manufactured solution b = A 1, generated on device)",
            "config": {**workload(a), "parallelism": f"slab x{world} (NCCL halo + all-gather)" if world > 1
                       else "single GPU"},
            "e2e": e2e, "gpu_launches": int(launches // max(1, a.steps)),
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
            "solve": {k: counts[k] for k in ("status", "outer", "inner_h", "inner_s", "norm_iters", "relres",
                                              "berr", "ferr")},
            "kernels": kernels, "fp64_inner_solve": fp64, "reference_rounding_solve": ref_round,
            "lib": _lib.load().gadi_build_info().decode()}
    if rank == 0:
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- reference arm
def run_reference(a, rank, world):
    """The reference's algorithm on the host cores (rank 0 only): the oracle
    port timed on bounded samples of the workload (one H-CG iteration, one
    CGNR iteration, one outer pass, one power iteration at cd3d cpu_ng^3 per
    step, after W warm-up samples), extrapolated per unknown to n = 512^3 and
    to the B200 solve's iteration counts; plus a measured full solve at 32^3
    that calibrates the model.  The reference itself (pure Python) cannot hold
    the 512^3 CSR (~100 GB) and is not on the GPU box."""
    if rank != 0:
        return
    counts = load_counts(a)
    if counts is None:
        print(json.dumps({"impl": "reference", "unavailable": f"no measured B200 iteration counts for this workload "
                                                              f"in {COUNTS_FILE.name}"}), flush=True)
        return
    for _ in range(a.warmup):
        cpu_units(a, a.cpu_ng, a.us)
    vals, detail, units = [], "", None
    t0 = time.perf_counter()
    for _ in range(max(1, a.steps)):
        est, detail, units = cpu_sample(a, counts)
        vals.append(est)
    wall_steps = time.perf_counter() - t0
    v = float(np.mean(vals))
    u64 = cpu_units(a, a.cpu_ng, "fp64")
    calib = cpu_calibration(a)
    line = {"metric": METRIC, "value": round(v, 2), "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(v * 1e3, 1), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": a.us + " inner (emulated) / fp64 outer", "data": "synthetic",
            "config": {**workload(a), "parallelism": "host CPU"}, "impl": "reference",
            "extrapolated": True,
            "extrapolation": {"per_unit_s": {k: round(units[k], 5) for k in ("h_it", "s_it", "outer", "power_it")},
                              "sample_n": units["n"], "target_n": counts["n"], "scale": counts["n"] / units["n"],
                              "counts": {k: counts[k] for k in ("outer", "inner_h", "inner_s", "norm_iters")},
                              "counts_source": counts.get("source", str(COUNTS_FILE.name)),
                              "sample_wall_s_per_step": round(wall_steps / max(1, a.steps), 3),
                              "fp64_per_unit_s": {k: round(u64[k], 5) for k in ("h_it", "s_it", "outer",
                                                                                "power_it")},
                              "fp64_same_counts_s": round(extrapolate(u64, counts), 1)},
            "calibration_full_solves": calib,
            "cpu_baseline": {"value": round(v, 2), "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                             "sample": detail, "extrapolated": True},
            "e2e": {"value": round(v, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- dist
_DIST = {"pg": False}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
        _DIST["pg"] = True
    return rank, world


def dist_barrier(world):
    if world > 1 and _DIST["pg"]:
        import torch.distributed as dist

        dist.barrier()


def dist_max(v, world):
    if world > 1 and _DIST["pg"]:
        import torch
        import torch.distributed as dist

        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return v


def relaunch(n):
    """--gpus N outside torchrun: run this script under torch.distributed.run
    with N ranks on 127.0.0.1 and return its exit code."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = parse()
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        raise SystemExit(relaunch(a.gpus))
    rank, world = dist_init()
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    if a.impl == "reference":
        run_reference(a, rank, world)
    else:
        run_ours(a, rank, world)
    if world > 1 and _DIST["pg"]:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
