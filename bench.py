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

N > 1 (torchrun): the grid is slab-partitioned along its slowest axis, one
slab per GPU, with NCCL halo exchanges and rank-ordered scalar all-gathers
(strong scaling: the same n = 512^3 system at every N); the reported time is
the max over ranks of the device-timed solve.  ``--compare-fp64 1`` also
times the same solve with fp64 inner arithmetic (the north-star ">= 2x over
the same code in full fp64"; minutes long, so off by default).  ``--impl reference``
times the CPU oracle port (oracle/gadi_oracle.py, the reference's algorithm
restated in numpy) on bounded samples of the same workload and extrapolates
to the solve's iteration counts.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GADI solve time (s) to fp64 accuracy, n~1.3e8; SpMV/inner HBM GB/s vs peak"
UNIT = "s"
# iteration counts of the benchmark workload measured on B200 (bench.py run,
# profiles/); the reference arm extrapolates its per-iteration CPU costs with
# them.  Updated from the last GPU measurement.
COUNTS_FILE = ROOT / "profiles" / "bench_counts.json"


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
    ap.add_argument("--compare-fp64", type=int, default=0,
                    help="also time the same solve with fp64 inner solves (slow: at this workload the fp64 "
                         "inner solves do not reach the tolerance within outer_maxit, see DESIGN.md)")
    return ap.parse_args()


def workload(a):
    return {"workload": f"{a.family} {a.ng}^{3 if a.family == 'cd3d' else 2}, u_s={a.us} inner, u=u_r=fp64",
            "family": a.family, "n_g": a.ng, "n": a.ng ** 3 if a.family == "cd3d" else a.ng ** 2,
            "alpha": a.alpha, "omega": 1.0, "u_s": a.us, "u": "fp64", "u_r": "fp64",
            "outer_tol": a.outer_tol, "inner_tol": a.inner_tol, "strict_model": False,
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
def cpu_sample(a, counts, threads_note=""):
    """Time the oracle (the reference's algorithm) per unit of work on a
    bounded cd3d(cpu_ng) problem, scale per unknown to the benchmark grid, and
    extrapolate with the solve's iteration counts.  Returns (seconds, detail)."""
    from oracle import gadi_oracle as O

    ng = a.cpu_ng
    op = O.build(a.family, ng)
    n = op.n
    H, S, ST = O.splitting(op, a.alpha, a.us)
    rng = np.random.default_rng(0)
    r = O.q(rng.standard_normal(n) * 1e-3, a.us)
    b = O.rhs_ones(op)

    def per(fn, reps):
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return (time.perf_counter() - t0) / reps

    t_h = per(lambda: O.cg_spd(H, r, 0.0, 2, a.us, True), 1) / 2        # per CG iteration (emulated u_s)
    t_s = per(lambda: O.cg_normal_skew(S, ST, r, 0.0, 2, a.us, True), 1) / 2
    x = np.ones(n)
    t_o = per(lambda: (O.stencil_residual(op, x, b), b - O.stencil_apply(op, x),
                       O.stencil_apply(op, x - 1.0)), 1)               # residual + monitor
    t_n = per(lambda: O.stencil_apply(op, O.stencil_apply(op, x)), 1)   # one power iteration
    scale = counts["n"] / n
    est = scale * (counts["outer"] * t_o + counts["inner_h"] * t_h + counts["inner_s"] * t_s
                   + counts["norm_iters"] * t_n)
    detail = (f"oracle port (numpy restatement of gadimp) on {a.family} {ng}^3 (n={n}): "
              f"{t_h:.3f} s/H-CG it, {t_s:.3f} s/CGNR it, {t_o:.3f} s/outer pass, {t_n:.3f} s/power it "
              f"(emulated {a.us} inner arithmetic, fp64 outer), scaled x{scale:.0f} per unknown and "
              f"extrapolated to {counts['outer']} outer / {counts['inner_h']} H / {counts['inner_s']} S / "
              f"{counts['norm_iters']} power iterations{threads_note}")
    return est, detail


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
    from paper_2512_21164_b200 import _lib

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    build = {"cd3d": g.build_cd_3d, "cdr2d": g.build_cdr_2d, "crd": g.build_complex_rd}[a.family]
    cfg = g.GadiConfig(alpha=a.alpha, u_s=a.us, outer_tol=a.outer_tol, inner_tol=a.inner_tol,
                       outer_maxit=a.outer_maxit, strict_model=False)
    comm = g.SlabComm.from_torch(device=dev) if world > 1 else None

    def solve(timer=None, problem=None, return_x=False, c=cfg):
        p = problem if problem is not None else build(a.ng)
        return g.gadi_solve(p, cfg=c, device=dev, return_x=return_x, hooks=timer, comm=comm, rounding=a.rounding)

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
    if rank == 0:
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
            "cgnr_p3": max(1, counts["inner_s"] - counts["outer"]), "outer": counts["outer"] + 1, "norm_b": counts["norm_iters"],
            "norm_a": counts["norm_iters"]}
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

    # end to end through the public API from host buffers
    e2e = None
    if not a.no_e2e:
        p = build(a.ng)
        b_host = np.ascontiguousarray(p.b)  # materialise b on the host (input preparation, untimed)
        p.b = b_host
        dist_barrier(world)
        t0 = time.perf_counter()
        r2 = solve(problem=p, return_x=True)
        t_e2e = time.perf_counter() - t0
        assert r2.x is not None and r2.x.shape == (rep_n,)
        t_e2e = dist_max(t_e2e, world)
        e2e = {"value": round(t_e2e, 4), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 8 * n + 48 * r2.iterations * world,
               "status": r2.status, "outer": r2.iterations,
               "path": "gadi_solve(problem with host b) -> H2D of b, D2H of x per rank's slab"}

    # the same solve with fp64 inner arithmetic (north star: >= 2x over full fp64)
    fp64 = None
    if a.compare_fp64 and a.us != "fp64":
        c64 = g.GadiConfig(alpha=a.alpha, u_s="fp64", outer_tol=a.outer_tol, inner_tol=a.inner_tol,
                           outer_maxit=a.outer_maxit, strict_model=False)
        solve(c=c64)  # warm-up (context + kernels)
        dist_barrier(world)
        t = Timer()
        r64 = solve(timer=t, c=c64)
        t64 = dist_max(t.ms / 1e3, world)
        fp64 = {"value": round(t64, 4), "unit": UNIT, "status": r64.status, "outer": r64.iterations,
                "inner_h": sum(h.inner_h_iterations for h in r64.history),
                "inner_s": sum(h.inner_s_iterations for h in r64.history),
                "berr": r64.history[-1].backward_error, "speedup_vs_fp64": round(t64 / t_solve, 3)}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:  # the CPU baseline: rank 0 at N = 1 only
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        est, detail = cpu_sample(a, counts, "; 1 thread")
        cpu = {"value": round(est, 2), "unit": UNIT, "cores": 1, "kind": "port", "sample": detail}

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
            "kernels": kernels, "fp64_inner_solve": fp64, "lib": _lib.load().gadi_build_info().decode()}
    if rank == 0:
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- reference arm
def run_reference(a, rank, world):
    if rank != 0:
        return
    counts = load_counts(a)
    if counts is None:
        # counts of the same workload measured on the GPU are needed to
        # extrapolate the CPU sample; fall back to the documented ones
        counts = {"n": a.ng ** 3, "outer": 60, "inner_h": 6000, "inner_s": 200, "norm_iters": 500}
    vals = []
    detail = ""
    for _ in range(a.warmup if a.warmup < 1 else 0):
        pass
    for _ in range(max(1, a.steps)):
        est, detail = cpu_sample(a, counts, f"; numpy elementwise single-threaded, BLAS {os.cpu_count()} threads")
        vals.append(est)
    v = float(np.mean(vals))
    line = {"metric": METRIC, "value": round(v, 2), "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(v * 1e3, 1), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": a.us + " inner (emulated) / fp64 outer", "data": "synthetic",
            "config": {**workload(a), "parallelism": "host CPU"}, "impl": "reference",
            "cpu_baseline": {"value": round(v, 2), "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                             "sample": detail},
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


def main():
    a = parse()
    rank, world = dist_init()
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
