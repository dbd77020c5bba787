#!/usr/bin/env python
"""Benchmark of the MAID hot path on B200 (contract: see README / DESIGN.md).

Workload (BASELINE.json configs[1], "c2"): 256x256x1 float64 image, 9x9
stencil, smoothed TV (nu 1e-4, alpha 0.6), adaptive AGD with gradient
restart, 1,200 lower iterations per solve (eps tiny so the budget is used).
One STEP = one ``solve_lower`` call exactly as MAID issues it: a fresh
operator (so the power iteration for L(b) runs), then the whole lower solve.

  value   lower-level Gpixel-iterations/s, inputs resident in HBM, device time
          (CUDA events around each step, L2 flushed between steps; the
          working set of c2 is L2-resident within a step).
  e2e     the same metric through the public API (paper_2502_09758_b200.solve_lower)
          with host NumPy inputs/outputs, H2D + D2H inside the timed region.
  N > 1   (torchrun) independent replicas, one instance per GPU ("replicas
          only": c2 does not shard); max time over ranks.

``--impl reference`` times the CPU oracle (the reference algorithm restated,
bitwise-pinned to it) on the host cores on a bounded sample of the same
workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "lower-level Gpixel-iters/s"
UNIT = "Gpx-it/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--mode", default="strict", choices=["strict", "fast", "fp32", "fft"],
                    help="fft: tile-FFT stencils (SURVEY.md §8 f2); single GPU for --workload c5")
    ap.add_argument("--iters", type=int, default=1200)
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--maid-steps", type=int, default=2, help="accepted MAID steps for upper iters/s (0: skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the fast-mode / fp32 / other-config side measurements")
    ap.add_argument("--workload", default="c2", choices=["c2", "c5"],
                    help="main-line workload (default c2 = BASELINE configs[1]); c5 under torchrun = row slabs")
    ap.add_argument("--c5-size", type=int, default=4096)
    ap.add_argument("--c5-iters", type=int, default=10)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_blur(x, kernel):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import adp_oracle as orc
    return orc.correlate(x, kernel.data)


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [t.strip() for t in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def cpu_sample(size, iters, seed=0):
    """Bounded oracle sample: one solve_lower with `iters` iterations on the
    c2 workload.  Returns (pixel-iterations, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import adp_oracle as orc
    from paper_2502_09758_b200 import configs
    up = configs.config2(seed, size=size, blur_fn=oracle_blur)
    p = orc.Lower(orc.Conv(up.b0.data, up.y_delta.shape), up.y_delta, 0.6, orc.TV(1e-4))
    # L(b)'s power iteration once, outside the sample: the GPU step amortises it over 1,200
    # iterations, a short CPU sample would otherwise be dominated by it
    orc.op_norm_sq(p.op, 300, 1e-4)
    t0 = time.perf_counter()
    _, _, it, _ = orc.solve_lower(p, up.y_delta, 1e-14, 10.0, iters, "agd", None, True)
    dt = time.perf_counter() - t0
    return up.y_delta.size * it, dt


def _cpu_worker(a):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    return cpu_sample(*a)


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    iters = 12
    rates, dts = [], []
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_worker, [(args.size, iters, k) for k in range(cores)])
            dt = time.perf_counter() - t0
            if s >= args.warmup:   # concurrent workers: sum of their solve-time rates (setup excluded)
                rates.append(sum(r[0] / r[1] for r in res) / 1e9)
                dts.append(max(r[1] for r in res))
    v = float(np.mean(rates))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(dts)), "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"c2: {args.size}x{args.size}x1 f64, 9x9 stencil, TV, adaptive AGD",
                       "sample": f"{iters} lower iterations per process per step"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{cores} concurrent processes x {iters} adaptive-AGD iterations of the CPU "
                                       "oracle (bitwise-pinned restatement of adp.solve_lower; L(b) precomputed)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_native(args):
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    import paper_2502_09758_b200 as adp
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs

    dtype, mode = ("float32", "fast") if args.mode == "fp32" else ("float64", args.mode)
    up = configs.config2(rank, size=args.size)
    adp.set_precision(dtype, mode)
    N = up.y_delta.size
    K = up.b0.data.shape[0]
    eps = 1e-14
    mu = 10.0
    x0 = nat.to_dev(up.x0)
    out = nat.empty_like_dev(up.x0.shape)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > L2

    def one_step(stats):
        p = up.lower_problem(up.b0)   # fresh operator: power iteration included
        return adp.solve_lower(p, x0, eps, mu, max_iters=args.iters, method="agd", adaptive=True, x_out=out,
                               stats=stats)

    for _ in range(args.warmup):
        one_step({})
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    times, units, vals, vgs = [], 0, 0, 0
    st = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            stats = {}
            r = one_step(stats)
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            units += N * r.iters
            vals += stats["value_evals"]
            vgs += stats["vg_evals"]
    if ws > 1:
        dist.barrier()
    t_dev = float(np.sum(times))
    if ws > 1:
        tt = torch.tensor([t_dev], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
    value = units * ws / t_dev / 1e9

    # ---- e2e through the public API with host buffers
    kern_host = up.b0.data.copy()
    y_host = np.asarray(up.y_delta)
    x0_host = np.asarray(up.x0)

    def e2e_step():
        b = adp.Kernel(kern_host, adp.DEPTHWISE2D)
        p = adp.LowerProblem(adp.ConvOperator(b, y_host.shape), y_host, up.alpha, up.reg)
        r = adp.solve_lower(p, x0_host, eps, mu, max_iters=args.iters, method="agd", adaptive=True)
        return r

    e2e_step()
    torch.cuda.synchronize()
    e2e_t, e2e_units = 0.0, 0
    for _ in range(max(1, args.steps)):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = e2e_step()
        assert isinstance(r.x_tilde, np.ndarray)
        e2e_t += time.perf_counter() - t0
        e2e_units += N * r.iters
    if ws > 1:
        tt = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
    esz = 8 if dtype == "float64" else 4
    e2e = {"value": e2e_units * ws / e2e_t / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": 2 * N * 8 + kern_host.size * 8, "d2h_bytes_per_step": N * esz,
           "note": "host float64 NumPy in/out through paper_2502_09758_b200.solve_lower"}

    # ---- roofline of the dominant (only) kernel: conv_solve_kernel
    iters_total = units / N
    value_per_it = vals / max(iters_total, 1)
    flop_px_it = 2.0 * K * K * (2.0 + value_per_it) + 50.0    # 6K^2+50 at one value pass
    achieved_tf = flop_px_it * units / t_dev / 1e12
    pk = nat.SolveArgs  # keep linter quiet
    import ctypes
    tf = ctypes.c_double()
    ms = ctypes.c_double()
    nat.check(nat.lib().adp_fp64_peak(ctypes.byref(tf), ctypes.byref(ms), nat.stream_ptr()), "fp64 peak")
    peak = tf.value
    bytes_px_it = 48.0 if dtype == "float64" else 24.0
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath) and args.size == 256 and args.iters == 1200 and mode == "strict":
        traffic = json.load(open(tpath))["conv_solve_kernel"]["dram_bytes_per_launch"]
    roof = {"bound": "fp64", "achieved": achieved_tf, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved_tf / peak, "traffic": traffic,
            "traffic_note": "DRAM bytes per conv_solve_kernel launch (one step) from the committed ncu capture; "
                            "the algorithmic bytes are 48 B/px-it = 3.77 GB per step, L2-resident",
            "peak_source": "measured live: DFMA microbenchmark (adp_fp64_peak), 2 flop/DFMA",
            "flop_per_px_it": flop_px_it, "kernel": "conv_solve_kernel",
            "note": ("strict mode issues DMUL+DADD per tap (reference rounding), so its attainable fraction "
                     "of the DFMA roof is <= 0.5" if mode == "strict" and dtype == "float64" else ""),
            "hbm": {"achieved_gbs": bytes_px_it * units / t_dev / 1e9, "peak_gbs": hbm,
                    "frac": bytes_px_it * units / t_dev / 1e9 / hbm,
                    "bytes_per_px_it": bytes_px_it}}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64" if dtype == "float64" else "f32",
            "data": "synthetic",
            "config": {"workload": f"c2: {args.size}x{args.size}x1 image, {K}x{K} stencil, smoothed TV, "
                                   f"adaptive AGD, {args.iters} lower iterations per solve",
                       "mode": mode, "l2": "flushed between steps (256 MB write)",
                       "parallelism": f"replicas x{ws}", "value_evals_per_iter": value_per_it,
                       "vg_evals": vgs},
            "roofline": roof, "e2e": e2e, "gpu_launches": args.steps, "clocks": clk.summary()}

    # ---- MAID upper iterations / s (c2, reference 2-D settings)
    if args.maid_steps > 0 and rank == 0:
        cfg = configs.maid_config("c2")
        cfg.max_upper_iters = args.maid_steps
        upm = configs.config2(0, size=args.size)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b, x, tr = adp.maid_run(upm, cfg)
        dt = time.perf_counter() - t0
        line["maid"] = {"metric": "MAID upper iters/s", "value": len(tr) / dt, "accepted": len(tr),
                        "seconds": dt, "lower_iters_cum": tr.lower_iters_cum[-1] if len(tr) else 0,
                        "cg_iters_cum": tr.cg_iters_cum[-1] if len(tr) else 0}

    # ---- side measurements: the other precision modes (device time)
    if not args.no_extra and rank == 0:
        side = {}
        for tag, (dt_, md) in {"fast_f64": ("float64", "fast"), "fp32": ("float32", "fast")}.items():
            if (dt_, md) == (dtype, mode):
                continue
            adp.set_precision(dt_, md)
            x0s = nat.to_dev(up.x0)
            outs = nat.empty_like_dev(up.x0.shape)
            p = up.lower_problem(up.b0)
            adp.solve_lower(p, x0s, eps, mu, max_iters=args.iters, method="agd", adaptive=True, x_out=outs)
            tt, uu = 0.0, 0
            for _ in range(3):
                p = up.lower_problem(up.b0)
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                r = adp.solve_lower(p, x0s, eps, mu, max_iters=args.iters, method="agd", adaptive=True, x_out=outs)
                e1.record()
                torch.cuda.synchronize()
                tt += e0.elapsed_time(e1) / 1e3
                uu += N * r.iters
            side[tag] = {"value": uu / tt / 1e9, "unit": UNIT}
        adp.set_precision(dtype, mode)
        line["other_modes"] = side

    # ---- the other BASELINE configs, one timed call each (rank 0, N = 1)
    if not args.no_extra and rank == 0 and ws == 1:
        adp.set_precision(dtype, mode)
        line["configs"] = other_configs(args, flush)

    # ---- CPU baseline (rank 0, N = 1 only): bounded oracle sample
    if not args.no_cpu and rank == 0 and ws == 1:
        iters = 40
        u, dt = cpu_sample(args.size, iters)
        line["cpu_baseline"] = {"value": u / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"one CPU-oracle solve_lower, {iters} adaptive-AGD iterations on c2 "
                                          f"({dt:.1f} s, 1 thread; L(b) precomputed)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _timed(fn):
    import torch
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1) / 1e3


def other_configs(args, flush):
    """c3 (one 512x512x3 image), c4 (8 c3 instances = one GPU's share of 64)
    and c5 (one 4096x4096x3 image, K = 31) through solve_lower, device time,
    power iteration included (fresh operator per solve, as MAID calls it)."""
    import paper_2502_09758_b200 as adp
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs
    out = {}
    eps, mu = 1e-14, 10.0

    dev = {}   # x0 and the output buffer stay resident in HBM (inputs resident before the timed region)

    def solve(up, iters, stats=None):
        if id(up) not in dev:
            dev[id(up)] = (nat.to_dev(up.x0), nat.empty_like_dev(up.x0.shape))
        x0, xo = dev[id(up)]
        p = up.lower_problem(up.b0)
        return adp.solve_lower(p, x0, eps, mu, max_iters=iters, method="agd", adaptive=True, x_out=xo, stats=stats)

    up3 = configs.config3(0)
    solve(up3, 50)
    flush.zero_()
    r, t = _timed(lambda: solve(up3, 1200))
    out["c3"] = {"value": up3.y_delta.size * r.iters / t / 1e9, "unit": UNIT, "iters": r.iters,
                 "ms_per_solve": 1e3 * t, "workload": "512x512x3, 15x15 line-Gaussian, 1200 AGD iterations"}
    ups = [configs.config3(seed) for seed in range(8)]
    for u in ups:
        solve(u, 2)
    flush.zero_()

    def c4():
        return [solve(u, 300) for u in ups]
    rs, t = _timed(c4)
    out["c4"] = {"value": sum(u.y_delta.size * q.iters for u, q in zip(ups, rs)) / t / 1e9, "unit": UNIT,
                 "instances": len(ups), "ms": 1e3 * t,
                 "workload": "8 c3 instances (seeds 0-7) = one GPU's share of 64, 300 AGD iterations each, "
                             "no collectives (weak scaling over GPUs)"}
    for u in ups:
        dev.pop(id(u), None)
    del ups
    # IFT baseline on c1 (baselines.py:58-90 with defaults.cfg [ift]): upper iters/s
    up1 = configs.config1(0)
    adp.run_ift(up1, adp.BaselineConfig(method="ift", upper_iters=1, upper_step=0.002))
    t0 = time.perf_counter()
    _, _, tr = adp.run_ift(up1, adp.BaselineConfig(method="ift", upper_iters=10, upper_step=0.002))
    dt = time.perf_counter() - t0
    out["ift_c1"] = {"metric": "IFT upper iters/s", "value": len(tr) / dt, "upper_iters": len(tr),
                     "lower_iters_per_upper": 500, "cg_iters_cum": tr.cg_iters_cum[-1],
                     "workload": "c1 (n=256 dense, elastic net): run_ift, 500 prox-gradient steps + CG(1e-10) "
                                 "per upper iteration, wall clock"}
    up5 = configs.config5(0, size=args.c5_size)
    solve(up5, 2)
    flush.zero_()
    st5 = {}
    r, t = _timed(lambda: solve(up5, args.c5_iters, st5))
    out["c5"] = {"value": up5.y_delta.size * r.iters / t / 1e9, "unit": UNIT, "iters": r.iters,
                 "ms_per_solve": 1e3 * t, "stats": {k: st5.get(k) for k in ("power_iters", "vg_evals", "value_evals")},
                 "workload": f"{args.c5_size}x{args.c5_size}x3, 31x31 Gaussian, {args.c5_iters} AGD iterations "
                             "(+ power iteration), one GPU"}
    out["c5_fft"] = c5_fft(args, up5, solve, flush)
    return out


def c5_fft(args, up5, solve, flush):
    """the c5 solve with the tile-FFT stencils (tolerance
    mode), and one stencil (ConvOperator.apply on a device image) direct
    strict vs FFT, with the FFT stencil's HBM roofline."""
    import paper_2502_09758_b200 as adp
    from paper_2502_09758_b200 import _native as nat
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    p = up5.lower_problem(up5.b0)
    xd = nat.to_dev(up5.x0)
    p.op.apply(xd)    # output buffer in the caching allocator before timing

    def stencil_ms(reps=3):
        p.op.apply(xd)
        flush.zero_()
        _, t = _timed(lambda: [p.op.apply(xd) for _ in range(reps)])
        return 1e3 * t / reps
    direct_ms = stencil_ms()
    with adp.precision("float64", "fft"):
        fft_ms = stencil_ms()
        solve(up5, 2)
        flush.zero_()
        stf = {}
        r, t = _timed(lambda: solve(up5, args.c5_iters, stf))
        plan = p.op.fft_plan()
    # Jacobi-PCG on the lower Hessian (the hypergradient's CG), 10 iterations: direct strict vs fft
    from paper_2502_09758_b200.hypergradient import hess_cg
    rhs = xd * 0.5
    cg_ms = {}
    for mode in ("strict", "fft"):
        with adp.precision("float64", mode):
            pc = up5.lower_problem(up5.b0)
            hess_cg(pc, xd, rhs, 1e-300, 2)
            flush.zero_()
            (cgr, _), tc = _timed(lambda: hess_cg(pc, xd, rhs, 1e-300, 10))
            cg_ms[mode] = 1e3 * tc / max(cgr.iters, 1)
    # one hypergradient (Algorithm 1: lower solve -> CG -> mixed derivative), budgets capped at 20 / 20
    import copy
    hg_ms = {}
    for mode in ("strict", "fft"):
        with adp.precision("float64", mode):
            uph = copy.copy(up5)
            uph.lower_max_iters = 20
            st = adp.WarmState(x=xd.clone())
            adp.inexact_hypergradient(uph, up5.b0, 1e-12, 1e-12, st, cg_max_iters=2)
            st = adp.WarmState(x=xd.clone())
            flush.zero_()
            _, th = _timed(lambda: adp.inexact_hypergradient(uph, up5.b0, 1e-12, 1e-12, st, cg_max_iters=20))
            hg_ms[mode] = 1e3 * th
    H, W, C = up5.x0.shape
    kh = up5.b0.data.shape[0]
    V = 512 - kh + 1
    npairs = (-(-H // V) * -(-W // V) + 1) // 2
    sbytes = 16 * C * npairs * 512 * 512
    traffic = 5 * sbytes + 16 * H * W * C      # K1 write, K2 read+write+spectrum, K3 read; image in + out
    n_sten = 2 * stf.get("power_iters", 0) + 2 * stf.get("vg_evals", 0) + stf.get("value_evals", 0)
    return {"value": up5.y_delta.size * r.iters / t / 1e9, "unit": UNIT, "iters": r.iters, "ms_per_solve": 1e3 * t,
            "stats": {k: stf.get(k) for k in ("power_iters", "vg_evals", "value_evals")},
            "stencils_per_solve": n_sten, "stencil_share": n_sten * fft_ms / (1e3 * t),
            "stencil_ms": {"direct_strict": direct_ms, "fft": fft_ms, "speedup": direct_ms / fft_ms},
            "hypergradient_ms": {"direct_strict": hg_ms["strict"], "fft": hg_ms["fft"],
                                 "note": "inexact_hypergradient with 20 lower iterations (+ power iteration) and "
                                         "20 CG iterations, mixed derivative included"},
            "cg_ms_per_iter": {"direct_strict": cg_ms["strict"], "fft": cg_ms["fft"],
                               "note": "hess_cg (hypergradient CG) incl. setup and true residual, 10 iterations"},
            "fft_stencil_roofline": {"bound": "hbm", "achieved": traffic / (fft_ms * 1e-3) / 1e9, "peak": hbm,
                                     "unit": "GB/s", "frac": traffic / (fft_ms * 1e-3) / 1e9 / hbm,
                                     "bytes_per_stencil": traffic,
                                     "note": "algorithmic bytes of the three tile-FFT passes (complex scratch "
                                             "written once, read+written by the column pass, read by the "
                                             "inverse row pass, spectrum read once) + image in/out"},
            "workspace_bytes": plan.workspace_bytes,
            "workload": f"c5 in FFT stencil mode (SURVEY.md §8 f2; tolerance parity): {H}x{W}x{C}, {kh}x{kh} "
                        f"Gaussian, {args.c5_iters} AGD iterations (+ power iteration), 512x512 overlap-save tiles"}


def run_c5(args):
    """c5 main line: one 4096x4096x3 image; N > 1 ranks hold one row slab each
    (3r+1 ghost rows, one exchange per iteration, NCCL over NVLink), strong
    scaling; the iterates are bitwise those of the unsplit solve."""
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    import paper_2502_09758_b200 as adp
    from paper_2502_09758_b200 import configs
    from paper_2502_09758_b200 import multigpu
    dtype, mode = ("float32", "fast") if args.mode == "fp32" else ("float64", args.mode)
    adp.set_precision(dtype, mode)
    up = configs.config5(0, size=args.c5_size)
    N = up.y_delta.size
    x0 = np.ascontiguousarray(up.x0)
    if mode == "fft" and ws > 1:
        raise SystemExit("--mode fft runs the c5 workload on one GPU (the row-slab path uses the direct stencils)")
    comm = multigpu.DistComm() if ws > 1 else multigpu.LocalComm()
    sv = None
    if mode != "fft":
        sv = multigpu.SlabSolver(up.lower_problem(up.b0), ws, ranks=[rank] if ws > 1 else None, comm=comm)
    from paper_2502_09758_b200 import _native as nat
    x0d, xo = nat.to_dev(x0), nat.empty_like_dev(x0.shape)
    fft_stats = {}

    def step():
        if sv is None:   # one GPU, tile-FFT stencils: the solve_lower drop-in in fft mode
            fft_stats.clear()
            r = adp.solve_lower(up.lower_problem(up.b0), x0d, 1e-14, 10.0, max_iters=args.c5_iters,
                                adaptive=True, x_out=xo, stats=fft_stats)
            return None, r.grad_norm, r.iters, r.converged
        sv.p = up.lower_problem(up.b0)      # fresh operator: power iteration included
        return sv.solve(x0, 1e-14, 10.0, max_iters=args.c5_iters)

    for _ in range(args.warmup):
        step()
    times, units, launches = [], 0, 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if ws > 1:
                torch.distributed.barrier()
            (xs, gn, it, conv), dt = _timed(step)
            times.append(dt)
            units += N * it
            if sv is None:   # fft: 3 row/column/inverse passes per stencil + folds and vector passes
                n_st = 2 * fft_stats.get("power_iters", 0) + fft_stats.get("vg_evals", 0) + \
                    fft_stats.get("value_evals", 0) + 1
                launches += 3 * n_st + 2 * fft_stats.get("vg_evals", 0) + fft_stats.get("value_evals", 0) + 2
                continue
            st = sv.stats
            n_steps = 1 + st["power_iters"] + st["value_evals"] + (0 if conv or it < args.c5_iters else 1)
            launches += 2 * n_steps          # one slab step + one unit fold per reduction point
    t_dev = float(np.sum(times))
    if ws > 1:
        tt = torch.tensor([t_dev], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_dev = float(tt.item())
    line = {"metric": METRIC, "value": units / t_dev / 1e9, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if dtype == "float64" else "f32",
            "data": "synthetic",
            "config": {"workload": f"c5: {args.c5_size}x{args.c5_size}x3 image, 31x31 stencil, smoothed TV, "
                                   f"adaptive AGD, {args.c5_iters} lower iterations per solve (+ power iteration)",
                       "mode": mode, "l2": "inputs larger than L2",
                       "parallelism": ("tile-FFT stencils, one GPU" if sv is None else
                                       f"row slabs x{ws} (ghost {sv.slabs[0].ghost_bot if ws > 1 else 0} rows)")},
            "gpu_launches": launches, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()



if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "c5":
        run_c5(a)
    else:
        run_native(a)
