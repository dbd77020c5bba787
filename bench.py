#!/usr/bin/env python
"""Benchmark of the MAID hot path on B200 (contract: README / DESIGN.md §Measurement).

Main line (N = 1): BASELINE.json configs[2], "c3" — the largest single-GPU
config: one 512x512x3 float64 image, 15x15 line-Gaussian stencil shared by
the channels, smoothed TV (nu 1e-4, alpha 0.6), adaptive AGD with gradient
restart, 1,200 lower iterations per solve (eps tiny so the budget is used).
One STEP = one ``solve_lower`` call exactly as MAID issues it: a fresh
operator (so the power iteration for L(b) runs), then the whole lower solve.

  value   lower-level Gpixel-iterations/s, inputs resident in HBM, device time
          (CUDA events on the launching stream around each step, L2 flushed
          between steps).
  e2e     the same metric through the public API (paper_2502_09758_b200.solve_lower)
          with host NumPy inputs/outputs: H2D of y, x0 and the kernel and D2H
          of x~ inside the timed region.
  N > 1   ``--gpus N`` (self-launched through torch.distributed.run when
          WORLD_SIZE is unset): configs[3], "c4" — independent c3-type
          instances sharded round-robin over the ranks (seed = rank + N*k,
          k = step mod 8: the rank's 8-instance share of the 64), no
          collective on the data path, weak scaling; max device time over
          ranks.  ``--workload c5`` runs the row-slab solve instead.

``--impl reference`` times the reference algorithm on the host cores: the CPU
oracle (bitwise-pinned restatement of adp.solve_lower; the reference is pure
Python and cannot travel to the GPU box), one process per core, on a bounded
sample of the same workload (see ``cpu_sample``).
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
FULL_ITERS = 1200          # lower_max_iters of the 2-D configs (defaults.cfg)
NOMINAL_FP64_TF = 148 * 64 * 2 * 1.965e9 / 1e12   # 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--mode", default="strict", choices=["strict", "fast", "fp32", "fft"],
                    help="fft: tile-FFT stencils (SURVEY.md §8 f2); single GPU for --workload c5")
    ap.add_argument("--iters", type=int, default=FULL_ITERS)
    ap.add_argument("--maid-steps", type=int, default=6, help="accepted c2 MAID steps for upper iters/s (0: skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the side measurements (other configs / modes)")
    ap.add_argument("--workload", default=None, choices=["c2", "c3", "c4", "c5"],
                    help="main line: default c3 at N = 1, c4 (instances sharded over ranks) at N > 1; "
                         "c5 = one 4096^2x3 image, row slabs over the ranks")
    ap.add_argument("--c5-size", type=int, default=4096)
    ap.add_argument("--c5-iters", type=int, default=10)
    a = ap.parse_args()
    if a.workload is None:
        a.workload = "c3" if a.gpus == 1 else "c4"
    return a


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def maybe_relaunch(args):
    """`python bench.py --gpus N` (N > 1) without torchrun: re-exec under
    torch.distributed.run, one rank per GPU, rendezvous on 127.0.0.1."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # communicator ranks on stderr, the JSON line alone on stdout
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execvpe(sys.executable, cmd, env)


def check_world(args):
    ws, _, _ = dist_env()
    if args.impl == "native" and ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch with torchrun --nproc-per-node "
                         f"{args.gpus} (or plain python, which self-launches)")


def oracle_blur(x, kernel):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import adp_oracle as orc
    return orc.correlate(x, kernel.data)


def workload_desc(wl, ws, iters):
    if wl == "c3":
        return {"workload": f"c3: 512x512x3 f64 image (seed 0), 15x15 line-Gaussian stencil shared by channels, "
                            f"smoothed TV (nu 1e-4, alpha 0.6), adaptive AGD + restart, {iters} lower iterations "
                            "per solve_lower, fresh operator per step (power iteration for L(b) included)",
                "parallelism": "one instance" if ws == 1 else f"replicas x{ws}"}
    if wl == "c4":
        return {"workload": f"c4: independent c3-type instances (512x512x3, 15x15 line-Gaussian, seeds "
                            f"rank + {ws}*k), one solve_lower of {iters} lower iterations per GPU per step, "
                            "k = step mod 8 (each rank's 8-instance share of the 64)",
                "parallelism": f"instances sharded over {ws} ranks, no collectives"}
    if wl == "c2":
        return {"workload": f"c2: 256x256x1 f64 image, 9x9 Gaussian stencil, smoothed TV, adaptive AGD, {iters} "
                            "lower iterations per solve_lower (power iteration included)",
                "parallelism": "one instance" if ws == 1 else f"replicas x{ws}"}
    raise ValueError(wl)


def instance_seed(wl, rank, ws, step):
    return rank + ws * (step % 8) if wl == "c4" else 0


def make_instance(wl, seed, blur_fn=None):
    from paper_2502_09758_b200 import configs
    if wl == "c2":
        return configs.config2(seed, blur_fn=blur_fn)
    return configs.config3(seed, blur_fn=blur_fn)


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
# CPU side: the oracle (test infrastructure) is executed here ONLY as the
# reported baseline (cpu_baseline leg and --impl reference), never as the
# measured product path.
_CPU_CACHE = {}


def cpu_sample(wl, seed, iters):
    """Bounded oracle sample of ONE step of workload `wl` (a fresh-operator
    solve_lower of FULL_ITERS adaptive-AGD iterations): the power iteration for
    L(b) is timed once per (process, instance) and `iters` AGD iterations from
    x0 are timed per call; the step time is extrapolated as
    t_power + FULL_ITERS * t_iteration.  Returns (pixel-iterations of a full
    step, extrapolated step seconds, measured sample seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import adp_oracle as orc
    key = wl     # a worker keeps the first instance it built (pool task -> worker mapping is arbitrary)
    if key not in _CPU_CACHE:
        up = make_instance(wl, seed, blur_fn=oracle_blur)
        p = orc.Lower(orc.Conv(up.b0.data, up.y_delta.shape), up.y_delta, up.alpha, orc.TV(1e-4))
        t0 = time.perf_counter()
        orc.op_norm_sq(p.op, 300, 1e-4)        # op_norm_sq as L_of_b calls it (lower_solvers.py:90-96)
        _CPU_CACHE[key] = (up, p, time.perf_counter() - t0)
    up, p, t_pow = _CPU_CACHE[key]
    t0 = time.perf_counter()
    _, _, it, _ = orc.solve_lower(p, up.y_delta, 1e-14, 10.0, iters, "agd", None, True)
    dt = time.perf_counter() - t0
    t_step = t_pow + FULL_ITERS * dt / max(it, 1)
    return up.y_delta.size * FULL_ITERS, t_step, dt + t_pow


def _cpu_worker(a):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    return cpu_sample(*a)


def run_reference(args):
    """The reference arm: rank 0 only; all host cores, one oracle process per
    core (OPENBLAS_NUM_THREADS=1, scipy.ndimage being single-threaded), each on
    its own instance of the same workload."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    wl = args.workload
    if wl not in ("c2", "c3", "c4"):
        print(json.dumps({"impl": "reference", "unavailable": f"no CPU sample defined for workload {wl}"}))
        return
    iters = 2 if wl != "c2" else 12
    rates, sample_s = [], []
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        for s in range(args.warmup + args.steps):
            seeds = [instance_seed(wl, k, cores, s) if wl == "c4" else 0 for k in range(cores)]
            res = pool.map(_cpu_worker, [(wl, sd, iters) for sd in seeds])
            if s >= args.warmup:   # concurrent independent processes: aggregate = sum of their rates
                rates.append(sum(u / t for u, t, _ in res) / 1e9)
                sample_s.append(max(m for _, _, m in res))
    v = float(np.mean(rates))
    cfg = workload_desc(wl, ws, FULL_ITERS)
    cfg["mode"] = "strict"
    cfg["parallelism"] = f"{cores} host processes (one per core)"
    sample = (f"{cores} concurrent processes, each: CPU oracle (bitwise-pinned restatement of adp.solve_lower) on "
              f"its own {wl} instance; power iteration for L(b) timed once per process, {iters} adaptive-AGD "
              f"iterations timed per step; step time = t_power + {FULL_ITERS} x t_iteration")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(sample_s)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_maid_c1():
    """The oracle's c1 MAID run (BASELINE configs[0], 60 accepted steps), 1
    thread: (upper iters/s, accepted steps, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import adp_oracle as orc
    from paper_2502_09758_b200 import configs
    up = configs.config1(0)
    A = np.array(up.A.matrix)
    ou = orc.Upper(A_kernel=A, a=A, y_delta=np.asarray(up.y_delta), beta=0.0, alpha=1.0,
                   reg=orc.ElasticNet(1.2e-3, 4e-3, 1e-4), b0=A, x0=np.zeros(A.shape[1]), dense=True)
    t0 = time.perf_counter()
    _, _, tr = orc.maid_run(ou, dict(max_upper_iters=60))
    dt = time.perf_counter() - t0
    return len(tr["k"]) / dt, len(tr["k"]), dt


# ---------------------------------------------------------------------------
def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return json.load(open(path)), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload, mode, iters, kernel="conv_solve_kernel"):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set
    full capture of the same workload (profiles/ncu_traffic.json), else None."""
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(tpath) or mode != "strict":
        return None, None
    tab = json.load(open(tpath))
    if kernel == "step_ca_kernel":
        ent = tab.get(f"{workload}_step_ca")
    else:
        ent = tab.get(workload)
        if ent and ent.get("iters") != iters:
            ent = None
    if not ent:
        return None, None
    return ent["dram_bytes_per_launch"], ent.get("source")


def run_native(args):
    import ctypes

    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2502_09758_b200 as adp
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs

    wl = args.workload
    dtype, mode = ("float32", "fast") if args.mode == "fp32" else ("float64", args.mode)
    adp.set_precision(dtype, mode)
    eps, mu = 1e-14, 10.0
    nsteps = args.warmup + args.steps
    seeds = sorted({instance_seed(wl, rank, ws, s) for s in range(nsteps)})
    ups = {sd: make_instance(wl, sd) for sd in seeds}
    dev = {sd: (nat.to_dev(u.x0), nat.empty_like_dev(u.x0.shape)) for sd, u in ups.items()}
    up0 = ups[seeds[0]]
    N = up0.y_delta.size
    K = up0.b0.data.shape[0]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > L2 (126 MB)
    st = torch.cuda.current_stream()

    def one_step(step, stats):
        up = ups[instance_seed(wl, rank, ws, step)]
        x0, out = dev[instance_seed(wl, rank, ws, step)]
        p = up.lower_problem(up.b0)   # fresh operator: power iteration included, as MAID calls it
        return adp.solve_lower(p, x0, eps, mu, max_iters=args.iters, method="agd", adaptive=True, x_out=out,
                               stats=stats)

    for s in range(args.warmup):
        one_step(s, {})
    torch.cuda.synchronize()
    plan = ups[seeds[0]].lower_problem(ups[seeds[0]].b0).op.plan()
    flags = plan.flags()
    # live timing of the dominant kernel: CUDA events around every 64th launch (sampled, so the host-side
    # event calls stay off the critical path of the timed steps; a sampled launch runs without the
    # stage-B overlap, i.e. the kernel alone)
    nat.check(nat.lib().adp_plan_profile(plan.handle, 64), "adp_plan_profile")
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times, units, vals, vgs, launches, dom_ms, dom_n = [], 0, 0, 0, 0, 0.0, 0
    with ClockSampler(local) as clk:
        for s in range(args.warmup, nsteps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            stats = {}
            r = one_step(s, stats)
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            units += N * r.iters
            vals += stats["value_evals"]
            vgs += stats["vg_evals"]
            launches += stats["launches"]
            dom_ms += stats["dominant_ms"]
            dom_n += stats["dominant_launches"]
    torch.cuda.synchronize()
    nat.check(nat.lib().adp_plan_profile(plan.handle, 0), "adp_plan_profile")
    if ws > 1:
        dist.barrier()
    t_dev = float(np.sum(times))
    units_all = units
    if ws > 1:
        tt = torch.tensor([t_dev], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev = float(tt.item())
        uu = torch.tensor([float(units)], device="cuda", dtype=torch.float64)
        dist.all_reduce(uu, op=dist.ReduceOp.SUM)
        units_all = float(uu.item())
    value = units_all / t_dev / 1e9

    # ---- e2e through the public API with host buffers (H2D + D2H inside the timed region)
    def e2e_step(step):
        up = ups[instance_seed(wl, rank, ws, step)]
        kern_host = np.array(up.b0.data)
        y_host = np.array(up.y_delta)
        x0_host = np.array(up.x0)
        t0 = time.perf_counter()
        b = adp.Kernel(kern_host, adp.DEPTHWISE2D)
        p = adp.LowerProblem(adp.ConvOperator(b, y_host.shape), y_host, up.alpha, up.reg)
        r = adp.solve_lower(p, x0_host, eps, mu, max_iters=args.iters, method="agd", adaptive=True)
        assert isinstance(r.x_tilde, np.ndarray)
        return r, time.perf_counter() - t0, kern_host.nbytes + y_host.nbytes + x0_host.nbytes

    e2e_step(0)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e2e_t, e2e_units, h2d = 0.0, 0, 0
    for s in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        r, dt, hb = e2e_step(args.warmup + s)
        e2e_t += dt
        e2e_units += N * r.iters
        h2d = hb
    e2e_all = e2e_units
    if ws > 1:
        tt = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())
        uu = torch.tensor([float(e2e_units)], device="cuda", dtype=torch.float64)
        dist.all_reduce(uu, op=dist.ReduceOp.SUM)
        e2e_all = float(uu.item())
    esz = 8 if dtype == "float64" else 4
    e2e = {"value": e2e_all / e2e_t / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": N * 8,
           "note": "host float64 NumPy y, x0, kernel in / x~ out through paper_2502_09758_b200.solve_lower "
                   "(wall clock, fresh operator per step)"}

    # ---- roofline.  Persistent solve (c2; ADP_STEP=0): the only kernel in the timed region is
    # conv_solve_kernel, one launch per step.  Host-stepped solve (c3-c5 default): the dominant kernel
    # is step_ca_kernel (the candidate's value pass + the speculative stage A at the next
    # extrapolation point: two stencil passes), timed live with CUDA events on its stream.
    iters_total = units / N
    value_per_it = vals / max(iters_total, 1)
    flop_px_it = 2.0 * K * K * (2.0 + value_per_it) + 50.0    # 6K^2+50 at one value pass
    step_total_tf = flop_px_it * units / sum(times) / 1e12     # whole solve (all kernels of the step)
    if flags["step"] and dom_n:
        dom_kernel = "step_ca_kernel"
        dom_flop = (2.0 * 2.0 * K * K + 50.0) * N              # two forward K x K passes + TV terms per launch
        achieved_tf = dom_flop * dom_n / (dom_ms * 1e-3) / 1e12
        dom_share = (dom_ms / dom_n) * 1e-3 * vgs / sum(times)   # one launch per lower iteration (vg evals)
    else:
        dom_kernel, dom_flop, dom_share = "conv_solve_kernel", flop_px_it * units / len(times), 1.0
        achieved_tf = step_total_tf
    tf = ctypes.c_double()
    ms = ctypes.c_double()
    nat.check(nat.lib().adp_fp64_peak(ctypes.byref(tf), ctypes.byref(ms), nat.stream_ptr()), "fp64 peak")
    peak = tf.value
    bytes_px_it = 48.0 if dtype == "float64" else 24.0
    peaks, peak_src = load_peaks()
    hbm = peaks["hbm_gbs"]
    traffic, tsrc = ncu_traffic(wl, mode, args.iters, dom_kernel)
    strict = mode == "strict" and dtype == "float64"
    roof = {"bound": "fp64", "achieved": achieved_tf, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved_tf / peak, "traffic": traffic,
            "traffic_note": (f"DRAM read+write bytes per {dom_kernel} launch from {tsrc}; algorithmic: "
                             f"{bytes_px_it:.0f} B/px-it = {bytes_px_it * units / len(times) / 1e9:.2f} GB per step "
                             "(the c3 working set is L2-resident)" if traffic else
                             "no committed ncu capture for this exact workload"),
            "peak_source": "measured live on this GPU: DFMA microbenchmark (adp_fp64_peak, 2 flop/DFMA); "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "peak_nominal_tflops": NOMINAL_FP64_TF,
            "kernel": dom_kernel, "flop_per_launch": dom_flop,
            "launch_ms": (dom_ms / max(dom_n, 1)) if dom_kernel == "step_ca_kernel" else 1e3 * sum(times) / len(times),
            "kernel_share_of_step": dom_share,
            "whole_step": {"achieved_tflops": step_total_tf, "flop_per_px_it": flop_px_it,
                           "frac": step_total_tf / peak,
                           "note": "all kernels of the timed steps: 2K^2 (2 + value passes per iteration) + 50 flop "
                                   "per lower pixel-iteration over the device time"},
            "solve_path": "host-stepped stage kernels (csrc/conv2d_step.cu)" if flags["step"] else
                          "persistent single-launch kernel" + (" with TMA tile boxes" if flags["tma"] else ""),
            "hbm": {"achieved_gbs": bytes_px_it * units / sum(times) / 1e9, "peak_gbs": hbm,
                    "frac": bytes_px_it * units / sum(times) / 1e9 / hbm, "bytes_per_px_it": bytes_px_it,
                    "peak_source": peak_src}}
    if strict:
        roof["strict_ceiling"] = {"frac": 2.0 * achieved_tf / peak, "whole_step_frac": 2.0 * step_total_tf / peak,
                                  "note": "strict mode reproduces scipy.ndimage rounding with DMUL + DADD per tap "
                                          "(2 FP64 issues per multiply-add), so its attainable fraction of the "
                                          "DFMA roof is 0.5; frac here is against that ceiling"}
    cfg = workload_desc(wl, ws, args.iters)
    cfg.update({"mode": mode, "l2": "flushed between steps (256 MB write); the c3 working set (~110 MB) is at "
                                    "the L2 size", "value_evals_per_iter": value_per_it, "vg_evals": vgs})
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64" if dtype == "float64" else "f32",
            "data": "synthetic (seeded generators of SURVEY.md Appendix A)", "config": cfg,
            "roofline": roof, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary()}

    # ---- MAID upper iterations / s: c1 (full 60-step run) and c2 (reference 2-D settings)
    if args.maid_steps > 0 and rank == 0:
        maid = {"metric": "MAID upper iters/s"}
        up1 = configs.config1(0)
        adp.maid_run(up1, configs.maid_config("c1"))   # warm (plans, caches)
        t0 = time.perf_counter()
        _, _, tr1 = adp.maid_run(up1, configs.maid_config("c1"))
        dt1 = time.perf_counter() - t0
        maid["c1"] = {"value": len(tr1) / dt1, "accepted": len(tr1), "seconds": dt1,
                      "lower_iters_cum": tr1.lower_iters_cum[-1], "cg_iters_cum": tr1.cg_iters_cum[-1],
                      "workload": "c1: n=256 dense, elastic net, MAIDConfig(max_upper_iters=60), wall clock"}
        cfg2 = configs.maid_config("c2")
        cfg2.max_upper_iters = args.maid_steps
        upm = configs.config2(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, tr = adp.maid_run(upm, cfg2)
        dt = time.perf_counter() - t0
        maid["c2"] = {"value": len(tr) / dt, "accepted": len(tr), "seconds": dt,
                      "lower_iters_cum": tr.lower_iters_cum[-1] if len(tr) else 0,
                      "cg_iters_cum": tr.cg_iters_cum[-1] if len(tr) else 0,
                      "workload": f"c2: 256x256x1, reference 2-D MAID settings, first {args.maid_steps} "
                                  "accepted upper steps, wall clock"}
        # c3 (the main line's instance): first 2 accepted upper steps of the same 2-D MAID settings
        cfg3 = configs.maid_config("c3")
        cfg3.max_upper_iters = min(2, args.maid_steps)
        up3 = configs.config3(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, tr3 = adp.maid_run(up3, cfg3)
        dt3 = time.perf_counter() - t0
        maid["c3"] = {"value": len(tr3) / dt3, "accepted": len(tr3), "seconds": dt3,
                      "lower_iters_cum": tr3.lower_iters_cum[-1] if len(tr3) else 0,
                      "cg_iters_cum": tr3.cg_iters_cum[-1] if len(tr3) else 0,
                      "workload": f"c3: 512x512x3, 15x15, reference 2-D MAID settings, first {cfg3.max_upper_iters} "
                                  "accepted upper steps, wall clock"}
        if not args.no_cpu and ws == 1:
            v, n, d = cpu_maid_c1()
            maid["c1"]["cpu_oracle"] = {"value": v, "accepted": n, "seconds": d, "cores": 1}
        line["maid"] = maid

    # ---- side measurements (rank 0, N = 1)
    if not args.no_extra and rank == 0 and ws == 1:
        side = {}
        for tag, (dt_, md) in {"fast_f64": ("float64", "fast"), "fp32": ("float32", "fast")}.items():
            if (dt_, md) == (dtype, mode):
                continue
            adp.set_precision(dt_, md)
            x0s = nat.to_dev(up0.x0)
            outs = nat.empty_like_dev(up0.x0.shape)
            p = up0.lower_problem(up0.b0)
            adp.solve_lower(p, x0s, eps, mu, max_iters=50, method="agd", adaptive=True, x_out=outs)
            tt, uu = 0.0, 0
            for _ in range(3):
                p = up0.lower_problem(up0.b0)
                flush.zero_()
                (r, t) = _timed(lambda: adp.solve_lower(p, x0s, eps, mu, max_iters=args.iters, method="agd",
                                                        adaptive=True, x_out=outs))
                tt += t
                uu += N * r.iters
            side[tag] = {"value": uu / tt / 1e9, "unit": UNIT, "workload": wl}
        adp.set_precision(dtype, mode)
        line["other_modes"] = side
        line["configs"] = other_configs(args, flush, wl)

    # ---- CPU baseline (rank 0, N = 1 only): bounded 1-thread oracle sample of the same step
    if not args.no_cpu and rank == 0 and ws == 1 and wl in ("c2", "c3"):
        iters = 3 if wl == "c3" else 12
        u, t_step, t_meas = cpu_sample(wl, 0, iters)
        line["cpu_baseline"] = {"value": u / t_step / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"CPU oracle (bitwise-pinned restatement of adp.solve_lower), 1 thread, "
                                          f"{wl} seed 0: power iteration + {iters} adaptive-AGD iterations "
                                          f"({t_meas:.1f} s), step time extrapolated to power iteration + "
                                          f"{FULL_ITERS} iterations"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def other_configs(args, flush, main_wl):
    """Side lines, device time, power iteration included (fresh operator per
    solve, as MAID calls it): c2 (256x256x1), c4 (8 c3 instances = one GPU's
    share of 64), c1 IFT, c5 (one 4096x4096x3 image, K = 31) direct and FFT."""
    import ctypes

    import paper_2502_09758_b200 as adp
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs
    out = {}
    eps, mu = 1e-14, 10.0
    tf_, ms_ = ctypes.c_double(), ctypes.c_double()
    nat.check(nat.lib().adp_fp64_peak(ctypes.byref(tf_), ctypes.byref(ms_), nat.stream_ptr()), "fp64 peak")
    fp64_peak = tf_.value   # measured DFMA TFLOP/s (2 flop per DFMA)

    dev = {}   # x0 and the output buffer stay resident in HBM (inputs resident before the timed region)

    def solve(up, iters, stats=None):
        if id(up) not in dev:
            dev[id(up)] = (nat.to_dev(up.x0), nat.empty_like_dev(up.x0.shape))
        x0, xo = dev[id(up)]
        p = up.lower_problem(up.b0)
        return adp.solve_lower(p, x0, eps, mu, max_iters=iters, method="agd", adaptive=True, x_out=xo, stats=stats)

    if main_wl != "c2":
        up2 = configs.config2(0)
        solve(up2, 50)
        tt, uu = 0.0, 0
        for _ in range(5):
            flush.zero_()
            r, t = _timed(lambda: solve(up2, 1200))
            tt += t
            uu += up2.y_delta.size * r.iters
        out["c2"] = {"value": uu / tt / 1e9, "unit": UNIT, "ms_per_solve": 1e3 * tt / 5,
                     "workload": "256x256x1, 9x9 Gaussian, 1200 AGD iterations (5 solves)"}
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
    # the same 8 instances on 2 host threads / CUDA streams (one instance's kernels fill the device while the
    # other waits on its host-side decisions); wall clock with a device-wide synchronisation on both sides
    import torch
    from paper_2502_09758_b200 import multigpu
    serial_x = [nat.to_host(q.x_tilde) for q in rs]
    multigpu.run_instances(list(range(2)), lambda k: solve(ups[k], 5), streams=2)   # per-thread plans
    torch.cuda.synchronize()
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rs2, _ = multigpu.run_instances(list(range(len(ups))), lambda k: solve(ups[k], 300), streams=2)
    torch.cuda.synchronize()
    t2 = time.perf_counter() - t0
    out["c4_2streams"] = {"value": sum(u.y_delta.size * q.iters for u, q in zip(ups, rs2)) / t2 / 1e9, "unit": UNIT,
                          "instances": len(ups), "ms": 1e3 * t2, "identical_to_serial": all(
                              np.array_equal(a, nat.to_host(b.x_tilde)) for a, b in zip(serial_x, rs2)),
                          "workload": "c4 share (8 instances, 300 AGD iterations each) on 2 host threads x 2 CUDA "
                                      "streams, wall clock"}
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
    # steady state of the direct c5 solve: a second solve 30 iterations longer, the difference per iteration
    # (the 10-iteration line above carries the power iteration for L(b))
    flush.zero_()
    r2, t2 = _timed(lambda: solve(up5, args.c5_iters + 30))
    if r2.iters > r.iters:
        per = (t2 - t) / (r2.iters - r.iters)
        out["c5"]["steady_state"] = {"ms_per_iter": 1e3 * per, "value": up5.y_delta.size / per / 1e9, "unit": UNIT,
                                     "flop_per_px_it": 2 * 31 * 31 * 3 + 50,
                                     "strict_ceiling_frac": (2 * 31 * 31 * 3 + 50) * up5.y_delta.size / per / 1e12
                                     / (0.5 * fp64_peak) if fp64_peak else None,
                                     "note": "solve of c5_iters + 30 iterations minus the solve above, per iteration; "
                                             "flop: three 31x31 strict stencils (1.0 value passes) + epilogues; "
                                             "ceiling: half the measured DFMA rate (DMUL + DADD per tap)"}
    out["c5_fft"] = c5_fft(args, up5, solve, flush)
    return out


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
    op_bytes = 16 * H * W * C
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
            "fft_stencil_roofline": {"bound": "hbm", "achieved": op_bytes / (fft_ms * 1e-3) / 1e9, "peak": hbm,
                                     "unit": "GB/s", "frac": op_bytes / (fft_ms * 1e-3) / 1e9 / hbm,
                                     "bytes_per_stencil": op_bytes,
                                     "note": "the operation's own bytes: 16 B per pixel-channel (image in + out)",
                                     "with_scratch": {"bytes_per_stencil": traffic,
                                                      "achieved": traffic / (fft_ms * 1e-3) / 1e9,
                                                      "frac": traffic / (fft_ms * 1e-3) / 1e9 / hbm,
                                                      "note": "incl. the complex scratch of the three tile-FFT "
                                                              "passes (written once, read+written by the column "
                                                              "pass, read by the inverse row pass) + spectrum"}},
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
    maybe_relaunch(a)
    check_world(a)
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "c5":
        run_c5(a)
    else:
        run_native(a)
