"""Profiling driver: one warm-up and one profiled c2 solve_lower (strict f64).

    python tools/prof_solve.py [--iters 100] [--size 256] [--mode strict|fast] [--config c2|c3|c5]

Used as the ncu target (the profiled launch is the 2nd conv_solve_kernel).
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--size", type=int, default=256)
ap.add_argument("--mode", default="strict")
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402

adp.set_precision("float64", a.mode)
up = configs.CONFIGS[a.config](0, size=a.size)
x0 = nat.to_dev(up.x0)
out = nat.empty_like_dev(up.x0.shape)
for rep in range(a.reps):
    p = up.lower_problem(up.b0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = {}
    r = adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=a.iters, method="agd", adaptive=True, x_out=out, stats=st)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {r.iters} iters, {dt * 1e3:.2f} ms, {dt / max(r.iters, 1) * 1e6:.1f} us/iter, stats {st}")
