"""A/B of the c3 solve: persistent single launch (ADP_STEP=0) vs host-stepped
high-occupancy stages (ADP_STEP=1): device time per lower iteration.

    python tools/step_ab.py [--iters 300]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=300)
ap.add_argument("--modes", default="0,1")
a = ap.parse_args()
import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402

up = configs.config3(0)
x0 = nat.to_dev(up.x0)
out = nat.empty_like_dev(up.x0.shape)
for mode in a.modes.split(","):
    os.environ["ADP_STEP"] = mode
    nat.clear_plans()
    p = up.lower_problem(up.b0)
    p.op._norm_sq = 1.0
    adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=20, adaptive=True, x_out=out)
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record()
        r = adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=a.iters, adaptive=True, x_out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1) * 1e3 / r.iters, (time.perf_counter() - w0) * 1e6 / r.iters))
    print(f"ADP_STEP={mode} flags {p.op.plan().flags()}: device {min(t[0] for t in ts):.1f} us/iter, "
          f"wall {min(t[1] for t in ts):.1f} us/iter", flush=True)
