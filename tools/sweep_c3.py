"""Tile-geometry sweep of the c3 solve (512x512x3, K = 15, strict f64):
device time per lower iteration for each (TH, TW) tile.

    python tools/sweep_c3.py [--iters 300]      (ADP_PIPE=0: unpipelined stages)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=300)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402

up = configs.config3(0)
x0 = nat.to_dev(up.x0)
out = nat.empty_like_dev(up.x0.shape)
key = (nat.LAYOUT_DEPTHWISE2D, tuple(up.x0.shape), (15, 15))
for tile in [(0, 0), (8, 32), (4, 64), (16, 32), (4, 128), (16, 64), (8, 128), (2, 128)]:
    nat.set_tile(key, tile)
    nat.clear_plans()
    try:
        geo = nat.probe_geometry(up.x0.shape, (15, 15), tile)
        p = up.lower_problem(up.b0)
        adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=20, adaptive=True, x_out=out)
        ts = []
        for rep in range(3):
            p = up.lower_problem(up.b0)
            p.op._norm_sq = 1.0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=a.iters, adaptive=True, x_out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / r.iters)
        print(f"tile {tile} geo {geo}: {min(ts):.2f} us/iter", flush=True)
    except Exception as ex:  # noqa: BLE001
        print(f"tile {tile}: {ex}", flush=True)
