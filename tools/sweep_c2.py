"""Tile-geometry sweep of the c2 solve (strict f64): device time per lower
iteration for each (TH, TW) tile at the plan's register blocking.

    python tools/sweep_c2.py [--iters 600]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=600)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402

up = configs.config2(0)
x0 = nat.to_dev(up.x0)
out = nat.empty_like_dev(up.x0.shape)
key = (nat.LAYOUT_DEPTHWISE2D, tuple(up.x0.shape), (9, 9))
tiles = [(0, 0), (2, 128), (4, 128), (8, 128), (1, 256), (2, 256), (4, 256), (1, 128)]
if os.environ.get("ADP_RW") == "1":
    tiles = [(2, 128), (4, 128), (1, 256), (2, 256), (1, 128)]
if os.environ.get("ADP_RW") == "4":   # host-stepped stage kernels on c2 (with ADP_STEP=1)
    tiles = [(0, 0), (4, 128), (8, 64), (8, 128), (16, 64), (4, 64), (2, 128), (16, 32)]
for tile in tiles:
    nat.set_tile(key, tile)
    nat.clear_plans()
    try:
        geo = nat.probe_geometry(up.x0.shape, (9, 9), tile)
        p = up.lower_problem(up.b0)
        adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=20, adaptive=True, x_out=out)
        ts = []
        for rep in range(3):
            p = up.lower_problem(up.b0)
            st = {}
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=a.iters, adaptive=True, x_out=out, stats=st)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / r.iters)
        print(f"tile {tile} geo {geo} flags {p.op.plan().flags()}: {min(ts):.2f} us/iter", flush=True)
    except Exception as ex:  # noqa: BLE001
        print(f"tile {tile}: {ex}")
