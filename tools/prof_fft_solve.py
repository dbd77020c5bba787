"""c5 solve in fft mode: stats and a time split (power iteration vs AGD).

    python tools/prof_fft_solve.py [--size 4096] [--iters 10]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=4096)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--config", default="c5")
a = ap.parse_args()

import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402

adp.set_precision("float64", os.environ.get("ADP_MODE", "fft"))
up = configs.config5(0, size=a.size) if a.config == "c5" else configs.CONFIGS[a.config](0)
x0 = nat.to_dev(up.x0)
out = nat.empty_like_dev(up.x0.shape)


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for rep in range(2):
    p = up.lower_problem(up.b0)
    lam, tp = timed(lambda: adp.op_norm_sq(p.op, 300, 1e-4))
    st = {}
    r, ts = timed(lambda: adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=a.iters, adaptive=True, x_out=out, stats=st))
    p2 = up.lower_problem(up.b0)
    st2 = {}
    r2, tt = timed(lambda: adp.solve_lower(p2, x0, 1e-14, 10.0, max_iters=a.iters, adaptive=True, x_out=out, stats=st2))
    _, t1 = timed(lambda: p.op.apply(x0))
    print(f"rep {rep}: power {tp:.1f} ms (lam {lam:.6f}); solve w/o power {ts:.1f} ms {st}; "
          f"solve with power {tt:.1f} ms {st2}; one stencil {t1:.2f} ms")
