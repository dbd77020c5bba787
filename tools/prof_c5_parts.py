"""c5 (4096x4096x3, K = 31) per-call device times of the hypergradient parts
in fft mode vs strict: mixed_second_transpose (kgc pair), upper terms, one
lower value+grad.

    python tools/prof_c5_parts.py [--size 4096]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=4096)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402
from paper_2502_09758_b200.hypergradient import _upper_terms  # noqa: E402

up = configs.config5(0, size=a.size)
xd = nat.to_dev(up.x0)
qd = xd * 0.1


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for mode in ("strict", "fft"):
    with adp.precision("float64", mode):
        p = up.lower_problem(up.b0)
        print(mode, "mixed_T %.2f ms" % t(lambda: adp.mixed_second_transpose(xd, up.b0, qd, p)),
              "upper_terms %.2f ms" % t(lambda: _upper_terms(up.A, xd, up.y_delta, want_grad=True)),
              "value_and_grad %.2f ms" % t(lambda: adp.lower_value_and_grad(p, xd)), flush=True)
