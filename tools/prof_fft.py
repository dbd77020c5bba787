"""ncu target for the FFT stencil path: one warm-up and one profiled
ConvOperator.apply in fft mode on the c5 image (4096x4096x3, K = 31).

    python tools/prof_fft.py [--size 4096] [--reps 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=4096)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()

import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402

adp.set_precision("float64", "fft")
up = configs.config5(0, size=a.size)
p = up.lower_problem(up.b0)
xd = nat.to_dev(up.x0)
for _ in range(a.reps):
    out = p.op.apply(xd)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    p.op.apply(xd)
e1.record()
torch.cuda.synchronize()
print(f"fft apply {e0.elapsed_time(e1) / 5:.3f} ms")
