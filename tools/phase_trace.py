"""Per-phase device timing of one c2/c3 solve (adp_debug_trace)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--size", type=int, default=256)
ap.add_argument("--mode", default="strict")
ap.add_argument("--tile", type=int, nargs=2, default=None, help="TH TW override")
a = ap.parse_args()
import torch  # noqa: E402
import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402

adp.set_precision("float64", a.mode)
up = configs.CONFIGS[a.config](0, size=a.size)
if a.tile:
    ks = tuple(up.b0.data.shape[:2])
    nat.set_tile((nat.LAYOUT_DEPTHWISE2D, tuple(up.x0.shape), ks), tuple(a.tile))
x0 = nat.to_dev(up.x0)
p = up.lower_problem(up.b0)
adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=64, method="agd", adaptive=True)
plan = p.op.plan()
print("geometry", plan.geometry())
nat.check(nat.lib().adp_debug_trace(plan.handle, 1, None))
p = up.lower_problem(up.b0)
adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=64, method="agd", adaptive=True)
buf = np.zeros(64 * 16 + 256, dtype=np.uint64)
nat.check(nat.lib().adp_debug_trace(plan.handle, 0, buf.ctypes.data))
cnt = max(int(buf[1024 + 63]), 1)
subs = [buf[1152 + 8 * w:1152 + 8 * w + 5].astype(np.float64) / cnt for w in range(16)]
tr = buf[:1024].reshape(64, 16).astype(np.int64)
names = ["A", "bar1", "B", "bar2", "C", "bar3", "reduce"]
d = np.diff(tr[:, :8], axis=1)[4:60]
print("phase means (us):", {n: round(float(v) / 1e3, 2) for n, v in zip(names, d.mean(axis=0))})
it = np.diff(tr[4:61, 0]) / 1e3
print(f"iteration mean {it.mean():.2f} us, median {np.median(it):.2f}")
rt = tr[:, 8:]
extra = [(rt[i][rt[i] > 0].max() - tr[i, 7]) / 1e3 for i in range(4, 60) if (rt[i] > 0).any()]
print(f"retries: {len(extra)} iterations, mean extra {np.mean(extra) if extra else 0:.2f} us")
print(f"stage B per warp, mean SM cycles over {cnt} calls: sync+issue+box / -> / sync / stencil / epilogue")
for w, sub in enumerate(subs):
    if sub.any():
        print(f"  warp {w:2d}:", " ".join(f"{float(v):6.0f}" for v in sub))
rc = max(int(buf[1088 + 7]), 1)
print(f"reduce sub-phases, CTA 0 mean SM cycles over {rc} calls:",
      {n: round(float(buf[1088 + k]) / rc) for k, n in enumerate(["phase1+bar", "issue", "wait+sync", "fold", "final"])})
