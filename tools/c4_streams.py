"""c4 share (8 c3-type instances, 300 adaptive-AGD iterations each) on 1-4 host threads / CUDA streams."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import _native as nat, configs, multigpu  # noqa: E402

ups = [configs.config3(seed) for seed in range(8)]
x0s = [nat.to_dev(u.x0) for u in ups]


def solve(k, iters):
    p = ups[k].lower_problem(ups[k].b0)
    return adp.solve_lower(p, x0s[k], 1e-14, 10.0, max_iters=iters, method="agd", adaptive=True)


ref = None
for streams in (1, 2, 3, 4, 2):
    multigpu.run_instances(list(range(min(streams, 8))), lambda k: solve(k, 5), streams=streams)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rs, _ = multigpu.run_instances(list(range(8)), lambda k: solve(k, 300), streams=streams)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    xs = [nat.to_host(r.x_tilde) for r in rs]
    if ref is None:
        ref = xs
    same = all(np.array_equal(a, b) for a, b in zip(ref, xs))
    units = sum(u.y_delta.size * r.iters for u, r in zip(ups, rs))
    print(f"streams {streams}: {dt*1e3:.1f} ms -> {units/dt/1e9:.2f} Gpx-it/s, identical {same}", flush=True)
