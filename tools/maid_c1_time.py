"""c1 MAID wall time (BASELINE config 1) and where the host time goes."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import configs  # noqa: E402

up = configs.config1(0)
cfg = configs.maid_config("c1")
adp.maid_run(up, cfg)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b, x, tr = adp.maid_run(up, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"c1 MAID {len(tr)} steps {dt:.3f} s -> {len(tr) / dt:.1f} upper it/s; lower iters {tr.lower_iters_cum[-1]}, "
          f"cg {tr.cg_iters_cum[-1]}", flush=True)
if len(sys.argv) > 1:
    pr = cProfile.Profile()
    pr.enable()
    adp.maid_run(up, cfg)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
