"""c3 MAID (first 2 accepted upper steps): wall time and the host-side profile."""
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

up = configs.config3(0)
cfg = configs.maid_config("c3")
cfg.max_upper_iters = 1
adp.maid_run(up, cfg)
cfg.max_upper_iters = 2
pr = cProfile.Profile()
torch.cuda.synchronize()
t0 = time.perf_counter()
pr.enable()
b, x, tr = adp.maid_run(up, cfg)
pr.disable()
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"c3 MAID {len(tr)} steps {dt:.3f} s; lower iters {tr.lower_iters_cum[-1]}, cg {tr.cg_iters_cum[-1]}")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
