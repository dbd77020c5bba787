import time, sys, dataclasses
sys.path.insert(0, '.')
import torch
import paper_2502_09758_b200 as adp
from paper_2502_09758_b200 import configs
up = configs.config1(0)
for alpha in (1.0, 0.0):
    up2 = dataclasses.replace(up, alpha=alpha)
    p = up2.lower_problem(up2.b0)
    adp.solve_lower(p, up.x0, 1e-14, 1e-3, max_iters=50, method="agd", adaptive=True)
    for ad in (True, False):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = {}
        r = adp.solve_lower(p, up.x0, 1e-300, 1e-3, max_iters=4000, method="agd", adaptive=ad, stats=st)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"alpha {alpha} adaptive {ad}: {r.iters} iterations {dt*1e6/r.iters:.2f} us/iter, value evals {st.get('value_evals')}, vg {st.get('vg_evals')}")
