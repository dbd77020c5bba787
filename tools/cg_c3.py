"""Time the hypergradient's Jacobi-PCG (hess_cg) on c3: ms per CG iteration."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2502_09758_b200 as adp
from paper_2502_09758_b200 import _native as nat, configs
from paper_2502_09758_b200.hypergradient import hess_cg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
up = configs.CONFIGS[cfg](0) if cfg != "c5" else configs.config5(0, size=int(sys.argv[2]) if len(sys.argv) > 2 else 4096)
xd = nat.to_dev(up.x0)
rhs = xd * 0.5
pc = up.lower_problem(up.b0)
hess_cg(pc, xd, rhs, 1e-300, 2)
for n in (10, 40):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    (r, _) = hess_cg(pc, xd, rhs, 1e-300, n)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{cfg}: hess_cg {r.iters} iterations {dt*1e3:.2f} ms -> {dt*1e6/max(r.iters,1):.1f} us/iter")
