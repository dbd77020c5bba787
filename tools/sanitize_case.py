"""Small invocations of every kernel family for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool racecheck python tools/sanitize_case.py

persistent solve (c2-type 9x9 and RW = 4 15x15 instances), the fused CG,
the per-call primitives (apply/adjoint/gram_diag/value/grad/Hv/diag/upper/
power/mixed), the kernel-gram correlation, the dense 1-D engine (solve, CG,
MAID step) and the row-slab steps."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2502_09758_b200 as adp  # noqa: E402
from paper_2502_09758_b200 import configs, multigpu  # noqa: E402
from paper_2502_09758_b200.hypergradient import hess_cg  # noqa: E402

adp.set_precision("float64", "strict")
rng = np.random.default_rng(0)
for shape, K in (((48, 64, 1), 9), ((40, 64, 3), 15)):
    k = configs.gaussian_kernel_2d(K, K / 4.0, shape[2])
    y = rng.uniform(0, 1, shape)
    p = adp.LowerProblem(adp.ConvOperator(k, shape), y, 0.6, adp.SmoothedTV(1e-4))
    r = adp.solve_lower(p, y, 1e-9, 10.0, max_iters=8, method="agd", adaptive=True)
    x = r.x_tilde
    v = rng.standard_normal(shape)
    p.op.apply(x), p.op.adjoint(v), p.op.gram_diag()
    adp.lower_value(p, x), adp.lower_value_and_grad(p, x), adp.lower_grad(p, x)
    adp.lower_hess_vec(p, x, v), adp.lower_hess_diag(p, x)
    hess_cg(p, x, v, 1e-12, 5)
    adp.mixed_second_transpose(x, k, v, p)
    print("2-D", shape, K, "ok", r.iters)
up1 = configs.config1(0)
cfg = configs.maid_config("c1")
cfg.max_upper_iters = 1
adp.maid_run(up1, cfg)
print("dense MAID step ok")
# row slabs (2 slabs in one process)
shape, K = (128, 128, 3), 9
k = configs.gaussian_kernel_2d(K, 2.0, 3)
y = rng.uniform(0, 1, shape)
p = adp.LowerProblem(adp.ConvOperator(k, shape), y, 0.6, adp.SmoothedTV(1e-4))
sv = multigpu.SlabSolver(p, 2)
sv.solve(y, 1e-14, 10.0, max_iters=3)
up = adp.UpperProblem(name="s", A=adp.ConvOperator(k, shape), a=k, y_delta=y, beta=0.3, alpha=0.6,
                      reg=adp.SmoothedTV(1e-4), b0=k, x0=y.copy(), mu_floor=10.0, lower_max_iters=5,
                      lower_adaptive=True)
sh = multigpu.SlabHypergradient(up, 2)
st = adp.WarmState(x=sh.sv.local(y))
sh.hypergradient(k, 0.5, 0.5, st, cg_max_iters=3)
torch.cuda.synchronize()
print("slabs ok")
