"""Diagnostic: device fused CG vs oracle CG per iteration budget, and the
oracle's own sensitivity to ddot rounding (perturbed-order oracle)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import adp_oracle as orc
import paper_2502_09758_b200 as adp
from paper_2502_09758_b200.hypergradient import hess_cg

d = np.load(os.path.join(ROOT, "tests/golden/hyper2d.npz"))
shape = d["y_delta"].shape
xt, rhs = d["x_tilde"], d["rhs"]
po = orc.Lower(orc.Conv(d["kern"], shape), d["y_delta"], 0.6, orc.TV(1e-4))
diag = orc.lower_hess_diag(po, xt)
p = adp.LowerProblem(adp.ConvOperator(adp.Kernel(d["kern"], adp.DEPTHWISE2D), shape), d["y_delta"], 0.6, adp.SmoothedTV(1e-4))
print("diag rel", np.abs(adp.lower_hess_diag(p, xt) - diag).max() / np.abs(diag).max())
print("rhs from device vs golden", np.abs(np.asarray(adp.upper_fit_grad(xt, adp.ConvOperator(adp.Kernel(d["a_kern"], adp.DEPTHWISE2D), shape), d["y_delta"])) - rhs).max())
real_ddot = orc.ddot
for k in [1, 2, 3, 5, 10, 20, 40, 60]:
    qo, reso, ito, _ = orc.cg_solve(lambda v: orc.lower_hess_vec(po, xt, v), rhs, 1e-12, k, None, diag)
    orc.ddot = lambda a, b: float(np.sum(np.asarray(a).ravel() * np.asarray(b).ravel()))
    qp, _, _, _ = orc.cg_solve(lambda v: orc.lower_hess_vec(po, xt, v), rhs, 1e-12, k, None, diag)
    orc.ddot = real_ddot
    cg, hv = hess_cg(p, xt, rhs, 1e-12, k)
    qd = cg.q.cpu().numpy()
    s = np.abs(qo).max()
    print(f"k={k:3d} dev-vs-oracle {np.abs(qd-qo).max()/s:.3e}  oracle-perturbed-ddot {np.abs(qp-qo).max()/s:.3e}  res dev {cg.residual:.6e} orc {reso:.6e}")
