"""Dense 1-D engine (c1): the single-cluster execution -- GEMV row results and
B^T partials exchanged through distributed shared memory, cluster barriers
(csrc/dense1d.cu) -- must be BITWISE the cooperative-grid execution (global
exchange buffers + grid barrier): same arithmetic in the same order, only the
transport differs."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _with_cluster(nat, on, fn):
    os.environ["ADP_DENSE_CLUSTER"] = "1" if on else "0"
    try:
        nat.clear_plans()
        return fn()
    finally:
        os.environ.pop("ADP_DENSE_CLUSTER", None)
        nat.clear_plans()


def test_dense_cluster_solve_and_hypergradient_bitwise(adp):
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs
    up = configs.config1(0)

    def run():
        p = up.lower_problem(up.b0)
        r = adp.solve_lower(p, up.x0, 1e-12, 1e-3, max_iters=400, method="agd", adaptive=True)
        v, g = adp.lower_value_and_grad(p, r.x_tilde)
        hv = adp.lower_hess_vec(p, r.x_tilde, g)
        d = adp.lower_hess_diag(p, r.x_tilde)
        return r.x_tilde, r.iters, r.grad_norm, p.op._norm_sq, v, g, hv, d

    a = _with_cluster(nat, True, run)
    b = _with_cluster(nat, False, run)
    assert a[1] == b[1] and a[2] == b[2] and a[3] == b[3] and a[4] == b[4]
    for u, w in zip((a[0], a[5], a[6], a[7]), (b[0], b[5], b[6], b[7])):
        assert np.array_equal(np.asarray(u), np.asarray(w))


def test_dense_cluster_maid_trace_bitwise(adp):
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs
    up = configs.config1(0)
    cfg = configs.maid_config("c1")
    cfg.max_upper_iters = 12

    def run():
        b, x, tr = adp.maid_run(up, cfg)
        return np.asarray(b.data), np.asarray(x), list(tr.loss), list(tr.lower_iters_cum), list(tr.cg_iters_cum)

    a = _with_cluster(nat, True, run)
    b = _with_cluster(nat, False, run)
    assert a[3] == b[3] and a[4] == b[4] and a[2] == b[2]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
