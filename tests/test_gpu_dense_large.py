"""The dense 1-D engine beyond shared-memory capacity (n = 4096: the
replicated signal vectors move to global memory): operator, objective and
solve against the CPU oracle (OpenBLAS dgemv order is a tolerance site)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def test_dense_4096(adp, orc):
    up = adp.build_deconv1d(seed=1, n=4096)
    resid = up.y_delta - up.A.apply(up.ground_truth)
    assert abs(np.std(resid) - 5e-3) <= 0.05 * 5e-3          # reference tests/test_problems.py:88-91
    m = np.array(up.A.matrix)
    x = np.random.default_rng(0).standard_normal(4096)
    assert rel(up.A.apply(x), m @ x) <= 1e-13
    assert rel(up.A.adjoint(x), m.T @ x) <= 1e-13
    p = up.lower_problem(up.b0)
    po = orc.Lower(orc.Dense(m), up.y_delta, 1.0, orc.ElasticNet(1.2e-3, 4e-3, 1e-4))
    v, g = adp.lower_value_and_grad(p, x)
    vo, go = orc.lower_value_and_grad(po, x)
    assert abs(v - vo) <= 1e-12 * abs(vo) and rel(g, go) <= 1e-12
    r = adp.solve_lower(p, up.x0, 1e-6, adp.mu_of_b(p, up.mu_floor), max_iters=40)
    xo, gno, ito, _ = orc.solve_lower(po, up.x0, 1e-6, adp.mu_of_b(p, up.mu_floor), max_iters=40)
    assert r.iters == ito and rel(r.x_tilde, xo) <= 1e-9
