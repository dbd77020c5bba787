"""Leaf-aligned ("fused") layouts: NumPy-pairwise leaves computed inside the
tiles, and the fused candidate-value + speculative next-stage-A pass
(ConvGeom.fuseCA).  The 2-D fixtures elsewhere are not leaf-aligned, so these
tests pin the fused kernels directly:
  * strict solve trajectories bitwise equal to the CPU oracle (the bitwise
    restatement of the reference),
  * the fused pass bitwise equal to the unfused stage order (ADP_FUSECA=0),
  * fast and fp32 modes within their tolerances."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [((256, 256, 1), 9, 60), ((128, 128, 3), 15, 30)]


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _case(shape, K, seed=0):
    from paper_2502_09758_b200 import configs
    rng = np.random.default_rng(seed)
    k = configs.gaussian_kernel_2d(K, 1.0 + K / 6.0, shape[2]).data
    y = rng.uniform(0.0, 1.0, shape)
    return k, y


def _solve(adp, k, y, iters, stats=None):
    p = adp.LowerProblem(adp.ConvOperator(adp.Kernel(k, adp.DEPTHWISE2D), y.shape), y, 0.6, adp.SmoothedTV(1e-4))
    return adp.solve_lower(p, y, 1e-14, 10.0, max_iters=iters, method="agd", adaptive=True, stats=stats)


@pytest.mark.parametrize("shape,K,iters", CASES)
def test_fused_layout_strict_solve_bitwise_vs_oracle(adp, orc, shape, K, iters):
    from paper_2502_09758_b200 import _native as nat
    k, y = _case(shape, K)
    plan = nat.plan_for(nat.LAYOUT_DEPTHWISE2D, shape, (K, K))
    assert plan.geometry()["fused"] == 1
    st = {}
    r = _solve(adp, k, y, iters, st)
    x_o, gn_o, it_o, conv_o = orc.solve_lower(orc.Lower(orc.Conv(k, shape), y, 0.6, orc.TV(1e-4)), y, 1e-14, 10.0,
                                              max_iters=iters, method="agd", adaptive=True)
    assert r.iters == it_o
    if shape[2] == 1:
        assert st["value_evals"] > iters   # backtracking retries (speculation discarded) happened
    assert np.array_equal(r.x_tilde, x_o)
    assert r.grad_norm == gn_o or abs(r.grad_norm - gn_o) <= 1e-12 * gn_o   # ddot site


@pytest.mark.parametrize("shape,K,iters", CASES)
def test_fused_candidate_pass_equals_unfused(adp, shape, K, iters):
    from paper_2502_09758_b200 import _native as nat
    k, y = _case(shape, K, seed=1)
    st1 = {}
    r1 = _solve(adp, k, y, iters, st1)
    old = os.environ.get("ADP_FUSECA")
    os.environ["ADP_FUSECA"] = "0"
    try:
        nat.clear_plans()
        st0 = {}
        r0 = _solve(adp, k, y, iters, st0)
    finally:
        if old is None:
            del os.environ["ADP_FUSECA"]
        else:
            os.environ["ADP_FUSECA"] = old
        nat.clear_plans()
    assert np.array_equal(r1.x_tilde, r0.x_tilde) and r1.grad_norm == r0.grad_norm
    assert st1 == st0


@pytest.mark.parametrize("shape,K,iters", CASES)
def test_fused_layout_fast_and_fp32(adp, shape, K, iters):
    k, y = _case(shape, K, seed=2)
    ref = _solve(adp, k, y, iters)
    with adp.precision("float64", "fast"):
        rf = _solve(adp, k, y, iters)
    # trajectories: per-primitive 1e-13 (fast) / 1e-4 (fp32) accumulated over
    # 30-60 accelerated iterations
    assert rel(rf.x_tilde, ref.x_tilde) <= 1e-7
    with adp.precision("float32", "fast"):
        r32 = _solve(adp, k, y, iters)
    # fp32 with TV nu = 1e-4 (nu^2 at fp32 resolution against d^2): the
    # iterates separate pixel-wise; the objective reached after 30-60
    # iterations agrees to 5e-4 (fp32 primitives themselves are within 1e-4)
    p = adp.LowerProblem(adp.ConvOperator(adp.Kernel(k, adp.DEPTHWISE2D), y.shape), y, 0.6, adp.SmoothedTV(1e-4))
    h64 = adp.lower_value(p, ref.x_tilde)
    h32 = adp.lower_value(p, np.asarray(r32.x_tilde, dtype=float))
    assert abs(h32 - h64) <= 5e-4 * abs(h64), (h32, h64)
