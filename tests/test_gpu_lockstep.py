"""P2 lockstep parity: the oracle's state at the start
of lower iteration k — (x, x_prev, t_mom, lip_t) — is injected into ONE
iteration of the production solve kernel (adp_lower_iter / lower_iteration),
whose output must match the oracle's state at iteration k + 1 with identical
decisions (backtracking retries, restart).  Strict mode: bitwise; fast:
1e-12; fft: 1e-11; fp32: 1e-4 (relative to the image scale)."""
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _record(orc, shape, k, seed, iters):
    rng = np.random.default_rng(seed)
    g = np.arange(k) - k // 2
    w = np.exp(-(g[:, None] ** 2 + g[None, :] ** 2) / (2 * (k / 4.0) ** 2))
    kern = np.repeat(w[:, :, None], shape[2], axis=2) * rng.uniform(0.7, 1.3, (k, k, shape[2]))
    kern /= kern.sum(axis=(0, 1), keepdims=True)
    xt = np.clip(np.cumsum(rng.standard_normal(shape), axis=0) * 0.05 + 0.5, 0, 1)
    y = orc.correlate(xt, kern) + 0.01 * rng.standard_normal(shape)
    po = orc.Lower(orc.Conv(kern, shape), y, 0.6, orc.TV(1e-4))
    rec = types.SimpleNamespace(gn=[], h_y=[], bt_tries=[], restart=[], states=[])
    orc.solve_lower(po, y, 1e-14, 10.0, max_iters=iters, method="agd", adaptive=True, record=rec)
    lam = po.op.norm_sq
    return kern, y, rec, lam


CASES = [("strict", (96, 80, 1), 9, 0.0), ("fast", (96, 80, 1), 9, 1e-12), ("fft", (90, 70, 3), 15, 1e-11),
         ("fp32", (96, 80, 1), 9, 1e-4), ("strict", (60, 64, 3), 15, 0.0)]


@pytest.mark.parametrize("mode,shape,k,tol", CASES)
def test_lower_iteration_lockstep(adp, orc, mode, shape, k, tol):
    kern, y, rec, lam = _record(orc, shape, k, 21 + k, 60)
    dtype, m = ("float32", "fast") if mode == "fp32" else ("float64", mode)
    with adp.precision(dtype, m):
        p = adp.LowerProblem(adp.ConvOperator(adp.Kernel(kern, adp.DEPTHWISE2D), shape), y, 0.6,
                             adp.SmoothedTV(1e-4))
        p.op._norm_sq = lam
        checked = retries = restarts = 0
        for it in range(0, 59, 3):
            x, xp, t_mom, lip_t = rec.states[it]
            out = adp.lower_iteration(p, x, xp, t_mom, lip_t, 1e-14, 10.0, adaptive=True)
            xn, xpn, tn, ln = rec.states[it + 1]
            assert out["bt_tries"] == rec.bt_tries[it], it
            assert out["restart"] == rec.restart[it], it
            assert out["t_mom"] == tn and out["lip_t"] == ln, it
            if tol == 0.0:
                assert np.array_equal(out["x"], xn), it
            else:
                assert rel(out["x"], xn) <= tol, (it, rel(out["x"], xn))
            retries += rec.bt_tries[it]
            restarts += rec.restart[it]
            checked += 1
    assert checked == 20 and retries > 0


@pytest.mark.parametrize("mode,tol", [("strict", 1e-11), ("fast", 1e-11)])
def test_cg_iteration_lockstep(adp, orc, mode, tol):
    """One Jacobi-PCG iteration of the production CG kernel from the oracle's
    state (q, r, p, rs) at iteration k reproduces the oracle's (q, r, rs) at
    k + 1 and its curvature <p, Hp>; the Jacobi diagonal (np.power in rho'')
    and the ddot order are tolerance sites (App. B), so the bar is 1e-11."""
    from paper_2502_09758_b200.hypergradient import cg_iteration
    shape, k = (80, 72, 2), 9
    kern, y, rec, lam = _record(orc, shape, k, 5, 5)
    rng = np.random.default_rng(3)
    xt = y + 0.02 * rng.standard_normal(shape)
    rhs = rng.standard_normal(shape)
    po = orc.Lower(orc.Conv(kern, shape), y, 0.6, orc.TV(1e-4))
    states = []
    orc.cg_solve(lambda v: orc.lower_hess_vec(po, xt, v), rhs, 1e-30, 30,
                 precond_diag=orc.lower_hess_diag(po, xt), record=states)
    with adp.precision("float64", mode):
        p = adp.LowerProblem(adp.ConvOperator(adp.Kernel(kern, adp.DEPTHWISE2D), shape), y, 0.6,
                             adp.SmoothedTV(1e-4))
        for it in (0, 1, 7, 18, 28):
            q, r, pd, rs, curv = states[it]
            out = cg_iteration(p, xt, q, r, pd, rs)
            qn, rn, _, rsn, _ = states[it + 1]
            assert abs(out["curv"] - curv) <= tol * abs(curv), it
            assert abs(out["rs"] - rsn) <= tol * abs(rsn), it
            assert rel(out["q"], qn) <= tol and rel(out["r"], rn) <= tol, it


@pytest.mark.parametrize("name,iters,check", [("c2", 30, (0, 7, 19, 28)), ("c3", 5, (1, 3))])
def test_lower_iteration_lockstep_at_config_shapes(adp, orc, name, iters, check):
    """P2 at the BASELINE config shapes (c2 256x256x1 K = 9, c3 512x512x3 K = 15)
    on the config's own data and initial kernel: strict mode bitwise."""
    from paper_2502_09758_b200 import configs
    up = configs.CONFIGS[name](0)
    y = np.asarray(up.y_delta, dtype=float)
    kern = up.b0.data
    po = orc.Lower(orc.Conv(kern, y.shape), y, up.alpha, orc.TV(up.reg.nu))
    rec = types.SimpleNamespace(gn=[], h_y=[], bt_tries=[], restart=[], states=[])
    orc.solve_lower(po, y, 1e-14, 10.0, max_iters=iters + 1, method="agd", adaptive=True, record=rec)
    p = up.lower_problem(up.b0)
    p.op._norm_sq = po.op.norm_sq
    for it in check:
        x, xp, t_mom, lip_t = rec.states[it]
        out = adp.lower_iteration(p, x, xp, t_mom, lip_t, 1e-14, 10.0, adaptive=True)
        xn, _, tn, ln = rec.states[it + 1]
        assert out["bt_tries"] == rec.bt_tries[it] and out["restart"] == rec.restart[it], it
        assert out["t_mom"] == tn and out["lip_t"] == ln, it
        assert np.array_equal(out["x"], xn), it
