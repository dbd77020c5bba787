"""Device solvers vs the reference (golden fixtures) and vs the CPU oracle.

Tolerances (north star): float64 within 1e-9 relative on iterates and
hypergradients, identical integer outputs (iterations, accepted steps).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def semiblind_problem(adp, d):
    shape = d["y_delta"].shape
    op = adp.ConvOperator(adp.Kernel(d["kern"], adp.DEPTHWISE2D), shape)
    return adp.LowerProblem(op, d["y_delta"], 0.6, adp.SmoothedTV(1e-4))


@pytest.mark.parametrize("tag,method,adaptive", [("agd_ad", "agd", True), ("agd_ad_conv", "agd", True),
                                                 ("gd_ad", "proxgrad", True), ("fista", "fista_sc", True),
                                                 ("agd_fixed", "agd", False)])
def test_solve_lower_2d_vs_reference(adp, golden, tag, method, adaptive):
    d = golden("solve2d.npz")
    eps, mu, iters = d[f"{tag}_args"]
    p = semiblind_problem(adp, d)
    r = adp.solve_lower(p, d["x0"], float(eps), float(mu), max_iters=int(iters), method=method, adaptive=adaptive)
    assert r.iters == int(d[f"{tag}_iters"])
    assert r.converged == bool(d[f"{tag}_conv"])
    assert rel(r.x_tilde, d[f"{tag}_x"]) <= 1e-9
    assert abs(r.grad_norm - float(d[f"{tag}_gn"])) <= 1e-9 * float(d[f"{tag}_gn"])


def test_solve_lower_2d_strict_is_bitwise(adp, golden):
    """Strict mode: identical stencils, np.sum trees and elementwise order
    make the whole adaptive AGD trajectory bit-identical to the reference
    (decisions only see ddot rounding, far from their margins here)."""
    d = golden("solve2d.npz")
    eps, mu, iters = d["agd_ad_args"]
    p = semiblind_problem(adp, d)
    r = adp.solve_lower(p, d["x0"], float(eps), float(mu), max_iters=int(iters), method="agd", adaptive=True)
    assert np.array_equal(r.x_tilde, d["agd_ad_x"])


def test_solve_lower_c2_small_vs_reference(adp, golden):
    d = golden("c2_small.npz")
    shape = d["y_delta"].shape
    op = adp.ConvOperator(adp.Kernel(d["a"], adp.DEPTHWISE2D), shape)
    p = adp.LowerProblem(op, d["y_delta"], 0.6, adp.SmoothedTV(1e-4))
    r = adp.solve_lower(p, d["y_delta"], 0.25, 10.0, max_iters=1200, method="agd", adaptive=True)
    assert r.iters == int(d["solve_iters"])
    assert r.converged == bool(d["solve_conv"])
    assert rel(r.x_tilde, d["solve_x"]) <= 1e-9


def test_cg_and_hypergradient_2d(adp, golden):
    d = golden("hyper2d.npz")
    shape = d["y_delta"].shape
    b = adp.Kernel(d["kern"], adp.DEPTHWISE2D)
    A = adp.ConvOperator(adp.Kernel(d["a_kern"], adp.DEPTHWISE2D), shape)
    up = adp.UpperProblem(name="s", A=A, a=adp.Kernel(d["a_kern"], adp.DEPTHWISE2D), y_delta=d["y_delta"],
                          beta=0.3, alpha=0.6, reg=adp.SmoothedTV(1e-4), b0=b, x0=d["x0"], mu_floor=1e-3,
                          lower_method="agd", lower_max_iters=300, lower_adaptive=True)
    st = adp.WarmState(x=d["x0"].copy())
    hg = adp.inexact_hypergradient(up, b, 0.5, 0.5, st, cg_max_iters=60)
    assert hg.lower_iters == int(d["lower_iters"])
    assert hg.cg_iters == int(d["cg_iters"])
    assert rel(hg.x_tilde, d["x_tilde"]) <= 1e-9
    assert abs(up.fit_value(d["x_tilde"]) - float(d["fit"])) == 0.0
    assert abs(up.loss(d["x_tilde"], b) - float(d["loss"])) == 0.0
    # P3 lockstep: given the reference's q, z = -mixed(x~, q) + grad r(b) within 1e-9
    p = up.lower_problem(b)
    z_ref_q = -adp.mixed_second_transpose(d["x_tilde"], b, d["q"], p) + adp.sobolev_grad(b, up.a, 0.3)
    assert rel(z_ref_q, d["z"]) <= 1e-9
    # Past ~20 iterations this PCG (TV Hessian, nu = 1e-4) amplifies last-bit
    # ddot differences to ~1e-3 (tools/diag_cg.py: the CPU oracle with a
    # different valid ddot order spreads the same way); full-run z is
    # therefore compared in the stable regime (15 CG iterations) at 1e-9.
    d15 = golden("hyper2d_cg15.npz")
    st = adp.WarmState(x=d["x0"].copy())
    hg15 = adp.inexact_hypergradient(up, b, 0.5, 0.5, st, cg_max_iters=15)
    assert hg15.cg_iters == int(d15["cg_iters"])
    assert rel(hg15.z, d15["z"]) <= 1e-9
    assert rel(st.q, d15["q"]) <= 1e-9
    assert abs(hg15.cg_residual - float(d15["cg_residual"])) <= 1e-9 * float(d15["cg_residual"])
    # generic cg_solve with a caller-supplied (numpy) hess_vec, stable regime
    cg = adp.cg_solve(lambda v: adp.lower_hess_vec(p, d["x_tilde"], v), d["rhs"], 1e-3, max_iters=15,
                      precond_diag=adp.lower_hess_diag(p, d["x_tilde"]))
    assert cg.iters == 15
    import adp_oracle as orc
    po = orc.Lower(orc.Conv(d["kern"], shape), d["y_delta"], 0.6, orc.TV(1e-4))
    qo, reso, ito, _ = orc.cg_solve(lambda v: orc.lower_hess_vec(po, d["x_tilde"], v), d["rhs"], 1e-3, 15, None,
                                    orc.lower_hess_diag(po, d["x_tilde"]))
    assert rel(cg.q, qo) <= 1e-9 and abs(cg.residual - reso) <= 1e-9 * reso


def test_dense_solve_hypergradient_maid(adp, golden):
    d = golden("dense1d_run.npz")
    up = adp.build_deconv1d(seed=1, n=80, num_pieces=5)
    assert np.array_equal(up.y_delta, d["y_delta"])
    p = up.lower_problem(up.b0)
    mu = adp.mu_of_b(p, up.mu_floor)
    r = adp.solve_lower(p, up.x0, 1e-6, mu, max_iters=300)
    assert r.iters == int(d["solve_iters"])
    assert rel(r.x_tilde, d["solve_x"]) <= 1e-9
    st = adp.WarmState(x=up.x0.copy())
    hg = adp.inexact_hypergradient(up, up.b0, 1e-2, 1e-2, st, cg_max_iters=200)
    assert hg.lower_iters == int(d["hg_lower_iters"]) and hg.cg_iters == int(d["hg_cg_iters"])
    assert rel(hg.z, d["z"]) <= 1e-9
    b, x, tr = adp.maid_run(up, adp.MAIDConfig(max_upper_iters=8))
    assert tr.lower_iters_cum == [int(v) for v in d["maid_lower_cum"]]
    assert tr.cg_iters_cum == [int(v) for v in d["maid_cg_cum"]]
    assert np.allclose(tr.alpha, d["maid_alpha"], rtol=1e-12, atol=0)
    assert rel(tr.loss, d["maid_loss"]) <= 1e-9
    assert rel(b.data, d["maid_b"]) <= 1e-9
    assert rel(x, d["maid_x"]) <= 1e-9


def test_config1_full_maid_run(adp, golden):
    """BASELINE c1 end to end: integer trace identical, loss / alpha / b / x
    within 1e-9."""
    from paper_2502_09758_b200 import configs
    d = golden("c1_maid.npz")
    up = configs.config1(0)
    assert np.array_equal(up.y_delta, d["y_delta"])
    b, x, tr = adp.maid_run(up, configs.maid_config("c1"))
    assert len(tr) == len(d["maid_loss"])
    assert tr.lower_iters_cum == [int(v) for v in d["maid_lower_cum"]]
    assert tr.cg_iters_cum == [int(v) for v in d["maid_cg_cum"]]
    e = {"alpha": rel(tr.alpha, d["maid_alpha"]), "loss": rel(tr.loss, d["maid_loss"]),
         "b": rel(b.data, d["maid_b"]), "x": rel(x, d["maid_x"]), "final": abs(tr.final_loss - float(d["maid_final"]))
         / abs(float(d["maid_final"]))}
    from _report import report
    report("c1_full_maid_run", **e)
    assert e["alpha"] <= 1e-12
    assert e["loss"] <= 1e-9 and e["final"] <= 1e-9
    assert e["b"] <= 1e-9
    # x: 1e-9 as the north star asks; SURVEY App. C measured the reference's own x reproducibility under
    # 1e-15 input noise at up to 1.06e-9 on c1, so the measured value is reported (parity_report.jsonl)
    assert e["x"] <= 1e-9, e["x"]
