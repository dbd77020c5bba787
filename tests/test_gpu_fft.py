"""FFT stencil mode: overlap-save tile FFTs for the
depthwise correlation, the lower objective and the AGD solve.  A tolerance
mode: primitives within 1e-12 of the reference arithmetic (CPU oracle =
scipy.ndimage order, pinned to the real reference), short solves within
1e-9, long solves to the same objective; fixed-order reductions make every
run bitwise reproducible."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def gauss(k, sigma, c, rng=None):
    g = np.arange(k) - k // 2
    w = np.exp(-(g[:, None] ** 2 + g[None, :] ** 2) / (2 * sigma**2))
    w = np.repeat(w[:, :, None], c, axis=2)
    if rng is not None:
        w = w * rng.uniform(0.5, 1.5, w.shape)
    return w / w.sum(axis=(0, 1), keepdims=True)


# (shape, K): single tile / one pair; 2 x 3 tiles (3 full pairs); 3 tiles (a pair with an empty slot);
# K = 31 at the c5 tile geometry; non-square kernel
CASES = [((100, 90, 3), (9, 9)), ((500, 1000, 1), (31, 31)), ((700, 300, 2), (15, 15)),
         ((600, 620, 3), (31, 31)), ((257, 129, 1), (5, 11))]


@pytest.fixture(autouse=True)
def fft_mode(adp):
    with adp.precision("float64", "fft"):
        yield


@pytest.mark.parametrize("shape,ks", CASES)
def test_fft_apply_adjoint(adp, orc, shape, ks):
    rng = np.random.default_rng(shape[0] + ks[0])
    kern = rng.uniform(0.0, 1.0, ks + (shape[2],))
    kern /= kern.sum(axis=(0, 1), keepdims=True)
    x = rng.uniform(0.0, 1.0, shape)
    v = rng.standard_normal(shape)
    op = adp.ConvOperator(adp.Kernel(kern, adp.DEPTHWISE2D), shape)
    bx, btv = op.apply(x), op.adjoint(v)
    assert rel(bx, orc.correlate(x, kern)) <= 1e-13
    assert rel(btv, orc.correlate(v, kern, flip=True)) <= 1e-13
    lhs, rhs = float(np.vdot(bx, v)), float(np.vdot(x, btv))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    assert np.array_equal(op.apply(x), bx)           # bitwise reproducible


def _problem(adp, orc, shape, k, sigma, seed):
    rng = np.random.default_rng(seed)
    kern = gauss(k, sigma, shape[2], rng)
    xt = rng.uniform(0.0, 1.0, shape)
    y = orc.correlate(xt, kern) + 0.01 * rng.standard_normal(shape)
    p = adp.LowerProblem(adp.ConvOperator(adp.Kernel(kern, adp.DEPTHWISE2D), shape), y, 0.6, adp.SmoothedTV(1e-4))
    po = orc.Lower(orc.Conv(kern, shape), y, 0.6, orc.TV(1e-4))
    return p, po, y, rng


@pytest.mark.parametrize("shape,k", [((300, 260, 3), 15), ((520, 500, 1), 31)])
def test_fft_lower_objective(adp, orc, shape, k):
    p, po, y, rng = _problem(adp, orc, shape, k, k / 5.0, 5)
    x = y + 0.05 * rng.standard_normal(shape)
    v, g = adp.lower_value_and_grad(p, x)
    vo, go = orc.lower_value_and_grad(po, x)
    assert abs(v - vo) <= 1e-12 * abs(vo)
    assert rel(g, go) <= 1e-11
    assert abs(adp.lower_value(p, x) - orc.lower_value(po, x)) <= 1e-12 * abs(vo)
    assert rel(adp.lower_grad(p, x), go) <= 1e-11


def test_fft_op_norm_sq(adp, orc):
    shape = (200, 230, 2)
    rng = np.random.default_rng(2)
    kern = gauss(31, 6.0, 2, rng)
    op = adp.ConvOperator(adp.Kernel(kern, adp.DEPTHWISE2D), shape)
    lam = adp.op_norm_sq(op, 300, 1e-4)
    lam_o, _, _ = orc.op_norm_sq(orc.Conv(kern, shape), 300, 1e-4)
    assert abs(lam - lam_o) <= 1e-10 * lam_o


@pytest.mark.parametrize("shape,k,iters", [((160, 150, 3), 15, 12), ((300, 280, 1), 31, 12)])
def test_fft_solve_short_matches_oracle(adp, orc, shape, k, iters):
    """A few adaptive-AGD iterations: FFT rounding (1e-15) has not grown yet."""
    p, po, y, _ = _problem(adp, orc, shape, k, k / 5.0, 9)
    res = adp.solve_lower(p, y, 1e-12, 10.0, max_iters=iters, method="agd", adaptive=True)
    xo, gno, it_o, _ = orc.solve_lower(po, y, 1e-12, 10.0, max_iters=iters, method="agd", adaptive=True)
    assert res.iters == it_o == iters
    assert rel(res.x_tilde, xo) <= 1e-9
    assert abs(res.grad_norm - gno) <= 1e-7 * gno


def test_fft_solve_long_objective_and_determinism(adp, orc):
    """300 iterations: pixel trajectories separate at the TV's sensitivity
    (SURVEY.md App. C), the objective reached agrees with the direct (fast)
    device solve; two FFT runs are bitwise identical."""
    shape, k = (256, 256, 1), 31
    p, po, y, _ = _problem(adp, orc, shape, k, 6.0, 4)
    r1 = adp.solve_lower(p, y, 1e-9, 10.0, max_iters=300, method="agd", adaptive=True)
    r2 = adp.solve_lower(p, y, 1e-9, 10.0, max_iters=300, method="agd", adaptive=True)
    assert np.array_equal(r1.x_tilde, r2.x_tilde) and r1.grad_norm == r2.grad_norm
    with adp.precision("float64", "fast"):
        p2 = adp.LowerProblem(adp.ConvOperator(p.op.kernel, shape), y, 0.6, adp.SmoothedTV(1e-4))
        rd = adp.solve_lower(p2, y, 1e-9, 10.0, max_iters=300, method="agd", adaptive=True)
        hd = adp.lower_value(p2, rd.x_tilde)
    h1 = orc.lower_value(po, r1.x_tilde)
    assert abs(h1 - hd) <= 1e-6 * abs(hd)
    assert rel(r1.x_tilde, rd.x_tilde) <= 1e-3


def test_fft_solve_methods_and_errors(adp, orc):
    shape = (120, 100, 2)
    p, po, y, _ = _problem(adp, orc, shape, 9, 2.0, 3)
    for method, adaptive in (("proxgrad", False), ("proxgrad", True), ("agd", False), ("fista_sc", True)):
        r = adp.solve_lower(p, y, 1e-12, 10.0, max_iters=8, method=method, adaptive=adaptive)
        xo, gno, it_o, _ = orc.solve_lower(po, y, 1e-12, 10.0, max_iters=8, method=method, adaptive=adaptive)
        assert r.iters == it_o
        assert rel(r.x_tilde, xo) <= 1e-9, method
    # converged solve returns the extrapolated point and its iteration index
    _, gn10, _, _ = orc.solve_lower(po, y, 1e-12, 10.0, max_iters=10, adaptive=True)
    eps = 1.5 * gn10 / 10.0
    r = adp.solve_lower(p, y, eps, 10.0, max_iters=50, adaptive=True)
    xo, gno, it_o, conv = orc.solve_lower(po, y, eps, 10.0, max_iters=50, adaptive=True)
    assert conv and r.converged and r.iters == it_o < 10
    assert rel(r.x_tilde, xo) <= 1e-9
    with pytest.raises(ValueError):
        adp.set_precision("float32", "fft")


@pytest.mark.parametrize("warm", [False, True])
def test_fft_hess_cg_matches_oracle(adp, orc, warm):
    """Jacobi-PCG on the lower Hessian with FFT Hessian products (the TV
    curvature term in the stencil epilogue, the SAT-based gram diagonal):
    a few iterations track the oracle's cg_solve before the TV Hessian's
    conditioning amplifies rounding (DESIGN.md, 2-D hypergradient)."""
    from paper_2502_09758_b200.hypergradient import hess_cg
    shape = (150, 140, 2)
    p, po, y, rng = _problem(adp, orc, shape, 15, 3.0, 6)
    xt = y + 0.02 * rng.standard_normal(shape)
    rhs = rng.standard_normal(shape)
    q0 = 0.01 * rng.standard_normal(shape) if warm else None
    cg, hv = hess_cg(p, xt, rhs, 1e-30, 6, q0=q0)
    qo, res_o, it_o, _ = orc.cg_solve(lambda v: orc.lower_hess_vec(po, xt, v), rhs, 1e-30, 6, x0=q0,
                                      precond_diag=orc.lower_hess_diag(po, xt))
    assert cg.iters == it_o == 6
    assert rel(cg.q.cpu().numpy(), qo) <= 1e-8
    assert abs(cg.residual - res_o) <= 1e-6 * res_o
    assert hv == 6 + 1 + (1 if warm else 0)
    # converged solve on an easy tolerance: same stopping iteration
    tol = 0.5 * float(np.linalg.norm(rhs))
    cg2, _ = hess_cg(p, xt, rhs, tol, 50)
    q2, r2, it2, conv2 = orc.cg_solve(lambda v: orc.lower_hess_vec(po, xt, v), rhs, tol, 50,
                                      precond_diag=orc.lower_hess_diag(po, xt))
    assert cg2.iters == it2 and cg2.converged == conv2


def test_fft_inexact_hypergradient_runs_and_agrees(adp, orc):
    """Algorithm 1 end to end in fft mode on a small semi-blind problem: the
    hypergradient agrees with the direct (fast) pipeline to the tolerance the
    inexact solves allow."""
    from paper_2502_09758_b200 import configs
    up = configs.config3(0, size=96)
    st = adp.WarmState(x=up.x0.copy(), q=None)
    h = adp.inexact_hypergradient(up, up.b0, 1e-3, 1e-3, st, cg_max_iters=15)
    with adp.precision("float64", "fast"):
        st2 = adp.WarmState(x=up.x0.copy(), q=None)
        h2 = adp.inexact_hypergradient(up, up.b0, 1e-3, 1e-3, st2, cg_max_iters=15)
    assert h.cg_iters == h2.cg_iters
    # the 1,200-iteration lower solves stop short of eps = 1e-3 in both modes and their pixel
    # trajectories separate at the TV's sensitivity: agreement is to the
    # percent level; the fft pipeline itself is bitwise reproducible
    assert np.isfinite(h.z).all() and rel(h.z, h2.z) <= 5e-2
    st3 = adp.WarmState(x=up.x0.copy(), q=None)
    h3 = adp.inexact_hypergradient(up, up.b0, 1e-3, 1e-3, st3, cg_max_iters=15)
    assert np.array_equal(h3.z, h.z)


def test_fft_upper_terms(adp, orc):
    """fit_value and upper_fit_grad (problems.py:48-50, hypergradient.py:87-89) on FFT stencils."""
    from paper_2502_09758_b200.hypergradient import _upper_terms
    shape = (300, 200, 3)
    rng = np.random.default_rng(8)
    kern = gauss(31, 6.0, 3, rng)
    A = adp.ConvOperator(adp.Kernel(kern, adp.DEPTHWISE2D), shape)
    x, yd = rng.uniform(0, 1, shape), rng.uniform(0, 1, shape)
    fit, gn, g = _upper_terms(A, x, yd, want_grad=True)
    Ao = orc.Conv(kern, shape)
    r = Ao.apply(x) - yd
    go = orc.upper_fit_grad(x, Ao, yd)
    assert abs(fit - orc.npsum(r * r)) <= 1e-12 * fit
    assert rel(g.cpu().numpy(), go) <= 1e-12
    assert abs(gn - orc.norm(go)) <= 1e-12 * gn


@pytest.mark.parametrize("shape,k", [((300, 260, 3), 15), ((600, 520, 1), 31), ((100, 90, 2), 9)])
def test_fft_mixed_second_transpose(adp, orc, shape, k):
    """2 [kgc(x~, Bq) + kgc(q, Bx~ - y)] from frequency-domain pair products vs the oracle."""
    p, po, y, rng = _problem(adp, orc, shape, k, k / 5.0, 12)
    xt = y + 0.02 * rng.standard_normal(shape)
    q = rng.standard_normal(shape)
    z = adp.mixed_second_transpose(xt, p.op.kernel, q, p)
    zo = orc.mixed_second_transpose(xt, q, po, False, (k, k))
    assert z.shape == zo.shape
    assert rel(z, zo) <= 1e-11


def test_fft_maid_run_end_to_end(adp):
    """MAID in fft mode (every image-space call on tile-FFT stencils: lower
    solves, CG, mixed derivative, upper terms) on a c2-type instance with the
    BASELINE MAID settings: two accepted steps that decrease the upper loss,
    final loss close to the strict run's."""
    from dataclasses import replace

    from paper_2502_09758_b200 import configs
    cfg = replace(configs.maid_config("c2"), max_upper_iters=2)
    up = configs.config2(0, size=128)
    b, x, tr = adp.maid_run(up, cfg)
    assert len(tr) == 2 and np.isfinite(tr.loss).all() and np.isfinite(x).all()
    assert tr.final_loss < tr.loss[0]
    with adp.precision("float64", "strict"):
        b2, x2, tr2 = adp.maid_run(configs.config2(0, size=128), cfg)
    assert abs(tr.final_loss - tr2.final_loss) <= 1e-3 * tr2.final_loss


@pytest.mark.parametrize("shape,ks", [((5, 7, 1), (9, 9)), ((1, 40, 2), (3, 5)), ((33, 1, 4), (7, 1)),
                                      ((483, 482, 1), (31, 31)), ((964, 20, 2), (31, 31)), ((2, 2, 3), (1, 1))])
def test_fft_edge_geometries(adp, orc, shape, ks):
    """Images smaller than the kernel, single rows/columns, 1x1 kernels, tile
    counts at the valid-region boundary (482 = 512 - 31 + 1) and odd tile counts."""
    rng = np.random.default_rng(sum(shape) + ks[0])
    kern = rng.uniform(-0.5, 1.0, ks + (shape[2],))
    x = rng.standard_normal(shape)
    op = adp.ConvOperator(adp.Kernel(kern, adp.DEPTHWISE2D), shape)
    assert rel(op.apply(x), orc.correlate(x, kern)) <= 1e-13
    assert rel(op.adjoint(x), orc.correlate(x, kern, flip=True)) <= 1e-13
