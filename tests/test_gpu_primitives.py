"""Device primitives vs the REAL reference's outputs (golden fixtures made by
tests/golden/make_golden.py from /root/reference).

Strict float64 mode claims bit-exactness wherever the reference's arithmetic
is deterministic (scipy.ndimage stencils, np.sum sites, elementwise NumPy);
ddot / dgemv / np.power sites are compared with the tolerance written in each
test.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CONV = ["conv_small.npz", "conv_k9.npz", "conv_k15.npz"]


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def conv_problem(adp, d):
    shape = d["x"].shape
    op = adp.ConvOperator(adp.Kernel(d["kern"], adp.DEPTHWISE2D), shape)
    return adp.LowerProblem(op, d["y"], float(d["alpha"]), adp.SmoothedTV(float(d["nu"])))


@pytest.mark.parametrize("name", CONV)
def test_conv_operator_bitwise(adp, golden, name):
    d = golden(name)
    p = conv_problem(adp, d)
    assert np.array_equal(p.op.apply(d["x"]), d["apply"])
    assert np.array_equal(p.op.adjoint(d["v"]), d["adjoint"])
    assert np.array_equal(p.op.gram_diag(), d["gram_diag"])


@pytest.mark.parametrize("name", CONV)
def test_conv_lower_value_grad_bitwise(adp, golden, name):
    d = golden(name)
    p = conv_problem(adp, d)
    assert adp.lower_value(p, d["x"]) == float(d["lower_value"])
    val, g = adp.lower_value_and_grad(p, d["x"])
    assert val == float(d["vg_val"])
    assert np.array_equal(g, d["vg_g"])
    assert np.array_equal(adp.lower_grad(p, d["x"]), d["lower_grad"])


@pytest.mark.parametrize("name", CONV)
def test_conv_tv_methods(adp, golden, name):
    d = golden(name)
    reg = adp.SmoothedTV(float(d["nu"]))
    assert reg.value(d["x"]) == float(d["tv_value"])
    v, g = reg.value_and_grad(d["x"])
    assert v == float(d["tv_vg_val"]) and np.array_equal(g, d["tv_vg_g"])
    assert np.array_equal(reg.grad(d["x"]), d["tv_grad"])
    # rho'' uses np.power (SVML on the reference host) vs CUDA: tolerance 1e-13
    assert rel(reg.hess_vec(d["x"], d["v"]), d["tv_hess_vec"]) <= 1e-13
    assert rel(reg.hess_diag(d["x"]), d["tv_hess_diag"]) <= 1e-13


@pytest.mark.parametrize("name", CONV)
def test_conv_hessian_and_mixed(adp, golden, name):
    d = golden(name)
    p = conv_problem(adp, d)
    assert rel(adp.lower_hess_vec(p, d["x"], d["v"]), d["hess_vec"]) <= 1e-13
    assert rel(adp.lower_hess_diag(p, d["x"]), d["hess_diag"]) <= 1e-13
    # kernel-gram correlations: fixed-order device reduction vs np.sum: 1e-12
    assert rel(adp.kernel_gram_correlation(d["x"], d["v"], p.op.kernel), d["kgc"]) <= 1e-12
    assert rel(adp.mixed_second_transpose(d["x"], p.op.kernel, d["v"], p), d["mixed"]) <= 1e-12


@pytest.mark.parametrize("name", CONV)
def test_conv_power_iteration(adp, golden, name):
    d = golden(name)
    op = adp.ConvOperator(adp.Kernel(d["kern"], adp.DEPTHWISE2D), d["x"].shape)
    lam = adp.op_norm_sq(op, 300, 1e-4)
    assert abs(lam - float(d["norm_sq"])) <= 1e-12 * float(d["norm_sq"])


def test_dense_primitives(adp, golden):
    d = golden("dense_small.npz")
    op = adp.DenseOperator(d["m"])
    reg = adp.SmoothedElasticNet(float(d["l1"]), float(d["l2"]), float(d["nu"]))
    p = adp.LowerProblem(op, d["y"], float(d["alpha"]), reg)
    # dgemv order differs (OpenBLAS vs warp tree): 1e-13
    assert rel(op.apply(d["x"]), d["apply"]) <= 1e-13
    assert rel(op.adjoint(d["v"]), d["adjoint"]) <= 1e-13
    assert rel(op.gram_diag(), d["gram_diag"]) <= 1e-13
    assert rel(adp.kernel_gram_correlation(d["x"], d["v"], op.kernel), d["kgc"]) == 0.0
    assert abs(adp.lower_value(p, d["x"]) - float(d["lower_value"])) <= 1e-13 * abs(float(d["lower_value"]))
    val, g = adp.lower_value_and_grad(p, d["x"])
    assert abs(val - float(d["vg_val"])) <= 1e-13 * abs(float(d["vg_val"]))
    assert rel(g, d["vg_g"]) <= 1e-12
    assert rel(adp.lower_grad(p, d["x"]), d["lower_grad"]) <= 1e-12
    assert rel(adp.lower_hess_vec(p, d["x"], d["v"]), d["hess_vec"]) <= 1e-12
    assert rel(adp.lower_hess_diag(p, d["x"]), d["hess_diag"]) <= 1e-12
    assert rel(adp.mixed_second_transpose(d["x"], op.kernel, d["v"], p), d["mixed"]) <= 1e-12
    # elastic net alone: elementwise + np.sum -> bitwise
    assert reg.value(d["x"]) == float(d["en_value"])
    assert np.array_equal(reg.grad(d["x"]), d["en_grad"])
    assert rel(reg.hess_vec(d["x"], d["v"]), d["en_hess_vec"]) <= 1e-13
    assert rel(reg.hess_diag(d["x"]), d["en_hess_diag"]) <= 1e-13
    lam = adp.op_norm_sq(adp.DenseOperator(d["m"]), 300, 1e-4)
    assert abs(lam - float(d["norm_sq"])) <= 1e-12 * float(d["norm_sq"])


@pytest.mark.parametrize("name", CONV)
def test_fast_and_fp32_modes(adp, golden, name):
    d = golden(name)
    for mode, dtype, tol in (("fast", "float64", 1e-13), ("fast", "float32", 1e-4)):
        with adp.precision(dtype, mode):
            p = conv_problem(adp, d)
            assert rel(p.op.apply(d["x"]), d["apply"]) <= tol
            val, g = adp.lower_value_and_grad(p, d["x"])
            assert abs(val - float(d["vg_val"])) <= tol * abs(float(d["vg_val"]))
            assert rel(g, d["vg_g"]) <= max(tol, 1e-12) * (1e3 if dtype == "float32" else 1.0)
