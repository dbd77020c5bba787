"""Lower-level problem h(x, b) = ||B x - y||^2 + alpha J(x) and its solvers
(drop-in for ``adp.lower_solvers``, reference ``pkg/src/adp/lower_solvers.py``).

``solve_lower`` is ONE persistent cooperative launch: power iteration for
L(b) (when the step is not given), then the whole GD / AGD-with-restart /
FISTA-SC loop including the Armijo backtracking, with all decisions taken on
the device from deterministic reductions.  Only (x~, ||grad||, iters,
converged) come back.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .operators import ConvOperator, DenseOperator, _op_kernel, op_norm_sq
from .regularizers import SmoothedElasticNet, SmoothedTV


class SolveDiverged(RuntimeError):
    """Objective became non-finite during a lower-level solve."""


@dataclass(frozen=True)
class LowerProblem:
    op: object  # ConvOperator | DenseOperator
    y: object   # numpy array or device tensor
    alpha: float
    reg: object  # SmoothedElasticNet | SmoothedTV


@dataclass
class LowerSolveResult:
    x_tilde: object
    grad_norm: float
    iters: int
    epsilon_achieved: float
    converged: bool


def _native_lower(p: LowerProblem):
    """(plan, adp_lower struct, keep-alive tensors) for a lower problem."""
    op = p.op
    reg = p.reg
    if isinstance(op, DenseOperator):
        if not isinstance(reg, SmoothedElasticNet):
            raise ValueError("the dense 1-D operator is paired with SmoothedElasticNet")
    elif isinstance(op, ConvOperator):
        if not isinstance(reg, SmoothedTV):
            raise ValueError("the depthwise 2-D operator is paired with SmoothedTV")
    else:
        raise TypeError(f"unsupported operator {type(op).__name__}")
    plan = None if (nat.is_fft() and isinstance(op, ConvOperator)) else op.plan()   # fft: tile-FFT plan instead
    s = reg.native()
    kd = _op_kernel(op).device()
    yd = _ydev(p)
    s.kernel = kd.data_ptr()
    s.y = yd.data_ptr()
    s.alpha = float(p.alpha)
    return plan, s, (kd, yd)


def _ydev(p: LowerProblem):
    """Device copy of the lower data, cached per (problem, precision)."""
    cache = p.__dict__.get("_ydev")
    key = nat.get_precision()["dtype"]
    if cache is None or cache[0] != key:
        cache = (key, nat.to_dev(p.y, p.op.signal_shape))
        object.__setattr__(p, "_ydev", cache)
    return cache[1]


def _check_reg_smooth(p: LowerProblem):
    reg = p.reg
    if p.alpha != 0:
        if isinstance(reg, SmoothedTV) and reg.nu <= 0:
            raise ValueError("gradient requested on the nonsmooth branch (nu = 0)")
        if isinstance(reg, SmoothedElasticNet):
            reg._check_smooth()


def _fft(p: LowerProblem) -> bool:
    """FFT stencil mode applies to the depthwise 2-D operator."""
    return nat.is_fft() and isinstance(p.op, ConvOperator)


def lower_value(p: LowerProblem, x) -> float:
    """h(x) = sum((Bx - y)^2) + alpha * J(x) (lower_solvers.py:37-39)."""
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x, p.op.signal_shape)
    val = ctypes.c_double()
    if _fft(p):
        nat.check(nat.lib().adp_fft_lower_value(p.op.fft_plan().handle, ctypes.byref(s), nat.ptr(xd),
                                                ctypes.byref(val), nat.stream_ptr()), "lower_value")
        return float(val.value)
    nat.check(nat.lib().adp_lower_value(plan.handle, ctypes.byref(s), nat.ptr(xd), ctypes.byref(val),
                                        nat.stream_ptr()), "lower_value")
    return float(val.value)


def lower_grad(p: LowerProblem, x):
    """2 B^T (Bx - y) + alpha grad J(x) (lower_solvers.py:42-47)."""
    _check_reg_smooth(p)
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x, p.op.signal_shape)
    g = nat.empty_like_dev(p.op.signal_shape)
    if _fft(p):
        nat.check(nat.lib().adp_fft_lower_value_and_grad(p.op.fft_plan().handle, ctypes.byref(s), nat.ptr(xd),
                                                         None, nat.ptr(g), nat.stream_ptr()), "lower_grad")
        return nat.like(g, x)
    nat.check(nat.lib().adp_lower_grad(plan.handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(g), nat.stream_ptr()),
              "lower_grad")
    return nat.like(g, x)


def lower_value_and_grad(p: LowerProblem, x):
    """Objective and gradient sharing one forward pass (lower_solvers.py:50-63)."""
    _check_reg_smooth(p)
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x, p.op.signal_shape)
    g = nat.empty_like_dev(p.op.signal_shape)
    val = ctypes.c_double()
    fn = nat.lib().adp_fft_lower_value_and_grad if _fft(p) else nat.lib().adp_lower_value_and_grad
    handle = p.op.fft_plan().handle if _fft(p) else plan.handle
    nat.check(fn(handle, ctypes.byref(s), nat.ptr(xd), ctypes.byref(val), nat.ptr(g), nat.stream_ptr()),
              "lower_value_and_grad")
    return float(val.value), nat.like(g, x)


def lower_hess_vec(p: LowerProblem, x, v):
    """(2 B^T B + alpha hess J(x)) v (lower_solvers.py:66-71)."""
    _check_reg_smooth(p)
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x, p.op.signal_shape)
    vd = nat.to_dev(v, p.op.signal_shape)
    out = nat.empty_like_dev(p.op.signal_shape)
    plan = plan or p.op.plan()   # fft mode: the Hessian product runs on the direct (fast) stencils
    nat.check(nat.lib().adp_lower_hess_vec(plan.handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(vd), nat.ptr(out),
                                           nat.stream_ptr()), "lower_hess_vec")
    return nat.like(out, v)


def lower_hess_diag(p: LowerProblem, x):
    """Jacobi diagonal of the lower Hessian, floored at 1e-12 max + 1e-300
    (lower_solvers.py:74-80)."""
    _check_reg_smooth(p)
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x, p.op.signal_shape)
    out = nat.empty_like_dev(p.op.signal_shape)
    plan = plan or p.op.plan()
    nat.check(nat.lib().adp_lower_hess_diag(plan.handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(out),
                                            nat.stream_ptr()), "lower_hess_diag")
    return nat.like(out, x)


def mu_of_b(p: LowerProblem, mu_floor: float) -> float:
    """Strong convexity constant max(alpha * mu_J, mu_floor) (lower_solvers.py:83-87)."""
    if mu_floor <= 0:
        raise ValueError("mu_floor must be > 0")
    return max(p.alpha * p.reg.mu, mu_floor)


def L_of_b(p: LowerProblem, norm_sq_max_iters: int = 300, norm_sq_tol: float = 1e-4) -> float:
    """2 ||B||^2 + alpha * C_J (lower_solvers.py:90-96)."""
    return 2.0 * op_norm_sq(p.op, norm_sq_max_iters, norm_sq_tol) + p.alpha * p.reg.curvature


def solve_lower(p: LowerProblem, x0, eps: float, mu: float, max_iters: int = 300, method: str = "agd",
                step_size: float | None = None, adaptive: bool = False, *, x_out=None,
                stats: dict | None = None) -> LowerSolveResult:
    """Drive ||grad_x h|| below eps * mu from the warm start x0
    (lower_solvers.py:104-146, _gradient_descent 154-167, _accelerated
    180-213).  ``x_tilde`` has the kind of ``x0`` (numpy or device tensor)."""
    if eps <= 0:
        raise ValueError("eps must be > 0")
    if mu <= 0:
        raise ValueError("mu must be > 0")
    if tuple(np.shape(x0)) != tuple(p.op.signal_shape):
        raise ValueError(f"x0 shape {tuple(np.shape(x0))} does not match {p.op.signal_shape}")
    if method not in nat.METHODS:
        raise ValueError(f"unknown lower solver method {method!r}")
    if step_size is None:
        p.reg.curvature  # raises for the nonsmooth branch exactly where L_of_b would
    _check_reg_smooth(p)
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x0, p.op.signal_shape)
    out = x_out if x_out is not None else nat.empty_like_dev(p.op.signal_shape)
    a = nat.SolveArgs()
    a.eps, a.mu = float(eps), float(mu)
    a.max_iters = int(max_iters)
    a.method = nat.METHODS[method]
    a.adaptive = 1 if adaptive else 0
    a.step_size = float(step_size) if step_size is not None else 0.0
    a.norm_sq = float(p.op._norm_sq) if p.op._norm_sq is not None else -1.0
    a.norm_max_iters = 300
    a.norm_tol = 1e-4
    v0 = nat.power_start(p.op.signal_shape)
    a.v0 = v0.data_ptr()
    r = nat.SolveResult()
    fn = nat.lib().adp_fft_lower_solve if _fft(p) else nat.lib().adp_lower_solve
    handle = p.op.fft_plan().handle if _fft(p) else plan.handle
    nat.check(fn(handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(out), ctypes.byref(a), ctypes.byref(r),
                 nat.stream_ptr()), "solve_lower")
    if step_size is None and p.op._norm_sq is None:
        if not r.power_converged:
            import warnings
            warnings.warn(f"power iteration did not converge in 300 iterations; returning best estimate "
                          f"{r.norm_sq:.6e}", RuntimeWarning)
        p.op._norm_sq = float(r.norm_sq)
    if r.status == nat.STATUS_DIVERGED:
        raise SolveDiverged(f"objective became non-finite at lower iteration {r.fail_iter}")
    if r.status == nat.STATUS_BT_FAIL:
        raise SolveDiverged("backtracking line search failed to find a decreasing step")
    if stats is not None:
        stats.update(vg_evals=int(r.vg_evals), value_evals=int(r.value_evals), restarts=int(r.restarts),
                     lip=float(r.lip), power_iters=int(r.power_iters), launches=int(r.launches),
                     dominant_ms=float(r.dominant_ms), dominant_launches=int(r.dominant_launches))
    gn = float(r.grad_norm)
    return LowerSolveResult(nat.like(out, x0), gn, int(r.iters), gn / mu, bool(r.converged))


def lower_iteration(p: LowerProblem, x, x_prev, t_mom: float, lip_t: float, eps: float, mu: float,
                    method: str = "agd", adaptive: bool = False, step_size: float | None = None) -> dict:
    """ONE iteration of _accelerated (lower_solvers.py:191-211) from an injected
    state (x, x_prev, t_mom, lip_t) — the P2 lockstep protocol of SURVEY.md
    Appendix C.  Runs the production solve kernel with max_iters = 1.  Returns
    the next state and the iteration's decisions: {"x", "x_prev", "t_mom",
    "lip_t", "bt_tries", "restart", "converged", "grad_norm"} (on convergence
    "x" is the extrapolated point y the solve would return)."""
    if method not in ("agd", "fista_sc"):
        raise ValueError("lower_iteration follows _accelerated (agd / fista_sc)")
    _check_reg_smooth(p)
    if step_size is None and p.op._norm_sq is None:
        op_norm_sq(p.op, 300, 1e-4)          # L(b) outside the iteration, as the solve caches it
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x, p.op.signal_shape)
    xpd = nat.to_dev(x_prev, p.op.signal_shape)
    out = nat.empty_like_dev(p.op.signal_shape)
    a = nat.SolveArgs()
    a.eps, a.mu = float(eps), float(mu)
    a.max_iters = 1
    a.method = nat.METHODS[method]
    a.adaptive = 1 if adaptive else 0
    a.step_size = float(step_size) if step_size is not None else 0.0
    a.norm_sq = float(p.op._norm_sq) if p.op._norm_sq is not None else -1.0
    a.norm_max_iters, a.norm_tol = 300, 1e-4
    a.v0 = nat.power_start(p.op.signal_shape).data_ptr()
    a.x_prev0 = xpd.data_ptr()
    a.t_mom0, a.lip_t0 = float(t_mom), float(lip_t)
    r = nat.SolveResult()
    if _fft(p):
        nat.check(nat.lib().adp_fft_lower_solve(p.op.fft_plan().handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(out),
                                                ctypes.byref(a), ctypes.byref(r), nat.stream_ptr()), "lower_iteration")
    else:
        nat.check(nat.lib().adp_lower_iter(plan.handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(xpd), float(t_mom),
                                           float(lip_t), ctypes.byref(a), nat.ptr(out), ctypes.byref(r),
                                           nat.stream_ptr()), "lower_iteration")
    if r.status == nat.STATUS_DIVERGED:
        raise SolveDiverged("objective became non-finite at lower iteration 0")
    if r.status == nat.STATUS_BT_FAIL:
        raise SolveDiverged("backtracking line search failed to find a decreasing step")
    converged = bool(r.converged) and r.iters == 0
    restart = r.restarts > 0
    xn = nat.like(out, x)
    return {"x": xn, "x_prev": xn if restart else x, "t_mom": float(r.t_mom), "lip_t": float(r.lip_t),
            "bt_tries": max(int(r.value_evals) - 1, 0) if adaptive else 0, "restart": restart,
            "converged": converged, "grad_norm": float(r.grad_norm)}
