"""Inexact hypergradient (drop-in for ``adp.hypergradient``, reference
``pkg/src/adp/hypergradient.py``).

``inexact_hypergradient`` issues four device calls: the persistent lower
solve, the upper fit gradient (CG right-hand side), the fused Jacobi-PCG on
the lower Hessian (diagonal, TV curvature weights, warm start, true residual
all inside one launch), and the mixed derivative (two stencils + two
kernel-gram correlations).  The Sobolev anchor and the kernel-space
combination z = -m + grad r(b) are computed on the host on <= 31x31x3 taps
(or the n x n dense kernel), as the reference does in NumPy.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .lower_solvers import LowerProblem, _native_lower, mu_of_b, solve_lower
from .operators import DENSE1D, DenseOperator, Kernel
from .regularizers import image_forward_diff, image_forward_diff_adjoint


class NegativeCurvatureError(RuntimeError):
    """CG met a direction of non-positive curvature; the lower-level Hessian
    is not positive definite, violating the strong convexity assumption."""


def _negcurv(curv: float) -> NegativeCurvatureError:
    return NegativeCurvatureError(
        f"non-positive curvature p^T H p = {curv:.3e} in CG: the lower-level "
        "Hessian is not positive definite (strong convexity assumption violated)")


@dataclass
class CGResult:
    q: object
    residual: float
    iters: int
    converged: bool


def _vec(op, n, a, x, y, out):
    dt = nat.DTYPE_F32 if nat.get_precision()["dtype"] == "float32" else nat.DTYPE_F64
    red = ctypes.c_double()
    nat.check(nat.lib().adp_vec(int(op), int(n), dt, float(a), nat.ptr(x), nat.ptr(y), nat.ptr(out),
                                ctypes.byref(red), nat.stream_ptr()), "vector op")
    return float(red.value)


def cg_solve(hess_vec, rhs, tol: float, max_iters: int = 200, x0=None, precond_diag=None) -> CGResult:
    """Conjugate gradients for H q = rhs with an arbitrary ``hess_vec``
    callable (hypergradient.py:35-84).  The vectors live on the device and
    every update / inner product runs in the library's vector kernels;
    ``hess_vec`` is called with arrays of the kind of ``rhs``.  (The hot path,
    inexact_hypergradient, uses the fused device CG instead.)"""
    if tol <= 0:
        raise ValueError("tol must be > 0")
    kind_ref = rhs
    rhs_d = nat.to_dev(rhs).reshape(-1)
    shape = tuple(np.shape(rhs))
    n = rhs_d.numel()

    def H(v):
        out = hess_vec(nat.like(v.reshape(shape), kind_ref))
        return nat.to_dev(out).reshape(-1)

    inv = None
    if precond_diag is not None:
        d = nat.to_dev(precond_diag).reshape(-1)
        if _vec(11, n, 0.0, d, d, None) > 0:
            raise ValueError("preconditioner diagonal must be positive")
        inv = nat.empty_like_dev((n,))
        _vec(3, n, 0.0, d, None, inv)
    r = nat.empty_like_dev((n,))
    if x0 is None:
        q = nat.zeros_dev((n,))
        _vec(5, n, 0.0, rhs_d, None, r)
    else:
        q = nat.to_dev(x0).reshape(-1).clone()
        _vec(4, n, 0.0, rhs_d, H(q), r)
    s = r.clone() if inv is None else nat.empty_like_dev((n,))
    if inv is not None:
        _vec(2, n, 0.0, inv, r, s)
    p = s.clone()
    rs = _vec(10, n, 0.0, r, s, None)
    iters = 0
    for iters in range(1, max_iters + 1):
        if np.sqrt(_vec(10, n, 0.0, r, r, None)) <= tol:
            iters -= 1
            break
        hp = H(p)
        curv = _vec(10, n, 0.0, p, hp, None)
        if curv <= 0:
            raise _negcurv(curv)
        a = rs / curv
        _vec(0, n, a, q, p, q)
        _vec(1, n, a, r, hp, r)
        if inv is None:
            _vec(5, n, 0.0, r, None, s)
        else:
            _vec(2, n, 0.0, inv, r, s)
        rs_new = _vec(10, n, 0.0, r, s, None)
        _vec(0, n, rs_new / rs, s, p, p)
        rs = rs_new
    res = nat.empty_like_dev((n,))
    _vec(4, n, 0.0, H(q), rhs_d, res)
    true_res = float(np.sqrt(_vec(10, n, 0.0, res, res, None)))
    return CGResult(nat.like(q.reshape(shape), kind_ref), true_res, iters, true_res <= tol)


def _upper_terms(A, x, y_delta, want_grad=False):
    """(sum((Ax - y)^2), ||2 A^T (Ax - y)||, optional grad) in one launch."""
    from .operators import ConvOperator, _op_kernel
    fft = nat.is_fft() and isinstance(A, ConvOperator)   # tile-FFT stencils
    plan = A.fft_plan() if fft else A.plan()
    xd = nat.to_dev(x, A.signal_shape)
    yd = y_delta if nat.is_torch(y_delta) and y_delta.is_cuda else _cached_dev(A, y_delta)
    g = nat.empty_like_dev(A.signal_shape) if want_grad else None
    fit = ctypes.c_double()
    gn = ctypes.c_double()
    fn = nat.lib().adp_fft_upper_terms if fft else nat.lib().adp_upper_terms
    nat.check(fn(plan.handle, nat.ptr(_op_kernel(A).device()), nat.ptr(xd), nat.ptr(yd), ctypes.byref(fit),
                 ctypes.byref(gn), nat.ptr(g), nat.stream_ptr()), "upper_terms")
    return float(fit.value), float(gn.value), g


def _cached_dev(owner, arr):
    """Device copy of a host array held by `owner` (e.g. y_delta), cached."""
    cache = owner.__dict__.setdefault("_devcache", {})
    key = (id(arr), nat.get_precision()["dtype"], nat.current_device())
    ver = arr._version if nat.is_torch(arr) else nat.host_fingerprint(arr)   # in-place edits re-copy
    hit = cache.get(key)
    if hit is None or hit[0] is not arr or hit[1] != ver:
        hit = (arr, ver, nat.to_dev(arr, owner.signal_shape))
        cache[key] = hit
    return hit[2]


def upper_fit_grad(x, A, y_delta):
    """2 A^T (Ax - y) (hypergradient.py:87-89)."""
    _, _, g = _upper_terms(A, x, y_delta, want_grad=True)
    return nat.like(g, x)


def mixed_second_transpose(x_tilde, b: Kernel, q, p: LowerProblem) -> np.ndarray:
    """(d^2_{xb} h)^T q = 2 kgc(x~, Bq) + 2 kgc(q, Bx~ - y); dense: the rank-2
    matrix 2[(Bx~ - y) q^T + (Bq) x~^T] (hypergradient.py:92-104).  Host array
    of the kernel's shape."""
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x_tilde, p.op.signal_shape)
    qd = nat.to_dev(q, p.op.signal_shape)
    out = nat.empty_like_dev(b.data.shape)
    if plan is None:   # fft mode: kernel-gradient correlations on tile FFTs
        fn, handle = nat.lib().adp_fft_mixed_T, p.op.fft_plan().handle
    else:
        fn, handle = nat.lib().adp_mixed_T, plan.handle
    nat.check(fn(handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(qd), nat.ptr(out), nat.stream_ptr()),
              "mixed_second_transpose")
    return nat.to_host(out).astype(float)


def sobolev_value(b: Kernel, a: Kernel, beta: float) -> float:
    """r(b) = beta (||b - a||^2 + ||D(b - a)||^2) on the kernel grid
    (hypergradient.py:107-113)."""
    if beta == 0:
        return 0.0
    d = b.data - a.data
    dd = image_forward_diff(d)
    return beta * (float(np.sum(d * d)) + float(np.sum(dd * dd)))


def sobolev_grad(b: Kernel, a: Kernel, beta: float) -> np.ndarray:
    """grad r(b) = 2 beta (I + D^T D)(b - a) (hypergradient.py:116-123)."""
    if b.data.shape != a.data.shape:
        raise ValueError(f"kernel shapes differ: {b.data.shape} vs {a.data.shape}")
    if beta == 0:
        return np.zeros_like(b.data)
    d = b.data - a.data
    return 2.0 * beta * (d + image_forward_diff_adjoint(image_forward_diff(d)))


@dataclass
class WarmState:
    """Warm-start caches owned by the outer loop (hypergradient.py:126-131)."""

    x: object
    q: object | None = None


@dataclass
class HypergradResult:
    z: np.ndarray
    x_tilde: object
    cg_iters: int
    lower_iters: int
    cg_residual: float
    epsilon_used: float
    delta_used: float
    lower_converged: bool = True
    cg_converged: bool = True
    mu: float = 0.0


def hess_cg(p: LowerProblem, x_tilde, rhs, tol: float, max_iters: int, q0=None):
    """Fused device Jacobi-PCG on the lower Hessian at x~ (cg_solve applied to
    lower_hess_vec with precond lower_hess_diag, hypergradient.py:171-176).
    Returns (CGResult with a device q, Hessian-vector products issued)."""
    if tol <= 0:
        raise ValueError("tol must be > 0")
    plan, s, keep = _native_lower(p)
    xd = nat.to_dev(x_tilde, p.op.signal_shape)
    rd = nat.to_dev(rhs, p.op.signal_shape)
    if q0 is None:
        q = nat.zeros_dev(p.op.signal_shape)
        warm = 0
    else:
        q = nat.to_dev(q0, p.op.signal_shape).clone()
        warm = 1
    r = nat.CGResultC()
    if plan is None:   # fft mode: Hessian products on the tile-FFT stencils
        fn, handle = nat.lib().adp_fft_hess_cg, p.op.fft_plan().handle
    else:
        fn, handle = nat.lib().adp_hess_cg, plan.handle
    nat.check(fn(handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(rd), nat.ptr(q), warm, ctypes.c_void_p(0), float(tol),
                 int(max_iters), ctypes.byref(r), nat.stream_ptr()), "hess_cg")
    if r.status == nat.STATUS_NEGCURV:
        raise _negcurv(float(r.curv))
    return CGResult(q, float(r.residual), int(r.iters), bool(r.converged)), int(r.hv)


def inexact_hypergradient(upper, b: Kernel, eps: float, delta: float, state: WarmState,
                          cg_max_iters: int = 200) -> HypergradResult:
    """Algorithm 1 (hypergradient.py:148-190).  ``state.x`` / ``state.q`` stay
    on the device between calls."""
    if eps <= 0 or delta <= 0:
        raise ValueError("eps and delta must be > 0")
    p = upper.lower_problem(b)
    mu = mu_of_b(p, upper.mu_floor)
    res = solve_lower(
        p, nat.to_dev(state.x, p.op.signal_shape), eps, mu,
        max_iters=upper.lower_max_iters,
        method=upper.lower_method,
        step_size=upper.lower_step,
        adaptive=upper.lower_adaptive,
    )
    host = not nat.is_torch(state.x)   # numpy state in -> numpy state out (reference types)
    x_t = res.x_tilde
    state.x = nat.to_host(x_t).astype(float) if host else x_t   # before the CG, as hypergradient.py:169
    _, _, rhs = _upper_terms(upper.A, x_t, upper.y_delta, want_grad=True)
    cg, _ = hess_cg(p, x_t, rhs, delta, cg_max_iters, q0=state.q)
    z = -mixed_second_transpose(x_t, b, cg.q, p) + sobolev_grad(b, upper.a, upper.beta)
    state.q = nat.to_host(cg.q).astype(float) if host else cg.q
    return HypergradResult(
        z=z,
        x_tilde=state.x,
        cg_iters=cg.iters,
        lower_iters=res.iters,
        cg_residual=cg.residual,
        epsilon_used=res.epsilon_achieved,
        delta_used=delta,
        lower_converged=res.converged,
        cg_converged=cg.converged,
        mu=mu,
    )


def cg_iteration(p: LowerProblem, x_tilde, q, r, p_dir, rs: float) -> dict:
    """ONE Jacobi-PCG iteration of cg_solve on lower_hess_vec
    (hypergradient.py:70-81) from an injected state (q, r, p, rs) — the P2
    lockstep protocol of SURVEY.md Appendix C — in the production CG kernel.
    Returns {"q", "r", "rs", "curv"} (q += a p, r -= a H p, rs = <r, M^-1 r>)."""
    plan, s, keep = _native_lower(p)
    plan = plan or p.op.plan()
    xd = nat.to_dev(x_tilde, p.op.signal_shape)
    qd = nat.to_dev(q, p.op.signal_shape).clone()
    rd = nat.to_dev(r, p.op.signal_shape).clone()
    pd = nat.to_dev(p_dir, p.op.signal_shape)
    res = nat.CGResultC()
    nat.check(nat.lib().adp_cg_iter(plan.handle, ctypes.byref(s), nat.ptr(xd), nat.ptr(qd), nat.ptr(rd), nat.ptr(pd),
                                    float(rs), ctypes.byref(res), nat.stream_ptr()), "cg_iteration")
    if res.status == nat.STATUS_NEGCURV:
        raise _negcurv(float(res.curv))
    return {"q": nat.like(qd, q), "r": nat.like(rd, r), "rs": float(res.rs), "curv": float(res.curv)}
