"""Lower-level regularizers (drop-in for ``adp.regularizers``, reference
``pkg/src/adp/regularizers.py``).

The classes carry the reference's parameters, constants (mu, curvature) and
validation.  Their array methods run on the device through ``adp_reg_op``:
the lower-level machinery with the operator term removed and alpha = 1,
which reproduces J's value / gradient / Hessian terms exactly (TV on
(h, w, c) images; elastic net on 1-D signals).  Inside the solvers J is
never called separately — it is fused into the stencil stages.

``image_forward_diff`` / ``image_forward_diff_adjoint`` and the scalar
helpers below act on kernel-space arrays (the Sobolev term of the upper
objective, <= 31x31x3 taps) on the host, as the hot-path plan prescribes
(hypergradient row).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat


def prox_l1(x, threshold: float):
    """Component-wise soft threshold sign(x) * max(|x| - threshold, 0)
    (regularizers.py:22-27), on the device (adp_vec op 6, NumPy's sign /
    maximum semantics).  Returns the kind of ``x``."""
    if threshold < 0:
        raise ValueError("threshold must be >= 0")
    from .hypergradient import _vec
    xd = nat.to_dev(x, tuple(np.shape(x)))
    out = nat.empty_like_dev(xd.shape)
    _vec(6, xd.numel(), float(threshold), xd, xd, out)
    return nat.like(out, x)


def image_forward_diff(x) -> np.ndarray:
    """Forward differences along the first two axes, zero last row/column,
    stacked as (2,) + x.shape (regularizers.py:46-58).  Kernel-space helper."""
    x = np.asarray(x, dtype=float)
    if x.ndim < 2:
        raise ValueError(f"need at least two grid axes, got shape {x.shape}")
    d = np.zeros((2,) + x.shape)
    d[0, :-1] = x[1:] - x[:-1]
    d[1, :, :-1] = x[:, 1:] - x[:, :-1]
    return d


def image_forward_diff_adjoint(d) -> np.ndarray:
    """Adjoint of image_forward_diff, accumulated in the reference's order
    (regularizers.py:61-67).  Kernel-space helper."""
    d = np.asarray(d, dtype=float)
    out = np.zeros(d.shape[1:])
    out[1:] += d[0, :-1]
    out[:-1] -= d[0, :-1]
    out[:, 1:] += d[1, :, :-1]
    out[:, :-1] -= d[1, :, :-1]
    return out


def _reg_call(reg_struct, layout, shape, ksize, op, x, v=None, want_out=True):
    plan = nat.plan_for(layout, shape, ksize)
    xd = nat.to_dev(x, shape)
    vd = nat.to_dev(v, shape) if v is not None else None
    out = nat.empty_like_dev(shape) if want_out else None
    val = ctypes.c_double(0.0)
    nat.check(nat.lib().adp_reg_op(plan.handle, ctypes.byref(reg_struct), int(op), nat.ptr(xd), nat.ptr(vd),
                                   nat.ptr(out), ctypes.byref(val), nat.stream_ptr()), "regularizer")
    return float(val.value), out


def _as_image(x):
    if tuple(np.shape(x)).__len__() != 3:
        raise ValueError(f"expected an (h, w, c) image, got shape {tuple(np.shape(x))}")
    return x


@dataclass(frozen=True)
class SmoothedElasticNet:
    """l1 * sum(rho_nu(x)) + l2 * ||x||^2 (regularizers.py:75-134)."""

    l1: float
    l2: float
    nu: float = 1e-4

    def __post_init__(self):
        if self.l1 < 0 or self.l2 < 0 or self.nu < 0:
            raise ValueError("elastic net parameters must be non-negative")

    @property
    def mu(self) -> float:
        return 2.0 * self.l2

    @property
    def curvature(self) -> float:
        c = 2.0 * self.l2
        if self.l1 > 0:
            if self.nu <= 0:
                raise ValueError("nonsmooth l1 part has no curvature bound; need nu > 0")
            c += self.l1 / self.nu
        return c

    def _check_smooth(self):
        if self.l1 > 0 and self.nu <= 0:
            raise ValueError("gradient requested on the nonsmooth branch (nu = 0)")

    def native(self) -> nat.Lower:
        s = nat.Lower()
        s.reg = nat.REG_ELASTIC
        s.l1, s.l2, s.nu = float(self.l1), float(self.l2), float(self.nu)
        return s

    def _call(self, op, x, v=None, want_out=True):
        """Elementwise on any shape, as the reference (regularizers.py:75-134):
        the C-order flattening is exactly what np.sum reduces over, so the
        device runs the 1-D form on the flat view and the result takes x's
        shape back."""
        shape = tuple(int(s) for s in np.shape(x))
        if v is not None and tuple(np.shape(v)) != shape:
            raise ValueError(f"shape mismatch: x {shape}, v {tuple(np.shape(v))}")
        n = int(np.prod(shape)) if shape else 1
        xf = x.reshape(n) if nat.is_torch(x) else np.ascontiguousarray(np.asarray(x, dtype=float)).reshape(n)
        vf = None if v is None else (v.reshape(n) if nat.is_torch(v) else
                                     np.ascontiguousarray(np.asarray(v, dtype=float)).reshape(n))
        val, out = _reg_call(self.native(), nat.LAYOUT_DENSE1D, (n,), (0, 0), op, xf, vf, want_out)
        return val, (out.reshape(shape) if out is not None else None)

    def value(self, x) -> float:
        return self._call(0, x, want_out=False)[0]

    def grad(self, x):
        self._check_smooth()
        return nat.like(self._call(2, x)[1], x)

    def hess_vec(self, x, v):
        self._check_smooth()
        return nat.like(self._call(3, x, v)[1], x)

    def hess_diag(self, x):
        self._check_smooth()
        return nat.like(self._call(4, x)[1], x)


@dataclass(frozen=True)
class SmoothedTV:
    """Smoothed anisotropic TV on (h, w, c) images (regularizers.py:137-199)."""

    nu: float = 1e-4

    def __post_init__(self):
        if self.nu < 0:
            raise ValueError("nu must be >= 0")

    @property
    def mu(self) -> float:
        return 0.0

    @property
    def curvature(self) -> float:
        if self.nu <= 0:
            raise ValueError("nonsmooth TV has no curvature bound; need nu > 0")
        return 8.0 / self.nu

    def native(self) -> nat.Lower:
        s = nat.Lower()
        s.reg = nat.REG_TV
        s.nu = float(self.nu)
        return s

    def _call(self, op, x, v=None, want_out=True):
        _as_image(x)
        shape = tuple(int(s) for s in np.shape(x))
        return _reg_call(self.native(), nat.LAYOUT_DEPTHWISE2D, shape, (1, 1), op, x, v, want_out)

    def value(self, x) -> float:
        """tv_value: sum(sqrt(d^2 + nu^2) - nu) over the difference stack."""
        return self._call(0, x, want_out=False)[0]

    def grad(self, x):
        if self.nu <= 0:
            raise ValueError("gradient requested on the nonsmooth branch (nu = 0)")
        return nat.like(self._call(2, x)[1], x)

    def value_and_grad(self, x):
        if self.nu <= 0:
            raise ValueError("gradient requested on the nonsmooth branch (nu = 0)")
        val, g = self._call(1, x)
        return val, nat.like(g, x)

    def hess_vec(self, x, v):
        if self.nu <= 0:
            raise ValueError("Hessian requested on the nonsmooth branch (nu = 0)")
        _as_image(v)
        return nat.like(self._call(3, x, v)[1], x)

    def hess_diag(self, x):
        if self.nu <= 0:
            raise ValueError("Hessian requested on the nonsmooth branch (nu = 0)")
        return nat.like(self._call(4, x)[1], x)


def tv_value(x, nu: float) -> float:
    """Smoothed anisotropic TV of an (h, w, c) image (regularizers.py:70-72)."""
    return SmoothedTV(nu).value(x)


def smoothed_abs_norm(x, nu: float) -> float:
    """sum(sqrt(x^2 + nu^2) - nu) of a 1-D signal (regularizers.py:15-19)."""
    if nu < 0:
        raise ValueError("nu must be >= 0")
    return SmoothedElasticNet(1.0, 0.0, nu).value(x)
