"""Seeded generators for the five BASELINE.json configurations.

The reference ships no builder for them; these
construct ``UpperProblem`` directly following the reference builders'
conventions: signal/image from ``default_rng(seed)``, noise from
``default_rng([seed, 1])``, further child streams ``[seed, 2]`` (random
kernel parts), ``[seed, 3]`` (piece count), ``[seed, 10 + c]`` (channel c
image).  Semi-blind semantics (problems.py:228-265): the data are blurred by
the TRUE kernel, ``A = a = b0`` = the assumed kernel.  Inputs are synthetic
(no dataset exists for these configs); the arrays are identical for the
device path and the CPU oracle.

  c1  1-D n=256, piecewise constant with 4..10 jumps, dense Gaussian
      sigma=3 (25 taps) truth, assumed sigma=3.9 (+30%), noise 0.01,
      build_deconv1d settings, MAID defaults with 60 upper iterations.
  c2  256x256x1: 20 random rectangles / ellipses with U[0,1] intensities
      plus a linear ramp; 9x9 Gaussian sigma=2 truth; assumed sigma=2.6.
  c3  512x512x3: the same generator per channel; one 15x15 kernel shared by
      the channels = normalised Gaussian sigma=3 convolved with a random 7-px
      line (seeded angle), centre-cropped and renormalised; assumed 15x15
      isotropic Gaussian sigma=3.
  c4  64 instances of c3, seeds 0..63.
  c5  4096x4096x3 with a 31x31 Gaussian sigma=6; A = a = b0 = that kernel
      (build_motion2d semantics; BASELINE.json gives no initial kernel).
  2-D MAID settings: defaults.cfg [motion2d] (alpha 0.6, beta 0.3, nu 1e-4,
  mu_floor 10, agd adaptive, 1200 lower iterations; eps0 = delta0 = 0.25,
  alpha0 = 2e-5, max_bt = 2, cg 100, 60 upper iterations).
"""
from __future__ import annotations

import numpy as np

from .maid import MAIDConfig
from .operators import DENSE1D, DEPTHWISE2D, Kernel, gaussian_conv_matrix
from .problems import UpperProblem, blur, gaussian_kernel_2d, piecewise_signal
from .regularizers import SmoothedElasticNet, SmoothedTV

NOISE = 0.01


def shapes_image(h: int, w: int, rng: np.random.Generator, n_shapes: int = 20) -> np.ndarray:
    """Linear ramp (random direction, amplitude 0.3) plus n_shapes painted
    rectangles / ellipses with U[0,1] intensities, clipped to [0, 1]."""
    yy, xx = np.mgrid[0:h, 0:w].astype(float)
    yy /= max(h - 1, 1)
    xx /= max(w - 1, 1)
    theta = rng.uniform(0.0, 2.0 * np.pi)
    ramp = 0.3 * (0.5 + 0.5 * (np.cos(theta) * (2 * xx - 1) + np.sin(theta) * (2 * yy - 1)) / np.sqrt(2.0))
    img = ramp.copy()
    for _ in range(n_shapes):
        kind = rng.integers(0, 2)
        cy, cx = rng.uniform(0.0, 1.0, size=2)
        ry, rx = rng.uniform(0.03, 0.2, size=2)
        val = rng.uniform(0.0, 1.0)
        if kind == 0:
            mask = (np.abs(yy - cy) <= ry) & (np.abs(xx - cx) <= rx)
        else:
            mask = ((yy - cy) / ry) ** 2 + ((xx - cx) / rx) ** 2 <= 1.0
        img[mask] = val + ramp[mask]
    return np.clip(img, 0.0, 1.0)


def line_gaussian_kernel(size: int, sigma: float, line_len: int, rng: np.random.Generator) -> np.ndarray:
    """Normalised Gaussian (size x size, sigma) convolved with a line_len-px
    line at a random angle, centre-cropped to size x size, sum 1."""
    g = gaussian_kernel_2d(size, sigma, 1).data[:, :, 0]
    ang = rng.uniform(0.0, np.pi)
    L = line_len
    line = np.zeros((L, L))
    c = (L - 1) / 2.0
    for t in np.linspace(-c, c, 4 * L):
        i = int(round(c + t * np.sin(ang)))
        j = int(round(c + t * np.cos(ang)))
        line[i, j] = 1.0
    line /= line.sum()
    full = np.zeros((size + L - 1, size + L - 1))
    for i in range(L):
        for j in range(L):
            if line[i, j]:
                full[i:i + size, j:j + size] += line[i, j] * g
    o = (L - 1) // 2
    k = full[o:o + size, o:o + size]
    return k / k.sum()


def _config_2d(seed, shape, true_kernel: Kernel, assumed: Kernel, name, blur_fn=None) -> UpperProblem:
    h, w, c = shape
    img = np.stack([shapes_image(h, w, np.random.default_rng([seed, 10 + ch])) for ch in range(c)], axis=2)
    noise = NOISE * np.random.default_rng([seed, 1]).standard_normal(shape)
    y_delta = (blur_fn or blur)(img, true_kernel) + noise
    from .operators import operator_from_kernel
    A = operator_from_kernel(assumed, shape)
    return UpperProblem(name=name, A=A, a=assumed, y_delta=y_delta, beta=0.3, alpha=0.6, reg=SmoothedTV(1e-4),
                        b0=assumed, x0=y_delta.copy(), ground_truth=img, mu_floor=10.0, lower_method="agd",
                        lower_max_iters=1200, lower_adaptive=True)


def config1(seed: int = 0) -> UpperProblem:
    n = 256
    pieces = int(np.random.default_rng([seed, 3]).integers(5, 12))   # 4..10 jumps
    x_true = piecewise_signal(n, pieces, seed)
    truth = gaussian_conv_matrix(n, 3.0)
    y_delta = truth.matrix @ x_true + NOISE * np.random.default_rng([seed, 1]).standard_normal(n)
    A = gaussian_conv_matrix(n, 3.9)
    a = Kernel(A.matrix.copy(), DENSE1D)
    return UpperProblem(name="c1_deconv1d", A=A, a=a, y_delta=y_delta, beta=0.0, alpha=1.0,
                        reg=SmoothedElasticNet(1.2e-3, 4e-3, 1e-4), b0=a, x0=np.zeros(n), ground_truth=x_true,
                        mu_floor=1e-3, lower_method="agd", lower_max_iters=300)


def config2(seed: int = 0, size: int = 256, blur_fn=None) -> UpperProblem:
    return _config_2d(seed, (size, size, 1), gaussian_kernel_2d(9, 2.0, 1), gaussian_kernel_2d(9, 2.6, 1),
                      "c2_gray256", blur_fn)


def config3(seed: int = 0, size: int = 512, blur_fn=None) -> UpperProblem:
    k = line_gaussian_kernel(15, 3.0, 7, np.random.default_rng([seed, 2]))
    truth = Kernel(np.repeat(k[:, :, None], 3, axis=2), DEPTHWISE2D)
    return _config_2d(seed, (size, size, 3), truth, gaussian_kernel_2d(15, 3.0, 3), "c3_rgb512", blur_fn)


def config4(n_instances: int = 64, blur_fn=None):
    return [config3(seed, blur_fn=blur_fn) for seed in range(n_instances)]


def config5(seed: int = 0, size: int = 4096, blur_fn=None) -> UpperProblem:
    k = gaussian_kernel_2d(31, 6.0, 3)
    return _config_2d(seed, (size, size, 3), k, k, "c5_rgb4096", blur_fn)


def maid_config(name: str) -> MAIDConfig:
    if name.startswith("c1"):
        return MAIDConfig(max_upper_iters=60)
    return MAIDConfig(eps0=0.25, delta0=0.25, alpha0=2e-5, max_bt=2, cg_max_iters=100, max_upper_iters=60)


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c5": config5}
