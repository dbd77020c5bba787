"""Quality metrics and run-trace CSV persistence (reference
``metrics_io.py:1-113``), drop-in names and behaviour.

PSNR, SSIM and the relative L2 error run on the device (``adp_np_sum``,
``adp_ssim``, ``adp_vec`` behind the C ABI); only the final scalar
arithmetic (division by the element count, ``10 log10``, the channel mean of
≤ 3 values) happens on the host, exactly as the reference writes it.
Rounding: PSNR and SSIM are bitwise equal to the reference (NumPy pairwise
sums, ndimage's tap order); the relative L2 error uses ``np.linalg.norm``
(an OpenBLAS ``ddot``) in the reference and the library's fixed-tree dot here,
so it agrees to ~1e-13 relative.

Inputs may be NumPy arrays or torch tensors (host or CUDA); results are
Python floats.  Plotting and PNG I/O (``render_plots``, ``save_png``,
``load_png``, ``save_kernel_image``) are outside the hot-path scope
 and are not provided.
"""
from __future__ import annotations

import csv
import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .maid import RunTrace

PSNR_CAP_DB = 99.0
TRACE_HEADER = ["k", "loss", "grad_norm", "eps", "delta", "alpha",
                "lower_iters_cum", "cg_iters_cum", "wall_s"]


@dataclass(frozen=True)
class MetricReport:
    psnr_db: float
    ssim: float
    rel_l2_error: float


def _shape(a):
    return tuple(a.shape) if nat.is_torch(a) else np.shape(np.asarray(a))


def _dev64(a):
    """Contiguous float64 CUDA tensor (metrics always run in float64)."""
    import torch
    if nat.is_torch(a):
        return a.detach().to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to("cuda")


def _np_sum(op, k, n, x, y=None):
    out = (ctypes.c_double * k)()
    nat.check(nat.lib().adp_np_sum(int(op), int(k), int(n), nat.ptr(x), nat.ptr(y), out, nat.stream_ptr()),
              "adp_np_sum")
    return [float(v) for v in out]


def psnr(x, ref, peak: float = 1.0, cap: float = PSNR_CAP_DB) -> float:
    """10 log10(peak^2 / MSE) over all channels, capped for identical inputs
    (metrics_io.py:26-37)."""
    if _shape(x) != _shape(ref):
        raise ValueError(f"shape mismatch: {_shape(x)} vs {_shape(ref)}")
    if peak <= 0:
        raise ValueError("peak must be > 0")
    xd, rd = _dev64(x), _dev64(ref)
    n = xd.numel()
    if n == 0:
        mse = float(np.mean(np.empty(0)))        # the reference's empty-mean nan (RuntimeWarning)
    else:
        mse = float(np.float64(_np_sum(1, 1, n, xd, rd)[0]) / n)
    if mse == 0.0:
        return cap
    return min(10.0 * np.log10(peak * peak / mse), cap)


def _ssim_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    """Normalised Gaussian window (metrics_io.py:40-44), a host constant."""
    half = size // 2
    g = np.arange(-half, half + 1, dtype=float)
    w = np.exp(-(g[:, None] ** 2 + g[None, :] ** 2) / (2.0 * sigma**2))
    return w / w.sum()


def ssim(x, ref) -> float:
    """Mean SSIM with an 11x11 Gaussian window (sigma 1.5), C1 = 0.01^2,
    C2 = 0.03^2, averaged over channels; windows fully inside the image
    (metrics_io.py:47-76).  The five correlations and the per-pixel ratio
    run in one device kernel per tile; the map's mean is a device pairwise
    sum."""
    if _shape(x) != _shape(ref):
        raise ValueError(f"shape mismatch: {_shape(x)} vs {_shape(ref)}")
    xd, rd = _dev64(x), _dev64(ref)
    if xd.ndim == 2:
        xd = xd[:, :, None].contiguous()
        rd = rd[:, :, None].contiguous()
    H, W, C = xd.shape[0], xd.shape[1], xd.shape[2]     # IndexError for 1-D input, as the reference
    win = _ssim_window()
    half = win.shape[0] // 2
    c1, c2 = 0.01**2, 0.03**2
    Ho, Wo = H - 2 * half, W - 2 * half
    if Ho <= 0 or Wo <= 0:
        vals = [np.mean(np.empty((0, 0))) for _ in range(C)]   # empty interior: nan, as the reference
        return float(np.mean(vals))
    wbuf = (ctypes.c_double * win.size)(*win.ravel())
    sums = (ctypes.c_double * C)()
    nat.check(nat.lib().adp_ssim(int(H), int(W), int(C), wbuf, int(win.shape[0]), float(c1), float(c2),
                                 nat.ptr(xd), nat.ptr(rd), ctypes.c_void_p(0), sums, nat.stream_ptr()), "adp_ssim")
    n = Ho * Wo
    vals = [np.float64(sums[c]) / n for c in range(C)]
    return float(np.mean(vals))


def rel_l2_error(x, ref) -> float:
    """||x - ref|| / ||ref|| (metrics_io.py:79-80)."""
    from .hypergradient import _vec
    if _shape(x) != _shape(ref):
        raise ValueError(f"operands could not be broadcast together with shapes {_shape(x)} {_shape(ref)}")
    with nat.precision("float64", nat.get_precision()["mode"]):
        xd, rd = _dev64(x), _dev64(ref)
        n = xd.numel()
        d = xd.new_empty(xd.shape)
        _vec(4, n, 0.0, xd, rd, d)
        num = np.sqrt(_vec(10, n, 0.0, d, d, None))
        den = np.sqrt(_vec(10, n, 0.0, rd, rd, None))
    return float(num / den)


def metric_report(x, ref, peak: float = 1.0) -> MetricReport:
    s = ssim(x, ref) if len(_shape(x)) >= 2 else float("nan")
    return MetricReport(psnr(x, ref, peak), s, rel_l2_error(x, ref))


def write_trace_csv(trace: RunTrace, path) -> None:
    """One row per accepted iteration, floats as repr (metrics_io.py:88-99)."""
    rows = zip(trace.k, trace.loss, trace.grad_norm, trace.eps, trace.delta,
               trace.alpha, trace.lower_iters_cum, trace.cg_iters_cum, trace.wall_s)
    try:
        with open(path, "w", newline="", encoding="utf-8") as fh:
            writer = csv.writer(fh)
            writer.writerow(TRACE_HEADER)
            for row in rows:
                writer.writerow([repr(v) if isinstance(v, float) else v for v in row])
    except OSError as exc:
        raise OSError(f"cannot write trace to {path}: {exc}") from exc


def read_trace_csv(path) -> RunTrace:
    """Inverse of write_trace_csv; rejects any other header (metrics_io.py:102-116)."""
    trace = RunTrace()
    try:
        with open(path, newline="", encoding="utf-8") as fh:
            reader = csv.reader(fh)
            header = next(reader)
            if header != TRACE_HEADER:
                raise ValueError(f"unexpected trace header {header} in {path}")
            for row in reader:
                trace.append(int(row[0]), *map(float, row[1:]))
    except OSError as exc:
        raise OSError(f"cannot read trace from {path}: {exc}") from exc
    return trace


def loss_axis_scale(losses) -> str:
    """Log scale when the (positive) losses span more than three decades (metrics_io.py:119-125)."""
    arr = np.asarray([v for trace_losses in losses for v in trace_losses], dtype=float)
    arr = arr[arr > 0]
    if arr.size >= 2 and arr.max() / arr.min() > 1e3:
        return "log"
    return "linear"
