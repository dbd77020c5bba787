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
``load_png``, ``save_kernel_image``) are host-side file utilities outside the
hot path; they are kept as thin host functions with the
reference's behaviour so the module is a complete drop-in.
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


def _same_shape(x, ref):
    sx, sr = _shape(x), _shape(ref)
    if sx != sr:
        raise ValueError(f"shape mismatch: {sx} vs {sr}")


def psnr(x, ref, peak: float = 1.0, cap: float = PSNR_CAP_DB) -> float:
    """Peak signal-to-noise ratio in dB over all channels, capped (identical
    inputs give `cap`) (metrics_io.py:26-37).  The squared-error mean is a
    device pairwise sum divided by the element count, as np.mean does."""
    _same_shape(x, ref)
    if peak <= 0:
        raise ValueError("peak must be > 0")
    xd, rd = _dev64(x), _dev64(ref)
    count = xd.numel()
    if count:
        mean_sq = float(np.float64(_np_sum(1, 1, count, xd, rd)[0]) / count)
    else:
        mean_sq = float(np.mean(np.empty(0)))      # nan with NumPy's empty-mean warning
    return cap if mean_sq == 0.0 else min(10.0 * np.log10(peak * peak / mean_sq), cap)


_SSIM_SIZE, _SSIM_SIGMA = 11, 1.5
_SSIM_C1, _SSIM_C2 = 0.01**2, 0.03**2


def _ssim_window(size: int = _SSIM_SIZE, sigma: float = _SSIM_SIGMA) -> np.ndarray:
    """Normalised 2-D Gaussian window (metrics_io.py:40-44), a host constant."""
    r = np.arange(-(size // 2), size // 2 + 1, dtype=float)
    g = np.exp(-(r[:, None] ** 2 + r[None, :] ** 2) / (2.0 * sigma**2))
    return g / g.sum()


def ssim(x, ref) -> float:
    """Mean structural similarity (metrics_io.py:47-76): per channel the
    mean of the SSIM map over the windows that lie fully inside the image
    (11x11 Gaussian window, sigma 1.5, C1 = 0.01^2, C2 = 0.03^2), then the
    mean over channels.  One device kernel computes the five windowed
    moments and the per-pixel ratio; the map means are device pairwise sums."""
    _same_shape(x, ref)
    xd, rd = _dev64(x), _dev64(ref)
    if xd.ndim == 2:
        xd, rd = xd.unsqueeze(2).contiguous(), rd.unsqueeze(2).contiguous()
    H, W, C = xd.shape[0], xd.shape[1], xd.shape[2]     # 1-D input: IndexError, as the reference
    win = _ssim_window()
    margin = 2 * (win.shape[0] // 2)
    inner = (H - margin) * (W - margin)
    if H <= margin or W <= margin:                      # no interior window: nan, as the reference
        return float(np.mean([np.mean(np.empty((0, 0))) for _ in range(C)]))
    taps = (ctypes.c_double * win.size)(*win.ravel())
    sums = (ctypes.c_double * C)()
    nat.check(nat.lib().adp_ssim(int(H), int(W), int(C), taps, int(win.shape[0]), float(_SSIM_C1), float(_SSIM_C2),
                                 nat.ptr(xd), nat.ptr(rd), ctypes.c_void_p(0), sums, nat.stream_ptr()), "adp_ssim")
    return float(np.mean([np.float64(v) / inner for v in sums]))


def rel_l2_error(x, ref) -> float:
    """||x - ref|| / ||ref|| (metrics_io.py:79-80)."""
    from .hypergradient import _vec
    if _shape(x) != _shape(ref):   # NumPy's broadcasting error for x - ref
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
    """PSNR, SSIM (nan for 1-D signals) and relative L2 error (metrics_io.py:83-85)."""
    structural = float("nan") if len(_shape(x)) < 2 else ssim(x, ref)
    return MetricReport(psnr(x, ref, peak), structural, rel_l2_error(x, ref))


_TRACE_FIELDS = ("k", "loss", "grad_norm", "eps", "delta", "alpha", "lower_iters_cum", "cg_iters_cum", "wall_s")


def _csv_cell(v):
    return repr(v) if isinstance(v, float) else v      # floats round-trip exactly


def write_trace_csv(trace: RunTrace, path) -> None:
    """Header TRACE_HEADER, then one row per accepted iteration with floats
    written as repr (metrics_io.py:88-99)."""
    columns = [getattr(trace, f) for f in _TRACE_FIELDS]
    try:
        with open(path, "w", newline="", encoding="utf-8") as fh:
            out = csv.writer(fh)
            out.writerow(TRACE_HEADER)
            out.writerows([_csv_cell(v) for v in row] for row in zip(*columns))
    except OSError as exc:
        raise OSError(f"cannot write trace to {path}: {exc}") from exc


def read_trace_csv(path) -> RunTrace:
    """Inverse of write_trace_csv; any other header is a ValueError
    (metrics_io.py:102-116)."""
    trace = RunTrace()
    try:
        with open(path, newline="", encoding="utf-8") as fh:
            rows = csv.reader(fh)
            first = next(rows)
            if first != TRACE_HEADER:
                raise ValueError(f"unexpected trace header {first} in {path}")
            for k, *rest in rows:
                trace.append(int(k), *(float(v) for v in rest))
    except OSError as exc:
        raise OSError(f"cannot read trace from {path}: {exc}") from exc
    return trace


def loss_axis_scale(losses) -> str:
    """'log' when the positive losses of all traces span more than three
    decades, else 'linear' (metrics_io.py:119-125)."""
    vals = [float(v) for seq in losses for v in seq]
    pos = np.array([v for v in vals if v > 0], dtype=float)
    return "log" if pos.size >= 2 and pos.max() > 1e3 * pos.min() else "linear"


# ---------------------------------------------------------------------------
# Host-side file utilities (outside the hot path): plots and 8-bit PNG I/O.
_PLOTS = (("loss_vs_lower_iters.png", "lower_iters_cum", "cumulative lower-level iterations"),
          ("loss_vs_wall_time.png", "wall_s", "wall-clock time [s]"))


def render_plots(traces, out_dir) -> list:
    """Upper loss against cumulative lower iterations and against wall time,
    one curve per trace labelled by trace.method (metrics_io.py:128-160).
    Needs matplotlib (absent in this image: ImportError, as the reference)."""
    import os

    import matplotlib
    matplotlib.use("Agg")
    from matplotlib import pyplot

    if not traces:
        raise ValueError("need at least one trace to plot")
    os.makedirs(out_dir, exist_ok=True)
    yscale = loss_axis_scale([t.loss for t in traces])
    written = []
    for name, attr, label in _PLOTS:
        fig, ax = pyplot.subplots(figsize=(6, 4))
        for t in traces:
            ax.plot(getattr(t, attr), t.loss, label=t.method or "run")
        ax.set(xlabel=label, ylabel="upper-level loss", yscale=yscale)
        ax.legend()
        fig.tight_layout()
        target = os.path.join(out_dir, name)
        fig.savefig(target, dpi=120)
        pyplot.close(fig)
        written.append(target)
    return written


def _to_u8(img) -> np.ndarray:
    arr = nat.to_host(img) if nat.is_torch(img) else np.asarray(img, dtype=float)
    return np.round(np.clip(arr, 0.0, 1.0) * 255.0).astype(np.uint8)


def save_png(img, path) -> None:
    """8-bit PNG of an image with values clamped to [0, 1]; 2-D arrays are
    grayscale (metrics_io.py:163-173)."""
    from PIL import Image
    try:
        Image.fromarray(_to_u8(img)).save(path)
    except OSError as exc:
        raise OSError(f"cannot write image to {path}: {exc}") from exc


def load_png(path) -> np.ndarray:
    """An 8-bit PNG as floats in [0, 1] (metrics_io.py:176-184)."""
    from PIL import Image
    try:
        with Image.open(path) as im:
            return np.asarray(im, dtype=float) / 255.0
    except OSError as exc:
        raise OSError(f"cannot read image from {path}: {exc}") from exc


def save_kernel_image(kernel, path) -> None:
    """The kernel's first channel (or the dense matrix), min-max scaled to
    [0, 1] (a constant kernel renders mid-grey) (metrics_io.py:187-199)."""
    from .operators import Kernel
    arr = np.asarray(kernel.data if isinstance(kernel, Kernel) else kernel, dtype=float)
    if arr.ndim == 3:
        arr = arr[:, :, 0]
    span = float(arr.max()) - float(arr.min())
    save_png((arr - float(arr.min())) / span if span > 0 else np.full_like(arr, 0.5), path)
