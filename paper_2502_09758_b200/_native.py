"""ctypes binding of ``libadpb200.so`` (the C ABI in ``include/adp_b200.h``).

PyTorch is used only to own device buffers and to name the current CUDA
stream; every arithmetic operation on the hot path runs in the hand-written
sm_100a kernels behind this ABI.  There is no CPU fallback: if the library or
a CUDA device is missing, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADP_LIB") or os.path.join(_HERE, "lib", "libadpb200.so")   # ADP_LIB: A/B builds

ADP_OK = 0
LAYOUT_DEPTHWISE2D = 0
LAYOUT_DENSE1D = 1
DTYPE_F64 = 0
DTYPE_F32 = 1
MODE_STRICT = 0
MODE_FAST = 1
REG_TV = 0
REG_ELASTIC = 1
METHODS = {"proxgrad": 0, "agd": 1, "fista_sc": 2}
STATUS_OK, STATUS_DIVERGED, STATUS_BT_FAIL, STATUS_NEGCURV = 0, 1, 2, 3


class PlanDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("layout", "dtype", "mode", "H", "W", "C", "kh", "kw", "tile_h", "tile_w", "rw",
                 "row0", "Hg", "own0", "own1")]


class Lower(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_void_p), ("y", ctypes.c_void_p), ("alpha", ctypes.c_double),
                ("reg", ctypes.c_int32), ("nu", ctypes.c_double), ("l1", ctypes.c_double),
                ("l2", ctypes.c_double)]


class SolveArgs(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("mu", ctypes.c_double), ("max_iters", ctypes.c_int32),
                ("method", ctypes.c_int32), ("adaptive", ctypes.c_int32), ("step_size", ctypes.c_double),
                ("norm_sq", ctypes.c_double), ("norm_max_iters", ctypes.c_int32),
                ("norm_tol", ctypes.c_double), ("v0", ctypes.c_void_p), ("x_prev0", ctypes.c_void_p),
                ("t_mom0", ctypes.c_double), ("lip_t0", ctypes.c_double)]


class SolveResult(ctypes.Structure):
    _fields_ = [("norm_sq", ctypes.c_double), ("lip", ctypes.c_double), ("grad_norm", ctypes.c_double),
                ("value", ctypes.c_double), ("iters", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("status", ctypes.c_int32), ("fail_iter", ctypes.c_int32), ("power_iters", ctypes.c_int32),
                ("power_converged", ctypes.c_int32), ("vg_evals", ctypes.c_int64),
                ("value_evals", ctypes.c_int64), ("restarts", ctypes.c_int64), ("t_mom", ctypes.c_double),
                ("lip_t", ctypes.c_double), ("launches", ctypes.c_int64), ("dominant_ms", ctypes.c_double),
                ("dominant_launches", ctypes.c_int64)]


class CGResultC(ctypes.Structure):
    _fields_ = [("residual", ctypes.c_double), ("curv", ctypes.c_double), ("iters", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("status", ctypes.c_int32), ("hv", ctypes.c_int32),
                ("rs", ctypes.c_double)]


# Exported symbols and their signatures (kept in sync with include/adp_b200.h).
_P = ctypes.c_void_p
_I = ctypes.c_int32
_D = ctypes.c_double
SIGNATURES = {
    "adp_plan_create": (_I, [ctypes.POINTER(_P), ctypes.POINTER(PlanDesc)]),
    "adp_plan_destroy": (None, [_P]),
    "adp_plan_workspace_bytes": (ctypes.c_size_t, [_P]),
    "adp_last_error": (ctypes.c_char_p, []),
    "adp_device_info": (_I, [ctypes.POINTER(_I)] * 3),
    "adp_apply": (_I, [_P, _P, _P, _P, _P]),
    "adp_adjoint": (_I, [_P, _P, _P, _P, _P]),
    "adp_gram_diag": (_I, [_P, _P, _P, _P]),
    "adp_op_norm_sq": (_I, [_P, _P, _P, _I, _D, ctypes.POINTER(_D), ctypes.POINTER(_I),
                            ctypes.POINTER(_I), _P]),
    "adp_kgc": (_I, [_P, _P, _P, _P, _P]),
    "adp_lower_value": (_I, [_P, ctypes.POINTER(Lower), _P, ctypes.POINTER(_D), _P]),
    "adp_lower_value_and_grad": (_I, [_P, ctypes.POINTER(Lower), _P, ctypes.POINTER(_D), _P, _P]),
    "adp_lower_grad": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P]),
    "adp_lower_hess_vec": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P, _P]),
    "adp_lower_hess_diag": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P]),
    "adp_lower_solve": (_I, [_P, ctypes.POINTER(Lower), _P, _P, ctypes.POINTER(SolveArgs),
                             ctypes.POINTER(SolveResult), _P]),
    "adp_lower_iter": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _D, _D, ctypes.POINTER(SolveArgs), _P,
                            ctypes.POINTER(SolveResult), _P]),
    "adp_hess_cg": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P, _I, _P, _D, _I,
                         ctypes.POINTER(CGResultC), _P]),
    "adp_cg_iter": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P, _P, _D, ctypes.POINTER(CGResultC), _P]),
    "adp_mixed_T": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P, _P]),
    "adp_upper_terms": (_I, [_P, _P, _P, _P, ctypes.POINTER(_D), ctypes.POINTER(_D), _P, _P]),
    "adp_dot": (_I, [_P, _P, _P, ctypes.POINTER(_D), _P]),
    "adp_reg_op": (_I, [_P, ctypes.POINTER(Lower), _I, _P, _P, _P, ctypes.POINTER(_D), _P]),
    "adp_vec": (_I, [_I, ctypes.c_int64, _I, _D, _P, _P, _P, ctypes.POINTER(_D), _P]),
    "adp_np_sum": (_I, [_I, _I, ctypes.c_int64, _P, _P, ctypes.POINTER(_D), _P]),
    "adp_ssim": (_I, [_I, _I, _I, ctypes.POINTER(_D), _I, _D, _D, _P, _P, _P, ctypes.POINTER(_D), _P]),
    "adp_fft_plan_create": (_I, [ctypes.POINTER(_P), _I, _I, _I, _I, _I]),
    "adp_fft_plan_destroy": (None, [_P]),
    "adp_fft_plan_workspace_bytes": (ctypes.c_size_t, [_P]),
    "adp_fft_apply": (_I, [_P, _P, _I, _P, _P, _P]),
    "adp_fft_lower_value": (_I, [_P, ctypes.POINTER(Lower), _P, ctypes.POINTER(_D), _P]),
    "adp_fft_lower_value_and_grad": (_I, [_P, ctypes.POINTER(Lower), _P, ctypes.POINTER(_D), _P, _P]),
    "adp_fft_op_norm_sq": (_I, [_P, _P, _P, _I, _D, ctypes.POINTER(_D), ctypes.POINTER(_I), ctypes.POINTER(_I), _P]),
    "adp_fft_hess_cg": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P, _I, _P, _D, _I, ctypes.POINTER(CGResultC), _P]),
    "adp_fft_upper_terms": (_I, [_P, _P, _P, _P, ctypes.POINTER(_D), ctypes.POINTER(_D), _P, _P]),
    "adp_fft_mixed_T": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P, _P]),
    "adp_fft_lower_solve": (_I, [_P, ctypes.POINTER(Lower), _P, _P, ctypes.POINTER(SolveArgs),
                                 ctypes.POINTER(SolveResult), _P]),
    "adp_debug_trace": (_I, [_P, _I, _P]),
    "adp_fp64_peak": (_I, [ctypes.POINTER(_D), ctypes.POINTER(_D), _P]),
    "adp_prox_grad": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _I, _D, _P]),
    "adp_plan_geometry": (_I, [_P, _P]),
    "adp_plan_probe": (_I, [ctypes.POINTER(PlanDesc), _P]),
    "adp_slab_step": (_I, [_P, ctypes.POINTER(Lower), _I, _P, _P, _P, _D, _D, _P]),
    "adp_slab_units": (_I, [_P, _I, ctypes.POINTER(ctypes.c_int64), _P, _P, _P]),
    "adp_fold_units": (_I, [_I, _P, _P, _P, _P]),
    "adp_slab_cg": (_I, [_P, ctypes.POINTER(Lower), _I, _P, _P, _P, _P, _D, _I, ctypes.POINTER(_D), _P]),
    "adp_slab_upper": (_I, [_P, _P, _P, _P, _P, _P]),
    "adp_slab_mixed": (_I, [_P, ctypes.POINTER(Lower), _P, _P, _P, _P]),
    "adp_kgc_groups": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "adp_plan_flags": (_I, [_P, ctypes.POINTER(_I)]),
    "adp_plan_profile": (_I, [_P, _I]),
    "adp_kgc_final": (_I, [_P, _P, _P, _D, _P]),
    "adp_sum_layout": (_I, [ctypes.c_int64, _I, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_I),
                            ctypes.POINTER(_I), _P, ctypes.c_int64, _P, _P, ctypes.c_int64, _P, ctypes.c_int64,
                            ctypes.POINTER(ctypes.c_int64)]),
}

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A C-ABI call failed (CUDA error or unsupported argument)."""


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and bind every signature (no device needed)."""
    if not os.path.exists(path):
        raise NativeError(
            f"{path} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    cdll = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(cdll, name)
        fn.restype = res
        fn.argtypes = args
    return cdll


def lib() -> ctypes.CDLL:
    """The bound library; requires a CUDA device (fails loudly otherwise)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch
                if not torch.cuda.is_available():
                    raise NativeError("paper_2502_09758_b200 requires a CUDA device (B200, sm_100a); "
                                      "there is no CPU fallback")
                torch.cuda.init()
                _lib = load_library()
    return _lib


def check(rc: int, what: str = ""):
    if rc != ADP_OK:
        msg = lib().adp_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed ({rc}): {msg}")


# ---------------------------------------------------------------------------
# precision settings
_settings = {"dtype": "float64", "mode": "strict"}


def set_precision(dtype: str = "float64", mode: str = "strict"):
    """Select the device arithmetic: float64 strict (bitwise reference order),
    float64 fast (FMA stencils), float64 fft (depthwise stencils of the
    lower-level objective and solver by overlap-save tile FFTs, SURVEY.md
    §8 f2; the other operations run as in fast mode) or float32."""
    if dtype not in ("float64", "float32") or mode not in ("strict", "fast", "fft"):
        raise ValueError("dtype in {float64, float32}, mode in {strict, fast, fft}")
    if mode == "fft" and dtype != "float64":
        raise ValueError("the FFT stencil mode is float64 only")
    _settings["dtype"] = dtype
    _settings["mode"] = mode


def get_precision():
    return dict(_settings)


class precision:
    """Context manager: temporarily switch the device arithmetic."""

    def __init__(self, dtype="float64", mode="strict"):
        self.new = (dtype, mode)

    def __enter__(self):
        self.old = (_settings["dtype"], _settings["mode"])
        set_precision(*self.new)
        return self

    def __exit__(self, *exc):
        set_precision(*self.old)
        return False


def torch_dtype():
    import torch
    return torch.float64 if _settings["dtype"] == "float64" else torch.float32


# ---------------------------------------------------------------------------
class Plan:
    """Owns one ``adp_plan`` (device workspace for one problem shape)."""

    def __init__(self, layout, shape, ksize, dtype, mode, tile=(0, 0), slab=None):
        d = PlanDesc()
        d.layout = layout
        d.dtype = DTYPE_F64 if dtype == "float64" else DTYPE_F32
        d.mode = MODE_STRICT if mode == "strict" else MODE_FAST   # fft: direct kernels in fast mode
        if layout == LAYOUT_DENSE1D:
            n = int(shape[0])
            d.H, d.W, d.C, d.kh, d.kw = 1, n, 1, n, n
        else:
            d.H, d.W, d.C = (int(s) for s in shape)
            d.kh, d.kw = int(ksize[0]), int(ksize[1])
        d.tile_h, d.tile_w = int(tile[0]), int(tile[1])
        if slab is not None:        # (row0, Hg, own0, own1): a row slab of a larger image
            d.row0, d.Hg, d.own0, d.own1 = (int(v) for v in slab)
        self.desc = d
        self.handle = ctypes.c_void_p()
        check(lib().adp_plan_create(ctypes.byref(self.handle), ctypes.byref(d)), "adp_plan_create")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            try:
                _lib.adp_plan_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def workspace_bytes(self) -> int:
        return int(lib().adp_plan_workspace_bytes(self.handle))

    def geometry(self) -> dict:
        """Tile geometry chosen by the plan (depthwise 2-D)."""
        out = (ctypes.c_int32 * 10)()
        check(lib().adp_plan_geometry(self.handle, out), "adp_plan_geometry")
        return dict(zip(GEOMETRY_KEYS, (int(v) for v in out)))

    def flags(self) -> dict:
        """Execution choices of the plan: TMA tile boxes, host-stepped solve, in-kernel decision sums,
        candidate launch overlapping stage B's last wave (tile flags), stage B overlapping the candidate
        launch's (opt-in)."""
        f = ctypes.c_int32()
        check(lib().adp_plan_flags(self.handle, ctypes.byref(f)), "adp_plan_flags")
        return {"tma": bool(f.value & 1), "step": bool(f.value & 2), "tail": bool(f.value & 4),
                "ovl": bool(f.value & 8), "ovl_b": bool(f.value & 16)}


_plans: dict = {}
_tile_override: dict = {}


def set_tile(shape_key, tile):
    _tile_override[shape_key] = tile


def host_fingerprint(arr) -> int:
    """Cheap content tag of a host array for device-copy caches: the bytes of
    4,096 strided samples (plus shape and address).  Catches reassignment and
    the usual in-place edits (y[:] = ..., y *= s) without reading the whole
    array; an edit that touches none of the sampled elements is not seen."""
    a = np.asarray(arr)
    flat = a.reshape(-1) if a.flags.c_contiguous else np.ascontiguousarray(a).reshape(-1)
    step = max(1, flat.size // 4096)
    return hash((a.shape, a.__array_interface__["data"][0], flat[::step].tobytes()))


def current_device() -> int:
    """CUDA device of the calling thread: every device-side cache is keyed by it."""
    import torch
    return torch.cuda.current_device()


def plan_for(layout, shape, ksize=(0, 0), slot=None) -> Plan:
    """Cached plan per (layout, shape, kernel size, precision, thread/slot)."""
    tile = _tile_override.get((layout, tuple(int(s) for s in shape), tuple(int(k) for k in ksize)), (0, 0))
    key = (layout, tuple(int(s) for s in shape), tuple(int(k) for k in ksize), _settings["dtype"],
           _settings["mode"], threading.get_ident() if slot is None else slot, tuple(tile), current_device())
    p = _plans.get(key)
    if p is None:
        p = Plan(layout, shape, ksize, _settings["dtype"], _settings["mode"], tile)
        _plans[key] = p
    return p


GEOMETRY_KEYS = ("TH", "TW", "tilesH", "tilesW", "fused", "leafL", "rw", "grid", "threads", "smem")


def probe_geometry(shape, ksize, tile=(0, 0)) -> dict:
    """Tile geometry a depthwise 2-D plan of this shape would use (no allocation)."""
    d = PlanDesc()
    d.layout = LAYOUT_DEPTHWISE2D
    d.dtype = DTYPE_F64 if _settings["dtype"] == "float64" else DTYPE_F32
    d.mode = MODE_STRICT if _settings["mode"] == "strict" else MODE_FAST
    d.H, d.W, d.C = (int(s) for s in shape)
    d.kh, d.kw = int(ksize[0]), int(ksize[1])
    d.tile_h, d.tile_w = int(tile[0]), int(tile[1])
    out = (ctypes.c_int32 * 10)()
    check(lib().adp_plan_probe(ctypes.byref(d), out), "adp_plan_probe")
    return dict(zip(GEOMETRY_KEYS, (int(v) for v in out)))


def clear_plans():
    _plans.clear()
    _fft_plans.clear()


def is_fft() -> bool:
    return _settings["mode"] == "fft"


class FFTPlan:
    """Owns one ``adp_fft_plan`` (tile-FFT stencils for one image shape and kernel size)."""

    def __init__(self, shape, ksize):
        H, W, C = (int(s) for s in shape)
        self.handle = ctypes.c_void_p()
        check(lib().adp_fft_plan_create(ctypes.byref(self.handle), H, W, C, int(ksize[0]), int(ksize[1])),
              "adp_fft_plan_create")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            try:
                _lib.adp_fft_plan_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def workspace_bytes(self) -> int:
        return int(lib().adp_fft_plan_workspace_bytes(self.handle))


_fft_plans: dict = {}


def fft_plan_for(shape, ksize, slot=None) -> FFTPlan:
    key = (tuple(int(s) for s in shape), tuple(int(k) for k in ksize),
           threading.get_ident() if slot is None else slot)
    p = _fft_plans.get(key)
    if p is None:
        p = FFTPlan(shape, ksize)
        _fft_plans[key] = p
    return p


def stream_ptr():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


# ---------------------------------------------------------------------------
# array helpers: accept numpy or torch; device tensors in the working dtype
def is_torch(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def to_dev(x, shape=None):
    """Contiguous device tensor of the working dtype (copies host data)."""
    import torch
    dt = torch_dtype()
    if is_torch(x):
        t = x
        if t.device.type != "cuda":
            t = t.to("cuda")
        if t.dtype != dt:
            t = t.to(dt)
        t = t.contiguous()
    else:
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        t = torch.from_numpy(a).to("cuda", non_blocking=False)
        if t.dtype != dt:
            t = t.to(dt)
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t


def empty_like_dev(shape):
    import torch
    return torch.empty(tuple(shape), dtype=torch_dtype(), device="cuda")


def zeros_dev(shape):
    import torch
    return torch.zeros(tuple(shape), dtype=torch_dtype(), device="cuda")


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def to_host(t) -> np.ndarray:
    return t.detach().to("cpu").numpy()


def like(t, ref):
    """Return device tensor t in the kind of `ref` (numpy -> numpy float64)."""
    if is_torch(ref):
        return t
    return np.asarray(to_host(t), dtype=np.float64)


_v0_cache: dict = {}


def power_start(shape):
    """The reference's power-iteration start vector (operators.py:145-149):
    ones + 0.01 * standard_normal from default_rng(0), un-normalised.  A
    constant of the algorithm generated once per shape and kept on device."""
    key = (tuple(shape), _settings["dtype"], current_device())
    t = _v0_cache.get(key)
    if t is None:
        rng = np.random.default_rng(0)
        v = np.ones(shape) + 0.01 * rng.standard_normal(shape)
        t = to_dev(v)
        _v0_cache[key] = t
    return t
