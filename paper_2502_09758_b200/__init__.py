"""B200-native MAID hot path for the analytic deep prior with a learned blur
kernel (arxiv 2502.09758) — drop-in for the reference package ``adp``.

Same module layout and public names as ``adp`` (reference
``pkg/src/adp/__init__.py``) for the hot path: operators, regularizers,
lower-level solvers, hypergradient and the MAID driver.  All image-space
arithmetic runs in hand-written sm_100a CUDA kernels behind the C ABI in
``include/adp_b200.h``; there is no CPU fallback.

Precision: ``set_precision("float64", "strict")`` (default; the
reference's own rounding order, bitwise on stencils and np.sum sites),
``("float64", "fast")`` (FMA stencils) or ``("float32", ...)``.
"""

from ._native import NativeError, get_precision, precision, set_precision
from .baselines import BaselineConfig, prox_grad_iterations, run_ift, run_unrolled, unrolled_gradient
from .hypergradient import (
    CGResult,
    HypergradResult,
    NegativeCurvatureError,
    WarmState,
    cg_solve,
    inexact_hypergradient,
    mixed_second_transpose,
    sobolev_grad,
    sobolev_value,
    upper_fit_grad,
)
from .lower_solvers import (
    L_of_b,
    LowerProblem,
    LowerSolveResult,
    SolveDiverged,
    lower_grad,
    lower_hess_diag,
    lower_hess_vec,
    lower_iteration,
    lower_value,
    lower_value_and_grad,
    mu_of_b,
    solve_lower,
)
from .metrics_io import MetricReport, metric_report, psnr, ssim
from .maid import BacktrackingStalled, MAIDConfig, RunTrace, lip_upper_x, maid_run, psi, psi_value
from .operators import (
    DENSE1D,
    DEPTHWISE2D,
    ConvOperator,
    DenseOperator,
    Kernel,
    gaussian_conv_matrix,
    kernel_gram_correlation,
    op_norm_sq,
    operator_from_kernel,
)
from .problems import (
    UpperProblem,
    build_deconv1d,
    build_motion2d,
    build_semiblind2d,
    piecewise_signal,
    solve_lower_at,
)
from .regularizers import (
    SmoothedElasticNet,
    SmoothedTV,
    image_forward_diff,
    image_forward_diff_adjoint,
    prox_l1,
    smoothed_abs_norm,
    tv_value,
)

__version__ = "0.1.0"

__all__ = [
    "BacktrackingStalled", "BaselineConfig", "CGResult", "ConvOperator", "DENSE1D", "DEPTHWISE2D", "DenseOperator",
    "HypergradResult", "Kernel", "L_of_b", "LowerProblem", "LowerSolveResult", "MAIDConfig", "MetricReport", "metric_report", "psnr", "ssim",
    "NativeError", "NegativeCurvatureError", "RunTrace", "SmoothedElasticNet", "SmoothedTV", "SolveDiverged",
    "UpperProblem", "WarmState", "build_deconv1d", "build_motion2d", "build_semiblind2d", "cg_solve",
    "gaussian_conv_matrix", "get_precision", "image_forward_diff", "image_forward_diff_adjoint",
    "inexact_hypergradient", "kernel_gram_correlation", "lip_upper_x", "lower_grad", "lower_hess_diag",
    "lower_hess_vec", "lower_iteration", "lower_value", "lower_value_and_grad", "maid_run", "mixed_second_transpose", "mu_of_b",
    "op_norm_sq", "operator_from_kernel", "piecewise_signal", "precision", "prox_grad_iterations", "prox_l1", "psi", "psi_value", "run_ift", "run_unrolled",
    "set_precision", "smoothed_abs_norm", "sobolev_grad", "sobolev_value", "solve_lower", "solve_lower_at",
    "tv_value", "unrolled_gradient", "upper_fit_grad",
]
