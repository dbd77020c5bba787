/*
 * adp_b200.h — C ABI of the B200-native MAID hot path.
 *
 * Drop-in boundary for the reference package `adp` (arxiv 2502.09758,
 * /root/reference/pkg/src/adp).  The reference is pure Python/NumPy with no
 * FFI; its seams are Python functions.  Each entry point
 * below replaces the NumPy/SciPy arithmetic behind one of those functions;
 * the Python package `paper_2502_09758_b200` binds them with ctypes and
 * keeps the reference's Python signatures, return types and exceptions.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers owned by the caller, C-order,
 *     element type given by the plan (float64, or float32 in fp32 mode).
 *     Images are (H, W, C); dense 1-D signals are (n,), dense kernels (n, n).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Scalar results are written to HOST memory; calls that return scalars
 *     synchronise `stream` before returning.
 *   - Return value: ADP_OK or a negative ADP_ERR_* code; adp_last_error()
 *     gives a message.  Numerical failures are reported through the result
 *     structs (status field), mirroring SolveDiverged / NegativeCurvatureError.
 *   - A plan owns its device workspace (allocated once at creation; no
 *     allocation in any hot call) and is not thread-safe: use one plan per
 *     concurrent stream.
 */
#ifndef ADP_B200_H
#define ADP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADP_OK 0
#define ADP_ERR_ARG (-1)
#define ADP_ERR_CUDA (-2)
#define ADP_ERR_UNSUPPORTED (-3)

#define ADP_LAYOUT_DEPTHWISE2D 0 /* operators.py:18, ConvOperator 83-122 */
#define ADP_LAYOUT_DENSE1D 1     /* operators.py:17, DenseOperator 49-80 */

#define ADP_DTYPE_F64 0
#define ADP_DTYPE_F32 1

#define ADP_MODE_STRICT 0 /* bitwise reference arithmetic order (f64) */
#define ADP_MODE_FAST 1   /* FMA stencils */

#define ADP_REG_TV 0      /* SmoothedTV, regularizers.py:137-199 */
#define ADP_REG_ELASTIC 1 /* SmoothedElasticNet, regularizers.py:75-134 */

#define ADP_METHOD_PROXGRAD 0 /* lower_solvers.py:154-167 */
#define ADP_METHOD_AGD 1      /* lower_solvers.py:180-213 */
#define ADP_METHOD_FISTA_SC 2

#define ADP_STATUS_OK 0
#define ADP_STATUS_DIVERGED 1  /* SolveDiverged("... at lower iteration t") */
#define ADP_STATUS_BT_FAIL 2   /* SolveDiverged("backtracking line search failed ...") */
#define ADP_STATUS_NEGCURV 3   /* NegativeCurvatureError */

typedef struct adp_plan adp_plan;

typedef struct {
  int32_t layout; /* ADP_LAYOUT_* */
  int32_t dtype;  /* ADP_DTYPE_* */
  int32_t mode;   /* ADP_MODE_* */
  int32_t H, W, C; /* depthwise2d image; dense1d: H = 1, W = n, C = 1 */
  int32_t kh, kw;  /* stencil size (odd); dense1d: kh = kw = n */
  int32_t tile_h, tile_w; /* 0 = auto */
  int32_t rw;             /* register blocking: outputs per thread (1, 2, 4); 0 = auto */
  /* row slab of a larger image (multi-GPU c5); Hg = 0: not a slab.
   * The plan covers local rows [0, H) = global rows [row0, row0 + H) (owned rows
   * plus ghost rows); only local rows [own0, own1) enter its sums, which keep the
   * GLOBAL image's trees (leaf and tile indices are global).  Tile geometry is
   * chosen from the global shape, so it equals the unsplit plan's; row0, own0 and
   * own1 must be multiples of the tile height (own1 may also be H at the global
   * bottom) and owned ranges of two-level sums must be subtree-aligned. */
  int32_t row0, Hg, own0, own1;
} adp_plan_desc;

/* Lower problem h(x, b) = ||B_b x - y||^2 + alpha J(x) (lower_solvers.py:20-25) */
typedef struct {
  const void* kernel; /* B_b: (kh, kw, C) stencil or (n, n) matrix */
  const void* y;      /* lower-level data */
  double alpha;
  int32_t reg;        /* ADP_REG_* */
  double nu, l1, l2;  /* TV: nu; elastic net: l1, l2, nu */
} adp_lower;

/* solve_lower arguments (lower_solvers.py:104-113) */
typedef struct {
  double eps, mu;
  int32_t max_iters;
  int32_t method;       /* ADP_METHOD_* */
  int32_t adaptive;
  double step_size;     /* <= 0: None (use 1 / L_of_b) */
  double norm_sq;       /* >= 0: cached op_norm_sq (op._norm_sq); < 0: compute */
  int32_t norm_max_iters; /* L_of_b: 300 */
  double norm_tol;        /* L_of_b: 1e-4 */
  const void* v0;       /* power-iteration start vector (un-normalised), device */
  /* injected AGD state (P2 lockstep): x_prev (NULL: x0), momentum t (<= 0: 1),
   * backtracking Lipschitz estimate lip_t (<= 0: L; proxgrad: 1 / step) at the first iteration */
  const void* x_prev0;
  double t_mom0;
  double lip_t0;
} adp_solve_args;

typedef struct {
  double norm_sq;       /* op_norm_sq used (computed or cached) */
  double lip;
  double grad_norm;
  double value;
  int32_t iters;
  int32_t converged;
  int32_t status;       /* ADP_STATUS_* */
  int32_t fail_iter;
  int32_t power_iters;
  int32_t power_converged;
  int64_t vg_evals, value_evals, restarts;
  double t_mom, lip_t;  /* AGD state at exit (momentum t; lip_t, or 1 / step for proxgrad) */
  int64_t launches;     /* kernel launches of the solve (1: the persistent single-launch kernel) */
  double dominant_ms;   /* with adp_plan_profile(p, 1): summed device time (CUDA events on the launching
                         * stream) of the dominant kernel (host-stepped solve: the candidate-value +
                         * speculative-stage-A kernel), and its launch count */
  int64_t dominant_launches;
} adp_solve_result;

typedef struct {
  double residual;
  double curv;
  int32_t iters;
  int32_t converged;
  int32_t status;
  int32_t hv;
  double rs;            /* <r, M^-1 r> at exit (the recurrence's rs) */
} adp_cg_result;

/* ---- plans ---- */
int adp_plan_create(adp_plan** out, const adp_plan_desc* desc);
void adp_plan_destroy(adp_plan* plan);
size_t adp_plan_workspace_bytes(const adp_plan* plan);
const char* adp_last_error(void);
int adp_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---- operators (operators.py) ---- */
/* ConvOperator.apply / DenseOperator.apply: out = B x      (operators.py:70-74, 108-112) */
int adp_apply(adp_plan* p, const void* kernel, const void* x, void* out, void* stream);
/* adjoint: out = B^T y                                      (operators.py:76-80, 114-118) */
int adp_adjoint(adp_plan* p, const void* kernel, const void* y, void* out, void* stream);
/* gram_diag: diag(B^T B)                                    (operators.py:66-68, 120-122) */
int adp_gram_diag(adp_plan* p, const void* kernel, void* out, void* stream);
/* op_norm_sq: power iteration on B^T B                      (operators.py:137-173) */
int adp_op_norm_sq(adp_plan* p, const void* kernel, const void* v0, int32_t max_iters, double tol,
                   double* lam, int32_t* converged, int32_t* iters, void* stream);
/* kernel_gram_correlation: out (kernel-shaped) = kgc(x, v)  (operators.py:198-220) */
int adp_kgc(adp_plan* p, const void* x, const void* v, void* out, void* stream);

/* ---- lower level (lower_solvers.py) ---- */
int adp_lower_value(adp_plan* p, const adp_lower* lp, const void* x, double* value, void* stream);          /* :37-39 */
int adp_lower_value_and_grad(adp_plan* p, const adp_lower* lp, const void* x, double* value, void* g,
                             void* stream);                                                              /* :50-63 */
int adp_lower_grad(adp_plan* p, const adp_lower* lp, const void* x, void* g, void* stream);                /* :42-47 */
int adp_lower_hess_vec(adp_plan* p, const adp_lower* lp, const void* x, const void* v, void* out,
                       void* stream);                                                                    /* :66-71 */
int adp_lower_hess_diag(adp_plan* p, const adp_lower* lp, const void* x, void* out, void* stream);         /* :74-80 */
/* solve_lower -> _gradient_descent / _accelerated, one persistent launch  (:104-213) */
int adp_lower_solve(adp_plan* p, const adp_lower* lp, const void* x0, void* x_out, const adp_solve_args* args,
                    adp_solve_result* res, void* stream);

/* one lower-level iteration from an injected state (x, x_prev, t_mom, lip_t): adp_lower_solve with
 * max_iters = 1 (P2 lockstep protocol).  x_out = the next x (or y when the
 * convergence test fires); res: decisions (value_evals - 1 = backtracking retries, restarts,
 * converged) and the next t_mom / lip_t.  args->max_iters is ignored. */
int adp_lower_iter(adp_plan* p, const adp_lower* lp, const void* x, const void* x_prev, double t_mom, double lip_t,
                   const adp_solve_args* args, void* x_out, adp_solve_result* res, void* stream);

/* ---- hypergradient (hypergradient.py) ---- */
/* cg_solve specialised to the lower Hessian at x_tilde with Jacobi preconditioner
 * lower_hess_diag (computed inside when precond == NULL); q in/out, warm start if warm != 0
 * (hypergradient.py:35-84 as called at 171-176) */
int adp_hess_cg(adp_plan* p, const adp_lower* lp, const void* x_tilde, const void* rhs, void* q, int32_t warm,
                const void* precond, double tol, int32_t max_iters, adp_cg_result* res, void* stream);
/* one PCG iteration from an injected state (q, r, p, rs) at iteration k of cg_solve (hypergradient.py:70-81):
 * hp = H p, curv = <p, hp>, q += a p, r -= a hp, rs' = <r, M^-1 r> (res->rs, res->curv); q and r are updated in
 * place (P2 lockstep protocol).  M = lower_hess_diag(x~) as in adp_hess_cg. */
int adp_cg_iter(adp_plan* p, const adp_lower* lp, const void* x_tilde, void* q, void* r, const void* p_dir, double rs,
                adp_cg_result* res, void* stream);
/* mixed_second_transpose: out = 2 [kgc(x~, B q) + kgc(q, B x~ - y)]   (hypergradient.py:92-104) */
int adp_mixed_T(adp_plan* p, const adp_lower* lp, const void* x_tilde, const void* q, void* out, void* stream);
/* UpperProblem.fit_value (problems.py:48-50) and ||upper_fit_grad|| (hypergradient.py:87-89);
 * grad_out may be NULL */
int adp_upper_terms(adp_plan* p, const void* A_kernel, const void* x, const void* y_delta, double* fit,
                    double* grad_norm, void* grad_out, void* stream);
/* ---- regularizer alone (regularizers.py SmoothedTV / SmoothedElasticNet methods) ----
 * op: 0 value (tv_value / ElasticNet.value), 1 value_and_grad (value -> *value, grad -> out),
 *     2 grad, 3 hess_vec(x, v), 4 hess_diag(x).  reg->kernel, reg->y, reg->alpha are ignored. */
int adp_reg_op(adp_plan* p, const adp_lower* reg, int32_t op, const void* x, const void* v, void* out,
               double* value, void* stream);
/* ddot-type inner product with the plan's fixed reduction tree (np.vdot sites) */
int adp_dot(adp_plan* p, const void* a, const void* b, double* out, void* stream);

/* ---- IFT baseline lower iteration (baselines.py:46-55, prox_grad_iterations) ----
 * n_iters steps of x = prox_l1(x - step (2 B^T (B x - y) + 2 alpha l2 x), step alpha l1) on a dense1d plan
 * with an elastic-net lower problem, one persistent launch; x0 -> x_out (device). */
int adp_prox_grad(adp_plan* p, const adp_lower* lp, const void* x0, void* x_out, int32_t n_iters, double step,
                  void* stream);

/* ---- plan-free vector primitives (generic cg_solve with a caller-supplied hess_vec) ----
 * op 0: out = x + a*y   1: out = x - a*y   2: out = x*y   3: out = 1/x   4: out = x - y   5: out = x
 * op 6: out = prox_l1(x, a) = sign(x) * max(|x| - a, 0)   (regularizers.py:22-27)
 * op 7: out = |y| > a ? x : 0   (soft-threshold activity mask, baselines.py:135)
 * op 10: *red_out = <x, y> (fixed-order tree)   11: *red_out = count(x <= 0) */
int adp_vec(int32_t op, int64_t n, int32_t dtype, double a, const void* x, const void* y, void* out,
            double* red_out, void* stream);

/* ---- quality metrics (metrics_io.py:26-85), float64 device arrays ----
 * adp_np_sum: np.sum of k contiguous segments of n elements each, in NumPy's pairwise order
 * (bitwise); op 0: the elements of x, op 1: (x - y) ** 2 (psnr's squared error, metrics_io.py:34).
 * Results to HOST out[k]; synchronises the stream. */
int adp_np_sum(int32_t op, int32_t k, int64_t n, const void* x, const void* y, double* out, void* stream);
/* ssim (metrics_io.py:47-76): for every channel c the map num/den over the interior windows
 * (H-10) x (W-10) of x, ref (H, W, C) with the ksize x ksize window `win` (HOST, row-major, the
 * reference's _ssim_window(): ksize must be 11) and constants c1, c2; chan_sum[c] (HOST) = np.sum of
 * channel c's map (pairwise order; the caller divides by its size as np.mean does).  map_out
 * (device, C x (H-10) x (W-10)) may be NULL.  Synchronises the stream. */
int adp_ssim(int32_t H, int32_t W, int32_t C, const double* win, int32_t ksize, double c1, double c2,
             const void* x, const void* ref, void* map_out, double* chan_sum, void* stream);

/* ---- FFT stencil path (float64, smoothed TV, depthwise 2-D) ----
 * The zero-padded depthwise correlation of operators.py:101-118 by overlap-save tile FFTs
 * (512 x 512 tiles, two tiles per complex transform) instead of K^2 direct taps: the cheaper
 * choice for large kernels (K = 31 at c5).  Tolerance mode (FFT rounding, ~1e-15 of the output
 * scale); reductions fixed-order (bitwise reproducible run to run).  The plan owns the complex
 * scratch, the kernel spectra (rebuilt from `kernel` at every call) and six image buffers. */
typedef struct adp_fft_plan adp_fft_plan;
int adp_fft_plan_create(adp_fft_plan** out, int32_t H, int32_t W, int32_t C, int32_t kh, int32_t kw);
void adp_fft_plan_destroy(adp_fft_plan* plan);
size_t adp_fft_plan_workspace_bytes(const adp_fft_plan* plan);
/* ConvOperator.apply (adjoint = 0) / .adjoint (adjoint = 1)     (operators.py:108-118) */
int adp_fft_apply(adp_fft_plan* p, const void* kernel, int32_t adjoint, const void* x, void* out, void* stream);
/* lower_value / lower_value_and_grad (lower_solvers.py:37-63); value may be NULL */
int adp_fft_lower_value(adp_fft_plan* p, const adp_lower* lp, const void* x, double* value, void* stream);
int adp_fft_lower_value_and_grad(adp_fft_plan* p, const adp_lower* lp, const void* x, double* value, void* g,
                                 void* stream);
/* op_norm_sq power iteration (operators.py:137-173) */
int adp_fft_op_norm_sq(adp_fft_plan* p, const void* kernel, const void* v0, int32_t max_iters, double tol,
                       double* lam, int32_t* converged, int32_t* iters, void* stream);
/* cg_solve on lower_hess_vec with the lower_hess_diag Jacobi preconditioner (hypergradient.py:35-84 as called
 * at 171-176): same arguments and result fields as adp_hess_cg */
int adp_fft_hess_cg(adp_fft_plan* p, const adp_lower* lp, const void* x_tilde, const void* rhs, void* q, int32_t warm,
                    const void* precond, double tol, int32_t max_iters, adp_cg_result* res, void* stream);
/* UpperProblem.fit_value and ||upper_fit_grad|| (problems.py:48-50, hypergradient.py:87-89): same arguments as
 * adp_upper_terms (grad_out may be NULL) */
int adp_fft_upper_terms(adp_fft_plan* p, const void* A_kernel, const void* x, const void* y_delta, double* fit,
                        double* grad_norm, void* grad_out, void* stream);
/* mixed_second_transpose 2 [kgc(x~, B q) + kgc(q, B x~ - y)] (hypergradient.py:92-104, operators.py:198-220):
 * same arguments as adp_mixed_T (out: device, kernel-shaped (kh, kw, C)) */
int adp_fft_mixed_T(adp_fft_plan* p, const adp_lower* lp, const void* x_tilde, const void* q, void* out, void* stream);
/* solve_lower (lower_solvers.py:104-213): same arguments and result fields as adp_lower_solve */
int adp_fft_lower_solve(adp_fft_plan* p, const adp_lower* lp, const void* x0, void* x_out, const adp_solve_args* args,
                        adp_solve_result* res, void* stream);

/* ---- FP64 roof: sustained DFMA throughput (TFLOP/s, 2 flop per DFMA) of this device ---- */
int adp_fp64_peak(double* tflops, double* ms, void* stream);

/* ---- debug: per-phase %globaltimer stamps of conv solves (enable=1 arms; enable=0 copies
 * 64 x 16 uint64 nanosecond stamps + 256 sub-phase cycle counters to host_out and disarms) ---- */
int adp_debug_trace(adp_plan* p, int32_t enable, uint64_t* host_out);

/* ---- plan geometry: out[0..9] = TH, TW, tilesH, tilesW, fused, leafL, rw, grid, threads, smem bytes;
 * adp_plan_probe computes the same for a descriptor without allocating (grid = 0) */
int adp_plan_geometry(const adp_plan* p, int32_t* out);
int adp_plan_probe(const adp_plan_desc* desc, int32_t* out);

/* ---- row slabs (multi-GPU c5).  One lower-level AGD iteration is split at its reductions:
 * op 0 (ABC): value+grad at y = x + beta (x - xp), first candidate out = y - g / L and its value,
 *             restart dot g.(out - x)                               (lower_solvers.py:196-207)
 * op 1 (C):   backtracking retry: out = y - g / L (g from the last op 0) and its value (:170-177)
 * op 2 (POWER): out = B^T B (x / L) and ||out||^2                   (operators.py:150-165)
 * op 3 (NORM0): ||x||^2                                              (operators.py:150)
 * op 4 (GRAD):  g = lower_grad(x), ||g||^2, fit and tv terms         (lower_solvers.py:212)
 * Each step leaves phase 1 of its sums in the plan; adp_slab_units exposes them. */
int adp_slab_step(adp_plan* p, const adp_lower* lp, int32_t op, const void* x, const void* xp, void* out,
                  double beta, double L, void* stream);
/* Sum units of a slab plan for sum `which` (0 fit, 1 tv, 2 fitc, 3 tvc, 4 ||g||^2 / norm / <p, Hp>,
 * 5 restart dot / <r, M^-1 r>, 6 ||r||^2):
 * the global tree has n_units units (leaf values, or subtree roots when the sum is two-level), of
 * which this plan produces [own[0], own[1]) and [own[2], own[3]).  If dst (device, n_units doubles)
 * is non-NULL those ranges are copied into it at their global offsets (stream-ordered).  Once every
 * rank's ranges are in place (the other entries zero: an all-reduce SUM assembles them exactly),
 * adp_fold_units gives the sum in the single-GPU tree order. */
int adp_slab_units(adp_plan* p, int32_t which, int64_t* n_units, int64_t* own, double* dst, void* stream);

/* ---- row-slab hypergradient (multi-GPU c5: inexact_hypergradient / maid_run on slabs).
 * adp_slab_cg: one step of the hypergradient's Jacobi-PCG (cg_solve, hypergradient.py:35-84, on
 * lower_hess_vec / lower_hess_diag, lower_solvers.py:66-80) over slab + ghosts, split at its sums:
 *   op 0: TV curvature weights and the unfloored Jacobi diagonal of H at x~ = in0; *scal = max over
 *         the owned pixels (the ranks take the max; floor = 1e-12 max + 1e-300, lower_solvers.py:80)
 *   op 1: DIAG = 1 / max(d, s); r = in0 (rhs) - (flag ? H q : 0); out0 = q (zeroed unless flag);
 *         out1 = M^-1 r; sums <r, M^-1 r> (units 5), ||r||^2 (units 6)          (hypergradient.py:55-63)
 *   op 2: flag 0 / 1: p = in0 (+ s * in1) -> out0, H p, <p, Hp> (units 4)       (:70-75, 81)
 *         flag 2: ||H in0 - in1||^2 (units 4), the true residual (:83); flag 3: H in0 (warm start)
 *   op 3: out0 (q) += s p (in0); r -= s H p; out1 = M^-1 r; sums units 5, 6     (:76-80)
 * adp_slab_upper: R = A x - y_delta, grad_out = 2 A^T R, sum(R^2) (units 0), ||grad||^2 (units 4)
 *                 (problems.py:48-50, hypergradient.py:87-89)
 * adp_slab_mixed: the two kernel_gram_correlation terms of mixed_second_transpose
 *                 (hypergradient.py:92-104, operators.py:198-220) for the slab's owned 16-row groups,
 *                 into part (ngroups x ntaps doubles, other groups untouched: zero them, sum over ranks,
 *                 then adp_kgc_final(scale 2) folds the groups in the unsplit order) */
int adp_slab_cg(adp_plan* p, const adp_lower* lp, int32_t op, const void* in0, const void* in1, void* out0,
                void* out1, double s, int32_t flag, double* scal, void* stream);
int adp_slab_upper(adp_plan* p, const void* A_kernel, const void* x, const void* y_delta, void* grad_out,
                   void* stream);
int adp_slab_mixed(adp_plan* p, const adp_lower* lp, const void* x_tilde, const void* q, double* part, void* stream);
int adp_kgc_groups(adp_plan* p, int32_t* ngroups, int32_t* ntaps);
/* plan execution flags: bit 0 = TMA tile boxes in the solve kernel (c2), bit 1 = host-stepped
 * high-occupancy solve_lower (c3-c5: stage kernels one tile per CTA, scalar control on the host),
 * bit 2 = its decision sums folded inside the stage kernels (no reduction launch; csrc/step_tail.h),
 * bit 3 = its candidate launch overlaps the stage-B launch's last wave (per-tile completion flags
 * instead of the grid dependency; ADP_OVL=0: off), bit 4 = stage B overlaps the candidate launch's
 * last wave as well (ADP_OVL=2; measured, off by default) */
int adp_plan_flags(adp_plan* p, int32_t* flags);
/* enable (period k >= 1) / disable (0) live timing of the dominant kernel of host-stepped solves:
 * every k-th iteration's launch is bracketed by CUDA events on its stream (result fields dominant_ms /
 * dominant_launches = the sampled launches' summed device time and count) */
int adp_plan_profile(adp_plan* p, int32_t enable);
int adp_kgc_final(adp_plan* p, const double* part, void* out, double scale, void* stream);
/* k (<= 8) perfect-tree folds (zero-padded to a power of two, <= 16384 units each) of device unit
 * vectors units[i] (n[i] doubles); results to HOST out[i]; synchronises the stream. */
int adp_fold_units(int32_t k, const double* const* units, const int64_t* n, double* out, void* stream);

/* ---- host-only introspection (no device): the deterministic-sum layout for n
 * elements (np_rule = 1: NumPy pairwise leaves of <= 128; 0: binary over n items):
 * leaf starts, subtree cut and the tree programs the kernels evaluate. */
int adp_sum_layout(int64_t n, int32_t np_rule, int64_t* n_leaves, int32_t* n_sub, int32_t* top_prog,
                   int64_t* leaf_start, int64_t leaf_cap, int32_t* sub_leaf, int32_t* sub_prog, int64_t sub_cap,
                   int32_t* words, int64_t words_cap, int64_t* n_words);

#ifdef __cplusplus
}
#endif
#endif /* ADP_B200_H */
