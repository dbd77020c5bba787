// Kernel-argument block of the depthwise 2-D engine (host + device).
#pragma once
#include <cuda.h>   // CUtensorMap
#include "adp_types.h"

namespace adp {

enum ConvMode : int {
  CM_APPLY = 0,          // out0 = B in0
  CM_ADJOINT = 1,        // out0 = B^T in0
  CM_GRAM_DIAG = 2,      // out0 = correlate(ones, flipped**2)
  CM_VALUE = 3,          // scal[0] = lower_value(in0)
  CM_VALUE_GRAD = 4,     // scal[0] = value, out0 = grad    (value_and_grad form)
  CM_GRAD = 5,           // out0 = lower_grad(in0)
  CM_HESS_VEC = 6,       // out0 = H(in0 = x) in1
  CM_HESS_DIAG = 7,      // out0 = lower_hess_diag(in0)
  CM_UPPER = 8,          // scal[0] = sum((B in0 - y)^2), scal[1] = ||2 B^T (B in0 - y)||, out0 = grad or null
  CM_POWER = 9,          // scal[0] = op_norm_sq, scal[1] = converged, scal[2] = iters
  CM_MIXED_PREP = 10,    // out0 = B in0 - y (residual), out1 = B in1 (B q)
  CM_DOT = 11,           // scal[0] = <in0, in1> (ddot-type, fixed tree)
  CM_SLAB_ABC = 12,      // row slab: A, B (+ candidate out0), C at out0; phase-1 sums
  CM_SLAB_C = 13,        // row slab: candidate retry at L -> out0; phase-1 sums
  CM_SLAB_POWER = 14,    // row slab: out0 = B^T B (in0 / sL); phase-1 of ||out0||^2
  CM_SLAB_NORM0 = 15,    // row slab: phase-1 of ||in0||^2
  CM_SLAB_GRAD = 16,     // row slab: lower_grad(in0) -> G; phase-1 of fit, tv, ||g||^2
  CM_BENCH_REDUCE = 17,  // micro-benchmark: the solve's 6-sum reduction, mode-param times back to back
  // row-slab hypergradient steps (multigpu.SlabHypergradient): each stops after phase 1 of its sums
  CM_SLAB_CG_DIAG = 18,  // TV weights + unfloored Jacobi diagonal of H(in0 = x~); scal[0] = max over owned pixels
  CM_SLAB_CG_INIT = 19,  // DIAG = 1 / max(d, sL); r = in0 (- HP if sflag); out0 = q (0 unless sflag); out1 = s
  CM_SLAB_CG_HV = 20,    // sflag 0/1: p = in0 (+ sbeta in1) -> out0, HP = H p, <p, Hp>; 2: (H in0 - in1)^2; 3: HP = H in0
  CM_SLAB_CG_UPD = 21,   // q (out0) += sbeta p (in0); r -= sbeta HP; s (out1) = DIAG r; <r, s>, <r, r>
  CM_SLAB_UPPER = 22,    // R = A in0 - y; out0 = 2 A^T R; leaves of R^2 (owned rows), <out0, out0>
  CM_SLAB_MIXED_PREP = 23,  // R = B in0 - y, BP = B in1 (every local row)
};


template <typename T>
struct ConvArgs {
  ConvGeom g;
  const T* kern;           // (kh, kw, C) stencil, C-order
  const T* ydat;           // lower-level data y (H, W, C)
  double alpha, nu, regcurv;  // alpha, TV nu, C_J
  int reg;                 // RegKind (conv path: REG_TV)
  int method, adaptive;
  int max_iters;
  double tol, mu;          // tol = eps * mu
  double step_given;       // > 0: step_size passed by the caller
  double lip_cached;       // > 0: op norm already known (op._norm_sq cache)
  int power_max_iters;
  double power_tol;
  const T* v0;             // power-iteration start (un-normalised)
  const T* x0;             // warm start
  const T* xprev0;         // injected x_prev (NULL: x0)
  double t_mom0, lip_t0;   // injected momentum / Lipschitz estimate (<= 0: defaults)
  T* out;                  // x_tilde
  // workspace
  T* X[3];
  T* R;  T* RC; T* G; T* TVG; T* TV2; T* TV2C;
  // CG / Hessian
  const T* xt;             // x_tilde (Hessian point)
  const T* rhs;
  T* Q;                    // q (in/out)
  const T* diag_in;        // optional precond diag
  T* DIAG;                 // inv diag workspace / diag output
  T* WV; T* WH;            // rho'' weights
  T* P[2]; T* BP; T* HP; T* CR; T* CS;
  int warm;
  // P2 lockstep of one CG iteration: injected r, p, rs (cg_p0 != NULL); r is written back to cg_r
  T* cg_r;
  const T* cg_p0;
  double cg_rs0;
  // sums
  SumDev s_fit, s_tv, s_fitc, s_tvc;   // numpy-pairwise element sums (N, 2N, N, 2N)
  SumDev s_t0, s_t1, s_t2;             // per-tile partial sums (ddot-type)
  SumDev s_fit2, s_tv2;                // second (fit, tv) set: speculative next value (fuseCA)
  unsigned int* bar;
  SolveOut* sres;
  CGOut* cres;
  double* scal;            // misc scalar outputs
  int mode;                // misc kernel mode
  int nofloor;             // hess_diag without the 1e-12*max floor (regularizer-only call)
  double sbeta, sL;        // row-slab steps: momentum beta, trial Lipschitz L (or power scale)
  double sbetaN;           // host-stepped solve: momentum of the next extrapolation point
  double* hscal;           // host-stepped solve: results also written to mapped pinned host memory,
  volatile int* hflag;     //   then the sequence number `hseq` to hflag (the host spins on it)
  int hseq;
  int sflag;               // row-slab CG steps: variant (see CM_SLAB_CG_*)
  unsigned int* tflag;     // host-stepped solve: per-tile completion flags of the stage-B launch (value tseq),
  unsigned int tseq;       //   polled by the overlapping candidate launch (conv2d_step.cu); NULL: off
  unsigned long long* trace;  // optional phase timestamps (CTA 0): [iter][16] %globaltimer ns
  const T* in0; const T* in1; T* out0; T* out1;
  // TMA descriptors of the plan's workspace images (KS = 9 single-channel
  // solve kernel): X[0..2], R, P[0] (the next extrapolation point)
  CUtensorMap tm[5];
};

// Host-stepped stage kernels: the launch's tap set as a kernel parameter
// (constant bank 0), channel-major [c][i][j] with ndimage's |w| <= DBL_EPSILON
// taps zeroed; forward taps for the value passes, flipped for the adjoint.
// Channel blocks are padded to an even tap count (16-byte aligned tap pairs).
// Two capacities: StepW (stencils up to 1024 padded taps: c2-c4) and StepWL (31 x 31 x 3: c5), so the
// common launches do not carry the large block; the host fills a StepWL and passes its address to either.
constexpr int kStepWSmall = 1024;
constexpr int kStepWMax = 3072;
template <int N>
struct alignas(16) StepWT {
  double w[N];
};
using StepW = StepWT<kStepWSmall>;
using StepWL = StepWT<kStepWMax>;

template <typename T>
struct KgcArgs {
  ConvGeom g;
  const T* xa; const T* va; const T* xb; const T* vb;
  double* part;   // [ngroups][kh*kw*C]
  int ngroups;    // (tile row of 16 image rows, column block) groups over the GLOBAL image
  int cblocks;    // column blocks per tile row
  T* out;         // (kh, kw, C)
  double scale;
};

struct ConvKernelSet {
  const void* solve;
  const void* cg;
  const void* misc;
  const void* kgc_part;
  const void* kgc_final;
};
ConvKernelSet conv_kernels_f64s();
ConvKernelSet conv_kernels_f64f();
ConvKernelSet conv_kernels_f32();
ConvKernelSet conv_kernels_f64s_rw2();
ConvKernelSet conv_kernels_f64f_rw2();
ConvKernelSet conv_kernels_f64s_rw1();
ConvKernelSet conv_kernels_f64f_rw1();
// solve kernels specialised to a 9x9 stencil at RW = 2 (c2), float64
const void* conv_solve_k9(int fast);
// the same with TMA tile boxes (dense plane layout, LDS.128 windows)
const void* conv_solve_k9_tma(int fast);
// host-stepped solve (conv2d_step.cu): stage kernels, one tile per CTA
struct StepKernels {
  const void* b;
  const void* c;
  const void* a;
  const void* red;
  const void* extrap;
  const void* ca;
  const void* cand;   // elementwise backtracking-retry candidate + its next extrapolation point
  int b_ep;        // stage-B epilogue operand variant (2: term buffers, two CTAs per SM)
};
// k: the plan's stencil size when square (instances specialised to 15 x 15 exist), else 0
StepKernels step_kernels(int fast, int k);
// thread bound of the compile-time-stencil solve kernel (the host selects it
// only for CTAs of at most this many threads)
constexpr int kSolveKSThreads = 256;
// RW = 4 solve kernels bounded at kSolveT384 threads (168 registers instead
// of 128; the host selects them for CTAs of at most that many threads)
constexpr int kSolveT384 = 384;
const void* conv_solve_t384(int dtype, int fast);
inline ConvKernelSet conv_kernels(int dtype, int mode, int rw) {
  if (dtype == 1) return conv_kernels_f32();
  const bool fast = mode == 1;
  if (rw == 1) return fast ? conv_kernels_f64f_rw1() : conv_kernels_f64s_rw1();
  if (rw == 2) return fast ? conv_kernels_f64f_rw2() : conv_kernels_f64s_rw2();
  return fast ? conv_kernels_f64f() : conv_kernels_f64s();
}

}  // namespace adp
