// FFT stencil path for large kernels: the depthwise
// zero-padded correlation of operators.py:101-118 computed by overlap-save
// tile FFTs instead of K^2 direct taps, and the lower-level AGD solve
// (lower_solvers.py:104-213) driven on top of it.
//
// Tiles.  The image (H, W, C) is cut into output tiles of Vh x Vw = (T-kh+1) x
// (T-kw+1) pixels, T = 512.  Tile input u[a][b] = x[h0-rh+a, w0-rw+b] (zero
// outside the image); the circular cross-correlation of u with the kernel
// zero-padded to T x T equals the linear one on the first Vh x Vw outputs.
// Two tiles of the same channel share one complex transform (tile a in the
// real part, tile b in the imaginary part): the kernel is real, so the
// correlation acts on both parts independently.
//
// Passes (one stencil = three launches, all in HBM-resident complex scratch):
//   K1 row pass     : load the two tiles' rows (zero padded), FFT-512 per row;
//                     a load prologue can produce the input on the fly (the
//                     AGD extrapolation, the backtracking candidate with the
//                     restart dot, the power iteration's w / lam, the CG
//                     direction) and store it for the later passes
//   K2 column pass  : FFT-512 per column, multiply by conj(FFT2(kernel)),
//                     inverse FFT-512 per column (registers + two padded
//                     shared-memory exchanges per transform)
//   K3 inverse rows : inverse FFT-512 per row, crop the valid outputs, fused
//                     epilogue (residual, gradient with the TV term, value
//                     terms, power-iteration norm, Hessian products, upper
//                     terms) with per-CTA partial sums
// The FFT is a register-resident radix-8 Stockham transform (3 stages for 512
// points; each of 64 threads owns elements j + 64 r) with an accurately
// rounded twiddle table.  Also here: the host-driven solvers on these passes
// (solve_lower, the hypergradient's PCG, op_norm_sq), the kernel-gradient
// correlation by frequency-domain pair products, the upper terms.
//
// Arithmetic: float64; complex multiplies use FMA and the TV terms use rsqrt
// (a tolerance-only mode, like "fast": results differ from the direct strict
// stencil by FFT rounding, ~1e-15 of the output scale).  Reductions are
// fixed-order (per-CTA trees, then a fixed fold), so every run is bitwise
// reproducible.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <string>
#include <vector>
#include "adp_device.cuh"
#include "../../include/adp_b200.h"

namespace adp {
int dense_fail(int code, const char* m);

namespace fft {

constexpr int T = 512;          // transform length (both axes)
constexpr int RROWS = 4;        // rows per CTA in the row passes (64 threads per row)
#ifndef FFT_CCOLS
#define FFT_CCOLS 4
#endif
constexpr int CCOLS = FFT_CCOLS;   // columns per CTA in the column pass (64 threads per column)
constexpr double kInvT2 = 1.0 / (512.0 * 512.0);   // exact power of two

struct Geo {
  int H, W, C, kh, kw, rh, rw, Vh, Vw, ntY, ntX, ntiles, npairs;
  // chunked stencil passes (see stencil()): this launch covers the global tile pairs pair0.., whose
  // scratch slots are spair0.. of an S laid out with spairs pairs per channel
  int pair0, spair0, spairs;
};

// ---------------------------------------------------------------------------
// radix-8 butterflies
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {   // FMA: this path is a tolerance mode
  return make_double2(fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x));
}
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {   // forward: * (-i); inverse: * (+i)
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// In-register 8-point DFT, natural order in and out (decimation in frequency).
template <bool INV>
__device__ __forceinline__ void dft8(double2* v) {
  constexpr double s = 0.70710678118654752440;
  double2 b0 = cadd(v[0], v[4]), b4 = csub(v[0], v[4]);
  double2 b1 = cadd(v[1], v[5]), b5 = csub(v[1], v[5]);
  double2 b2 = cadd(v[2], v[6]), b6 = csub(v[2], v[6]);
  double2 b3 = cadd(v[3], v[7]), b7 = csub(v[3], v[7]);
  // b5 *= w8^1, b6 *= w8^2, b7 *= w8^3  (w8 = exp(-+2 pi i / 8))
  b5 = INV ? make_double2(s * (b5.x - b5.y), s * (b5.x + b5.y)) : make_double2(s * (b5.x + b5.y), s * (b5.y - b5.x));
  b6 = mul_mi<INV>(b6);
  b7 = INV ? make_double2(-s * (b7.x + b7.y), s * (b7.x - b7.y)) : make_double2(s * (b7.y - b7.x), -s * (b7.x + b7.y));
  double2 c0 = cadd(b0, b2), c2 = csub(b0, b2);
  double2 c1 = cadd(b1, b3), c3 = mul_mi<INV>(csub(b1, b3));
  double2 c4 = cadd(b4, b6), c6 = csub(b4, b6);
  double2 c5 = cadd(b5, b7), c7 = mul_mi<INV>(csub(b5, b7));
  v[0] = cadd(c0, c1);
  v[4] = csub(c0, c1);
  v[2] = cadd(c2, c3);
  v[6] = csub(c2, c3);
  v[1] = cadd(c4, c5);
  v[5] = csub(c4, c5);
  v[3] = cadd(c6, c7);
  v[7] = csub(c6, c7);
}

// Register-resident 512-point FFT (radix-8 Stockham, 3 stages) of one batch.
// The batch's 64 threads (j = 0..63) hold v[r] = element j + 64 r on entry
// and output element j + 64 r on exit, so global loads and stores around it
// are direct and coalesced; the two inter-stage exchanges go through the
// batch's shared buffer `sm` (>= kPadB double2) with one pad slot per 8
// elements (conflict-free 16-byte accesses).  Every thread of the CTA must
// call it together (it contains CTA barriers; on return `sm` is free).
// padded batch stride = 2 mod 8 (16-byte units): the 8 threads of each quarter-warp phase of a
// column pass (2 rows x 4 columns) land on 8 distinct bank groups
constexpr int kPadB = 512 + 64 + 2;
__device__ __forceinline__ int pad8(int i) { return i + (i >> 3); }

template <bool INV>
__device__ __forceinline__ void twiddle(double2* v, int step, const double2* __restrict__ tw) {
#pragma unroll
  for (int r = 1; r < 8; ++r) {
    double2 w = __ldg(tw + ((r * step) & 511));   // exp(-2 pi i m / 512), m = r * step
    if (INV) w.y = -w.y;
    v[r] = cmul(v[r], w);
  }
}

template <bool INV>
__device__ __forceinline__ void fft512_reg(double2* v, double2* sm, int j, const double2* __restrict__ tw) {
  dft8<INV>(v);                                   // stage 0 (Ns = 1): outputs to 8 j + r
#pragma unroll
  for (int r = 0; r < 8; ++r) sm[pad8(8 * j + r)] = v[r];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = sm[pad8(j + 64 * r)];
  __syncthreads();
  const int k = j & 7;                            // stage 1 (Ns = 8): outputs to (j - k) 8 + k + 8 r
  twiddle<INV>(v, 8 * k, tw);
  dft8<INV>(v);
#pragma unroll
  for (int r = 0; r < 8; ++r) sm[pad8((j - k) * 8 + k + 8 * r)] = v[r];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = sm[pad8(j + 64 * r)];
  __syncthreads();
  twiddle<INV>(v, j, tw);                         // stage 2 (Ns = 64): outputs to j + 64 r
  dft8<INV>(v);
}

// Block index -> (pair, row/column group, channel); channel fastest so the
// C CTAs that read (write) the same interleaved image rows run together.
__device__ __forceinline__ void block_coords(int groups, int C, int& p, int& grp, int& c) {
  const int b = blockIdx.x;
  c = b % C;
  const int q = b / C;
  p = q / groups;
  grp = q - p * groups;
}

// ---------------------------------------------------------------------------
// K1: row pass.  grid npairs * (T / RROWS) * C, 256 threads (64 per row).
// mode 0: image tiles of x; mode 1: kernel embedding (spectrum setup; pair p:
// p = 0 the kernel, p = 1 the flipped kernel).
// Row-pass prologues: the elementwise solver step that produces the stencil's
// input is computed while loading it (no separate pass over HBM).  The tile's
// valid-region pixels (each image pixel exactly once) store the produced
// iterate for the later passes.
enum Pro {
  P_NONE = 0,    // input = x
  P_EXTRAP = 1,  // input = y = x + coef (x - x2), stored to wout        (lower_solvers.py:197)
  P_STEP = 2,    // input = xc = x - x2 * coef (x = y, x2 = g, coef = 1 / L), stored; partial sum g (xc - xold)
                 // (:173, :209)
  P_SCALE = 3,   // input = x * coef (power iteration v = w / lam with coef = 1 / lam, operators.py:162)
  P_CGDIR = 4    // input = p' = minv * r + coef * p (x = r, x2 = minv, xold = p), stored to wout (hypergradient.py:79-80)
};

struct RowArgs {
  Geo g;
  const double* x;
  double2* S;       // scratch (C, npairs, T, T)
  const double2* tw;
  int mode;
  const double* kern;   // (kh, kw, C)
  int pro;
  const double* x2;
  const double* xold;
  double coef;
  double* wout;
  double* part;         // P_STEP: one partial per CTA
};

__device__ __forceinline__ void tile_origin(const Geo& g, int t, int& h0, int& w0) {
  const int ty = t / g.ntX, tx = t - ty * g.ntX;
  h0 = ty * g.Vh;
  w0 = tx * g.Vw;
}

__device__ __forceinline__ double row_input(const RowArgs& A, int64_t o, bool valid, double& dot) {
  const double xv = A.x[o];
  switch (A.pro) {
    case P_EXTRAP: {
      const double u = xv + A.coef * (xv - A.x2[o]);
      if (valid) A.wout[o] = u;
      return u;
    }
    case P_STEP: {   // coef = 1 / L: a multiply instead of the reference's division (tolerance mode)
      const double gv = A.x2[o];
      const double u = xv - gv * A.coef;
      if (valid) {
        A.wout[o] = u;
        dot = dot + gv * (u - A.xold[o]);
      }
      return u;
    }
    case P_SCALE: return xv * A.coef;   // coef = 1 / lam
    case P_CGDIR: {
      const double u = A.x2[o] * xv + A.coef * A.xold[o];
      if (valid) A.wout[o] = u;
      return u;
    }
    default: return xv;
  }
}

#ifndef FFT_ROW_MINB
#define FFT_ROW_MINB 3
#endif
__global__ void __launch_bounds__(256, FFT_ROW_MINB) row_fwd_kernel(const __grid_constant__ RowArgs A) {
  __shared__ __align__(16) double2 sm[RROWS * kPadB];
  __shared__ double red[40];
  const Geo& g = A.g;
  int p, rg, c;
  block_coords(T / RROWS, g.C, p, rg, c);
  const int j = threadIdx.x & 63, rr = threadIdx.x >> 6, row = rg * RROWS + rr;
  double2 v[8];
  double dot = 0.0;
  if (A.mode == 0) {
    int h0a, w0a, h0b = 0, w0b = 0;
    const int pg = p + g.pair0;   // global pair
    tile_origin(g, 2 * pg, h0a, w0a);
    const bool hasb = 2 * pg + 1 < g.ntiles;
    if (hasb) tile_origin(g, 2 * pg + 1, h0b, w0b);
    const int ha = h0a - g.rh + row, hb = h0b - g.rh + row;
    const bool rowa = ha >= 0 && ha < g.H, rowb = hasb && hb >= 0 && hb < g.H;
    const bool vrow = row >= g.rh && row - g.rh < g.Vh;     // valid-region row of both tiles
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int col = j + 64 * r;
      const int wa = w0a - g.rw + col, wb = w0b - g.rw + col;
      const bool vcol = vrow && col >= g.rw && col - g.rw < g.Vw;
      double re = 0.0, im = 0.0;
      if (rowa && wa >= 0 && wa < g.W) re = row_input(A, ((int64_t)ha * g.W + wa) * g.C + c, vcol, dot);
      if (rowb && wb >= 0 && wb < g.W) im = row_input(A, ((int64_t)hb * g.W + wb) * g.C + c, vcol, dot);
      v[r] = make_double2(re, im);
    }
    if (A.pro == P_STEP) {
      const double s = block_sum(dot, red);
      if (threadIdx.x == 0) A.part[blockIdx.x + g.pair0 * (T / RROWS) * g.C] = s;   // global CTA index
    }
  } else if (A.mode == 2) {   // kgc: the tiles' own valid-region pixels v[h0 + a, w0 + b] (zero elsewhere)
    int h0a, w0a, h0b = 0, w0b = 0;
    tile_origin(g, 2 * p, h0a, w0a);
    const bool hasb = 2 * p + 1 < g.ntiles;
    if (hasb) tile_origin(g, 2 * p + 1, h0b, w0b);
    const bool vrow = row < g.Vh;
    const bool rowa = vrow && h0a + row < g.H, rowb = vrow && hasb && h0b + row < g.H;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int col = j + 64 * r;
      double re = 0.0, im = 0.0;
      if (rowa && col < g.Vw && w0a + col < g.W) re = A.x[((int64_t)(h0a + row) * g.W + w0a + col) * g.C + c];
      if (rowb && col < g.Vw && w0b + col < g.W) im = A.x[((int64_t)(h0b + row) * g.W + w0b + col) * g.C + c];
      v[r] = make_double2(re, im);
    }
  } else {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int col = j + 64 * r;
      double val = 0.0;
      if (row < g.kh && col < g.kw) {
        const int ii = p ? g.kh - 1 - row : row, jj = p ? g.kw - 1 - col : col;
        val = A.kern[(ii * g.kw + jj) * g.C + c];
      }
      v[r] = make_double2(val, 0.0);
    }
  }
  fft512_reg<false>(v, sm + rr * kPadB, j, A.tw);
  double2* S = A.S + (((int64_t)c * g.spairs + g.spair0 + p) * T + row) * T;
#pragma unroll
  for (int r = 0; r < 8; ++r) S[j + 64 * r] = v[r];
}

// ---------------------------------------------------------------------------
// K2: column pass.  grid npairs * (T / CCOLS) * C, 64 * CCOLS threads.
// mode 0: forward, multiply by the spectrum, inverse (a stencil);
// mode 1: forward only, store conj (spectrum setup: S -> spec).
struct ColArgs {
  Geo g;
  double2* S;
  const double2* spec;   // (C, T, T): conj(FFT2(kernel pad)), this direction
  double2* spec_out;     // mode 1: (2, C, T, T)
  const double2* tw;
  int mode;
  int npairs;            // pairs held in S for this pass
};

#ifndef FFT_COL_MINB
#define FFT_COL_MINB 3
#endif
__global__ void __launch_bounds__(64 * CCOLS, FFT_COL_MINB) col_kernel(const __grid_constant__ ColArgs A) {
  __shared__ __align__(16) double2 sm[CCOLS * kPadB];
  int p, strip, c;
  block_coords(T / CCOLS, A.g.C, p, strip, c);
  const int bi = threadIdx.x % CCOLS, j = threadIdx.x / CCOLS;
  const int col = strip * CCOLS + bi;
  double2* S = A.S + ((int64_t)c * A.npairs + A.g.spair0 + p) * T * T + col;
  double2 v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = S[(int64_t)(j + 64 * r) * T];
  if (A.mode == 2) {   // inverse column FFTs only (kgc accumulator)
    fft512_reg<true>(v, sm + bi * kPadB, j, A.tw);
#pragma unroll
    for (int r = 0; r < 8; ++r) S[(int64_t)(j + 64 * r) * T] = v[r];
    return;
  }
  fft512_reg<false>(v, sm + bi * kPadB, j, A.tw);
  if (A.mode == 1) {
    double2* o = A.spec_out + ((int64_t)p * A.g.C + c) * T * T + col;
#pragma unroll
    for (int r = 0; r < 8; ++r) o[(int64_t)(j + 64 * r) * T] = make_double2(v[r].x, -v[r].y);
    return;
  }
  const double2* K = A.spec + (int64_t)c * T * T + col;
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = cmul(v[r], __ldg(K + (int64_t)(j + 64 * r) * T));
  fft512_reg<true>(v, sm + bi * kPadB, j, A.tw);
#pragma unroll
  for (int r = 0; r < 8; ++r) S[(int64_t)(j + 64 * r) * T] = v[r];
}

// kernel_gram_correlation by tile FFTs (operators.py:198-220, hypergradient.py:92-104):
//   kgc(x, v)[i, j] = sum_tiles sum_{a,b} u_t[a + i, b + j] vt_t[a, b]
// with u_t the tile's input window of x (the stencil row pass, mode 0) and vt_t the tile's own
// pixels of v (mode 2): per pair Z_u conj(Z_v), whose inverse transform's real part is the sum
// of the pair's two correlations (the cross terms are purely imaginary), summed over pairs in
// the frequency domain; one inverse transform per channel gives the K^2 lags.
__global__ void __launch_bounds__(64 * CCOLS, 2) col_corr_kernel(const __grid_constant__ ColArgs A,
                                                                 const double2* __restrict__ Sv) {
  __shared__ __align__(16) double2 sm[CCOLS * kPadB];
  int p, strip, c;
  block_coords(T / CCOLS, A.g.C, p, strip, c);
  const int bi = threadIdx.x % CCOLS, j = threadIdx.x / CCOLS;
  const int col = strip * CCOLS + bi;
  const int64_t off = ((int64_t)c * A.npairs + p) * T * T + col;
  double2* S = A.S + off;
  double2 u[8], v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) u[r] = S[(int64_t)(j + 64 * r) * T];
  fft512_reg<false>(u, sm + bi * kPadB, j, A.tw);
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = Sv[off + (int64_t)(j + 64 * r) * T];
  fft512_reg<false>(v, sm + bi * kPadB, j, A.tw);
#pragma unroll
  for (int r = 0; r < 8; ++r) S[(int64_t)(j + 64 * r) * T] = cmul(u[r], make_double2(v[r].x, -v[r].y));
}

// acc[c][i] (+)= sum over pairs p (in order) of S[c][p][i]
__global__ void __launch_bounds__(256) pair_sum_kernel(const double2* __restrict__ S, int npairs, int C, int accumulate,
                                                       double2* acc) {
  const int64_t n = (int64_t)C * T * T;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / ((int64_t)T * T), i = e - c * T * T;
    double2 s = accumulate ? acc[e] : make_double2(0.0, 0.0);
    const double2* src = S + c * npairs * T * T + i;
    for (int p = 0; p < npairs; ++p) s = cadd(s, src[(int64_t)p * T * T]);
    acc[e] = s;
  }
}

// rows i < kh of the column-inverted accumulator: inverse row FFT, out[i, j, c] = scale Re(.) for j < kw
__global__ void __launch_bounds__(256) kgc_final_kernel(Geo g, const double2* __restrict__ acc,
                                                        const double2* __restrict__ tw, double scale, double* out) {
  __shared__ __align__(16) double2 sm[RROWS * kPadB];
  const int groups = (g.kh + RROWS - 1) / RROWS;
  const int c = blockIdx.x / groups, i0 = (blockIdx.x - c * groups) * RROWS;
  const int j = threadIdx.x & 63, rr = threadIdx.x >> 6, i = i0 + rr;
  const double2* row = acc + ((int64_t)c * T + min(i, T - 1)) * T;
  double2 v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = row[j + 64 * r];
  fft512_reg<true>(v, sm + rr * kPadB, j, tw);
  if (i < g.kh) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int jj = j + 64 * r;
      if (jj < g.kw) out[((int64_t)i * g.kw + jj) * g.C + c] = scale * v[r].x;
    }
  }
}

// ---------------------------------------------------------------------------
// K3: inverse row pass + crop + epilogue.  grid npairs * (T / RROWS) * C, 256 threads.
enum Epi {
  E_STORE = 0, E_RESID = 1, E_GRAD = 2, E_VALUE = 3, E_POWER = 4,
  E_HESS = 5,     // out = hv = 2 adj + alpha tvhess(v); partial <v, hv>     (lower_solvers.py:66-71)
  E_HESSRES = 6,  // d = hv - rhs: out = -d (r = rhs - H q) when out != NULL; partial ||d||^2 (hypergradient.py:56,83)
  E_TWICE = 7     // out = 2 v (when out != NULL); partial ||2 v||^2 (upper_fit_grad, hypergradient.py:87-89)
};

struct InvArgs {
  Geo g;
  const double2* S;
  const double2* tw;
  double* out;          // E_STORE / E_RESID / E_GRAD / E_POWER
  const double* y;      // data (E_RESID, E_VALUE)
  const double* xp;     // point of the TV term (E_GRAD, E_VALUE)
  double alpha, nu;
  int epi;
  double* part;         // 2 partial sums per CTA: part[2 * cta + {0, 1}]
  const double* w0;     // E_HESS*: TV curvature weights rho''(D x~), vertical / horizontal
  const double* w1;
};

struct TvTerms {
  double root0, root1, grad;
};

// Smoothed anisotropic TV at pixel (h, w, c) of xp (regularizers.py:46-67, 158-175).
__device__ __forceinline__ TvTerms tv_at(const Geo& g, const double* __restrict__ X, int h, int w, int c, double nu,
                                         bool want_grad) {
  const int64_t o = ((int64_t)h * g.W + w) * g.C + c;
  const int64_t rs = (int64_t)g.W * g.C;
  const double nu2 = nu * nu;
  const double x0 = X[o];
  const double d0 = (h + 1 < g.H) ? X[o + rs] - x0 : 0.0;
  const double d1 = (w + 1 < g.W) ? X[o + g.C] - x0 : 0.0;
  // one reciprocal square root per difference: root = s * rsqrt(s), rho' = d * rsqrt(s)
  // (a few ulp from sqrt / division; this path is a tolerance mode)
  TvTerms t;
  const double s0 = d0 * d0 + nu2, s1 = d1 * d1 + nu2;
  const double i0 = rsqrt(s0), i1 = rsqrt(s1);
  t.root0 = s0 * i0;
  t.root1 = s1 * i1;
  t.grad = 0.0;
  if (want_grad) {
    double acc = 0.0;
    if (h > 0) {
      const double du = x0 - X[o - rs];
      acc = acc + du * rsqrt(du * du + nu2);
    }
    acc = acc - d0 * i0;
    if (w > 0) {
      const double dl = x0 - X[o - g.C];
      acc = acc + dl * rsqrt(dl * dl + nu2);
    }
    acc = acc - d1 * i1;
    t.grad = acc;
  }
  return t;
}


__global__ void __launch_bounds__(256, FFT_ROW_MINB) row_inv_kernel(const __grid_constant__ InvArgs A) {
  __shared__ __align__(16) double2 sm[RROWS * kPadB];
  __shared__ double red[40];
  const Geo& g = A.g;
  int p, rg, c;
  block_coords(T / RROWS, g.C, p, rg, c);
  const int j = threadIdx.x & 63, rr = threadIdx.x >> 6, row = rg * RROWS + rr;
  const double2* S = A.S + (((int64_t)c * g.spairs + g.spair0 + p) * T + row) * T;
  double2 v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = S[j + 64 * r];
  fft512_reg<true>(v, sm + rr * kPadB, j, A.tw);
  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    const int t = 2 * (p + g.pair0) + half;
    if (t >= g.ntiles || row >= g.Vh) break;
    int h0, w0;
    tile_origin(g, t, h0, w0);
    const int h = h0 + row;
    if (h >= g.H) continue;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int q = j + 64 * r, w = w0 + q;
      if (q >= g.Vw || w >= g.W) continue;
      const double val = (half ? v[r].y : v[r].x) * kInvT2;
      const int64_t o = ((int64_t)h * g.W + w) * g.C + c;
      switch (A.epi) {
        case E_STORE: A.out[o] = val; break;
        case E_POWER: A.out[o] = val; acc0 = acc0 + val * val; break;
        case E_TWICE: {
          const double gv = 2.0 * val;
          if (A.out) A.out[o] = gv;
          acc0 = acc0 + gv * gv;
          break;
        }
        case E_RESID: {
          const double rs = val - A.y[o];
          A.out[o] = rs;
          acc0 = acc0 + rs * rs;
          break;
        }
        case E_GRAD: {   // g = 2 adj + alpha grad J (lower_solvers.py:54-62); vg TV form (regularizers.py:173-174)
          const TvTerms tv = tv_at(g, A.xp, h, w, c, A.nu, true);
          const double gv = 2.0 * val + A.alpha * tv.grad;
          A.out[o] = gv;
          acc0 = acc0 + gv * gv;
          acc1 = acc1 + (tv.root0 + tv.root1);
          break;
        }
        case E_HESS:
        case E_HESSRES: {   // TV hess_vec = D^T (w * D v), v = A.xp (regularizers.py:177-183)
          const int64_t rs = (int64_t)g.W * g.C;
          const double v0 = A.xp[o];
          const double dv0 = (h + 1 < g.H) ? A.xp[o + rs] - v0 : 0.0;
          const double dv1 = (w + 1 < g.W) ? A.xp[o + g.C] - v0 : 0.0;
          double tvh = 0.0;
          if (h > 0) tvh = tvh + A.w0[o - rs] * (v0 - A.xp[o - rs]);
          tvh = tvh - A.w0[o] * dv0;
          if (w > 0) tvh = tvh + A.w1[o - g.C] * (v0 - A.xp[o - g.C]);
          tvh = tvh - A.w1[o] * dv1;
          const double hv = 2.0 * val + A.alpha * tvh;
          if (A.epi == E_HESS) {
            A.out[o] = hv;
            acc0 = acc0 + v0 * hv;
          } else {
            const double d = hv - A.y[o];
            if (A.out) A.out[o] = -d;
            acc0 = acc0 + d * d;
          }
          break;
        }
        case E_VALUE: {  // sum (Bx - y)^2 and tv_value = sum(sqrt(d^2 + nu^2) - nu) (regularizers.py:70-72)
          if (A.out) A.out[o] = val;   // keep B x (the solver's linear extrapolation of B y)
          const double rs = val - A.y[o];
          acc0 = acc0 + rs * rs;
          const TvTerms tv = tv_at(g, A.xp, h, w, c, A.nu, false);
          acc1 = acc1 + ((tv.root0 - A.nu) + (tv.root1 - A.nu));
          break;
        }
        default: break;
      }
    }
  }
  if (A.part) {
    const double s0 = block_sum(acc0, red);
    const double s1 = block_sum(acc1, red);
    if (threadIdx.x == 0) {
      const int cta = blockIdx.x + g.pair0 * (T / RROWS) * g.C;   // global CTA index
      A.part[2 * cta] = s0;
      A.part[2 * cta + 1] = s1;
    }
  }
}

// ---------------------------------------------------------------------------
// elementwise steps of the solvers + fixed-order partials
enum VecOp {
  V_EXTRAP = 0,   // out = x + beta * (x - xp)                 (lower_solvers.py:197)
  V_STEPDIV = 1,  // out = y - g / L                           (:173, :207)
  V_STEPMUL = 2,  // out = x - step * g                        (:165)
  V_DIVNORM = 3,  // out = x / a                               (operators.py:150, 162)
  V_DOTDIFF = 4,  // partial: sum g * (x - xp)                 (:209)
  V_NORM2 = 5,    // partial: sum x * x
  V_COPY = 6
};
constexpr int kVecGrid = 1184;   // 8 x 148

__global__ void __launch_bounds__(256) vec_kernel(int op, int64_t n, double a, const double* __restrict__ x,
                                                  const double* __restrict__ xp, const double* __restrict__ gg,
                                                  double* __restrict__ out, double* part) {
  __shared__ double red[40];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    switch (op) {
      case V_EXTRAP: out[i] = x[i] + a * (x[i] - xp[i]); break;
      case V_STEPDIV: out[i] = x[i] - gg[i] / a; break;
      case V_STEPMUL: out[i] = x[i] - a * gg[i]; break;
      case V_DIVNORM: out[i] = x[i] / a; break;
      case V_DOTDIFF: acc = acc + gg[i] * (x[i] - xp[i]); break;
      case V_NORM2: acc = acc + x[i] * x[i]; break;
      case V_COPY: out[i] = x[i]; break;
      default: break;
    }
  }
  if (part) {
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) part[2 * blockIdx.x] = s;
  }
}

// Residual by linearity (the adaptive accelerated FFT solve): y = x + beta (x - xp) and
// B y = Bx + beta (Bx - Bxp) from the kept B x / B x_prev, r = B y - data; partial sum r^2.
// (B y is a linear combination of two fresh transforms: no error accumulates over iterations.)
__global__ void __launch_bounds__(256) resid_lin_kernel(int64_t n, double beta, const double* __restrict__ x,
                                                        const double* __restrict__ xp, const double* __restrict__ bx,
                                                        const double* __restrict__ bxp,
                                                        const double* __restrict__ data, double* y, double* r,
                                                        double* part) {
  __shared__ double red[40];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double xv = x[i], bv = bx[i];
    y[i] = xv + beta * (xv - xp[i]);
    const double rv = (bv + beta * (bv - bxp[i])) - data[i];
    r[i] = rv;
    acc = acc + rv * rv;
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[2 * blockIdx.x] = s;
}

// Fixed-order folds of up to three partial buffers in one launch: source i
// holds k_i interleaved streams (p[k_i * n + j], n < n_i); results in order.
// One CTA, per-thread strided (coalesced) chains in a fixed order, then block_sum.
struct FoldSrc {
  const double* p;
  int n, k;
};

__global__ void __launch_bounds__(1024) fold_kernel(FoldSrc a, FoldSrc b, FoldSrc c, double* out) {
  __shared__ double red[40];
  int o = 0;
  for (int si = 0; si < 3; ++si) {
    const FoldSrc f = si == 0 ? a : (si == 1 ? b : c);
    for (int j = 0; j < f.k; ++j) {
      double acc = 0.0;
#pragma unroll 8
      for (int i = threadIdx.x; i < f.n; i += blockDim.x) acc = acc + f.p[(int64_t)f.k * i + j];
      const double s = block_sum(acc, red);
      if (threadIdx.x == 0) out[o] = s;
      ++o;
    }
  }
}

// ---------------------------------------------------------------------------
// CG support (hypergradient.py:35-84 on lower_hess_vec / lower_hess_diag)
// rho''(D x~) per pixel: w0 vertical, w1 horizontal (regularizers.py:34-36, 177-199)
__global__ void __launch_bounds__(256) curv_kernel(Geo g, const double* __restrict__ x, double nu, double* w0,
                                                   double* w1) {
  const int64_t N = (int64_t)g.H * g.W * g.C, rs = (int64_t)g.W * g.C;
  const double nu2 = nu * nu;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < N; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t hw = o / g.C;
    const int h = (int)(hw / g.W), w = (int)(hw - (int64_t)h * g.W);
    const double x0 = x[o];
    const double d0 = (h + 1 < g.H) ? x[o + rs] - x0 : 0.0;
    const double d1 = (w + 1 < g.W) ? x[o + g.C] - x0 : 0.0;
    w0[o] = nu2 / pow(d0 * d0 + nu2, 1.5);
    w1[o] = nu2 / pow(d1 * d1 + nu2, 1.5);
  }
}

// Summed-area table of the flipped kernel squared, per channel: sat[(i * (kw + 1) + j) * C + c] =
// sum_{i' < i, j' < j} kf[i', j', c]^2, kf = kernel[::-1, ::-1] (operators.py:98, 120-122)
__global__ void sat_kernel(Geo g, const double* __restrict__ kern, double* sat) {
  const int W1 = g.kw + 1;
  for (int c = threadIdx.x; c < g.C; c += blockDim.x) {
  for (int j = 0; j < W1; ++j) sat[j * g.C + c] = 0.0;
  for (int i = 1; i <= g.kh; ++i) {
    double row = 0.0;
    sat[(i * W1) * g.C + c] = 0.0;
    for (int j = 1; j <= g.kw; ++j) {
      const double k = kern[((g.kh - i) * g.kw + (g.kw - j)) * g.C + c];   // kf[i-1, j-1]
      row = row + k * k;
      sat[(i * W1 + j) * g.C + c] = sat[((i - 1) * W1 + j) * g.C + c] + row;
    }
  }
  }
}

// d = 2 gram_diag + alpha hess_diag_TV (lower_solvers.py:74-79); partial max per CTA.
// gram_diag = correlate(ones, kf^2): the in-image taps form an i- and a j-interval -> 4 SAT lookups.
__global__ void __launch_bounds__(256) diag_kernel(Geo g, const double* __restrict__ sat, const double* __restrict__ w0,
                                                   const double* __restrict__ w1, double alpha, double* d,
                                                   double* part) {
  __shared__ double red[40];
  const int64_t N = (int64_t)g.H * g.W * g.C, rs = (int64_t)g.W * g.C;
  const int W1 = g.kw + 1;
  double mx = -INFINITY;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < N; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t hw = o / g.C;
    const int c = (int)(o - hw * g.C);
    const int h = (int)(hw / g.W), w = (int)(hw - (int64_t)h * g.W);
    const int i0 = max(0, g.rh - h), i1 = min(g.kh, g.H - h + g.rh);   // 0 <= h + i - rh < H
    const int j0 = max(0, g.rw - w), j1 = min(g.kw, g.W - w + g.rw);
    const double gram = sat[(i1 * W1 + j1) * g.C + c] - sat[(i0 * W1 + j1) * g.C + c] -
                        sat[(i1 * W1 + j0) * g.C + c] + sat[(i0 * W1 + j0) * g.C + c];
    double tv = 0.0;
    if (h + 1 < g.H) tv = tv + w0[o];
    if (h > 0) tv = tv + w0[o - rs];
    if (w + 1 < g.W) tv = tv + w1[o];
    if (w > 0) tv = tv + w1[o - g.C];
    const double v = 2.0 * gram + alpha * tv;
    d[o] = v;
    mx = fmax(mx, v);
  }
  const double m = block_max(mx, red);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

// minv = 1 / max(d, floor) in place (lower_solvers.py:80; hypergradient.py:52-54)
__global__ void __launch_bounds__(256) minv_kernel(int64_t n, double floor_, double* d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = 1.0 / fmax(d[i], floor_);
}

// CG step (hypergradient.py:75-78): q += a p; r -= a hp; partials <r, minv r> and <r, r>.
// With first != 0 (the start): r given, partials only.
__global__ void __launch_bounds__(256) cg_update_kernel(int64_t n, double a, double* q, double* r,
                                                        const double* __restrict__ p, const double* __restrict__ hp,
                                                        const double* __restrict__ minv, int first, double* part) {
  __shared__ double red[40];
  double rz = 0.0, rr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double ri = r[i];
    if (!first) {
      q[i] = q[i] + a * p[i];
      ri = ri - a * hp[i];
      r[i] = ri;
    }
    rz = rz + ri * (minv[i] * ri);
    rr = rr + ri * ri;
  }
  const double s0 = block_sum(rz, red);
  const double s1 = block_sum(rr, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
}

}  // namespace fft
}  // namespace adp

// ===========================================================================
// host side
using namespace adp;
using namespace adp::fft;

struct adp_fft_plan {
  Geo g;
  int chunk = 0;               // tile pairs per chunk of the stencil passes (0: whole image)
  int64_t N = 0;
  double2* S = nullptr;        // (C, npairs, T, T)
  double2* spec = nullptr;     // (2, C, T, T): [0] apply, [1] adjoint
  double2* tw = nullptr;       // T twiddles exp(-2 pi i m / T)
  double* partR = nullptr;     // residual-pass partials (2 per row CTA)
  double* partG = nullptr;     // gradient / value / power-pass partials (2 per row CTA)
  double* partK1 = nullptr;    // row-pass prologue partials (1 per row CTA)
  double* partV = nullptr;     // vector-kernel partials (2 per CTA)
  double* red = nullptr;       // fold results (device)
  double* hred = nullptr;      // pinned host copy
  double* buf[6] = {};         // solver images
  double* cgbuf[7] = {};       // CG images (allocated at first use): r, p0, p1, hp, minv, w0, w1
  double* lin[3] = {};         // adaptive accelerated solve: B x, B x_prev, B x_candidate (first use)
  double* sat = nullptr;       // summed-area table of the flipped kernel squared
  double2* S2 = nullptr;       // kgc: second complex scratch (first use)
  double2* acc = nullptr;      // kgc: (C, T, T) frequency-domain accumulator
  int nrow_ctas = 0;
  const void* spec_kernel = nullptr;   // kernel pointer the spectra were built from (this call)
  size_t bytes = 0;
};

namespace {

int setup_attrs() { return ADP_OK; }   // static shared memory only

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dense_fail(ADP_ERR_CUDA, (std::string(what) + ": " + cudaGetErrorString(e)).c_str());
  return ADP_OK;
}

// Spectra of the kernel and of the flipped kernel (conj(FFT2(pad))), into P->spec.
int build_spectra(adp_fft_plan* P, const double* kern, cudaStream_t st) {
  const Geo& g = P->g;
  Geo kg = g;
  kg.npairs = 2;   // S slots: pair 0 = kernel, pair 1 = flipped kernel
  kg.spairs = 2;
  RowArgs ra{kg, nullptr, P->S, P->tw, 1, kern, P_NONE, nullptr, nullptr, 0.0, nullptr, nullptr};
  row_fwd_kernel<<<2 * (T / RROWS) * g.C, 256, 0, st>>>(ra);
  ColArgs ca{kg, P->S, nullptr, P->spec, P->tw, 1, 2};
  col_kernel<<<2 * (T / CCOLS) * g.C, 64 * CCOLS, 0, st>>>(ca);
  return check_launch("fft spectra");
}

// Row-pass prologue of one stencil (see enum Pro).
struct ProArgs {
  int pro = P_NONE;
  const double* x2 = nullptr;
  const double* xold = nullptr;
  double coef = 0.0;
  double* wout = nullptr;
};

// One stencil: out/epilogue from (the prologue of) x with the apply (adj = 0) or adjoint (adj = 1)
// spectrum; K3 partials to part3 (2 per CTA) when non-NULL, K1 partials (P_STEP) to P->partK1.
// Optional (ADP_FFT_PB > 0, off by default: measured slower, see the plan set-up): the passes run over
// chunks of P->chunk tile pairs (row pass, column pass, inverse rows per chunk) through ONE chunk-sized
// scratch region, so the complex scratch of a chunk (12 MB per pair at C = 3) is written, transformed
// and consumed while it is L2-resident instead of making three round trips to HBM.  Partial sums are indexed by the global CTA, so the results are those of the unchunked
// passes bit for bit.  A stencil whose inverse-row epilogue reads neighbours of the iterate its own
// row-pass prologue stores (the candidate's value pass) runs the row pass over the whole image first
// (the later chunks' tiles must exist), then the other two passes per chunk.
int stencil(adp_fft_plan* P, int adj, const double* x, const ProArgs& pa, int epi, double* out, const double* y,
            const double* xp, double alpha, double nu, double* part3, cudaStream_t st) {
  Geo g = P->g;
  const int PB = P->chunk > 0 ? std::min(P->chunk, g.npairs) : g.npairs;
  const bool reads_nb = epi == E_VALUE || epi == E_GRAD || epi == E_HESS || epi == E_HESSRES;
  const bool hazard = pa.wout != nullptr && reads_nb && xp == pa.wout && PB < g.npairs;
  const double2* spec = P->spec + (size_t)adj * g.C * T * T;
  if (hazard) {
    g.pair0 = g.spair0 = 0;
    g.spairs = g.npairs;
    RowArgs ra{g, x, P->S, P->tw, 0, nullptr, pa.pro, pa.x2, pa.xold, pa.coef, pa.wout, P->partK1};
    row_fwd_kernel<<<g.npairs * (T / RROWS) * g.C, 256, 0, st>>>(ra);
  }
  for (int p0 = 0; p0 < g.npairs; p0 += PB) {
    const int np = std::min(PB, g.npairs - p0);
    g.pair0 = p0;
    g.spair0 = hazard ? p0 : 0;
    g.spairs = hazard ? g.npairs : PB;
    const int rgrid = np * (T / RROWS) * g.C;
    if (!hazard) {
      RowArgs ra{g, x, P->S, P->tw, 0, nullptr, pa.pro, pa.x2, pa.xold, pa.coef, pa.wout, P->partK1};
      row_fwd_kernel<<<rgrid, 256, 0, st>>>(ra);
    }
    ColArgs ca{g, P->S, spec, nullptr, P->tw, 0, g.spairs};
    col_kernel<<<np * (T / CCOLS) * g.C, 64 * CCOLS, 0, st>>>(ca);
    InvArgs ia{g, P->S, P->tw, out, y, xp, alpha, nu, epi, part3, P->cgbuf[5], P->cgbuf[6]};
    row_inv_kernel<<<rgrid, 256, 0, st>>>(ia);
  }
  return check_launch("fft stencil");
}

int rowctas(const adp_fft_plan* P) { return P->g.npairs * (T / RROWS) * P->g.C; }

// Fold up to three partial sources (one launch, one device->host read, one sync).
int fold(adp_fft_plan* P, FoldSrc a, FoldSrc b, FoldSrc c, double* host, cudaStream_t st) {
  const int k = a.k + b.k + c.k;
  fold_kernel<<<1, 1024, 0, st>>>(a, b, c, P->red);
  cudaMemcpyAsync(P->hred, P->red, k * sizeof(double), cudaMemcpyDeviceToHost, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return dense_fail(ADP_ERR_CUDA, cudaGetErrorString(e));
  for (int j = 0; j < k; ++j) host[j] = P->hred[j];
  return ADP_OK;
}
FoldSrc src3(const adp_fft_plan* P, const double* part) { return FoldSrc{part, rowctas(P), 2}; }
constexpr FoldSrc kNoSrc{nullptr, 0, 0};

int vec(adp_fft_plan* P, int op, double a, const double* x, const double* xp, const double* g, double* out,
        double* host_red, cudaStream_t st) {
  const bool red = (op == V_DOTDIFF || op == V_NORM2);
  vec_kernel<<<kVecGrid, 256, 0, st>>>(op, P->N, a, x, xp, g, out, red ? P->partV : nullptr);
  int rc = check_launch("fft vec");
  if (rc != ADP_OK || !red) return rc;
  double r[2];
  rc = fold(P, FoldSrc{P->partV, kVecGrid, 2}, kNoSrc, kNoSrc, r, st);
  *host_red = r[0];
  return rc;
}

// value and gradient of the lower objective (lower_solvers.py:50-63) at the stencil input
// produced by `pa` from x (the point itself, or y = x + beta (x - x_prev) stored to pa.wout):
// r = Bz - y (buf R), g = 2 B^T r + alpha grad TV(z); value = sum r^2 + alpha (sum root - nu * 2N)
int vg(adp_fft_plan* P, const adp_lower* lp, const double* x, const ProArgs& pa, double* g, double* value,
       double* gn2, cudaStream_t st) {
  double* R = P->buf[5];
  const double* z = pa.pro == P_NONE ? x : pa.wout;
  int rc = stencil(P, 0, x, pa, E_RESID, R, (const double*)lp->y, nullptr, 0.0, 0.0, P->partR, st);
  if (rc) return rc;
  rc = stencil(P, 1, R, ProArgs{}, E_GRAD, g, nullptr, z, lp->alpha, lp->nu, P->partG, st);
  if (rc) return rc;
  double t[4];
  if ((rc = fold(P, src3(P, P->partR), src3(P, P->partG), kNoSrc, t, st))) return rc;
  const double tv = t[3] - lp->nu * (double)(2 * P->N);
  if (value) *value = t[0] + lp->alpha * tv;
  if (gn2) *gn2 = t[2];
  return ADP_OK;
}

// value and gradient at y = x + beta (x - xp) with B y from the kept B x, B xp (resid_lin_kernel):
// one elementwise pass + the adjoint stencil instead of two stencils
int vg_lin(adp_fft_plan* P, const adp_lower* lp, double beta, const double* x, const double* xp, const double* bx,
           const double* bxp, double* y, double* g, double* value, double* gn2, cudaStream_t st) {
  double* R = P->buf[5];
  resid_lin_kernel<<<kVecGrid, 256, 0, st>>>(P->N, beta, x, xp, bx, bxp, (const double*)lp->y, y, R, P->partV);
  int rc = check_launch("fft resid_lin");
  if (rc) return rc;
  rc = stencil(P, 1, R, ProArgs{}, E_GRAD, g, nullptr, y, lp->alpha, lp->nu, P->partG, st);
  if (rc) return rc;
  double t[4];
  if ((rc = fold(P, FoldSrc{P->partV, kVecGrid, 2}, src3(P, P->partG), kNoSrc, t, st))) return rc;
  const double tv = t[3] - lp->nu * (double)(2 * P->N);
  if (value) *value = t[0] + lp->alpha * tv;
  if (gn2) *gn2 = t[2];
  return ADP_OK;
}

// lower_value (lower_solvers.py:37-39) at the stencil input produced by `pa`:
// sum (Bz - y)^2 + alpha tv_value(z); with P_STEP also the restart dot sum g (xc - xold)
int value(adp_fft_plan* P, const adp_lower* lp, const double* x, const ProArgs& pa, double* val, double* dot,
          cudaStream_t st, double* bx_out = nullptr) {
  const double* z = pa.pro == P_NONE ? x : pa.wout;
  int rc = stencil(P, 0, x, pa, E_VALUE, bx_out, (const double*)lp->y, z, 0.0, lp->nu, P->partG, st);
  if (rc) return rc;
  double t[3];
  const bool step = pa.pro == P_STEP;
  if ((rc = fold(P, src3(P, P->partG), step ? FoldSrc{P->partK1, rowctas(P), 1} : kNoSrc, kNoSrc, t, st)))
    return rc;
  *val = t[0] + lp->alpha * t[1];
  if (dot) *dot = step ? t[2] : 0.0;
  return ADP_OK;
}

// op_norm_sq (operators.py:137-173); v = w / lam is the next row pass's prologue
int power(adp_fft_plan* P, const double* v0, int max_iters, double tol, double* lam_out, int* conv_out,
          int* iters_out, cudaStream_t st) {
  double* Wb = P->buf[4];
  double* Bv = P->buf[5];
  double n2 = 0.0;
  int rc = vec(P, V_NORM2, 0.0, v0, nullptr, nullptr, nullptr, &n2, st);
  if (rc) return rc;
  const double* vin = v0;      // v = vin / scale
  double scale = std::sqrt(n2);
  double lam = 0.0;
  int converged = 0, it = 0;
  for (; it < max_iters; ++it) {
    ProArgs pa;
    pa.pro = P_SCALE;
    pa.coef = 1.0 / scale;
    if ((rc = stencil(P, 0, vin, pa, E_STORE, Bv, nullptr, nullptr, 0.0, 0.0, nullptr, st))) return rc;
    if ((rc = stencil(P, 1, Bv, ProArgs{}, E_POWER, Wb, nullptr, nullptr, 0.0, 0.0, P->partG, st))) return rc;
    double w2[2];
    if ((rc = fold(P, src3(P, P->partG), kNoSrc, kNoSrc, w2, st))) return rc;
    const double lam_new = std::sqrt(w2[0]);
    if (lam_new == 0.0) {
      lam = 0.0;
      converged = 1;
      ++it;
      break;
    }
    vin = Wb;
    scale = lam_new;
    if (std::fabs(lam_new - lam) <= tol * std::max(lam_new, 1e-300)) {
      lam = lam_new;
      converged = 1;
      ++it;
      break;
    }
    lam = lam_new;
  }
  *lam_out = lam;
  if (conv_out) *conv_out = converged;
  if (iters_out) *iters_out = it;
  return ADP_OK;
}

int prepare(adp_fft_plan* P, const void* kernel, cudaStream_t st) {
  int rc = setup_attrs();
  if (rc) return rc;
  return build_spectra(P, (const double*)kernel, st);
}

}  // namespace

extern "C" int adp_fft_plan_create(adp_fft_plan** out, int32_t H, int32_t W, int32_t C, int32_t kh, int32_t kw) {
  if (!out || H < 1 || W < 1 || C < 1 || kh < 1 || kw < 1 || kh % 2 == 0 || kw % 2 == 0)
    return dense_fail(ADP_ERR_ARG, "fft plan: bad shape");
  if (kh > T / 2 || kw > T / 2) return dense_fail(ADP_ERR_UNSUPPORTED, "fft plan: kernel larger than 256 taps");
  adp_fft_plan* P = new adp_fft_plan();
  Geo& g = P->g;
  g.H = H; g.W = W; g.C = C; g.kh = kh; g.kw = kw; g.rh = kh / 2; g.rw = kw / 2;
  g.Vh = T - kh + 1; g.Vw = T - kw + 1;
  g.ntY = (H + g.Vh - 1) / g.Vh; g.ntX = (W + g.Vw - 1) / g.Vw;
  g.ntiles = g.ntY * g.ntX;
  g.npairs = (g.ntiles + 1) / 2;
  g.pair0 = g.spair0 = 0;
  g.spairs = g.npairs;
  {
    // tile pairs per chunk of the stencil passes (see stencil()); default 0: whole-image passes -- the
    // chunked, L2-resident order measured slower on B200 (c5 stencil 1.05 ms whole-image, 1.15 / 1.26 /
    // 1.56 ms at 12 / 6 / 2 pairs per chunk: the passes are issue-latency bound, not HBM bound, and the
    // extra kernel boundaries cost more than the scratch traffic saves; profiles/r02zf_fft_chunks.txt)
    const char* ev = getenv("ADP_FFT_PB");
    P->chunk = ev ? atoi(ev) : 0;
  }
  P->N = (int64_t)H * W * C;
  // >= 2 pair slots: the spectrum setup transforms the kernel and its flip together
  const size_t sbytes = (size_t)C * std::max(2, g.npairs) * T * T * sizeof(double2);
  const size_t specb = (size_t)2 * C * T * T * sizeof(double2);
  const int nparts = rowctas(P);
  bool ok = cudaMalloc(&P->S, sbytes) == cudaSuccess && cudaMalloc(&P->spec, specb) == cudaSuccess &&
            cudaMalloc(&P->tw, T * sizeof(double2)) == cudaSuccess &&
            cudaMalloc(&P->partR, (size_t)2 * nparts * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&P->partG, (size_t)2 * nparts * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&P->partK1, (size_t)nparts * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&P->partV, (size_t)2 * kVecGrid * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&P->red, 8 * sizeof(double)) == cudaSuccess &&
            cudaMallocHost(&P->hred, 8 * sizeof(double)) == cudaSuccess;
  for (int i = 0; ok && i < 6; ++i) ok = cudaMalloc(&P->buf[i], (size_t)P->N * sizeof(double)) == cudaSuccess;
  if (!ok) {
    adp_fft_plan_destroy(P);
    return dense_fail(ADP_ERR_CUDA, "fft plan: device allocation failed");
  }
  P->bytes = sbytes + specb + (size_t)6 * P->N * sizeof(double) + (size_t)(5 * nparts + 2 * kVecGrid) * sizeof(double);
  // accurately rounded twiddles exp(-2 pi i m / T)
  std::vector<double2> tw(T);
  for (int m = 0; m < T; ++m) {
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)T;
    tw[m] = make_double2((double)cosl(a), (double)sinl(a));
  }
  cudaMemcpy(P->tw, tw.data(), T * sizeof(double2), cudaMemcpyHostToDevice);
  *out = P;
  return ADP_OK;
}

extern "C" void adp_fft_plan_destroy(adp_fft_plan* P) {
  if (!P) return;
  cudaFree(P->S);
  cudaFree(P->spec);
  cudaFree(P->tw);
  cudaFree(P->partR);
  cudaFree(P->partG);
  cudaFree(P->partK1);
  cudaFree(P->partV);
  cudaFree(P->red);
  if (P->hred) cudaFreeHost(P->hred);
  for (double* b : P->buf) cudaFree(b);
  for (double* b : P->cgbuf) cudaFree(b);
  for (double* b : P->lin) cudaFree(b);
  cudaFree(P->sat);
  cudaFree(P->S2);
  cudaFree(P->acc);
  delete P;
}

extern "C" size_t adp_fft_plan_workspace_bytes(const adp_fft_plan* P) { return P ? P->bytes : 0; }

extern "C" int adp_fft_apply(adp_fft_plan* P, const void* kernel, int32_t adjoint, const void* x, void* out,
                             void* stream) {
  if (!P || !kernel || !x || !out) return dense_fail(ADP_ERR_ARG, "fft apply: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = prepare(P, kernel, st);
  if (rc) return rc;
  return stencil(P, adjoint ? 1 : 0, (const double*)x, ProArgs{}, E_STORE, (double*)out, nullptr, nullptr, 0.0, 0.0,
                 nullptr, st);
}

extern "C" int adp_fft_lower_value(adp_fft_plan* P, const adp_lower* lp, const void* x, double* val, void* stream) {
  if (!P || !lp || !x || !val) return dense_fail(ADP_ERR_ARG, "fft lower_value: null argument");
  if (lp->reg != ADP_REG_TV) return dense_fail(ADP_ERR_UNSUPPORTED, "fft path: smoothed TV only");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = prepare(P, lp->kernel, st);
  if (rc) return rc;
  return value(P, lp, (const double*)x, ProArgs{}, val, nullptr, st);
}

extern "C" int adp_fft_lower_value_and_grad(adp_fft_plan* P, const adp_lower* lp, const void* x, double* val,
                                            void* g, void* stream) {
  if (!P || !lp || !x || !g) return dense_fail(ADP_ERR_ARG, "fft lower_value_and_grad: null argument");
  if (lp->reg != ADP_REG_TV) return dense_fail(ADP_ERR_UNSUPPORTED, "fft path: smoothed TV only");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = prepare(P, lp->kernel, st);
  if (rc) return rc;
  double v = 0.0, gn2 = 0.0;
  rc = vg(P, lp, (const double*)x, ProArgs{}, (double*)g, &v, &gn2, st);
  if (val) *val = v;
  return rc;
}

extern "C" int adp_fft_op_norm_sq(adp_fft_plan* P, const void* kernel, const void* v0, int32_t max_iters, double tol,
                                  double* lam, int32_t* converged, int32_t* iters, void* stream) {
  if (!P || !kernel || !v0 || !lam) return dense_fail(ADP_ERR_ARG, "fft op_norm_sq: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = prepare(P, kernel, st);
  if (rc) return rc;
  int c = 0, it = 0;
  rc = power(P, (const double*)v0, max_iters, tol, lam, &c, &it, st);
  if (converged) *converged = c;
  if (iters) *iters = it;
  return rc;
}

// solve_lower (lower_solvers.py:104-213) on the FFT stencils; the scalar
// control flow runs here on the host in the reference's order, one small
// device->host read per reduction (negligible next to three 2-D FFT
// stencils per iteration at the sizes this path is for).
extern "C" int adp_fft_lower_solve(adp_fft_plan* P, const adp_lower* lp, const void* x0, void* x_out,
                                   const adp_solve_args* a, adp_solve_result* res, void* stream) {
  if (!P || !lp || !x0 || !x_out || !a || !res) return dense_fail(ADP_ERR_ARG, "fft solve: null argument");
  if (lp->reg != ADP_REG_TV) return dense_fail(ADP_ERR_UNSUPPORTED, "fft path: smoothed TV only");
  if (!(a->eps > 0) || !(a->mu > 0)) return dense_fail(ADP_ERR_ARG, "eps and mu must be > 0");
  cudaStream_t st = (cudaStream_t)stream;
  *res = adp_solve_result{};
  int rc = prepare(P, lp->kernel, st);
  if (rc) return rc;
  const double tol = a->eps * a->mu;
  const int64_t nbytes = P->N * (int64_t)sizeof(double);
  // --- step size / Lipschitz constant (L_of_b, lower_solvers.py:90-96)
  double lip, step;
  res->norm_sq = a->norm_sq;
  if (a->step_size > 0) {
    step = a->step_size;
    lip = 1.0 / step;
  } else {
    if (a->norm_sq < 0) {
      if (!a->v0) return dense_fail(ADP_ERR_ARG, "fft solve: power-iteration start vector missing");
      int pc = 0, pit = 0;
      if ((rc = power(P, (const double*)a->v0, a->norm_max_iters, a->norm_tol, &res->norm_sq, &pc, &pit, st)))
        return rc;
      res->power_converged = pc;
      res->power_iters = pit;
    }
    lip = 2.0 * res->norm_sq + lp->alpha * (8.0 / lp->nu);
    step = 1.0 / lip;
  }
  res->lip = lip;
  // buffers: X (iterate), XP (previous), Y (extrapolation), XC (candidate), G; buf[5] = residual
  double* X = P->buf[0];
  double* XP = P->buf[1];
  double* Y = P->buf[2];
  double* XC = P->buf[3];
  double* G = P->buf[4];
  cudaMemcpyAsync(X, x0, nbytes, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(XP, a->x_prev0 ? a->x_prev0 : x0, nbytes, cudaMemcpyDeviceToDevice, st);
  // injected state (P2 lockstep): momentum and backtracking estimate at the first iteration
  double t_mom = a->t_mom0 > 0 ? a->t_mom0 : 1.0;
  double lip_t = a->lip_t0 > 0 ? a->lip_t0 : lip;
  if (a->method == ADP_METHOD_PROXGRAD && a->lip_t0 > 0) step = 1.0 / a->lip_t0;
  auto finish = [&](const double* xr, double gn2, int t, int conv) {
    res->t_mom = t_mom;
    res->lip_t = a->method == ADP_METHOD_PROXGRAD ? 1.0 / step : lip_t;
    cudaMemcpyAsync(x_out, xr, nbytes, cudaMemcpyDeviceToDevice, st);
    res->grad_norm = std::sqrt(gn2);
    res->iters = t;
    res->converged = conv;
    const cudaError_t e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? ADP_OK : dense_fail(ADP_ERR_CUDA, cudaGetErrorString(e));
  };
  auto diverged = [&](int t) {
    res->status = ADP_STATUS_DIVERGED;
    res->fail_iter = t;
    return ADP_OK;
  };
  // backtracked step from y (lower_solvers.py:170-177): XC = y - g / L_try
  // backtracked step from y (lower_solvers.py:170-177): XC = y - g / L_try is the value pass's
  // row prologue, which also sums the restart dot g . (XC - X) (X = the current iterate)
  double last_dot = 0.0;
  double* bx_keep = nullptr;   // set: each candidate's B x_c is stored there (the linear B y path)
  auto backtrack = [&](const double* yv, double h_y, double gn, double lip_try, double* step_out, int* ok) -> int {
    for (int k = 0; k < 60; ++k) {
      ProArgs pa;
      pa.pro = P_STEP;
      pa.x2 = G;
      pa.xold = X;
      pa.coef = 1.0 / lip_try;
      pa.wout = XC;
      double hv = 0.0;
      int r = value(P, lp, yv, pa, &hv, &last_dot, st, bx_keep);
      if (r) return r;
      res->value_evals++;
      if (hv <= h_y - 0.5 * gn * gn / lip_try + 1e-15 * std::fabs(h_y)) {
        *step_out = 1.0 / lip_try;
        *ok = 1;
        return ADP_OK;
      }
      lip_try *= 2.0;
    }
    *ok = 0;
    return ADP_OK;
  };
  if (a->method == ADP_METHOD_PROXGRAD) {   // _gradient_descent (:154-167)
    double h_x = 0.0, gn2 = 0.0;
    if ((rc = vg(P, lp, X, ProArgs{}, G, &h_x, &gn2, st))) return rc;
    res->vg_evals++;
    for (int t = 0; t < a->max_iters; ++t) {
      const double gn = std::sqrt(gn2);
      if (!std::isfinite(gn)) return diverged(t);
      if (gn <= tol) return finish(X, gn2, t, 1);
      if (a->adaptive) {
        int ok = 0;
        double s = 0.0;
        if ((rc = backtrack(X, h_x, gn, 1.0 / step, &s, &ok))) return rc;
        if (!ok) { res->status = ADP_STATUS_BT_FAIL; return ADP_OK; }
        step = s;
        std::swap(X, XC);
      } else {
        if ((rc = vec(P, V_STEPMUL, step, X, nullptr, G, XC, nullptr, st))) return rc;
        std::swap(X, XC);
      }
      if ((rc = vg(P, lp, X, ProArgs{}, G, &h_x, &gn2, st))) return rc;
      res->vg_evals++;
    }
    return finish(X, gn2, a->max_iters, std::sqrt(gn2) <= tol);
  }
  // _accelerated (:180-213)
  double theta = 0.0;
  if (a->method == ADP_METHOD_FISTA_SC) {
    const double q = std::min(a->mu / lip, 1.0);
    theta = (1.0 - std::sqrt(q)) / (1.0 + std::sqrt(q));
  }
  bool xp_is_x = a->x_prev0 == nullptr;   // x_prev == x (start, and after a restart)
  // Adaptive: every accepted x is a backtracking candidate whose B x_c the value pass already
  // computed, so B y = B x + beta (B x - B x_prev) needs no forward stencil (vg_lin).
  const bool lin = a->adaptive != 0;
  double *BX = nullptr, *BXP = nullptr, *BXC = nullptr;
  if (lin) {
    for (double*& b : P->lin)
      if (!b && cudaMalloc(&b, (size_t)P->N * sizeof(double)) != cudaSuccess)
        return dense_fail(ADP_ERR_CUDA, "fft solve: device allocation failed");
    BX = P->lin[0];
    BXP = P->lin[1];
    BXC = P->lin[2];
    if ((rc = stencil(P, 0, X, ProArgs{}, E_STORE, BX, nullptr, nullptr, 0.0, 0.0, nullptr, st))) return rc;
    if (!xp_is_x && (rc = stencil(P, 0, XP, ProArgs{}, E_STORE, BXP, nullptr, nullptr, 0.0, 0.0, nullptr, st)))
      return rc;
    bx_keep = BXC;
  }
  for (int t = 0; t < a->max_iters; ++t) {
    double beta;
    if (a->method == ADP_METHOD_FISTA_SC) {
      beta = theta;
    } else {
      const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t_mom * t_mom));
      beta = (t_mom - 1.0) / t_next;
      t_mom = t_next;
    }
    // y = x + beta (x - x_prev) is the residual pass's row prologue (stored to Y)
    ProArgs pe;
    pe.pro = P_EXTRAP;
    pe.x2 = xp_is_x ? X : XP;
    pe.coef = beta;
    pe.wout = Y;
    double h_y = 0.0, gn2 = 0.0;
    if (lin) rc = vg_lin(P, lp, beta, X, xp_is_x ? X : XP, BX, xp_is_x ? BX : BXP, Y, G, &h_y, &gn2, st);
    else rc = vg(P, lp, X, pe, G, &h_y, &gn2, st);
    if (rc) return rc;
    res->vg_evals++;
    const double gn = std::sqrt(gn2);
    if (!std::isfinite(gn)) return diverged(t);
    if (gn <= tol) return finish(Y, gn2, t, 1);
    // x_prev = x; x = step from y
    double d = 0.0;
    if (a->adaptive) {
      int ok = 0;
      double s = 0.0;
      if ((rc = backtrack(Y, h_y, gn, lip_t, &s, &ok))) return rc;
      if (!ok) { res->status = ADP_STATUS_BT_FAIL; return ADP_OK; }
      lip_t = std::max(1.0 / s * 0.9, lip * 1e-8);
      d = last_dot;
    } else {
      if ((rc = vec(P, V_STEPDIV, lip_t, Y, nullptr, G, XC, nullptr, st))) return rc;
      if (a->method == ADP_METHOD_AGD && (rc = vec(P, V_DOTDIFF, 0.0, XC, X, G, nullptr, &d, st))) return rc;
    }
    // rotate: XP <- X, X <- XC (and their images under B)
    std::swap(XP, X);
    std::swap(X, XC);
    if (lin) {
      std::swap(BXP, BX);
      std::swap(BX, BXC);
      bx_keep = BXC;
    }
    xp_is_x = false;
    if (a->method == ADP_METHOD_AGD && d > 0) {   // gradient restart: vdot(g, x - x_prev) > 0
      t_mom = 1.0;
      xp_is_x = true;
      res->restarts++;
    }
  }
  double gn2 = 0.0;
  if (lin) rc = vg_lin(P, lp, 0.0, X, X, BX, BX, Y, G, nullptr, &gn2, st);
  else rc = vg(P, lp, X, ProArgs{}, G, nullptr, &gn2, st);
  if (rc) return rc;
  return finish(X, gn2, a->max_iters, std::sqrt(gn2) <= tol);
}

// cg_solve on lower_hess_vec with the lower_hess_diag Jacobi preconditioner (hypergradient.py:35-84 as
// called at 171-176), every Hessian product = two tile-FFT stencils with the TV term in the epilogue;
// the next search direction p = minv r + beta p rides in the first stencil's row prologue.
extern "C" int adp_fft_hess_cg(adp_fft_plan* P, const adp_lower* lp, const void* x_tilde, const void* rhs, void* q,
                               int32_t warm, const void* precond, double tol, int32_t max_iters, adp_cg_result* res,
                               void* stream) {
  if (!P || !lp || !x_tilde || !rhs || !q || !res) return dense_fail(ADP_ERR_ARG, "fft hess_cg: null argument");
  if (lp->reg != ADP_REG_TV) return dense_fail(ADP_ERR_UNSUPPORTED, "fft path: smoothed TV only");
  if (!(tol > 0)) return dense_fail(ADP_ERR_ARG, "tol must be > 0");
  cudaStream_t st = (cudaStream_t)stream;
  *res = adp_cg_result{};
  int rc = prepare(P, lp->kernel, st);
  if (rc) return rc;
  for (int i = 0; i < 7; ++i)
    if (!P->cgbuf[i] && cudaMalloc(&P->cgbuf[i], (size_t)P->N * sizeof(double)) != cudaSuccess)
      return dense_fail(ADP_ERR_CUDA, "fft hess_cg: device allocation failed");
  if (!P->sat && cudaMalloc(&P->sat, (size_t)(P->g.kh + 1) * (P->g.kw + 1) * P->g.C * sizeof(double)) != cudaSuccess)
    return dense_fail(ADP_ERR_CUDA, "fft hess_cg: device allocation failed");
  const Geo& g = P->g;
  const int64_t n = P->N;
  double* R = P->cgbuf[0];
  double* Pb[2] = {P->cgbuf[1], P->cgbuf[2]};
  double* HP = P->cgbuf[3];
  double* MINV = P->cgbuf[4];
  double* Bp = P->buf[5];
  double* Q = (double*)q;
  const double* RHS = (const double*)rhs;
  // curvature weights of x~ and the Jacobi diagonal
  curv_kernel<<<kVecGrid, 256, 0, st>>>(g, (const double*)x_tilde, lp->nu, P->cgbuf[5], P->cgbuf[6]);
  double floor_ = -1e308;
  if (precond) {
    cudaMemcpyAsync(MINV, precond, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  } else {
    sat_kernel<<<1, 32, 0, st>>>(g, (const double*)lp->kernel, P->sat);
    diag_kernel<<<kVecGrid, 256, 0, st>>>(g, P->sat, P->cgbuf[5], P->cgbuf[6], lp->alpha, MINV, P->partV);
    if ((rc = check_launch("fft hess_cg diag"))) return rc;
    // max over the per-CTA maxima (exact in any order)
    std::vector<double> pm(kVecGrid);
    cudaMemcpyAsync(pm.data(), P->partV, kVecGrid * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return dense_fail(ADP_ERR_CUDA, "fft hess_cg: diag");
    double mx = -INFINITY;
    for (double v : pm) mx = std::max(mx, v);
    floor_ = 1e-12 * mx + 1e-300;
  }
  minv_kernel<<<kVecGrid, 256, 0, st>>>(n, floor_, MINV);
  // r = rhs - H q (warm start) or q = 0, r = rhs
  if (warm) {
    if ((rc = stencil(P, 0, Q, ProArgs{}, E_STORE, Bp, nullptr, nullptr, 0.0, 0.0, nullptr, st))) return rc;
    if ((rc = stencil(P, 1, Bp, ProArgs{}, E_HESSRES, R, RHS, Q, lp->alpha, lp->nu, P->partG, st))) return rc;
    res->hv++;
  } else {
    cudaMemsetAsync(Q, 0, n * sizeof(double), st);
    cudaMemcpyAsync(R, RHS, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  cg_update_kernel<<<kVecGrid, 256, 0, st>>>(n, 0.0, Q, R, nullptr, nullptr, MINV, 1, P->partV);
  double t2[2];
  if ((rc = fold(P, FoldSrc{P->partV, kVecGrid, 2}, kNoSrc, kNoSrc, t2, st))) return rc;
  double rs = t2[0], rr = t2[1], beta = 0.0;
  int iters = 0, cur = 0;
  const double* pold = MINV;   // p_1 = s_0 = minv r (+ 0 * a finite vector)
  for (iters = 1; iters <= max_iters; ++iters) {
    if (std::sqrt(rr) <= tol) {
      iters -= 1;
      break;
    }
    ProArgs pa;
    pa.pro = P_CGDIR;
    pa.x2 = MINV;
    pa.xold = pold;
    pa.coef = beta;
    pa.wout = Pb[cur];
    if ((rc = stencil(P, 0, R, pa, E_STORE, Bp, nullptr, nullptr, 0.0, 0.0, nullptr, st))) return rc;
    if ((rc = stencil(P, 1, Bp, ProArgs{}, E_HESS, HP, nullptr, Pb[cur], lp->alpha, lp->nu, P->partG, st))) return rc;
    res->hv++;
    double cv[2];
    if ((rc = fold(P, src3(P, P->partG), kNoSrc, kNoSrc, cv, st))) return rc;
    const double curv = cv[0];
    if (curv <= 0) {
      res->status = ADP_STATUS_NEGCURV;
      res->curv = curv;
      res->iters = iters;
      return ADP_OK;
    }
    const double a = rs / curv;
    cg_update_kernel<<<kVecGrid, 256, 0, st>>>(n, a, Q, R, Pb[cur], HP, MINV, 0, P->partV);
    if ((rc = fold(P, FoldSrc{P->partV, kVecGrid, 2}, kNoSrc, kNoSrc, t2, st))) return rc;
    beta = t2[0] / rs;
    rs = t2[0];
    rr = t2[1];
    pold = Pb[cur];
    cur ^= 1;
  }
  if (iters > max_iters) iters = max_iters;
  // true residual ||H q - rhs|| (hypergradient.py:83)
  if ((rc = stencil(P, 0, Q, ProArgs{}, E_STORE, Bp, nullptr, nullptr, 0.0, 0.0, nullptr, st))) return rc;
  if ((rc = stencil(P, 1, Bp, ProArgs{}, E_HESSRES, nullptr, RHS, Q, lp->alpha, lp->nu, P->partG, st))) return rc;
  res->hv++;
  double tr[2];
  if ((rc = fold(P, src3(P, P->partG), kNoSrc, kNoSrc, tr, st))) return rc;
  res->residual = std::sqrt(tr[0]);
  res->iters = iters;
  res->converged = res->residual <= tol;
  return ADP_OK;
}

// UpperProblem.fit_value and ||upper_fit_grad|| (problems.py:48-50, hypergradient.py:87-89):
// r = A x - y_delta (residual pass), grad = 2 A^T r (adjoint pass with the doubling in the epilogue)
extern "C" int adp_fft_upper_terms(adp_fft_plan* P, const void* A_kernel, const void* x, const void* y_delta,
                                   double* fit, double* grad_norm, void* grad_out, void* stream) {
  if (!P || !A_kernel || !x || !y_delta || !fit || !grad_norm) return dense_fail(ADP_ERR_ARG, "fft upper_terms: null");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = prepare(P, A_kernel, st);
  if (rc) return rc;
  double* R = P->buf[5];
  if ((rc = stencil(P, 0, (const double*)x, ProArgs{}, E_RESID, R, (const double*)y_delta, nullptr, 0.0, 0.0, P->partR,
                    st)))
    return rc;
  if ((rc = stencil(P, 1, R, ProArgs{}, E_TWICE, (double*)grad_out, nullptr, nullptr, 0.0, 0.0, P->partG, st))) return rc;
  double t[4];
  if ((rc = fold(P, src3(P, P->partR), src3(P, P->partG), kNoSrc, t, st))) return rc;
  *fit = t[0];
  *grad_norm = std::sqrt(t[2]);
  return ADP_OK;
}

// mixed_second_transpose (hypergradient.py:92-104): 2 [kgc(x~, B q) + kgc(q, B x~ - y)] on tile FFTs;
// out is the kernel-shaped (kh, kw, C) device array.
extern "C" int adp_fft_mixed_T(adp_fft_plan* P, const adp_lower* lp, const void* x_tilde, const void* q, void* out,
                               void* stream) {
  if (!P || !lp || !x_tilde || !q || !out) return dense_fail(ADP_ERR_ARG, "fft mixed_T: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = prepare(P, lp->kernel, st);
  if (rc) return rc;
  const Geo& g = P->g;
  const size_t sbytes = (size_t)g.C * std::max(2, g.npairs) * T * T * sizeof(double2);
  if (!P->S2 && cudaMalloc(&P->S2, sbytes) != cudaSuccess) return dense_fail(ADP_ERR_CUDA, "fft mixed_T: allocation");
  if (!P->acc && cudaMalloc(&P->acc, (size_t)g.C * T * T * sizeof(double2)) != cudaSuccess)
    return dense_fail(ADP_ERR_CUDA, "fft mixed_T: allocation");
  double* Bq = P->buf[3];
  double* R = P->buf[4];
  if ((rc = stencil(P, 0, (const double*)q, ProArgs{}, E_STORE, Bq, nullptr, nullptr, 0.0, 0.0, nullptr, st))) return rc;
  if ((rc = stencil(P, 0, (const double*)x_tilde, ProArgs{}, E_RESID, R, (const double*)lp->y, nullptr, 0.0, 0.0, nullptr,
                    st)))
    return rc;
  const int rgrid = g.npairs * (T / RROWS) * g.C;
  const double* us[2] = {(const double*)x_tilde, (const double*)q};
  const double* vs[2] = {Bq, R};
  for (int k = 0; k < 2; ++k) {
    RowArgs ru{g, us[k], P->S, P->tw, 0, nullptr, P_NONE, nullptr, nullptr, 0.0, nullptr, nullptr};
    row_fwd_kernel<<<rgrid, 256, 0, st>>>(ru);
    RowArgs rv{g, vs[k], P->S2, P->tw, 2, nullptr, P_NONE, nullptr, nullptr, 0.0, nullptr, nullptr};
    row_fwd_kernel<<<rgrid, 256, 0, st>>>(rv);
    ColArgs ca{g, P->S, nullptr, nullptr, P->tw, 0, g.npairs};
    col_corr_kernel<<<g.npairs * (T / CCOLS) * g.C, 64 * CCOLS, 0, st>>>(ca, P->S2);
    pair_sum_kernel<<<kVecGrid, 256, 0, st>>>(P->S, g.npairs, g.C, k, P->acc);
  }
  Geo ag = g;
  ag.npairs = 1;
  ColArgs ci{ag, P->acc, nullptr, nullptr, P->tw, 2, 1};
  col_kernel<<<(T / CCOLS) * g.C, 64 * CCOLS, 0, st>>>(ci);
  kgc_final_kernel<<<g.C * ((g.kh + RROWS - 1) / RROWS), 256, 0, st>>>(g, P->acc, P->tw, 2.0 * kInvT2, (double*)out);
  return check_launch("fft mixed_T");
}
