// Depthwise 2-D engine: the MAID lower-level machinery for
//   h(x, b) = ||B_b x - y||^2 + alpha * TV_nu(x)          (lower_solvers.py:37-96)
// on (H, W, C) images with a (kh, kw, C) zero-padded "same" correlation
// stencil (operators.py:83-122) and smoothed anisotropic TV
// (regularizers.py:137-199).
//
// Design (B200-first):
//   * One cooperative persistent kernel per call; all CTAs run the same
//     scalar control flow (AGD momentum, backtracking, restart, CG
//     coefficients) redundantly from identical deterministic reductions, so
//     decisions need no broadcast and no host round trip.
//   * Each stage walks fixed image tiles (TH x TW pixels, all channels) and
//     stages the tile plus halo in shared memory as channel planes with a
//     skewed row layout (one pad per RW elements) so the register-blocked
//     stencil (RW outputs per thread, sliding window) is bank-conflict free.
//   * Strict mode reproduces scipy.ndimage.correlate bit for bit: taps in
//     row-major order, acc = 0.0 then acc + x*w (no FMA), taps with
//     |w| <= DBL_EPSILON skipped.  Fast mode uses FMA.
//   * Element sums the reference takes with np.sum use NumPy's pairwise
//     tree (bitwise); ddot-type sums (norms, vdot) use fixed per-tile trees.
#pragma once
#include "adp_device.cuh"
#include "conv2d_args.h"

namespace adp {

// ---------------------------------------------------------------------------
// value sources used by the tile loaders (all compute exactly the reference
// expression for one element)
template <typename T> struct SrcZero { __device__ T operator()(int64_t) const { return T(0); } };
template <typename T> struct SrcOnes { __device__ T operator()(int64_t) const { return T(1); } };
template <typename T> struct SrcLin {
  const T* x;
  __device__ T operator()(int64_t i) const { return ldcg(x + i); }
};
// y = x + beta * (x - x_prev)                      (lower_solvers.py:196)
template <typename T> struct SrcExtrap {
  const T* x; const T* xp; T beta;
  __device__ T operator()(int64_t i) const {
    const T a = ldcg(x + i), b = ldcg(xp + i);
    return a + beta * (a - b);
  }
};
// x = y - g / L                                    (lower_solvers.py:173, 207)
template <typename T> struct SrcCand {
  const T* x; const T* xp; const T* g; T beta; T L;
  __device__ T operator()(int64_t i) const {
    const T a = ldcg(x + i), b = ldcg(xp + i);
    const T y = a + beta * (a - b);
    return y - ldcg(g + i) / L;
  }
};
// x = x - step * g                                 (lower_solvers.py:165)
template <typename T> struct SrcStep {
  const T* x; const T* g; T step;
  __device__ T operator()(int64_t i) const { return ldcg(x + i) - step * ldcg(g + i); }
};
// v = w / s                                        (operators.py:150, 160)
template <typename T> struct SrcScaled {
  const T* w; T s;
  __device__ T operator()(int64_t i) const { return ldcg(w + i) / s; }
};
// p = s + beta * p_old (first: p = s)              (hypergradient.py:75, 81)
template <typename T> struct SrcCGDir {
  const T* s; const T* p; T beta; int first;
  __device__ T operator()(int64_t i) const {
    const T sv = ldcg(s + i);
    return first ? sv : sv + beta * ldcg(p + i);
  }
};

// ---------------------------------------------------------------------------
template <typename T, bool FAST, int RW>
struct Conv {
  static_assert((RW & (RW - 1)) == 0, "RW must be a power of two");
  static constexpr int kShift = RW == 1 ? 0 : RW == 2 ? 1 : RW == 4 ? 2 : 3;

  const ConvArgs<T>& a;
  const ConvGeom& g;
  T* ws;       // C x kh x kw  (taps, tiny taps zeroed)
  T* wf;       // flipped
  T* pa;       // plane set A: C x SH x SWP
  T* pb;       // small planes (1-halo) C x YSH x YSWP, or Q planes
  T* pq;       // Q planes 2 x C x (TH+1) x QP
  double* sv;  // tree scratch
  double* red; // 33 doubles
  int QP;
  int ty, tx;

  __device__ static __forceinline__ int sk(int col) { return col + (col >> kShift); }

  __device__ Conv(const ConvArgs<T>& a_, unsigned char* smem) : a(a_), g(a_.g) {
    const int nk = g.kh * g.kw * g.C;
    size_t off = 0;
    red = reinterpret_cast<double*>(smem);
    off += 64 * sizeof(double);
    ws = reinterpret_cast<T*>(smem + off);
    off += ((size_t)nk * sizeof(T) + 15) & ~size_t(15);
    wf = reinterpret_cast<T*>(smem + off);
    off += ((size_t)nk * sizeof(T) + 15) & ~size_t(15);
    unsigned char* region = smem + off;
    sv = reinterpret_cast<double*>(region);
    pa = reinterpret_cast<T*>(region);
    const size_t pa_elems = (size_t)g.C * g.SH * g.SWP;
    pb = pa + pa_elems;
    QP = (g.TW + 1) + ((g.TW + 1) >> kShift) + 1;
    pq = pb;  // Q planes live after plane set A (stage A only)
    const int tpr = g.TW / RW;
    ty = threadIdx.x / tpr;
    tx = threadIdx.x % tpr;
  }

  // ---- weights: ws[c][i][j] = kern[i][j][c] (|w| <= eps -> 0), wf flipped
  __device__ void load_weights(const T* kern) {
    const int kh = g.kh, kw = g.kw, C = g.C, nk = kh * kw * C;
    for (int e = threadIdx.x; e < nk; e += blockDim.x) {
      const int c = e % C, ij = e / C, i = ij / kw, j = ij % kw;
      T w = kern[e];
      if (!(fabs((double)w) > kDblEps)) w = T(0);  // ndimage: only |w| > DBL_EPSILON taps
      ws[(c * kh + i) * kw + j] = w;
      wf[(c * kh + (kh - 1 - i)) * kw + (kw - 1 - j)] = w;
    }
    __syncthreads();
  }
  // squared flipped taps (gram_diag: correlate(ones, flipped**2), operators.py:120-122)
  __device__ void load_weights_sq(const T* kern) {
    const int kh = g.kh, kw = g.kw, C = g.C, nk = kh * kw * C;
    for (int e = threadIdx.x; e < nk; e += blockDim.x) {
      const int c = e % C, ij = e / C, i = ij / kw, j = ij % kw;
      T w = kern[e];
      w = w * w;
      if (!(fabs((double)w) > kDblEps)) w = T(0);
      wf[(c * kh + (kh - 1 - i)) * kw + (kw - 1 - j)] = w;
    }
    __syncthreads();
  }

  __device__ __forceinline__ void tile_origin(int tile, int& h0, int& w0) const {
    h0 = (tile / g.tilesW) * g.TH;
    w0 = (tile % g.tilesW) * g.TW;
  }
  __device__ __forceinline__ T* plane(T* base, int c) const { return base + (size_t)c * g.SH * g.SWP; }

  // ---- load tile + (r+1) halo of all channels into plane set `dst`
  template <class Src>
  __device__ void load_full(T* dst, int h0, int w0, const Src& src) const {
    const int C = g.C, SWL = g.TW + 2 * g.rw + 2, rowE = SWL * C;
    const int total = g.SH * rowE;
    const int gh0 = h0 - g.rh - 1, gw0 = w0 - g.rw - 1;
    for (int k = threadIdx.x; k < total; k += blockDim.x) {
      const int sr = k / rowE, e = k - sr * rowE;
      const int px = e / C, c = e - px * C;
      const int gh = gh0 + sr, gw = gw0 + px;
      T v = T(0);
      if (gh >= 0 && gh < g.H && gw >= 0 && gw < g.W) v = src(((int64_t)gh * g.W + gw) * C + c);
      dst[(size_t)c * g.SH * g.SWP + sr * g.SWP + sk(px)] = v;
    }
  }
  // ---- load tile + 1 halo into small planes (pitch YSWP)
  template <class Src>
  __device__ void load_small(T* dst, int h0, int w0, const Src& src) const {
    const int C = g.C, SWL = g.TW + 2, rowE = SWL * C;
    const int total = g.YSH * rowE;
    for (int k = threadIdx.x; k < total; k += blockDim.x) {
      const int sr = k / rowE, e = k - sr * rowE;
      const int px = e / C, c = e - px * C;
      const int gh = h0 - 1 + sr, gw = w0 - 1 + px;
      T v = T(0);
      if (gh >= 0 && gh < g.H && gw >= 0 && gw < g.W) v = src(((int64_t)gh * g.W + gw) * C + c);
      dst[(size_t)c * g.YSH * g.YSWP + sr * g.YSWP + sk(px)] = v;
    }
  }

  // ---- register-blocked correlation: RW consecutive outputs (row ty, cols
  // tx*RW..) of one channel plane with stencil w (kh x kw).  Per output the
  // taps are accumulated in row-major order starting from 0.
  __device__ __forceinline__ void stencil(const T* __restrict__ pl, const T* __restrict__ w, T (&acc)[RW]) const {
#pragma unroll
    for (int o = 0; o < RW; ++o) acc[o] = T(0);
    const int kh = g.kh, kw = g.kw;
    const T* base = pl + (ty + 1) * g.SWP + tx * (RW + 1);
    for (int i = 0; i < kh; ++i) {
      const T* row = base + i * g.SWP;
      const T* wr = w + i * kw;
      T win[RW];
#pragma unroll
      for (int q = 0; q < RW - 1; ++q) win[q] = row[(1 + q) + ((1 + q) >> kShift)];
      int j = 0;
      for (; j + RW <= kw; j += RW) {
        const T* rj = row + j + (j >> kShift);
#pragma unroll
        for (int jj = 0; jj < RW; ++jj) {
          const int q = jj + RW - 1;
          win[(jj + RW - 1) % RW] = rj[(1 + q) + ((1 + q) >> kShift)];
          const T wt = wr[j + jj];
#pragma unroll
          for (int o = 0; o < RW; ++o) acc[o] = madd<FAST>(acc[o], win[(o + jj) % RW], wt);
        }
      }
      if (j < kw) {
        const T* rj = row + j + (j >> kShift);
#pragma unroll
        for (int jj = 0; jj < RW - 1; ++jj) {
          if (j + jj < kw) {
            const int q = jj + RW - 1;
            win[(jj + RW - 1) % RW] = rj[(1 + q) + ((1 + q) >> kShift)];
            const T wt = wr[j + jj];
#pragma unroll
            for (int o = 0; o < RW; ++o) acc[o] = madd<FAST>(acc[o], win[(o + jj) % RW], wt);
          }
        }
      }
    }
  }

  __device__ __forceinline__ int64_t gidx(int h, int w, int c) const { return ((int64_t)h * g.W + w) * g.C + c; }

  // small-plane accessor: pixel (tile row r, tile col q), r,q in [-1, TH]/[-1, TW]
  __device__ __forceinline__ T sp(const T* base, int c, int r, int q) const {
    return base[(size_t)c * g.YSH * g.YSWP + (r + 1) * g.YSWP + sk(q + 1)];
  }
  // full-plane accessor for pixel (tile row r, tile col q)
  __device__ __forceinline__ T fp(const T* base, int c, int r, int q) const {
    return base[(size_t)c * g.SH * g.SWP + (r + g.rh + 1) * g.SWP + sk(q + g.rw + 1)];
  }

  // =========================================================================
  // Stage A: r = B y - ydat (write R); TV at y: terms (root) -> TV2, grad -> TVG
  // (lower_value_and_grad, lower_solvers.py:50-63; SmoothedTV.value_and_grad,
  // regularizers.py:167-175).  `tv` false when alpha == 0.
  template <class Src>
  __device__ void stageA(const Src& src, T* Rout, const T* ydat, bool tv, T* TV2out, T* TVGout) {
    const T nu = T(a.nu), nu2 = nu * nu;
    for (int tile = blockIdx.x; tile < g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      load_full(pa, h0, w0, src);
      __syncthreads();
      const int h = h0 + ty;
      for (int c = 0; c < g.C; ++c) {
        T acc[RW];
        stencil(plane(pa, c), ws + c * g.kh * g.kw, acc);
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + tx * RW + o;
          if (h < g.H && w < g.W) {
            const int64_t i = gidx(h, w, c);
            Rout[i] = acc[o] - ydat[i];
          }
        }
      }
      if (!tv) continue;
      // Q planes over tile rows -1..TH-1, cols -1..TW-1: q = d / sqrt(d^2 + nu^2)
      T* q0 = pq;
      T* q1 = pq + (size_t)g.C * (g.TH + 1) * QP;
      const int qrE = (g.TW + 1) * g.C, qtot = (g.TH + 1) * qrE;
      for (int k = threadIdx.x; k < qtot; k += blockDim.x) {
        const int qr = k / qrE, e = k - qr * qrE;
        const int qc = e / g.C, c = e - qc * g.C;
        const int r = qr - 1, q = qc - 1;   // tile-relative pixel
        const int hh = h0 + r, ww = w0 + q;
        const T yc = fp(pa, c, r, q);
        const T d0 = (hh < g.H - 1) ? fp(pa, c, r + 1, q) - yc : T(0);
        const T d1 = (ww < g.W - 1) ? fp(pa, c, r, q + 1) - yc : T(0);
        const T rt0 = sqrt(d0 * d0 + nu2), rt1 = sqrt(d1 * d1 + nu2);
        q0[(size_t)c * (g.TH + 1) * QP + qr * QP + sk(qc)] = d0 / rt0;
        q1[(size_t)c * (g.TH + 1) * QP + qr * QP + sk(qc)] = d1 / rt1;
        if (r >= 0 && q >= 0 && hh < g.H && ww < g.W) {
          const int64_t i = gidx(hh, ww, c);
          TV2out[i] = rt0;
          TV2out[g.N + i] = rt1;
        }
      }
      __syncthreads();
      for (int c = 0; c < g.C; ++c) {
        const T* Q0 = q0 + (size_t)c * (g.TH + 1) * QP;
        const T* Q1 = q1 + (size_t)c * (g.TH + 1) * QP;
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int qcol = tx * RW + o;
          const int w = w0 + qcol;
          if (h < g.H && w < g.W) {
            // image_forward_diff_adjoint (regularizers.py:61-67), per-pixel order
            T t = T(0);
            if (h >= 1) t = t + Q0[ty * QP + sk(qcol + 1)];
            if (h <= g.H - 2) t = t - Q0[(ty + 1) * QP + sk(qcol + 1)];
            if (w >= 1) t = t + Q1[(ty + 1) * QP + sk(qcol)];
            if (w <= g.W - 2) t = t - Q1[(ty + 1) * QP + sk(qcol + 1)];
            TVGout[gidx(h, w, c)] = t;
          }
        }
      }
    }
  }

  // Stage B: g = 2 * B^T r (+ alpha * tvg); tile partial of g.g -> sgg
  __device__ void stageB(const T* Rin, bool tv, const T* TVGin, T* Gout, const SumDev* sgg) {
    const T two = T(2), alpha = T(a.alpha);
    for (int tile = blockIdx.x; tile < g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      load_full(pa, h0, w0, SrcLin<T>{Rin});
      __syncthreads();
      const int h = h0 + ty;
      double part = 0.0;
      for (int c = 0; c < g.C; ++c) {
        T acc[RW];
        stencil(plane(pa, c), wf + c * g.kh * g.kw, acc);
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + tx * RW + o;
          if (h < g.H && w < g.W) {
            const int64_t i = gidx(h, w, c);
            T gv = two * acc[o];
            if (tv) gv = gv + alpha * ldcg(TVGin + i);
            Gout[i] = gv;
            part += (double)gv * (double)gv;
          }
        }
      }
      if (sgg) store_tile_partial(*sgg, tile, part, red);
    }
  }

  // Stage C (value at a candidate): xc = src; rc = B xc - y -> RCout; TV
  // terms sqrt(d^2+nu^2) - nu -> TV2Cout (tv_value, regularizers.py:70-72);
  // optional tile partial of g.(xc - xold); xc written to Xout.
  template <class Src>
  __device__ void stageC(const Src& src, T* RCout, bool tv, T* TV2Cout, T* Xout, const T* Gin, const T* Xold,
                         const SumDev* sdot) {
    const T nu = T(a.nu), nu2 = nu * nu;
    for (int tile = blockIdx.x; tile < g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      load_full(pa, h0, w0, src);
      __syncthreads();
      const int h = h0 + ty;
      double part = 0.0;
      for (int c = 0; c < g.C; ++c) {
        T acc[RW];
        stencil(plane(pa, c), ws + c * g.kh * g.kw, acc);
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int q = tx * RW + o;
          const int w = w0 + q;
          if (h < g.H && w < g.W) {
            const int64_t i = gidx(h, w, c);
            RCout[i] = acc[o] - a.ydat[i];
            const T xc = fp(pa, c, ty, q);
            if (tv) {
              const T d0 = (h < g.H - 1) ? fp(pa, c, ty + 1, q) - xc : T(0);
              const T d1 = (w < g.W - 1) ? fp(pa, c, ty, q + 1) - xc : T(0);
              TV2Cout[i] = sqrt(d0 * d0 + nu2) - nu;
              TV2Cout[g.N + i] = sqrt(d1 * d1 + nu2) - nu;
            }
            if (Xout) Xout[i] = xc;
            if (sdot) part += (double)ldcg(Gin + i) * (double)(xc - ldcg(Xold + i));
          }
        }
      }
      if (sdot) store_tile_partial(*sdot, tile, part, red);
    }
  }

  // Light candidate (non-adaptive step): xc = src per own pixel, dot partial.
  template <class Src>
  __device__ void stageCLight(const Src& src, T* Xout, const T* Gin, const T* Xold, const SumDev* sdot) {
    for (int tile = blockIdx.x; tile < g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      const int h = h0 + ty;
      double part = 0.0;
      for (int c = 0; c < g.C; ++c) {
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + tx * RW + o;
          if (h < g.H && w < g.W) {
            const int64_t i = gidx(h, w, c);
            const T xc = src(i);
            Xout[i] = xc;
            part += (double)ldcg(Gin + i) * (double)(xc - ldcg(Xold + i));
          }
        }
      }
      store_tile_partial(*sdot, tile, part, red);
    }
  }

  // Plain correlation pass: out = B src (or B^T src with flipped taps),
  // optional ydat subtraction and tile partial of out.out.
  template <class Src>
  __device__ void stage_corr(const Src& src, bool flipped, T* Out, const T* sub, T scale, const SumDev* ssq) {
    for (int tile = blockIdx.x; tile < g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      load_full(pa, h0, w0, src);
      __syncthreads();
      const int h = h0 + ty;
      double part = 0.0;
      for (int c = 0; c < g.C; ++c) {
        T acc[RW];
        stencil(plane(pa, c), (flipped ? wf : ws) + c * g.kh * g.kw, acc);
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + tx * RW + o;
          if (h < g.H && w < g.W) {
            const int64_t i = gidx(h, w, c);
            T v = acc[o];
            if (sub) v = v - sub[i];
            v = scale * v;
            Out[i] = v;
            part += (double)v * (double)v;
          }
        }
      }
      if (ssq) store_tile_partial(*ssq, tile, part, red);
    }
  }

  // Elementwise over own pixels of every tile (grid-stride by tiles).
  template <class F>
  __device__ void foreach_pixel(const F& f) {
    for (int tile = blockIdx.x; tile < g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      const int h = h0 + ty;
      for (int c = 0; c < g.C; ++c)
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + tx * RW + o;
          if (h < g.H && w < g.W) f(gidx(h, w, c), h, w, c);
        }
    }
  }
  // Same, with a per-tile partial accumulated by f's return value.
  template <class F>
  __device__ void foreach_pixel_sum(const F& f, const SumDev& s) {
    for (int tile = blockIdx.x; tile < g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      const int h = h0 + ty;
      double part = 0.0;
      for (int c = 0; c < g.C; ++c)
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + tx * RW + o;
          if (h < g.H && w < g.W) part += f(gidx(h, w, c), h, w, c);
        }
      store_tile_partial(s, tile, part, red);
    }
  }
};

template <typename T> struct SqOf {
  const T* p;
  __device__ double operator()(int64_t i) const {
    const T v = ldcg(p + i);
    return (double)(v * v);
  }
};
template <typename T> struct Plain {
  const T* p;
  __device__ double operator()(int64_t i) const { return (double)ldcg(p + i); }
};

}  // namespace adp
