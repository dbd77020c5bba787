// Dense 1-D engine: DenseOperator (operators.py:49-80) with the smoothed
// elastic net (regularizers.py:75-134) — the reference's 1-D deconvolution
// path (config 1, build_deconv1d problems.py:156-191).
//
// B200 design: a small cooperative grid; CTA c keeps rows [c*R, (c+1)*R) of
// B resident in shared memory for the whole call.  Every signal-length
// vector (x, x_prev, g, candidate, CG state) is replicated in every CTA's
// shared memory and updated redundantly and identically, so the only data
// exchanged per GEMV is the row results (B v) or the per-CTA column
// partials (B^T u), each followed by one grid barrier.
// Grids of <= 16 CTAs whose state fits (c1: n = 256, 16 CTAs) run as ONE
// thread-block cluster: every CTA stores its row results / column partials
// straight into all CTAs' shared memory (distributed shared memory) and the
// exchange ends with a cluster barrier -- no global round trip, no grid
// barrier; same arithmetic in the same order (bitwise equal to the grid path,
// tests/test_gpu_dense_cluster.py).
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <algorithm>
#include <cstring>
#include <string>
#include "adp_device.cuh"
#include "adp_plan.h"
#include "dense1d_args.h"

namespace adp {
namespace cg = cooperative_groups;

enum DenseMode : int {
  DM_APPLY = 0, DM_ADJOINT, DM_GRAM, DM_VALUE, DM_VG, DM_GRAD, DM_HV, DM_HDIAG, DM_UPPER, DM_POWER, DM_MIXED,
  DM_DOT, DM_KGC, DM_PROX
};

constexpr int kDenseVecs = 12;

// np_leaf_warp (adp_device.cuh: NumPy's pairwise leaf, n <= 128) with the terms evaluated by all 32
// lanes at once -- lane (k, g) computes rows g, g + 4, g + 8, g + 12 of accumulator k -- and only the
// ordered additions r[k] += a[8 m + k] left as a serial chain fed by shuffles.  The dense engine's sums
// are latency chains of a few hundred elements whose terms hold square roots: evaluating them inside
// the 8-lane chain cost 1.8 us per sum.  Same additions in the same order: bitwise equal.
template <class Src>
__device__ __forceinline__ double np_leaf_warp32(const Src& src, int64_t s, int n) {
  const int lane = threadIdx.x & 31;
  if (n < 8 || n > 128) return np_leaf_warp(src, s, n);
  const int nfull = n - (n % 8), M = nfull >> 3;   // rows of 8 terms
  const int k = lane & 7, g = lane >> 3;
  double v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int m = g + 4 * j;
    v[j] = m < M ? src(s + 8 * m + k) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const double x = __shfl_sync(kFull, v[m >> 2], k + 8 * (m & 3));   // row m of accumulator k
    if (m == 0) acc = x;
    else if (m < M) acc = acc + x;
  }
  double t = acc + __shfl_down_sync(kFull, acc, 1);
  t = t + __shfl_down_sync(kFull, t, 2);
  t = t + __shfl_down_sync(kFull, t, 4);
  if (lane == 0) {
    for (int i = nfull; i < n; ++i) t = t + src(s + i);
  }
  return t;
}

template <typename T>
struct Dense {
  const DenseArgs<T>& a;
  GridBarrier gb;
  int n, r0, r1;
  const T* Bs;      // row slice (smem) or global rows
  T* v[kDenseVecs];
  double* sv;
  double* sv2;
  double* red;
  int64_t* lstart;  // smem copy of s_n.leaf_start
  int* sprog;       // smem copy of s_n's tree program
  int rb;           // rowbuf ping-pong index
  bool cl;          // single-cluster launch: exchanges through distributed shared memory
  T* rowv[2];       // cluster: this CTA's copy of the gathered row results (ping-pong)
  double* partv[2]; // cluster: [G][n] column partials of all CTAs (ping-pong)
  int pb;

  __device__ Dense(const DenseArgs<T>& a_, unsigned char* smem) : a(a_) {
    gb.counter = a.bar;
    gb.nblocks = gridDim.x;
    gb.target = 0;
    n = a.n;
    r0 = blockIdx.x * a.rows_per;
    r1 = min(n, r0 + a.rows_per);
    size_t off = 0;
    red = reinterpret_cast<double*>(smem);
    off += 64 * sizeof(double);
    sv = reinterpret_cast<double*>(smem + off);
    off += (size_t)(2 * a.s_n.nLeaves + 2) * sizeof(double);
    sv2 = reinterpret_cast<double*>(smem + off);   // second tree workspace (two sums folded in one pass)
    off += (size_t)(2 * a.s_n.nLeaves + 2) * sizeof(double);
    // the sum's leaf starts and tree program, read on every npsum: cached in shared memory (each sum
    // was a chain of four dependent global loads before)
    lstart = reinterpret_cast<int64_t*>(smem + off);
    off += (size_t)(a.s_n.nLeaves + 1) * sizeof(int64_t);
    sprog = reinterpret_cast<int*>(smem + off);
    off += (size_t)a.plen * sizeof(int);
    for (int k = threadIdx.x; k <= a.s_n.nLeaves; k += blockDim.x) lstart[k] = a.s_n.leaf_start[k];
    for (int k = threadIdx.x; k < a.plen; k += blockDim.x) sprog[k] = a.s_n.progs[a.s_n.top_prog + k];
    off = (off + 15) & ~size_t(15);
    for (int k = 0; k < kDenseVecs; ++k) {
      if (a.gvec) {   // large n: this CTA's private copies in global memory (L1/L2-resident)
        v[k] = a.gvec + ((int64_t)blockIdx.x * kDenseVecs + k) * a.vpitch;
      } else {
        v[k] = reinterpret_cast<T*>(smem + off);
        off += ((size_t)n * sizeof(T) + 15) & ~size_t(15);
      }
    }
    if (a.b_smem && a.B) {
      T* bs = reinterpret_cast<T*>(smem + off);
      for (int64_t e = threadIdx.x; e < (int64_t)(r1 - r0) * n; e += blockDim.x) bs[e] = a.B[(int64_t)r0 * n + e];
      Bs = bs;
    } else {
      Bs = a.B + (int64_t)r0 * n;
    }
    rb = 0;
    cl = a.cluster != 0;
    pb = 0;
    if (cl) {
      if (a.b_smem) off += (size_t)a.rows_per * n * sizeof(T);
      off = (off + 15) & ~size_t(15);
      for (int k = 0; k < 2; ++k) {
        rowv[k] = reinterpret_cast<T*>(smem + off);
        off += ((size_t)n * sizeof(T) + 15) & ~size_t(15);
      }
      for (int k = 0; k < 2; ++k) {
        partv[k] = reinterpret_cast<double*>(smem + off);
        off += (size_t)gridDim.x * n * sizeof(double);
      }
      cg::this_cluster().sync();   // every CTA of the cluster runs before anyone writes into its shared memory
    }
    __syncthreads();
  }

  // split form of xsync(): local work placed between the two runs inside the cluster barrier's latency
  // (the grid barrier has no split form: it all happens in xwait)
  __device__ __forceinline__ void xarrive() {
    if (cl) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }
  __device__ __forceinline__ void xwait() {
    if (cl) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    else gb.sync();
  }
  // the barrier that ends an exchange (after gemv_rows / gemvT_partial / gram_partial)
  __device__ __forceinline__ void xsync() {
    if (cl) cg::this_cluster().sync();   // arrive.release + wait.acquire: the remote shared-memory stores are visible
    else gb.sync();
  }

  __device__ __forceinline__ T* rowbuf() { return a.rowbuf + (size_t)rb * n; }

  // own rows of (B u) (- sub) -> rowbuf[rb]; warp per row, fixed lane order
  __device__ void gemv_rows(const T* u, const T* sub) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T* out = cl ? rowv[rb] : rowbuf();
    cg::cluster_group cluster = cg::this_cluster();
    for (int i = r0 + warp; i < r1; i += nw) {
      const T* row = Bs + (int64_t)(i - r0) * n;
      T acc = T(0);
      for (int k = lane; k < n; k += 32) acc = acc + row[k] * u[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc = acc + __shfl_xor_sync(kFull, acc, o);
      const T val = sub ? acc - sub[i] : acc;   // (every lane holds the sum)
      if (cl) {
        if (lane < (int)gridDim.x) cluster.map_shared_rank(out, lane)[i] = val;   // lane c -> CTA c's copy
      } else if (lane == 0) {
        out[i] = val;
      }
    }
  }
  // after a barrier: dst = full rowbuf; flip the ping-pong buffer
  __device__ void gather_rows(T* dst) {
    if (cl) {
      const T* src = rowv[rb];
      for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = src[k];
    } else {
      const T* src = rowbuf();
      for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = ldcg(src + k);
    }
    rb ^= 1;
    __syncthreads();
  }
  // this CTA's column partial j -> part[cta][j] (global), or into every CTA's partv (cluster)
  __device__ __forceinline__ void put_part(int j, double v) {
    if (cl) {
      cg::cluster_group cluster = cg::this_cluster();
      double* mine = partv[pb] + (size_t)blockIdx.x * n + j;
      for (int c = 0; c < (int)gridDim.x; ++c) *cluster.map_shared_rank(mine, c) = v;
    } else {
      a.part[(size_t)blockIdx.x * n + j] = v;
    }
  }
  // part[cta][j] = sum_{i in own rows} B[i][j] * u[i]
  __device__ void gemvT_partial(const T* u) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      T acc = T(0);
      for (int i = r0; i < r1; ++i) acc = acc + Bs[(int64_t)(i - r0) * n + j] * u[i];
      put_part(j, (double)acc);
    }
  }
  // column sums of squares over own rows (gram_diag partial)
  __device__ void gram_partial() {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      T acc = T(0);
      for (int i = r0; i < r1; ++i) {
        const T b = Bs[(int64_t)(i - r0) * n + j];
        acc = acc + b * b;
      }
      put_part(j, (double)acc);
    }
  }
  // after a barrier: dst[j] = scale * sum_c part[c][j]  (fixed CTA order)
  __device__ void gemvT_finish(T* dst, T scale) {
    if (cl) {
      const double* p = partv[pb];
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        T s = T(0);
        for (int c = 0; c < gridDim.x; ++c) s = s + T(p[(size_t)c * n + j]);
        dst[j] = scale * s;
      }
      pb ^= 1;
    } else {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        T s = T(0);
        for (int c = 0; c < gridDim.x; ++c) s = s + T(ldcg(a.part + (size_t)c * n + j));
        dst[j] = scale * s;
      }
    }
    __syncthreads();
  }

  // NumPy pairwise sum of f(k), k < n (bitwise np.sum order)
  template <class F>
  __device__ double npsum(const F& f) {
    const SumDev& s = a.s_n;
    const int wpb = blockDim.x >> 5;
    for (int l = threadIdx.x >> 5; l < s.nLeaves; l += wpb) {
      const int64_t st = lstart[l];
      const int len = (int)(lstart[l + 1] - st);
      const double r = np_leaf_warp32(f, st, len);
      if ((threadIdx.x & 31) == 0) sv[l] = r;
    }
    __syncthreads();
    return eval_prog(sprog, sv);
  }
  // two sums in one pass (their leaves on different warps, one barrier, both trees folded level by level
  // together): each bitwise npsum's value
  template <class F0, class F1>
  __device__ void npsum2(const F0& f0, const F1& f1, double& o0, double& o1) {
    const int nL = a.s_n.nLeaves;
    const int wpb = blockDim.x >> 5;
    for (int l = threadIdx.x >> 5; l < 2 * nL; l += wpb) {
      const int w = l >= nL, ll = l - w * nL;
      const int64_t st = lstart[ll];
      const int len = (int)(lstart[ll + 1] - st);
      const double r = w ? np_leaf_warp32(f1, st, len) : np_leaf_warp32(f0, st, len);
      if ((threadIdx.x & 31) == 0) (w ? sv2 : sv)[ll] = r;
    }
    __syncthreads();
    const int* prog = sprog;
    const int nI = prog[1], nLev = prog[2];
    const int* lev = prog + 3;
    const int* left = lev + nLev + 1;
    const int* right = left + nI;
    for (int lv = 0; lv < nLev; ++lv) {
      const int b0 = lev[lv], b1 = lev[lv + 1];
      for (int k = b0 + threadIdx.x; k < b1; k += blockDim.x) {
        sv[nL + k] = sv[left[k]] + sv[right[k]];
        sv2[nL + k] = sv2[left[k]] + sv2[right[k]];
      }
      __syncthreads();
    }
    o0 = nI ? sv[nL + nI - 1] : sv[0];
    o1 = nI ? sv2[nL + nI - 1] : sv2[0];
    __syncthreads();
  }
  // ddot-type sum (fixed thread-strided order then block tree)
  template <class F>
  __device__ double dsum(const F& f) {
    double p = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) p += f(k);
    return block_sum(p, red);
  }

  // ---- smoothed elastic net pieces (regularizers.py:75-134)
  __device__ double reg_value(const T* x) {
    if (a.l1 > 0) {
      const T nu = T(a.nu), nu2 = nu * nu;
      double s1, s2;
      npsum2([&](int64_t k) { const T t = x[k]; return (double)(t * t); },
             [&](int64_t k) { const T t = x[k]; return (double)(sqrt(t * t + nu2) - nu); }, s1, s2);
      double val = a.l2 * s1;
      val = val + a.l1 * s2;
      return val;
    }
    const double s1 = npsum([&](int64_t k) { const T t = x[k]; return (double)(t * t); });
    return a.l2 * s1;
  }
  // g[k] = g[k] + alpha * grad J(x)[k]
  __device__ void add_reg_grad(T* g, const T* x) {
    const T two_l2 = T(2.0 * a.l2), l1 = T(a.l1), nu = T(a.nu), nu2 = nu * nu, al = T(a.alpha);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const T t = x[k];
      T rg = two_l2 * t;
      if (a.l1 > 0) rg = rg + l1 * (t / sqrt(t * t + nu2));
      g[k] = g[k] + al * rg;
    }
    __syncthreads();
  }
  __device__ __forceinline__ T rho_curv(T t) const {
    const T nu = T(a.nu), nu2 = nu * nu, s = t * t + nu2;
    return nu2 / (s * sqrt(s));
  }

  // value (and optionally gradient) of the lower problem at x (smem).
  // r into v[4]; g into gout (if non-null).  Uses barriers.
  __device__ double value_grad(const T* x, T* gout, bool vg_form) {
    double val = 0.0, rv = 0.0;
    const bool need_reg = !vg_form || a.alpha != 0.0;
    if (a.reg_only) {
      if (gout) {
        for (int k = threadIdx.x; k < n; k += blockDim.x) gout[k] = T(0);
        __syncthreads();
      }
      if (need_reg) rv = reg_value(x);
    } else {
      // the sums that need no remote data run between the arrive and the wait of the exchange barriers
      gemv_rows(x, a.ydat);
      xarrive();
      if (need_reg) rv = reg_value(x);
      xwait();
      T* r = v[4];
      gather_rows(r);
      if (gout) {
        gemvT_partial(r);
        xarrive();
        val = npsum([&](int64_t k) { const T t = r[k]; return (double)(t * t); });
        xwait();
        gemvT_finish(gout, T(2));
      } else {
        val = npsum([&](int64_t k) { const T t = r[k]; return (double)(t * t); });
      }
    }
    if (need_reg) {
      val = val + a.alpha * rv;
      if (gout && a.alpha != 0.0) add_reg_grad(gout, x);
    }
    return val;
  }

  // H u = 2 B^T B u + alpha * (2 l2 u + l1 rho''(xt) u); wcur = l1*rho''(xt) in smem
  __device__ void hess_vec(const T* u, T* out, const T* wcur) {
    if (a.reg_only) {
      for (int k = threadIdx.x; k < n; k += blockDim.x) out[k] = T(0);
      __syncthreads();
    } else {
      gemv_rows(u, nullptr);
      xsync();
      T* bu = v[4];
      gather_rows(bu);
      gemvT_partial(bu);
      xsync();
      gemvT_finish(out, T(2));
    }
    if (a.alpha != 0.0) {
      const T two_l2 = T(2.0 * a.l2), al = T(a.alpha);
      for (int k = threadIdx.x; k < n; k += blockDim.x) {
        T h = two_l2 * u[k];
        if (a.l1 > 0) h = h + wcur[k] * u[k];
        out[k] = out[k] + al * h;
      }
      __syncthreads();
    }
  }

  __device__ double power(const T* v0, int max_iters, double tol, int& iters, int& conv) {
    T* vv = v[0];
    T* w = v[1];
    T* u = v[2];
    for (int k = threadIdx.x; k < n; k += blockDim.x) vv[k] = v0[k];
    __syncthreads();
    const double nv = sqrt(dsum([&](int k) { const double t = vv[k]; return t * t; }));
    for (int k = threadIdx.x; k < n; k += blockDim.x) vv[k] = vv[k] / T(nv);
    __syncthreads();
    double lam = 0.0;
    conv = 0;
    iters = 0;
    for (int it = 0; it < max_iters; ++it) {
      iters = it + 1;
      gemv_rows(vv, nullptr);
      xsync();
      gather_rows(u);
      gemvT_partial(u);
      xsync();
      gemvT_finish(w, T(1));
      const double lam_new = sqrt(dsum([&](int k) { const double t = w[k]; return t * t; }));
      if (lam_new == 0.0) { lam = 0.0; conv = 1; break; }
      for (int k = threadIdx.x; k < n; k += blockDim.x) vv[k] = w[k] / T(lam_new);
      __syncthreads();
      if (fabs(lam_new - lam) <= tol * fmax(lam_new, 1e-300)) { lam = lam_new; conv = 1; break; }
      lam = lam_new;
    }
    return lam;
  }
};

// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) dense_solve_kernel(const __grid_constant__ DenseArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  Dense<T> E(a, smem);
  const int n = a.n;
  T* X[3] = {E.v[0], E.v[1], E.v[2]};
  T* Y = E.v[3];
  T* G = E.v[5];
  double lip, step = 0.0, lam = a.lip_cached;
  int pit = 0, pconv = 1;
  if (a.step_given > 0.0) {
    step = a.step_given;
    lip = 1.0 / a.step_given;
  } else {
    if (!(a.lip_cached >= 0.0)) lam = E.power(a.v0, a.power_max_iters, a.power_tol, pit, pconv);
    lip = 2.0 * lam + a.alpha * a.regcurv;
    step = 1.0 / lip;
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) X[0][k] = a.x0[k];
  __syncthreads();
  int ix = 0, ixp = 0, ic = 1;
  double t_mom = 1.0, lip_t = lip, theta = 0.0, gd_step = step;
  if (a.method == M_FISTA_SC) {
    const double q = fmin(a.mu / lip, 1.0);
    theta = (1.0 - sqrt(q)) / (1.0 + sqrt(q));
  }
  int status = ST_OK, fail_iter = -1, iters = a.max_iters, converged = 0;
  double gn = 0.0, h_y = 0.0;
  long long vg = 0, vals = 0, restarts = 0;
  bool done = false;
  for (int t = 0; t < a.max_iters; ++t) {
    double beta;
    if (a.method == M_AGD) {
      const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t_mom * t_mom));
      beta = (t_mom - 1.0) / t_next;
      t_mom = t_next;
    } else if (a.method == M_FISTA_SC) {
      beta = theta;
    } else {
      beta = 0.0;
      ixp = ix;
    }
    const T tb = T(beta);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const T xv = X[ix][k], xpv = X[ixp][k];
      Y[k] = xv + tb * (xv - xpv);
    }
    __syncthreads();
    h_y = E.value_grad(Y, G, true);
    ++vg;
    gn = sqrt(E.dsum([&](int k) { const double g = G[k]; return g * g; }));
    if (!isfinite(gn)) { status = ST_DIVERGED; fail_iter = t; done = true; break; }
    if (gn <= a.tol) {
      if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < n; k += blockDim.x) a.out[k] = Y[k];
      iters = t;
      converged = 1;
      done = true;
      break;
    }
    T* XC = X[ic];
    if (a.adaptive) {
      double L_try = (a.method == M_PROXGRAD) ? 1.0 / gd_step : lip_t;
      int kk = 0;
      while (true) {
        const T tL = T(L_try);
        for (int k = threadIdx.x; k < n; k += blockDim.x) XC[k] = Y[k] - G[k] / tL;
        __syncthreads();
        const double val = E.value_grad(XC, nullptr, false);
        ++vals;
        if (val <= h_y - 0.5 * gn * gn / L_try + 1e-15 * fabs(h_y)) break;
        L_try *= 2.0;
        if (++kk >= 60) { status = ST_BT_FAIL; fail_iter = t; break; }
      }
      if (status != ST_OK) { done = true; break; }
      const double bstep = 1.0 / L_try;
      if (a.method == M_PROXGRAD) gd_step = bstep;
      else lip_t = fmax(1.0 / bstep * 0.9, lip * 1e-8);
    } else if (a.method == M_PROXGRAD) {
      const T ts = T(gd_step);
      for (int k = threadIdx.x; k < n; k += blockDim.x) XC[k] = X[ix][k] - ts * G[k];
      __syncthreads();
    } else {
      const T tL = T(lip_t);
      for (int k = threadIdx.x; k < n; k += blockDim.x) XC[k] = Y[k] - G[k] / tL;
      __syncthreads();
    }
    const T* XO = X[ix];
    const double dot = E.dsum([&](int k) { return (double)G[k] * (double)(XC[k] - XO[k]); });
    ixp = ix;
    ix = ic;
    if (a.method == M_AGD && dot > 0.0) {
      t_mom = 1.0;
      ixp = ix;
      ++restarts;
    }
    for (int b = 0; b < 3; ++b)
      if (b != ix && b != ixp) { ic = b; break; }
  }
  if (!done) {
    E.value_grad(X[ix], G, true);
    gn = sqrt(E.dsum([&](int k) { const double g = G[k]; return g * g; }));
    if (blockIdx.x == 0)
      for (int k = threadIdx.x; k < n; k += blockDim.x) a.out[k] = X[ix][k];
    iters = a.max_iters;
    converged = gn <= a.tol;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    SolveOut* r = a.sres;
    r->lam = lam; r->lip = lip; r->grad_norm = gn; r->value = h_y; r->iters = iters; r->converged = converged;
    r->status = status; r->fail_iter = fail_iter; r->power_iters = pit; r->power_converged = pconv;
    r->vg_evals = vg; r->value_evals = vals; r->restarts = restarts;
  }
}

// ---------------------------------------------------------------------------
template <typename T>
__device__ void dense_hess_diag(Dense<T>& E, const T* xt, T* d) {
  const int n = E.n;
  const DenseArgs<T>& a = E.a;
  if (a.reg_only) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) d[k] = T(0);
    __syncthreads();
  } else {
    E.gram_partial();
    E.xsync();
    E.gemvT_finish(d, T(2));   // 2.0 * gram_diag
  }
  if (a.alpha != 0.0) {
    const T two_l2 = T(2.0 * a.l2), l1 = T(a.l1), al = T(a.alpha);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      T hd = two_l2;
      if (a.l1 > 0) hd = hd + l1 * E.rho_curv(xt[k]);
      d[k] = d[k] + al * hd;
    }
    __syncthreads();
  }
  if (a.nofloor) return;
  double mx = -INFINITY;
  for (int k = threadIdx.x; k < n; k += blockDim.x) mx = fmax(mx, (double)d[k]);
  mx = block_max(mx, E.red);
  const T fl = T(1e-12 * mx + 1e-300);
  for (int k = threadIdx.x; k < n; k += blockDim.x) d[k] = d[k] > fl ? d[k] : fl;
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(256) dense_cg_kernel(const __grid_constant__ DenseArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  Dense<T> E(a, smem);
  const int n = a.n;
  T* XT = E.v[0]; T* Q = E.v[1]; T* R = E.v[2]; T* S = E.v[3]; T* P = E.v[5]; T* HP = E.v[6];
  T* DI = E.v[7]; T* WC = E.v[8];
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    XT[k] = a.xt[k];
    WC[k] = a.l1 > 0 ? T(a.l1) * E.rho_curv(a.xt[k]) : T(0);
  }
  __syncthreads();
  if (a.diag_in) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) DI[k] = T(1) / a.diag_in[k];
  } else {
    dense_hess_diag(E, XT, DI);
    for (int k = threadIdx.x; k < n; k += blockDim.x) DI[k] = T(1) / DI[k];
  }
  __syncthreads();
  int hv = 0, status = ST_OK;
  double curv = 0.0;
  if (a.warm) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) Q[k] = a.Q[k];
    __syncthreads();
    E.hess_vec(Q, HP, WC);
    ++hv;
    for (int k = threadIdx.x; k < n; k += blockDim.x) R[k] = a.rhs[k] - HP[k];
  } else {
    for (int k = threadIdx.x; k < n; k += blockDim.x) { Q[k] = T(0); R[k] = a.rhs[k]; }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) { S[k] = DI[k] * R[k]; P[k] = S[k]; }
  __syncthreads();
  double rs = E.dsum([&](int k) { return (double)R[k] * (double)S[k]; });
  int iters;
  for (iters = 1; iters <= a.max_iters; ++iters) {
    const double rr = E.dsum([&](int k) { const double t = R[k]; return t * t; });
    if (sqrt(rr) <= a.tol) { iters -= 1; break; }
    E.hess_vec(P, HP, WC);
    ++hv;
    curv = E.dsum([&](int k) { return (double)P[k] * (double)HP[k]; });
    if (curv <= 0.0) { status = ST_NEGCURV; break; }
    const T al = T(rs / curv);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      Q[k] = Q[k] + al * P[k];
      R[k] = R[k] - al * HP[k];
      S[k] = DI[k] * R[k];
    }
    __syncthreads();
    const double rs_new = E.dsum([&](int k) { return (double)R[k] * (double)S[k]; });
    const T be = T(rs_new / rs);
    for (int k = threadIdx.x; k < n; k += blockDim.x) P[k] = S[k] + be * P[k];
    __syncthreads();
    rs = rs_new;
  }
  if (iters > a.max_iters) iters = a.max_iters;
  double res = 0.0;
  int conv = 0;
  if (status == ST_OK) {
    E.hess_vec(Q, HP, WC);
    ++hv;
    res = sqrt(E.dsum([&](int k) { const double t = (double)(HP[k] - a.rhs[k]); return t * t; }));
    conv = res <= a.tol;
  }
  if (blockIdx.x == 0) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) a.Q[k] = Q[k];
    if (threadIdx.x == 0) {
      CGOut* r = a.cres;
      r->residual = res; r->curv = curv; r->rs = rs; r->iters = iters; r->converged = conv; r->status = status;
      r->hv = hv;
    }
  }
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) dense_misc_kernel(const __grid_constant__ DenseArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  Dense<T> E(a, smem);
  const int n = a.n;
  T* U = E.v[0]; T* V = E.v[1]; T* W = E.v[2]; T* Z = E.v[3];
  const bool lead = blockIdx.x == 0;
  auto load = [&](T* dst, const T* src) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = src[k];
    __syncthreads();
  };
  auto store = [&](T* dst, const T* src) {
    if (lead)
      for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = src[k];
  };
  switch (a.mode) {
    case DM_APPLY:
      load(U, a.in0);
      E.gemv_rows(U, nullptr);
      E.xsync();
      E.gather_rows(V);
      store(a.out0, V);
      break;
    case DM_ADJOINT:
      load(U, a.in0);
      E.gemvT_partial(U);
      E.xsync();
      E.gemvT_finish(V, T(1));
      store(a.out0, V);
      break;
    case DM_GRAM:
      E.gram_partial();
      E.xsync();
      E.gemvT_finish(V, T(1));
      store(a.out0, V);
      break;
    case DM_VALUE: {
      load(U, a.in0);
      const double v = E.value_grad(U, nullptr, false);
      if (lead && threadIdx.x == 0) a.scal[0] = v;
      break;
    }
    case DM_VG:
    case DM_GRAD: {
      load(U, a.in0);
      const double v = E.value_grad(U, V, true);
      store(a.out0, V);
      if (lead && threadIdx.x == 0) a.scal[0] = v;
      break;
    }
    case DM_HV: {
      load(U, a.in0);   // x
      load(V, a.in1);   // v
      for (int k = threadIdx.x; k < n; k += blockDim.x) Z[k] = a.l1 > 0 ? T(a.l1) * E.rho_curv(U[k]) : T(0);
      __syncthreads();
      E.hess_vec(V, W, Z);
      store(a.out0, W);
      break;
    }
    case DM_HDIAG:
      load(U, a.in0);
      dense_hess_diag(E, U, W);
      store(a.out0, W);
      break;
    case DM_UPPER: {
      load(U, a.in0);
      E.gemv_rows(U, a.ydat);
      E.xsync();
      E.gather_rows(V);
      const double fit = E.npsum([&](int64_t k) { const T t = V[k]; return (double)(t * t); });
      E.gemvT_partial(V);
      E.xsync();
      E.gemvT_finish(W, T(2));
      const double gn = sqrt(E.dsum([&](int k) { const double t = W[k]; return t * t; }));
      if (a.out0) store(a.out0, W);
      if (lead && threadIdx.x == 0) { a.scal[0] = fit; a.scal[1] = gn; }
      break;
    }
    case DM_POWER: {
      int it = 0, cv = 0;
      const double lam = E.power(a.v0, a.power_max_iters, a.power_tol, it, cv);
      if (lead && threadIdx.x == 0) { a.scal[0] = lam; a.scal[1] = cv; a.scal[2] = it; }
      break;
    }
    case DM_MIXED: {
      // 2 [(B x~ - y) q^T + (B q) x~^T]   (hypergradient.py:92-104, dense branch)
      load(U, a.in0);   // x~
      load(V, a.in1);   // q
      E.gemv_rows(U, a.ydat);
      E.xsync();
      E.gather_rows(W);  // residual
      E.gemv_rows(V, nullptr);
      E.xsync();
      E.gather_rows(Z);  // B q
      for (int i = E.r0; i < E.r1; ++i)
        for (int j = threadIdx.x; j < n; j += blockDim.x)
          a.out0[(int64_t)i * n + j] = T(2) * (Z[i] * U[j] + W[i] * V[j]);
      break;
    }
    case DM_DOT: {
      load(U, a.in0);
      load(V, a.in1);
      const double d = E.dsum([&](int k) { return (double)U[k] * (double)V[k]; });
      if (lead && threadIdx.x == 0) a.scal[0] = d;
      break;
    }
    case DM_PROX: {
      // prox_grad_iterations (baselines.py:46-55): piters steps of
      //   x = prox_l1(x - step * (2 B^T (B x - y) + 2 alpha l2 x), step alpha l1)
      // with the reference's expression order; prox_l1 = sign(u) * max(|u| - thr, 0)
      // (regularizers.py:22-27, np.sign / np.maximum semantics incl. NaN)
      T* x = U;
      load(x, a.in0);
      const T step = T(a.pstep), thr = T(a.pthr), c2al2 = T((2.0 * a.alpha) * a.l2);
      for (int it = 0; it < a.piters; ++it) {
        E.gemv_rows(x, a.ydat);
        E.xsync();
        T* r = E.v[4];
        E.gather_rows(r);
        E.gemvT_partial(r);
        E.xsync();
        E.gemvT_finish(V, T(2));
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
          const T g = V[k] + c2al2 * x[k];
          const T u = x[k] - step * g;
          const T m = fabs(u) - thr;
          const T mx = (m > T(0) || m != m) ? m : T(0);
          const T sg = u > T(0) ? T(1) : (u < T(0) ? T(-1) : (u == T(0) ? T(0) : u));
          x[k] = sg * mx;
        }
        __syncthreads();
      }
      store(a.out0, x);
      break;
    }
    case DM_KGC: {
      // np.outer(v, x)  (operators.py:208-209)
      load(U, a.in0);
      load(V, a.in1);
      for (int i = E.r0; i < E.r1; ++i)
        for (int j = threadIdx.x; j < n; j += blockDim.x) a.out0[(int64_t)i * n + j] = V[i] * U[j];
      break;
    }
    default:
      break;
  }
}

DenseKernelSet dense_kernels_f64() {
  return {(const void*)dense_solve_kernel<double>, (const void*)dense_cg_kernel<double>,
          (const void*)dense_misc_kernel<double>};
}
DenseKernelSet dense_kernels_f32() {
  return {(const void*)dense_solve_kernel<float>, (const void*)dense_cg_kernel<float>,
          (const void*)dense_misc_kernel<float>};
}

// ===========================================================================
// host side
int dense_fail(int code, const char* m);  // adp_host.cu

struct DenseState {
  int cluster;       // the grid is one thread-block cluster (distributed-shared-memory exchanges)
  int plen;          // words of the top sum program
  int G, rows_per, b_smem;
  size_t smem;
  void* d_gvec;      // large n: replicated vectors in global memory
  int64_t vpitch;
  SumHost sn;
  int* d_progs;
  int64_t* d_leaf;
  void* d_rowbuf;
  double* d_part;
  KernelInfo ks, kc, km;
};

#define DCK(x)                                                                              \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) return dense_fail(ADP_ERR_CUDA, cudaGetErrorString(e_));          \
  } while (0)

int dense_plan_init(PlanImpl& P) {
  const int n = P.d.W;
  int dev = 0;
  DCK(cudaGetDevice(&dev));
  DCK(cudaDeviceGetAttribute(&P.sm_count, cudaDevAttrMultiProcessorCount, dev));
  int optin = 0;
  DCK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  DenseState* S = new DenseState();
  P.ws[0] = S;
  ProgPool pool;
  build_sum(S->sn, n, true, pool, false);   // in-CTA program evaluation (signal-length vectors)
  if (S->sn.nSub != 1) return dense_fail(ADP_ERR_UNSUPPORTED, "dense1d signal too long");
  const size_t es = (size_t)P.esize;
  const int* tw = pool.words.data() + S->sn.top_prog;
  S->plen = 3 + (tw[2] + 1) + 2 * tw[1];   // nL, nI, nLev, level bounds, left / right children
  size_t base = 64 * sizeof(double) + 2 * (size_t)(2 * S->sn.nLeaves + 2) * sizeof(double);
  base += (size_t)(S->sn.nLeaves + 1) * sizeof(int64_t) + (size_t)S->plen * sizeof(int);
  base = (base + 15) & ~size_t(15);
  const size_t vecs = (size_t)kDenseVecs * (((size_t)n * es + 15) & ~size_t(15));
  const bool gvec = base + vecs > (size_t)optin;   // large n: vectors in global memory instead of smem
  if (!gvec) base += vecs;
  int G = std::max(1, std::min((n + 15) / 16, P.sm_count));
  int rows_per = (n + G - 1) / G;
  G = (n + rows_per - 1) / rows_per;
  S->d_gvec = nullptr;
  S->vpitch = (int64_t)((n + 1) & ~1);
  if (gvec) DCK(cudaMalloc(&S->d_gvec, (size_t)G * kDenseVecs * S->vpitch * es));
  const size_t bslice = (size_t)rows_per * n * es;
  S->b_smem = (base + bslice <= (size_t)optin) ? 1 : 0;
  S->smem = base + (S->b_smem ? bslice : 0);
  S->G = G;
  S->rows_per = rows_per;
  // one thread-block cluster (<= 16 CTAs; > 8 is the non-portable size) when the vectors and the B slice are in
  // shared memory and the exchange buffers fit next to them; ADP_DENSE_CLUSTER=0: the cooperative grid
  S->cluster = 0;
  {
    const char* ev = getenv("ADP_DENSE_CLUSTER");
    size_t cs = (S->smem + 15) & ~size_t(15);
    cs += 2 * (((size_t)n * es + 15) & ~size_t(15)) + 2 * (size_t)G * n * sizeof(double);
    if (!(ev && atoi(ev) == 0) && G >= 2 && G <= 16 && !gvec && S->b_smem && cs <= (size_t)optin) {
      S->cluster = 1;
      S->smem = cs;
    }
  }
  DCK(cudaMalloc(&S->d_progs, pool.words.size() * sizeof(int)));
  DCK(cudaMemcpy(S->d_progs, pool.words.data(), pool.words.size() * sizeof(int), cudaMemcpyHostToDevice));
  DCK(cudaMalloc(&S->d_leaf, S->sn.leaf_start.size() * sizeof(int64_t)));
  DCK(cudaMemcpy(S->d_leaf, S->sn.leaf_start.data(), S->sn.leaf_start.size() * sizeof(int64_t),
                 cudaMemcpyHostToDevice));
  DCK(cudaMalloc(&S->d_rowbuf, 2 * (size_t)n * es));
  DCK(cudaMalloc(&S->d_part, (size_t)G * n * sizeof(double)));
  DCK(cudaMalloc(&P.dmem, 4096));
  P.dbytes = 4096;
  P.d_bar = (unsigned int*)P.dmem;
  P.d_sres = (SolveOut*)((char*)P.dmem + 256);
  P.d_cres = (CGOut*)((char*)P.dmem + 1024);
  P.d_scal = (double*)((char*)P.dmem + 2048);
  DCK(cudaMallocHost(&P.h_sres, sizeof(SolveOut)));
  DCK(cudaMallocHost(&P.h_cres, sizeof(CGOut)));
  DCK(cudaMallocHost(&P.h_scal, 64 * sizeof(double)));
  DenseKernelSet k = P.d.dtype == ADP_DTYPE_F32 ? dense_kernels_f32() : dense_kernels_f64();
  const void* fns[3] = {k.solve, k.cg, k.misc};
  KernelInfo* kis[3] = {&S->ks, &S->kc, &S->km};
  for (int i = 0; i < 3; ++i) DCK(cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  for (int i = 0; i < 3 && S->cluster; ++i) {   // can one cluster of G CTAs be scheduled?  else the cooperative grid
    if (G > 8 && cudaFuncSetAttribute(fns[i], cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      (void)cudaGetLastError();
      S->cluster = 0;
      break;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = S->smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, fns[i], &cfg) != cudaSuccess || nc < 1) {
      (void)cudaGetLastError();
      S->cluster = 0;
    }
  }
  for (int i = 0; i < 3; ++i) {
    int nb = 0;
    DCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fns[i], 256, S->smem));
    if (nb * P.sm_count < G) return dense_fail(ADP_ERR_UNSUPPORTED, "dense grid not co-resident");
    kis[i]->fn = fns[i];
    kis[i]->grid = G;
  }
  P.dense_grid = G;
  P.dense_smem = S->smem;
  P.ws[0] = S;
  return ADP_OK;
}

void dense_plan_free(PlanImpl& P) {
  DenseState* S = (DenseState*)P.ws[0];
  if (!S) return;
  cudaFree(S->d_progs);
  cudaFree(S->d_leaf);
  cudaFree(S->d_rowbuf);
  cudaFree(S->d_part);
  if (S->d_gvec) cudaFree(S->d_gvec);
  delete S;
  P.ws[0] = nullptr;
}

template <typename T>
static DenseArgs<T> dense_base(PlanImpl& P) {
  DenseState* S = (DenseState*)P.ws[0];
  DenseArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.n = P.d.W;
  a.G = S->G;
  a.rows_per = S->rows_per;
  a.b_smem = S->b_smem;
  a.rowbuf = (T*)S->d_rowbuf;
  a.part = S->d_part;
  a.gvec = (T*)S->d_gvec;
  a.vpitch = S->vpitch;
  a.cluster = S->cluster;
  a.plen = S->plen;
  a.s_n.nLeaves = S->sn.nLeaves;
  a.s_n.nSub = 1;
  a.s_n.sub_own0 = 0;
  a.s_n.sub_own1 = 1;
  a.s_n.sub_own2 = a.s_n.sub_own3 = 0;
  a.s_n.top_prog = S->sn.top_prog;
  a.s_n.leaf_start = S->d_leaf;
  a.s_n.progs = S->d_progs;
  a.bar = P.d_bar;
  a.sres = P.d_sres;
  a.cres = P.d_cres;
  a.scal = P.d_scal;
  return a;
}

template <typename T>
static void dense_set_lower(DenseArgs<T>& a, const adp_lower* lp) {
  if (!lp) return;
  a.B = (const T*)lp->kernel;
  a.ydat = (const T*)lp->y;
  a.alpha = lp->alpha;
  a.l1 = lp->l1;
  a.l2 = lp->l2;
  a.nu = lp->nu;
  a.reg = lp->reg;
  double c = 2.0 * lp->l2;               // SmoothedElasticNet.curvature (regularizers.py:92-99)
  if (lp->l1 > 0) c += lp->l1 / lp->nu;
  a.regcurv = c;
}

template <typename T>
static int dense_launch(PlanImpl& P, KernelInfo& k, DenseArgs<T>& a, cudaStream_t st) {
  DenseState* S = (DenseState*)P.ws[0];
  void* args[] = {&a};
  if (S->cluster) {   // the whole grid is one cluster: no grid barrier, no counter
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(k.grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = S->smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = k.grid;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    DCK(cudaLaunchKernelExC(&cfg, k.fn, args));
    return ADP_OK;
  }
  DCK(cudaMemsetAsync(P.d_bar, 0, sizeof(unsigned int), st));
  DCK(cudaLaunchCooperativeKernel(k.fn, dim3(k.grid), dim3(256), args, S->smem, st));
  return ADP_OK;
}

template <typename T>
static int dense_call_t(PlanImpl& P, int op, const void* kernel, const adp_lower* lp, const void* a0, const void* a1,
                        void* o0, void* o1, const void* ydat, double* scal, cudaStream_t st) {
  DenseState* S = (DenseState*)P.ws[0];
  DenseArgs<T> a = dense_base<T>(P);
  dense_set_lower(a, lp);
  if (kernel) a.B = (const T*)kernel;
  if (ydat) a.ydat = (const T*)ydat;
  a.in0 = (const T*)a0;
  a.in1 = (const T*)a1;
  a.out0 = (T*)o0;
  a.out1 = (T*)o1;
  int nscal = 0;
  if (op >= 100) {
    op -= 100;
    a.reg_only = 1;
    a.nofloor = 1;
  }
  switch (op) {
    case 0: a.mode = DM_APPLY; break;
    case 1: a.mode = DM_ADJOINT; break;
    case 2: a.mode = DM_GRAM; break;
    case 3: a.mode = DM_VALUE; nscal = 1; break;
    case 4: a.mode = DM_VG; nscal = 1; break;
    case 5: a.mode = DM_GRAD; break;
    case 6: a.mode = DM_HV; break;
    case 7: a.mode = DM_HDIAG; break;
    case 8: a.mode = DM_UPPER; nscal = 2; break;
    case 9:
      a.mode = DM_POWER;
      nscal = 3;
      a.v0 = (const T*)a0;
      a.power_max_iters = (int)lp->alpha;
      a.power_tol = lp->l1;
      a.alpha = 0.0;
      a.l1 = 0.0;
      break;
    case 10: a.mode = DM_MIXED; break;
    case 11: a.mode = DM_DOT; nscal = 1; break;
    case 12: a.mode = DM_KGC; break;
    default: return dense_fail(ADP_ERR_ARG, "bad dense op");
  }
  if (int e = dense_launch(P, S->km, a, st)) return e;
  if (nscal) {
    DCK(cudaMemcpyAsync(P.h_scal, P.d_scal, nscal * sizeof(double), cudaMemcpyDeviceToHost, st));
    DCK(cudaStreamSynchronize(st));
    for (int i = 0; i < nscal; ++i) scal[i] = P.h_scal[i];
  }
  return ADP_OK;
}

int dense_call(PlanImpl& P, int op, const void* kernel, const adp_lower* lp, const void* a0, const void* a1, void* o0,
               void* o1, const void* ydat, double* scal, cudaStream_t st) {
  if (lp && op % 100 != 9 && lp->reg != ADP_REG_ELASTIC)
    return dense_fail(ADP_ERR_UNSUPPORTED, "dense1d path supports SmoothedElasticNet");
  return P.d.dtype == ADP_DTYPE_F32 ? dense_call_t<float>(P, op, kernel, lp, a0, a1, o0, o1, ydat, scal, st)
                                    : dense_call_t<double>(P, op, kernel, lp, a0, a1, o0, o1, ydat, scal, st);
}

template <typename T>
static int dense_solve_t(PlanImpl& P, const adp_lower* lp, const void* x0, void* x_out, const adp_solve_args* sa,
                         adp_solve_result* res, cudaStream_t st) {
  DenseState* S = (DenseState*)P.ws[0];
  DenseArgs<T> a = dense_base<T>(P);
  dense_set_lower(a, lp);
  a.method = sa->method;
  a.adaptive = sa->adaptive;
  a.max_iters = sa->max_iters;
  a.mu = sa->mu;
  a.tol = sa->eps * sa->mu;
  a.step_given = sa->step_size > 0 ? sa->step_size : 0.0;
  a.lip_cached = sa->norm_sq;
  a.power_max_iters = sa->norm_max_iters;
  a.power_tol = sa->norm_tol;
  a.v0 = (const T*)sa->v0;
  a.x0 = (const T*)x0;
  a.out = (T*)x_out;
  if (int e = dense_launch(P, S->ks, a, st)) return e;
  DCK(cudaMemcpyAsync(P.h_sres, P.d_sres, sizeof(SolveOut), cudaMemcpyDeviceToHost, st));
  DCK(cudaStreamSynchronize(st));
  const SolveOut& o = *P.h_sres;
  res->norm_sq = o.lam; res->lip = o.lip; res->grad_norm = o.grad_norm; res->value = o.value;
  res->iters = o.iters; res->converged = o.converged; res->status = o.status; res->fail_iter = o.fail_iter;
  res->power_iters = o.power_iters; res->power_converged = o.power_converged;
  res->vg_evals = o.vg_evals; res->value_evals = o.value_evals; res->restarts = o.restarts;
  return ADP_OK;
}

int dense_solve(PlanImpl& P, const adp_lower* lp, const void* x0, void* x_out, const adp_solve_args* sa,
                adp_solve_result* res, cudaStream_t st) {
  if (lp->reg != ADP_REG_ELASTIC) return dense_fail(ADP_ERR_UNSUPPORTED, "dense1d path supports SmoothedElasticNet");
  return P.d.dtype == ADP_DTYPE_F32 ? dense_solve_t<float>(P, lp, x0, x_out, sa, res, st)
                                    : dense_solve_t<double>(P, lp, x0, x_out, sa, res, st);
}

template <typename T>
static int dense_cg_t(PlanImpl& P, const adp_lower* lp, const void* xt, const void* rhs, void* q, int warm,
                      const void* precond, double tol, int max_iters, adp_cg_result* res, cudaStream_t st) {
  DenseState* S = (DenseState*)P.ws[0];
  DenseArgs<T> a = dense_base<T>(P);
  dense_set_lower(a, lp);
  a.xt = (const T*)xt;
  a.rhs = (const T*)rhs;
  a.Q = (T*)q;
  a.warm = warm;
  a.diag_in = (const T*)precond;
  a.tol = tol;
  a.max_iters = max_iters;
  if (int e = dense_launch(P, S->kc, a, st)) return e;
  DCK(cudaMemcpyAsync(P.h_cres, P.d_cres, sizeof(CGOut), cudaMemcpyDeviceToHost, st));
  DCK(cudaStreamSynchronize(st));
  const CGOut& o = *P.h_cres;
  res->residual = o.residual; res->curv = o.curv; res->iters = o.iters; res->converged = o.converged;
  res->status = o.status; res->hv = o.hv;
  return ADP_OK;
}

template <typename T>
static int dense_prox_t(PlanImpl& P, const adp_lower* lp, const void* x0, void* x_out, int n_iters, double step,
                        cudaStream_t st) {
  DenseState* S = (DenseState*)P.ws[0];
  DenseArgs<T> a = dense_base<T>(P);
  dense_set_lower(a, lp);
  a.mode = DM_PROX;
  a.in0 = (const T*)x0;
  a.out0 = (T*)x_out;
  a.piters = n_iters;
  a.pstep = step;
  a.pthr = (step * lp->alpha) * lp->l1;    // threshold = step * alpha * l1
  return dense_launch(P, S->km, a, st);
}

int dense_prox(PlanImpl& P, const adp_lower* lp, const void* x0, void* x_out, int n_iters, double step,
               cudaStream_t st) {
  if (lp->reg != ADP_REG_ELASTIC) return dense_fail(ADP_ERR_UNSUPPORTED, "prox-gradient: SmoothedElasticNet");
  return P.d.dtype == ADP_DTYPE_F32 ? dense_prox_t<float>(P, lp, x0, x_out, n_iters, step, st)
                                    : dense_prox_t<double>(P, lp, x0, x_out, n_iters, step, st);
}

int dense_cg(PlanImpl& P, const adp_lower* lp, const void* xt, const void* rhs, void* q, int warm, const void* precond,
             double tol, int max_iters, adp_cg_result* res, cudaStream_t st) {
  if (lp->reg != ADP_REG_ELASTIC) return dense_fail(ADP_ERR_UNSUPPORTED, "dense1d path supports SmoothedElasticNet");
  return P.d.dtype == ADP_DTYPE_F32 ? dense_cg_t<float>(P, lp, xt, rhs, q, warm, precond, tol, max_iters, res, st)
                                    : dense_cg_t<double>(P, lp, xt, rhs, q, warm, precond, tol, max_iters, res, st);
}

}  // namespace adp
