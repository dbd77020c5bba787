// Cooperative persistent kernels of the depthwise 2-D engine.
#pragma once
#include "conv2d_engine.cuh"

namespace adp {

template <typename T, bool FAST, int RW, int KS = 0, bool TMA = false>
struct ConvOps : Conv<T, FAST, RW, KS, TMA> {
  using Base = Conv<T, FAST, RW, KS, TMA>;
  using Base::a;
  GridBarrier gb;
  SumDev* ssm;   // shared-memory copies of a.s_fit .. a.s_tv2 (read at every decision point)
  unsigned long long* mbar = nullptr;   // TMA: two transaction barriers (one per plane region)

  __device__ explicit ConvOps(const ConvArgs<T>& a_) : Base(a_) {
    gb.counter = a_.bar;
    gb.nblocks = gridDim.x;
    gb.target = 0;
    if constexpr (TMA) {
      __shared__ __align__(8) unsigned long long sh_mbar[2];
      mbar = sh_mbar;
      if (threadIdx.x == 0) {
        for (int k = 0; k < 2; ++k)
          asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(Base::smem_u32(sh_mbar + k)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
    }
    __shared__ SumDev sh_sums[kNumSums];
    static_assert(offsetof(ConvArgs<T>, s_tv2) - offsetof(ConvArgs<T>, s_fit) == (kNumSums - 1) * sizeof(SumDev),
                  "sum descriptors must be contiguous");
    if (threadIdx.x < kNumSums) sh_sums[threadIdx.x] = (&a_.s_fit)[threadIdx.x];
    ssm = sh_sums;
    __syncthreads();
  }
  static constexpr int kNumSums = 9;

  template <int K>
  __device__ void reduce(const SumDev* const (&l)[K], double* out) {
    const SumDev* ss[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const ptrdiff_t j = l[i] - &a.s_fit;
      ss[i] = (j >= 0 && j < kNumSums) ? ssm + j : l[i];
    }
    reduce_k<K, (KS > 0)>(ss, out, this->sv(), gb, a.trace ? a.trace + 1088 : nullptr);
  }
  // phase 1 only (subtrees of two-level sums), for the row-slab steps
  template <int K>
  __device__ void phase1(const SumDev* const (&l)[K]) {
    int off = 0;
#pragma unroll 1
    for (int i = 0; i < K; ++i) {
      const ptrdiff_t j = l[i] - &a.s_fit;
      const SumDev& s = (j >= 0 && j < kNumSums) ? ssm[j] : *l[i];
      if (s.nSub > 1) {
        sum_phase1(s, this->sv(), off);
        off += s.nSub;
      }
    }
  }
  __device__ double reduce1(const SumDev& s) {
    double o;
    reduce({&s}, &o);
    return o;
  }
  // NumPy-pairwise leaves of an element sum over the OWNED rows of a row
  // slab (regular, row-aligned layout), at their GLOBAL leaf indices; the
  // same per-leaf arithmetic as np_leaves_regular (unsplit plans: all rows).
  template <class Src>
  __device__ void slab_leaves(const SumDev& s, const Src& src) {
    const int L = s.leaf_len;
    const int64_t rowL = (int64_t)a.g.W * a.g.C / L;
    const int64_t l0 = (int64_t)(a.g.row0 + a.g.own0) * rowL;
    const int64_t l1 = (int64_t)(a.g.row0 + min(a.g.own1, a.g.H)) * rowL;
    const int64_t ebase = (int64_t)a.g.row0 * a.g.W * a.g.C;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t total = (l1 - l0) * 8;
    const int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t g0 = 0; g0 < total; g0 += nthreads) {
      const int64_t g = g0 + base;
      const bool act = g < total;
      const int64_t leaf = l0 + (g >> 3);
      const int k = (int)(g & 7);
      double acc = 0.0;
      if (act) {
        const int64_t e0 = leaf * L + k - ebase;
        double v[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = (8 * m < L) ? src(e0 + 8 * m) : 0.0;
        acc = v[0];
#pragma unroll
        for (int m = 1; m < 16; ++m)
          if (8 * m < L) acc = acc + v[m];
      }
      acc = acc + __shfl_xor_sync(kFull, acc, 1);
      acc = acc + __shfl_xor_sync(kFull, acc, 2);
      acc = acc + __shfl_xor_sync(kFull, acc, 4);
      if (act && k == 0) s.leaf_vals[leaf] = acc;
    }
  }
  // element-sum leaves for the non-fused layout (after a barrier)
  __device__ void leaves_if_unfused(const SumDev& s, const T* terms, bool square) {
    if (a.g.fused) return;
    if (square) np_leaves(s, SqOf<T>{terms});
    else np_leaves(s, Plain<T>{terms});
  }

  // Power iteration on B^T B (op_norm_sq, operators.py:137-173).  Uses R
  // (B v) and G (w) as scratch.  Returns lambda; sets iters / converged.
  __device__ double power(int max_iters, double tol, int& iters, int& conv) {
    this->foreach_pixel_sum([&](int64_t i, int, int, int) {
      const double v = (double)a.v0[i];
      return v * v;
    }, a.s_t0);
    gb.sync();
    const double nv = sqrt(reduce1(a.s_t0));      // v /= ||v||  (operators.py:150)
    double lam = 0.0;
    conv = 0;
    iters = 0;
    const T* src = a.v0;
    double scale = nv;
    for (int it = 0; it < max_iters; ++it) {
      iters = it + 1;
      this->stage_corr(SrcScaled<T>{src, T(scale)}, false, a.R, nullptr, T(1), nullptr);
      gb.sync();
      this->stage_corr(SrcLin<T>{a.R}, true, a.G, nullptr, T(1), &a.s_t0);
      gb.sync();
      const double lam_new = sqrt(reduce1(a.s_t0));
      if (lam_new == 0.0) { lam = 0.0; conv = 1; break; }
      src = a.G;
      scale = lam_new;
      if (fabs(lam_new - lam) <= tol * fmax(lam_new, 1e-300)) { lam = lam_new; conv = 1; break; }
      lam = lam_new;
    }
    return lam;
  }

  // value + gradient at a source point: stage A, barrier, stage B (+ leaves
  // when unfused).  Caller syncs afterwards.
  template <class Src>
  __device__ void value_grad(const Src& src, bool tv, T* Gout, const T* Xs = nullptr, const T* XPs = nullptr,
                             T beta = T(0), T L = T(1), T* Xc = nullptr) {
    this->stageA(src, a.R, a.ydat, tv, a.TV2, a.TVG, &a.s_fit, &a.s_tv);
    gb.sync();
    this->stageB(a.R, tv, a.TVG, Gout, &a.s_t0, Xs, XPs, beta, L, Xc);
    leaves_if_unfused(a.s_fit, a.R, true);
    if (tv) leaves_if_unfused(a.s_tv, a.TV2, false);
  }
  // value at a candidate (lower_value form) + restart-dot partial; caller syncs.
  template <class Src>
  __device__ void value_cand(const Src& src, bool tv, T* Xout, const T* Gin, const T* Xold, const SumDev* sdot) {
    this->stageC(src, a.RC, tv, a.TV2C, Xout, Gin, Xold, sdot, &a.s_fitc, &a.s_tvc);
    if (!a.g.fused) {
      gb.sync();
      np_leaves(a.s_fitc, SqOf<T>{a.RC});
      if (tv) np_leaves(a.s_tvc, Plain<T>{a.TV2C});
    }
  }
};

#define ADP_TRACE(it, k)                                                               \
  do {                                                                                 \
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && (it) < 64) a.trace[(it) * 16 + (k)] = gtimer(); \
  } while (0)

// ---------------------------------------------------------------------------
// solve_lower (lower_solvers.py:104-213) as one persistent kernel.
// The compile-time-stencil instance (KS > 0: the c2 kernel, <= 256 threads,
// see kSolveKSThreads) is bounded at 256 threads so it gets the full
// 255-register file instead of spilling at the 512-thread cap of 128.
// MAXT < 512: instances for CTAs of at most MAXT threads (c3-c5 run 384),
// more registers per thread for the same reason.
template <typename T, bool FAST, int RW, int KS = 0, int MAXT = 512, bool TMA = false>
__global__ void __launch_bounds__(KS > 0 ? kSolveKSThreads : MAXT, 1) conv_solve_kernel(const __grid_constant__ ConvArgs<T> a) {
  ConvOps<T, FAST, RW, KS, TMA> E(a);
  unsigned tph[2] = {0u, 0u};   // TMA: mbarrier phases
  if constexpr (TMA) {
    // the five tile-box descriptors into the descriptor cache before the first box needs them
    if (threadIdx.x < 5) asm volatile("prefetch.tensormap [%0];" ::"l"(&a.tm[threadIdx.x]) : "memory");
  }
  const ConvGeom& g = a.g;
  E.load_weights(a.kern);
  const bool tv = (a.alpha != 0.0);
  const double twoN = 2.0 * (double)g.N;

  // ---- step size / Lipschitz constant (solve_lower lines 135-140, L_of_b 90-96)
  double lip, step = 0.0;
  int pit = 0, pconv = 1;
  double lam = a.lip_cached;
  if (a.step_given > 0.0) {
    step = a.step_given;
    lip = 1.0 / a.step_given;
  } else {
    if (!(a.lip_cached >= 0.0)) lam = E.power(a.power_max_iters, a.power_tol, pit, pconv);
    lip = 2.0 * lam + a.alpha * a.regcurv;
    step = 1.0 / lip;
  }

  // ---- x = x_prev = x0 (or an injected x_prev, t_mom, lip_t: P2 lockstep)
  E.foreach_pixel([&](int64_t i, int, int, int) {
    a.X[0][i] = a.x0[i];
    if (a.xprev0) a.X[1][i] = a.xprev0[i];
  });
  E.gb.sync();

  int ix = 0, ixp = a.xprev0 ? 1 : 0, ic = a.xprev0 ? 2 : 1;
  double t_mom = a.t_mom0 > 0.0 ? a.t_mom0 : 1.0, lip_t = a.lip_t0 > 0.0 ? a.lip_t0 : lip;
  double theta = 0.0;
  if (a.method == M_FISTA_SC) {
    const double q = fmin(a.mu / lip, 1.0);
    theta = (1.0 - sqrt(q)) / (1.0 + sqrt(q));
  }
  double gd_step = (a.method == M_PROXGRAD && a.lip_t0 > 0.0) ? 1.0 / a.lip_t0 : step;   // _gradient_descent's `step`
  int status = ST_OK, fail_iter = -1, iters = a.max_iters, converged = 0;
  double gn = 0.0, h_y = 0.0, beta = 0.0;
  long long vg = 0, vals = 0, restarts = 0;
  bool done = false;
  // fuseCA (adaptive AGD with TV): the candidate's value pass also computes
  // stage A at the NEXT extrapolation point, assuming the first candidate is
  // accepted without restart; when that holds (the common case) the next
  // iteration skips stage A and one grid barrier.  Stage-A sums alternate
  // between two sets (par).  Same arithmetic as the unfused order.
  const bool spec = a.adaptive && tv && g.fuseCA && a.method == M_AGD;
  // pipelined stages (asynchronous double-buffered tile copies; RW = 4 plans
  // with the Q scratch): stage B also writes the next extrapolation point to P[0]
  const bool pipe = KS == 0 && spec && g.o_q > 0;
  bool a_ready = false;
  int par = 0;

  for (int t = 0; t < a.max_iters; ++t) {
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
    // first candidate, computed speculatively before the convergence test
    double L_try = (a.method == M_PROXGRAD) ? 1.0 / gd_step : lip_t;
    // value and gradient at y (stages A, B); stage B also writes the own
    // pixels of the first candidate y - g / L_try (adaptive path)
    ADP_TRACE(t, 0);
    const SumDev* sfit = par ? &a.s_fit2 : &a.s_fit;
    const SumDev* stv = par ? &a.s_tv2 : &a.s_tv;
    if (a.adaptive) {
      if (!a_ready) {
        E.stageA(SrcExtrap<T>{a.X[ix], a.X[ixp], tb}, a.R, a.ydat, tv, a.TV2, a.TVG, sfit, stv);
        ADP_TRACE(t, 1);
        E.gb.sync();
      } else {
        ADP_TRACE(t, 1);
      }
      ADP_TRACE(t, 2);
      const double t_nextB = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t_mom * t_mom));   // as in the stage-CA branch
      const double betaB = (t_mom - 1.0) / t_nextB;
      if constexpr (TMA) {
        if (spec)
          E.stageB_tma(&a.tm[3], tv, a.TVG, a.G, &a.s_t0, a.X[ix], a.X[ixp], tb, T(L_try), a.X[ic], T(betaB),
                       a.P[0], E.mbar, tph[0]);
        else
          E.stageB(a.R, tv, a.TVG, a.G, &a.s_t0, a.X[ix], a.X[ixp], tb, T(L_try), a.X[ic]);
      } else {
        if (pipe)
          E.stageB_pipe(a.R, tv, a.TVG, a.G, &a.s_t0, a.X[ix], a.X[ixp], tb, T(L_try), a.X[ic], T(betaB), a.P[0]);
        else
          E.stageB(a.R, tv, a.TVG, a.G, &a.s_t0, a.X[ix], a.X[ixp], tb, T(L_try), a.X[ic]);
      }
      E.leaves_if_unfused(a.s_fit, a.R, true);
      if (tv) E.leaves_if_unfused(a.s_tv, a.TV2, false);
    } else {
      E.value_grad(SrcExtrap<T>{a.X[ix], a.X[ixp], tb}, tv, a.G);
    }
    ++vg;
    ADP_TRACE(t, 3);
    E.gb.sync();
    ADP_TRACE(t, 4);
    if (spec) {
      // next iteration's momentum if this one ends without restart
      const double t_next2 = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t_mom * t_mom));
      const double beta2 = (t_mom - 1.0) / t_next2;
      if constexpr (TMA) {
        E.stageCA_tma(&a.tm[ic], &a.tm[4], a.X[ix], a.G, tv, a.R, a.TVG, &a.s_t1, &a.s_fitc, &a.s_tvc,
                      par ? &a.s_fit : &a.s_fit2, par ? &a.s_tv : &a.s_tv2, E.mbar, tph);
      } else {
        if (pipe)
          E.stageCA_pipe(a.X[ic], a.P[0], a.X[ix], a.G, tv, a.R, a.TVG, &a.s_t1, &a.s_fitc, &a.s_tvc,
                         par ? &a.s_fit : &a.s_fit2, par ? &a.s_tv : &a.s_tv2);
        else
          E.stageCA(a.X[ic], a.X[ix], T(beta2), a.G, tv, a.R, a.TVG, &a.s_t1, &a.s_fitc, &a.s_tvc,
                    par ? &a.s_fit : &a.s_fit2, par ? &a.s_tv : &a.s_tv2);
      }
      ++vals;
    } else if (a.adaptive) {
      E.value_cand(SrcLin<T>{a.X[ic]}, tv, nullptr, a.G, a.X[ix], &a.s_t1);
      ++vals;
    } else if (a.method == M_PROXGRAD) {
      E.stageCLight(SrcStep<T>{a.X[ix], a.G, T(gd_step)}, a.X[ic], a.G, a.X[ix], &a.s_t1);
    } else {
      E.stageCLight(SrcCand<T>{a.X[ix], a.X[ixp], a.G, tb, T(lip_t)}, a.X[ic], a.G, a.X[ix], &a.s_t1);
    }
    ADP_TRACE(t, 5);
    E.gb.sync();
    ADP_TRACE(t, 6);
    // fit(y), tv(y), g.g, dot, [fit(xc), tv(xc)]
    double o[6] = {0, 0, 0, 0, 0, 0};
    if (a.adaptive && tv) E.reduce({sfit, stv, &a.s_t0, &a.s_t1, &a.s_fitc, &a.s_tvc}, o);
    else if (a.adaptive) { E.reduce({&a.s_fit, &a.s_t0, &a.s_t1, &a.s_fitc}, o + 2); o[0] = o[2]; o[2] = o[3]; o[3] = o[4]; o[4] = o[5]; o[5] = 0.0; }
    else if (tv) E.reduce({&a.s_fit, &a.s_tv, &a.s_t0, &a.s_t1}, o);
    else { E.reduce({&a.s_fit, &a.s_t0, &a.s_t1}, o + 1); o[0] = o[1]; o[1] = 0.0; }
    ADP_TRACE(t, 7);
    const double fit = o[0];
    h_y = fit;
    if (tv) h_y = fit + a.alpha * (o[1] - a.nu * twoN);
    gn = sqrt(o[2]);
    double dot = o[3];
    if (!isfinite(gn)) { status = ST_DIVERGED; fail_iter = t; done = true; break; }
    if (gn <= a.tol) {
      // converged: return y (lower_solvers.py:200-201)
      E.foreach_pixel([&](int64_t i, int, int, int) {
        const T xv = ldcg(a.X[ix] + i), xpv = ldcg(a.X[ixp] + i);
        a.out[i] = xv + tb * (xv - xpv);
      });
      iters = t;
      converged = 1;
      done = true;
      break;
    }
    int k = 0;   // backtracking retries of this iteration
    if (a.adaptive) {
      // _backtracked_step (lower_solvers.py:170-177)
      double fitc = o[4], tvc = o[5];
      while (true) {
        const double val = tv ? fitc + a.alpha * tvc : fitc + a.alpha * 0.0;
        if (val <= h_y - 0.5 * gn * gn / L_try + 1e-15 * fabs(h_y)) break;
        L_try *= 2.0;
        if (++k >= 60) { status = ST_BT_FAIL; fail_iter = t; break; }
        E.gb.sync();   // every CTA has finished reading the previous candidate sums
        E.value_cand(SrcCand<T>{a.X[ix], a.X[ixp], a.G, tb, T(L_try)}, tv, a.X[ic], a.G, a.X[ix], &a.s_t1);
        ++vals;
        E.gb.sync();
        double o3[3] = {0, 0, 0};
        if (tv) E.reduce({&a.s_fitc, &a.s_tvc, &a.s_t1}, o3);
        else { E.reduce({&a.s_fitc, &a.s_t1}, o3); o3[2] = o3[1]; o3[1] = 0.0; }
        fitc = o3[0]; tvc = o3[1]; dot = o3[2];
        ADP_TRACE(t, 8 + min(k, 7));
      }
      if (status != ST_OK) { done = true; break; }
      const double bstep = 1.0 / L_try;
      if (a.method == M_PROXGRAD) gd_step = bstep;
      else lip_t = fmax(1.0 / bstep * 0.9, lip * 1e-8);
    }
    // x_prev = x; x = candidate; restart (lower_solvers.py:202-211)
    ixp = ix;
    ix = ic;
    const bool restart = a.method == M_AGD && dot > 0.0;
    if (restart) {
      t_mom = 1.0;
      ixp = ix;
      ++restarts;
    }
    for (int b = 0; b < 3; ++b)
      if (b != ix && b != ixp) { ic = b; break; }
    // the speculative stage A of stageCA is valid iff its assumptions held
    a_ready = spec && k == 0 && !restart;
    if (a_ready) par ^= 1;
  }

  if (!done) {
    // max_iters reached: g = lower_grad(p, x) (lower_solvers.py:212-213)
    E.value_grad(SrcLin<T>{a.X[ix]}, tv, a.G);
    E.foreach_pixel([&](int64_t i, int, int, int) { a.out[i] = ldcg(a.X[ix] + i); });
    E.gb.sync();
    gn = sqrt(E.reduce1(a.s_t0));
    iters = a.max_iters;
    converged = gn <= a.tol;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    SolveOut* r = a.sres;
    r->lam = lam;
    r->lip = lip;
    r->grad_norm = gn;
    r->value = h_y;
    r->iters = iters;
    r->converged = converged;
    r->status = status;
    r->fail_iter = fail_iter;
    r->power_iters = pit;
    r->power_converged = pconv;
    r->vg_evals = vg;
    r->value_evals = vals;
    r->restarts = restarts;
    r->t_mom = t_mom;
    r->lip_t = (a.method == M_PROXGRAD) ? 1.0 / gd_step : lip_t;
  }
}

// ---------------------------------------------------------------------------
// Hessian of the lower problem (lower_hess_vec, lower_solvers.py:66-71):
//   H v = 2 B^T (B v) + alpha * D^T (rho''(D x) . D v)
template <typename T, bool FAST, int RW>
struct HessOps : ConvOps<T, FAST, RW> {
  using Base = ConvOps<T, FAST, RW>;
  using Base::a;
  __device__ explicit HessOps(const ConvArgs<T>& a_) : Base(a_) {}

  // rho'' weights of x: WV (vertical edges), WH (horizontal); _rho_curv
  // (regularizers.py:34-36): nu^2 / (t^2 + nu^2)^1.5
  __device__ void hess_weights(const T* x) {
    const T nu = T(a.nu), nu2 = nu * nu;
    const int H = a.g.H, W = a.g.W, C = a.g.C;
    this->foreach_pixel([&](int64_t i, int h, int w, int) {
      const T xc = ldcg(x + i);
      const T d0 = this->below(h) ? ldcg(x + i + (int64_t)W * C) - xc : T(0);
      const T d1 = (w < W - 1) ? ldcg(x + i + C) - xc : T(0);
      const T s0 = d0 * d0 + nu2, s1 = d1 * d1 + nu2;
      a.WV[i] = nu2 / (s0 * sqrt(s0));
      a.WH[i] = nu2 / (s1 * sqrt(s1));
    });
  }

  // out = H v, given BP = B v already computed; v read with 1-halo from
  // global.  Optional tile partial of <pdot, out> (curvature) or of
  // (out - sub)^2 (true residual).
  __device__ void hess_stage2(const T* V, bool tv, T* Out, const T* pdot, const T* sub, const SumDev* s) {
    const T two = T(2), alpha = T(a.alpha);
    const int C = a.g.C, H = a.g.H, W = a.g.W;
    const int64_t rowS = (int64_t)W * C;
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      this->tile_origin(tile, h0, w0);
      __syncthreads();
      this->load_full(h0, w0, SrcLin<T>{a.BP});
      __syncthreads();
      const int h = h0 + this->ty;
      double part = 0.0;
      {
        T acc[RW];
        this->stencil_adj(acc);
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + this->tx * RW + o;
          if (h < H && w < W) {
            const int64_t i = this->gidx(h, w, this->ch);
            T hv = two * acc[o];
            if (tv) {
              // D^T (W . D v) at pixel i, image_forward_diff_adjoint order
              const T vc = ldcg(V + i);
              T t = T(0);
              if (this->above(h)) t = t + ldcg(a.WV + i - rowS) * (vc - ldcg(V + i - rowS));
              if (this->below(h)) t = t - ldcg(a.WV + i) * (ldcg(V + i + rowS) - vc);
              if (w >= 1) t = t + ldcg(a.WH + i - C) * (vc - ldcg(V + i - C));
              if (w <= W - 2) t = t - ldcg(a.WH + i) * (ldcg(V + i + C) - vc);
              hv = hv + alpha * t;
            }
            Out[i] = hv;
            if (s) {
              if (pdot) {
                part += (double)ldcg(pdot + i) * (double)hv;
              } else {
                const double d = (double)(hv - ldcg(sub + i));
                part += d * d;
              }
            }
          }
        }
      }
      if (s) this->tile_partial(*s, tile, part);
    }
  }

  // H v with v = src (materialised into Vbuf by stage 1).
  template <class Src>
  __device__ void hess_vec(const Src& src, T* Vbuf, bool tv, T* Out, const T* pdot, const T* sub, const SumDev* s) {
    const int H = a.g.H, W = a.g.W;
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      this->tile_origin(tile, h0, w0);
      __syncthreads();
      this->load_full(h0, w0, src);
      __syncthreads();
      const int h = h0 + this->ty;
      T acc[RW];
      this->stencil_fwd(acc);
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int q = this->tx * RW + o;
        const int w = w0 + q;
        if (h < H && w < W) {
          const int64_t i = this->gidx(h, w, this->ch);
          a.BP[i] = acc[o];
          if (Vbuf) Vbuf[i] = this->fp(this->ty, q);
        }
      }
    }
    this->gb.sync();
    hess_stage2(Vbuf, tv, Out, pdot, sub, s);
  }

  // lower_hess_diag (lower_solvers.py:74-80) into Out; TV part:
  // SmoothedTV.hess_diag (regularizers.py:185-199).
  // the global-row TV edge AND inside the local array (a row slab's outer rows are ghosts)
  __device__ __forceinline__ bool below(int h) const { return this->has_below(h) && h + 1 < a.g.H; }
  __device__ __forceinline__ bool above(int h) const { return this->has_above(h) && h >= 1; }

  // slab = true (row-slab CG setup): no floor; the max over the OWNED pixels
  // goes to scal[0] (the ranks all-reduce it and floor in CM_SLAB_CG_INIT)
  __device__ void hess_diag(const T* x, bool tv, T* Out, bool slab = false) {
    this->load_weights_sq(a.kern);
    const T nu = T(a.nu), nu2 = nu * nu, two = T(2), alpha = T(a.alpha);
    const int C = a.g.C, H = a.g.H, W = a.g.W;
    const int64_t rowS = (int64_t)W * C;
    double mx = -INFINITY;
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      this->tile_origin(tile, h0, w0);
      __syncthreads();
      this->load_full(h0, w0, SrcOnes<T>{});
      __syncthreads();
      const int h = h0 + this->ty;
      {
        T acc[RW];
        this->stencil_adj(acc);
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + this->tx * RW + o;
          if (h < H && w < W) {
            const int64_t i = this->gidx(h, w, this->ch);
            T d = two * acc[o];
            if (tv) {
              const T xc = ldcg(x + i);
              T t = T(0);
              // diag[:-1] += wv; diag[1:] += wv; diag[:, :-1] += wh; diag[:, 1:] += wh
              if (this->below(h)) { const T dd = ldcg(x + i + rowS) - xc, s = dd * dd + nu2; t = t + nu2 / (s * sqrt(s)); }
              if (this->above(h)) { const T dd = xc - ldcg(x + i - rowS), s = dd * dd + nu2; t = t + nu2 / (s * sqrt(s)); }
              if (w <= W - 2) { const T dd = ldcg(x + i + C) - xc, s = dd * dd + nu2; t = t + nu2 / (s * sqrt(s)); }
              if (w >= 1) { const T dd = xc - ldcg(x + i - C), s = dd * dd + nu2; t = t + nu2 / (s * sqrt(s)); }
              d = d + alpha * t;
            }
            Out[i] = d;
            if (!slab || this->tile_owned(h0)) mx = fmax(mx, (double)d);
          }
        }
      }
    }
    // global max -> floor (np.maximum(d, 1e-12 * d.max() + 1e-300))
    mx = block_max(mx, this->red());
    if (threadIdx.x == 0) a.s_t2.leaf_vals[blockIdx.x] = mx;
    this->gb.sync();
    double gmx = -INFINITY;
    for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) gmx = fmax(gmx, ldcg(a.s_t2.leaf_vals + b));
    gmx = block_max(gmx, this->red());
    if (slab) {
      if (blockIdx.x == 0 && threadIdx.x == 0) a.scal[0] = gmx;
      this->load_weights(a.kern);
      return;
    }
    const T fl = T(1e-12 * gmx + 1e-300);
    if (!a.nofloor) this->foreach_pixel([&](int64_t i, int, int, int) {
      const T d = ldcg(Out + i);
      Out[i] = d > fl ? d : fl;   // np.maximum (d is never NaN here)
    });
    this->load_weights(a.kern);
  }
};

// ---------------------------------------------------------------------------
// Jacobi-preconditioned CG on the lower Hessian at x_tilde
// (cg_solve, hypergradient.py:35-84, as specialised by inexact_hypergradient
// 171-176).  Q in/out (warm start when a.warm), DIAG gets the preconditioner.
template <typename T, bool FAST, int RW>
__global__ void __launch_bounds__(512, 1) conv_cg_kernel(const __grid_constant__ ConvArgs<T> a) {
  HessOps<T, FAST, RW> E(a);
  if (a.kern) E.load_weights(a.kern);
  const bool tv = (a.alpha != 0.0);
  const double tol = a.tol;
  int status = ST_OK, hv = 0;
  double curv = 0.0;

  if (tv) E.hess_weights(a.xt);
  if (a.diag_in) {
    E.foreach_pixel([&](int64_t i, int, int, int) { a.DIAG[i] = T(1) / a.diag_in[i]; });
  } else {
    E.gb.sync();
    E.hess_diag(a.xt, tv, a.DIAG);
    E.gb.sync();
    E.foreach_pixel([&](int64_t i, int, int, int) { a.DIAG[i] = T(1) / ldcg(a.DIAG + i); });
  }
  E.gb.sync();
  // r = rhs - H q0 (warm) or rhs; q = q0 or 0; or the injected state (q, r, p) of a lockstep step,
  // the direction entering as the "first" direction p = s
  if (a.cg_p0) {
    E.foreach_pixel([&](int64_t i, int, int, int) { a.CR[i] = a.cg_r[i]; a.CS[i] = a.cg_p0[i]; });
  } else if (a.warm) {
    E.hess_vec(SrcLin<T>{a.Q}, a.P[1], tv, a.HP, nullptr, nullptr, nullptr);
    ++hv;
    E.gb.sync();
    E.foreach_pixel([&](int64_t i, int, int, int) { a.CR[i] = a.rhs[i] - ldcg(a.HP + i); });
  } else {
    E.foreach_pixel([&](int64_t i, int, int, int) { a.Q[i] = T(0); a.CR[i] = a.rhs[i]; });
  }
  // s = inv_diag * r ; rs = <r, s> ; rr = <r, r>
  E.foreach_pixel_sum([&](int64_t i, int, int, int) {
    const T r = ldcg(a.CR + i), s = ldcg(a.DIAG + i) * r;
    if (!a.cg_p0) a.CS[i] = s;
    return (double)r * (double)s;
  }, a.s_t1);
  E.foreach_pixel_sum([&](int64_t i, int, int, int) {
    const double r = (double)ldcg(a.CR + i);
    return r * r;
  }, a.s_t2);
  E.gb.sync();
  double rs, rr;
  {
    double o[2];
    E.reduce({&a.s_t1, &a.s_t2}, o);
    rs = a.cg_p0 ? a.cg_rs0 : o[0];
    rr = o[1];
  }
  int iters = 0;
  int cur = 0;          // P[cur] holds the current direction
  int first = 1;        // p = s.copy() on the first direction
  double beta = 0.0;
  for (iters = 1; iters <= a.max_iters; ++iters) {
    if (sqrt(rr) <= tol) { iters -= 1; break; }
    const int nxt = first ? cur : cur ^ 1;
    E.hess_vec(SrcCGDir<T>{a.CS, a.P[cur], T(beta), first}, a.P[nxt], tv, a.HP, a.P[nxt], nullptr, &a.s_t0);
    ++hv;
    cur = nxt;
    first = 0;
    E.gb.sync();
    curv = E.reduce1(a.s_t0);
    if (curv <= 0.0) { status = ST_NEGCURV; break; }
    const double al = rs / curv;
    const T ta = T(al);
    E.foreach_pixel_sum([&](int64_t i, int, int, int) {
      const T p = ldcg(a.P[cur] + i);
      a.Q[i] = ldcg(a.Q + i) + ta * p;
      const T r = ldcg(a.CR + i) - ta * ldcg(a.HP + i);
      a.CR[i] = r;
      const T s = ldcg(a.DIAG + i) * r;
      a.CS[i] = s;
      return (double)r * (double)s;
    }, a.s_t1);
    E.foreach_pixel_sum([&](int64_t i, int, int, int) {
      const double r = (double)ldcg(a.CR + i);
      return r * r;
    }, a.s_t2);
    E.gb.sync();
    double o[2];
    E.reduce({&a.s_t1, &a.s_t2}, o);
    beta = o[0] / rs;
    rs = o[0];
    rr = o[1];
  }
  if (iters > a.max_iters) iters = a.max_iters;
  if (a.cg_p0) {
    E.gb.sync();
    E.foreach_pixel([&](int64_t i, int, int, int) { a.cg_r[i] = ldcg(a.CR + i); });
  }
  double res = 0.0;
  int conv = 0;
  if (status == ST_OK) {
    // true residual ||H q - rhs|| (hypergradient.py:83)
    E.gb.sync();
    E.hess_vec(SrcLin<T>{a.Q}, a.P[cur ^ 1], tv, a.HP, nullptr, a.rhs, &a.s_t0);
    ++hv;
    E.gb.sync();
    res = sqrt(E.reduce1(a.s_t0));
    conv = res <= tol;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    CGOut* r = a.cres;
    r->residual = res;
    r->curv = curv;
    r->rs = rs;
    r->iters = iters;
    r->converged = conv;
    r->status = status;
    r->hv = hv;
  }
}

// ---------------------------------------------------------------------------
// Per-call primitives (one cooperative launch each).
template <typename T, bool FAST, int RW>
__global__ void __launch_bounds__(512, 1) conv_misc_kernel(const __grid_constant__ ConvArgs<T> a) {
  HessOps<T, FAST, RW> E(a);
  const ConvGeom& g = a.g;
  if (a.kern) E.load_weights(a.kern);
  const bool tv = (a.alpha != 0.0);
  switch (a.mode) {
    case CM_APPLY:
      E.stage_corr(SrcLin<T>{a.in0}, false, a.out0, nullptr, T(1), nullptr);
      break;
    case CM_ADJOINT:
      E.stage_corr(SrcLin<T>{a.in0}, true, a.out0, nullptr, T(1), nullptr);
      break;
    case CM_GRAM_DIAG:
      E.load_weights_sq(a.kern);
      E.stage_corr(SrcOnes<T>{}, true, a.out0, nullptr, T(1), nullptr);
      break;
    case CM_VALUE: {
      // lower_value (lower_solvers.py:37-39): sum(r*r) + alpha * tv_value(x)
      E.value_cand(SrcLin<T>{a.in0}, true, nullptr, nullptr, nullptr, nullptr);
      E.gb.sync();
      double o[2];
      E.reduce({&a.s_fitc, &a.s_tvc}, o);
      if (blockIdx.x == 0 && threadIdx.x == 0) a.scal[0] = o[0] + a.alpha * o[1];
      break;
    }
    case CM_VALUE_GRAD:
    case CM_GRAD: {
      E.value_grad(SrcLin<T>{a.in0}, tv, a.out0);
      E.gb.sync();
      double o[3] = {0, 0, 0};
      if (tv) E.reduce({&a.s_fit, &a.s_tv, &a.s_t0}, o);
      else { E.reduce({&a.s_fit, &a.s_t0}, o); o[2] = o[1]; o[1] = 0.0; }
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        double v = o[0];
        if (tv) v = o[0] + a.alpha * (o[1] - a.nu * (2.0 * (double)g.N));
        a.scal[0] = v;
        a.scal[1] = sqrt(o[2]);
      }
      break;
    }
    case CM_HESS_VEC:
      if (tv) { E.hess_weights(a.in0); E.gb.sync(); }
      E.hess_vec(SrcLin<T>{a.in1}, a.P[0], tv, a.out0, nullptr, nullptr, nullptr);
      break;
    case CM_HESS_DIAG:
      E.hess_diag(a.in0, tv, a.out0);
      break;
    case CM_UPPER: {
      // UpperProblem.fit_value (problems.py:48-50) and ||upper_fit_grad||
      // (hypergradient.py:87-89): r = A x - y; sum(r*r); u = 2 A^T r
      E.stage_corr(SrcLin<T>{a.in0}, false, a.R, a.ydat, T(1), nullptr);
      E.gb.sync();
      E.stage_corr(SrcLin<T>{a.R}, true, a.out0 ? a.out0 : a.G, nullptr, T(2), &a.s_t0);
      np_leaves(a.s_fit, SqOf<T>{a.R});
      E.gb.sync();
      double o[2];
      E.reduce({&a.s_fit, &a.s_t0}, o);
      if (blockIdx.x == 0 && threadIdx.x == 0) { a.scal[0] = o[0]; a.scal[1] = sqrt(o[1]); }
      break;
    }
    case CM_POWER: {
      int it = 0, cv = 0;
      const double lam = E.power(a.power_max_iters, a.power_tol, it, cv);
      if (blockIdx.x == 0 && threadIdx.x == 0) { a.scal[0] = lam; a.scal[1] = cv; a.scal[2] = it; }
      break;
    }
    case CM_MIXED_PREP:
      E.stage_corr(SrcLin<T>{a.in0}, false, a.out0, a.ydat, T(1), nullptr);
      E.stage_corr(SrcLin<T>{a.in1}, false, a.out1, nullptr, T(1), nullptr);
      break;
    case CM_DOT: {
      E.foreach_pixel_sum([&](int64_t i, int, int, int) { return (double)a.in0[i] * (double)a.in1[i]; }, a.s_t0);
      E.gb.sync();
      const double d = E.reduce1(a.s_t0);
      if (blockIdx.x == 0 && threadIdx.x == 0) a.scal[0] = d;
      break;
    }
    // ---- row-slab steps (multi-GPU c5, multigpu.SlabSolver): each stops
    // after phase 1 of its sums; the ranks all-gather the sum units and fold
    // the tops on the host, in the single-GPU tree order.
    case CM_SLAB_ABC: {
      // value + grad at y = x + beta (x - xp), first candidate xc = y - g / L
      // and its value, restart dot g.(xc - x)   (lower_solvers.py:196-207)
      E.stageA(SrcExtrap<T>{a.in0, a.in1, T(a.sbeta)}, a.R, a.ydat, tv, a.TV2, a.TVG, &a.s_fit, &a.s_tv);
      E.gb.sync();
      E.stageB(a.R, tv, a.TVG, a.G, &a.s_t0, a.in0, a.in1, T(a.sbeta), T(a.sL), a.out0);
      E.gb.sync();
      E.value_cand(SrcLin<T>{a.out0}, tv, nullptr, a.G, a.in0, &a.s_t1);
      E.gb.sync();
      E.phase1({&a.s_fit, &a.s_tv, &a.s_t0, &a.s_t1, &a.s_fitc, &a.s_tvc});
      break;
    }
    case CM_SLAB_C:
      // backtracking retry: xc = y - g / L and its value   (lower_solvers.py:170-177)
      E.value_cand(SrcCand<T>{a.in0, a.in1, a.G, T(a.sbeta), T(a.sL)}, tv, a.out0, a.G, a.in0, &a.s_t1);
      E.gb.sync();
      E.phase1({&a.s_fitc, &a.s_tvc, &a.s_t1});
      break;
    case CM_SLAB_POWER:
      // power step: out = B^T B (src / scale), partials of ||out||^2   (operators.py:150-165)
      E.stage_corr(SrcScaled<T>{a.in0, T(a.sL)}, false, a.R, nullptr, T(1), nullptr);
      E.gb.sync();
      E.stage_corr(SrcLin<T>{a.R}, true, a.out0, nullptr, T(1), &a.s_t0);
      E.gb.sync();
      E.phase1({&a.s_t0});
      break;
    case CM_SLAB_NORM0:
      E.foreach_pixel_sum([&](int64_t i, int, int, int) {
        const double v = (double)a.in0[i];
        return v * v;
      }, a.s_t0);
      E.gb.sync();
      E.phase1({&a.s_t0});
      break;
    case CM_BENCH_REDUCE: {
      double o[6], acc = 0.0;
      for (int r = 0; r < a.max_iters; ++r) {
        E.reduce({&a.s_fit, &a.s_tv, &a.s_t0, &a.s_t1, &a.s_fitc, &a.s_tvc}, o);
        acc += o[0] + o[5];
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) a.scal[0] = acc;
      break;
    }
    // ---- row-slab hypergradient (multigpu.SlabHypergradient): the steps of
    // conv_cg_kernel / CM_UPPER / adp_mixed_T split at their reductions, over
    // slab + ghosts, sums over the owned rows only (same tiles / leaves / trees
    // as the unsplit plan, so the folded scalars are bitwise those of one GPU)
    case CM_SLAB_CG_DIAG:
      if (tv) { E.hess_weights(a.in0); E.gb.sync(); }
      E.hess_diag(a.in0, tv, a.DIAG, true);
      break;
    case CM_SLAB_CG_INIT: {
      const T fl = T(a.sL);
      E.foreach_pixel([&](int64_t i, int, int, int) {
        const T d = ldcg(a.DIAG + i);
        a.DIAG[i] = T(1) / (d > fl ? d : fl);
      });
      E.foreach_pixel_sum([&](int64_t i, int, int, int) {
        T r;
        if (a.sflag) {
          r = a.in0[i] - ldcg(a.HP + i);
        } else {
          a.out0[i] = T(0);
          r = a.in0[i];
        }
        a.CR[i] = r;
        const T sv = ldcg(a.DIAG + i) * r;
        a.out1[i] = sv;
        return (double)r * (double)sv;
      }, a.s_t1);
      E.foreach_pixel_sum([&](int64_t i, int, int, int) {
        const double r = (double)ldcg(a.CR + i);
        return r * r;
      }, a.s_t2);
      E.gb.sync();
      E.phase1({&a.s_t1, &a.s_t2});
      break;
    }
    case CM_SLAB_CG_HV:
      if (a.sflag <= 1) {
        E.hess_vec(SrcCGDir<T>{a.in0, a.in1, T(a.sbeta), a.sflag == 0}, a.out0, tv, a.HP, a.out0, nullptr, &a.s_t0);
      } else if (a.sflag == 2) {
        E.hess_vec(SrcLin<T>{a.in0}, a.out0, tv, a.HP, nullptr, a.in1, &a.s_t0);
      } else {
        E.hess_vec(SrcLin<T>{a.in0}, a.out0, tv, a.HP, nullptr, nullptr, nullptr);
        break;
      }
      E.gb.sync();
      E.phase1({&a.s_t0});
      break;
    case CM_SLAB_CG_UPD: {
      const T ta = T(a.sbeta);
      E.foreach_pixel_sum([&](int64_t i, int, int, int) {
        const T p = ldcg(a.in0 + i);
        a.out0[i] = ldcg(a.out0 + i) + ta * p;
        const T r = ldcg(a.CR + i) - ta * ldcg(a.HP + i);
        a.CR[i] = r;
        const T sv = ldcg(a.DIAG + i) * r;
        a.out1[i] = sv;
        return (double)r * (double)sv;
      }, a.s_t1);
      E.foreach_pixel_sum([&](int64_t i, int, int, int) {
        const double r = (double)ldcg(a.CR + i);
        return r * r;
      }, a.s_t2);
      E.gb.sync();
      E.phase1({&a.s_t1, &a.s_t2});
      break;
    }
    case CM_SLAB_UPPER:
      E.stage_corr(SrcLin<T>{a.in0}, false, a.R, a.ydat, T(1), nullptr);
      E.gb.sync();
      E.stage_corr(SrcLin<T>{a.R}, true, a.out0 ? a.out0 : a.G, nullptr, T(2), &a.s_t0);
      E.slab_leaves(a.s_fit, SqOf<T>{a.R});
      E.gb.sync();
      E.phase1({&a.s_fit, &a.s_t0});
      break;
    case CM_SLAB_MIXED_PREP:
      E.stage_corr(SrcLin<T>{a.in0}, false, a.R, a.ydat, T(1), nullptr);
      E.stage_corr(SrcLin<T>{a.in1}, false, a.BP, nullptr, T(1), nullptr);
      break;
    case CM_SLAB_GRAD:
      // g = lower_grad(x) partials (final gradient norm, lower_solvers.py:212)
      E.stageA(SrcLin<T>{a.in0}, a.R, a.ydat, tv, a.TV2, a.TVG, &a.s_fit, &a.s_tv);
      E.gb.sync();
      E.stageB(a.R, tv, a.TVG, a.G, &a.s_t0);
      E.gb.sync();
      E.phase1({&a.s_fit, &a.s_tv, &a.s_t0});
      break;
    default:
      break;
  }
}

// ---------------------------------------------------------------------------
// kernel_gram_correlation (operators.py:198-220), summed over pairs:
//   out[i,j,c] = sum_{h,w} xa[h+i-r, w+j-r, c] * va[h,w,c] (+ same for xb, vb)
// Non-cooperative.  Work groups are (tile row of KT GLOBAL image rows,
// column block): group g = tr * cblocks + cb owns the 16x16 tiles of tile row
// tr in columns [cb * per, (cb + 1) * per); per-group partials, then a
// fixed-order final sum over the groups (deterministic, grid-independent).
// A row slab (rows KT-aligned) computes exactly the groups of its owned tile
// rows, so assembling the per-rank partial vectors and the same final sum is
// bitwise the unsplit result.
template <typename T>
__global__ void __launch_bounds__(256) kgc_partial_kernel(const __grid_constant__ KgcArgs<T> a) {
  const ConvGeom& g = a.g;
  constexpr int KT = 16;
  const int SHx = KT + g.kh - 1, SWx = KT + g.kw - 1;
  T* xs = reinterpret_cast<T*>(dsm());
  T* vs = xs + SHx * SWx;
  const int ntap = g.kh * g.kw;
  const int thW = (g.W + KT - 1) / KT;
  const int per = (thW + a.cblocks - 1) / a.cblocks;
  for (int grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    const int tr = grp / a.cblocks, cb = grp - tr * a.cblocks;
    const int h0 = tr * KT - g.row0;            // local row of the tile row
    if (h0 < g.own0 || h0 >= g.own1) continue;  // not this slab's (CTA-uniform)
    const int tc0 = cb * per, tc1 = min(thW, tc0 + per);
    for (int c = 0; c < g.C; ++c) {
      double acc[12];
#pragma unroll
      for (int k = 0; k < 12; ++k) acc[k] = 0.0;
      for (int pair = 0; pair < 2; ++pair) {
        const T* X = pair ? a.xb : a.xa;
        const T* V = pair ? a.vb : a.va;
        if (!X) continue;
        for (int tc = tc0; tc < tc1; ++tc) {
          const int w0 = tc * KT;
          __syncthreads();
          for (int e = threadIdx.x; e < SHx * SWx; e += blockDim.x) {
            const int r = e / SWx, q = e % SWx;
            const int gh = h0 - g.rh + r, gw = w0 - g.rw + q;
            xs[e] = (gh >= 0 && gh < g.H && gw >= 0 && gw < g.W) ? X[((int64_t)gh * g.W + gw) * g.C + c] : T(0);
          }
          for (int e = threadIdx.x; e < KT * KT; e += blockDim.x) {
            const int r = e / KT, q = e % KT;
            const int gh = h0 + r, gw = w0 + q;
            vs[e] = (gh < g.H && gw < g.W) ? V[((int64_t)gh * g.W + gw) * g.C + c] : T(0);
          }
          __syncthreads();
#pragma unroll
          for (int k = 0; k < 12; ++k) {
            const int t = threadIdx.x + k * blockDim.x;
            if (t < ntap) {
              const int i = t / g.kw, j = t % g.kw;
              double s = 0.0;
              for (int r = 0; r < KT; ++r)
                for (int q = 0; q < KT; ++q) s += (double)xs[(r + i) * SWx + q + j] * (double)vs[r * KT + q];
              acc[k] += s;
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const int t = threadIdx.x + k * blockDim.x;
        if (t < ntap) a.part[(size_t)grp * ntap * g.C + t * g.C + c] = acc[k];
      }
    }
  }
}

template <typename T>
__global__ void kgc_final_kernel(const __grid_constant__ KgcArgs<T> a) {
  const int n = a.g.kh * a.g.kw * a.g.C;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < a.ngroups; ++k) s += a.part[(size_t)k * n + e];
    a.out[e] = T(a.scale * s);
  }
}

}  // namespace adp
