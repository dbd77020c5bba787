// Host-stepped, high-occupancy lower solve for the large RW = 4 plans (c3,
// c4, c5): the stages of conv_solve_kernel (adaptive AGD with restart on
// smoothed TV, lower_solvers.py:180-213) as separate non-cooperative kernels,
// one tile per CTA and two CTAs per SM, so one CTA's tile loads, epilogues
// and leaf sums overlap the other's stencil; the deterministic reductions run
// in a small cooperative kernel and the scalar AGD decisions on the host (the
// same IEEE double expressions in the same order as the persistent kernel).
// Every stage computes exactly the persistent kernel's arithmetic (same stage
// methods, tiles, fused leaves, tile partials and trees), so iterates and
// decisions are bitwise identical to it.
// Taps: a StepW kernel parameter (see Conv's PW), not shared memory.
#include <cstdlib>
#include "conv2d_kernels.cuh"
#include "step_tail.h"

namespace adp {

// Perfect-tree folds of K runs of units read from L2 (n[i] <= 4 T units, T the largest power of two
// <= blockDim): reduce_k's register path -- chunks of <= 4 contiguous units per folding thread, zero
// padding to the next power of two, xor-shuffles, then the warp partials.  out valid in every thread.
template <int K>
__device__ __forceinline__ void fold_many(const double* const (&src)[K], const int (&n)[K], double (&out)[K],
                                          double* red) {
  const int BD = blockDim.x, lgT = 31 - __clz(BD), T = 1 << lgT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = BD >> 5;
  double root[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int P = n[i] <= 1 ? 1 : 1 << (32 - __clz(n[i] - 1));
    const int chunk = P > T ? P >> lgT : 1;
    const int e0 = threadIdx.x * chunk;
    double v[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int e = e0 + m;
      v[m] = (m < chunk && e < n[i] && (int)threadIdx.x < T) ? ldcg(src[i] + e) : 0.0;
    }
    root[i] = chunk == 1 ? v[0] : chunk == 2 ? v[0] + v[1] : (v[0] + v[1]) + (v[2] + v[3]);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < K; ++i) root[i] = root[i] + __shfl_xor_sync(kFull, root[i], o);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) red[i * 32 + warp] = root[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < K; ++i) root[i] = lane < nw ? red[i * 32 + lane] : 0.0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < K; ++i) root[i] = root[i] + __shfl_xor_sync(kFull, root[i], o);
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = root[i];
  __syncthreads();
}

// Tail of a leaf-producing stage CTA (see step_tail.h): ticket of the tile row; its last CTA folds the
// row's leaves; candidate half (isC): the last tile row folds all six sums and publishes them to the host.
// sf / st: the (fit, tv) sums the stage-A pass of this launch wrote (isC false).
template <class Eng, typename T>
__device__ __forceinline__ void tail_fold(Eng& E, const ConvArgs<T>& a, const StepTail& tl, bool isC, int tile,
                                          const SumDev* sf, const SumDev* st) {
  __shared__ int s_last;
  const int grp = E.tile_row(tile);
  const int GL = tl.GL, tW = tl.tW, nG = tl.nG;
  unsigned int* cnt = tl.cnt + (isC ? 0 : nG) + grp;
  // the CTA's leaves / partial are ordered before the ticket by the barrier and thread 0's
  // (cumulative) fence; the folding CTA reads them from L2 (ldcg) after its own fence + barrier
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(cnt, 1u) == (unsigned)tW - 1;
    __threadfence();
  }
  __syncthreads();
  if (!s_last) return;
  double* red = E.tm();   // the term buffers are free by now
  const int koff = (int)(a.g.Ng / a.g.leafL);
  if (!isC) {
    const double* src[3] = {sf->leaf_vals + (size_t)grp * GL, st->leaf_vals + (size_t)grp * GL,
                            st->leaf_vals + koff + (size_t)grp * GL};
    const int n[3] = {GL, GL, GL};
    double o[3];
    fold_many<3>(src, n, o, red);
    if (threadIdx.x == 0) {
      tl.sub[tl.o_fit(tl.setA) + grp] = o[0];
      tl.sub[tl.o_tv(tl.setA) + grp] = o[1];
      tl.sub[tl.o_tv(tl.setA) + nG + grp] = o[2];
      *cnt = 0;
    }
    return;
  }
  {
    const double* src[5] = {a.s_fitc.leaf_vals + (size_t)grp * GL, a.s_tvc.leaf_vals + (size_t)grp * GL,
                            a.s_tvc.leaf_vals + koff + (size_t)grp * GL, a.s_t1.leaf_vals + (size_t)grp * tW,
                            a.s_t0.leaf_vals + (size_t)grp * tW};
    const int n[5] = {GL, GL, GL, tW, tW};
    double o[5];
    fold_many<5>(src, n, o, red);
    if (threadIdx.x == 0) {
      tl.sub[tl.o_fitc() + grp] = o[0];
      tl.sub[tl.o_tvc() + grp] = o[1];
      tl.sub[tl.o_tvc() + nG + grp] = o[2];
      tl.sub[tl.o_t1() + grp] = o[3];
      tl.sub[tl.o_t0() + grp] = o[4];
      *cnt = 0;
      __threadfence();
      s_last = atomicAdd(tl.cnt + 2 * nG, 1u) == (unsigned)nG - 1;
      __threadfence();
    }
  }
  __syncthreads();
  if (!s_last) return;
  const double* src[6] = {tl.sub + tl.o_fit(tl.setR), tl.sub + tl.o_tv(tl.setR), tl.sub + tl.o_t0(),
                          tl.sub + tl.o_t1(),         tl.sub + tl.o_fitc(),      tl.sub + tl.o_tvc()};
  const int n[6] = {nG, 2 * nG, nG, nG, nG, 2 * nG};
  double o[6];
  fold_many<6>(src, n, o, red);
  if (threadIdx.x == 0) {
    tl.cnt[2 * nG] = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      a.scal[i] = o[i];
      if (a.hscal) a.hscal[i] = o[i];
    }
    if (a.hflag) {
      __threadfence_system();   // the results are visible to the host before the flag
      *a.hflag = a.hseq;
    }
  }
}

// Stage B on one tile (stageB_pipe's arithmetic, expression for expression):
// g = 2 B^T r + alpha tvg -> G, tile partial of g.g, the first candidate
// x_c = (x + beta (x - x_prev)) - g / L -> out0 and the next extrapolation
// point y' = x_c + betaN (x_c - x) -> out1.  wt: flipped taps.  EP selects
// where the epilogue operands (tvg, x, x_prev) come from: 0 registers loaded
// before the stencil, 1 registers loaded after it, 2 term buffers filled by
// asynchronous copies with the tile box (two CTAs per SM instead of three;
// the default: c3 4.86 / 4.83 / 4.99 Gpx-it/s for EP = 0 / 1 / 2).
template <typename T, bool FAST, int EP>
__global__ void __launch_bounds__(384, EP == 2 ? 2 : 3) step_b_kernel(const __grid_constant__ ConvArgs<T> a,
                                                                      const __grid_constant__ StepW wt) {
  Conv<T, FAST, 4, 0, false, true> E(a);
  E.pw = wt.w;
  const bool tv = a.alpha != 0.0;
  const T two = T(2), alpha = T(a.alpha), beta = T(a.sbeta), L = T(a.sL), betaN = T(a.sbetaN);
  const int H = a.g.H, W = a.g.W;
  const int tile = blockIdx.x;
  int h0, w0;
  E.tile_origin(tile, h0, w0);
  if (EP == 2) {
    if (tv) {
      const T* const ops[3] = {a.TVG, a.in0, a.in1};
      E.template stage_own_n<3>(h0, w0, ops, 0);
    } else {
      const T* const ops[2] = {a.in0, a.in1};
      E.template stage_own_n<2>(h0, w0, ops, 1);
    }
  }
  E.load_async(h0, w0, a.R, E.pa());
  cp_commit();
  const int h = h0 + E.ty;
  T tpre[4], xpre[4], xppre[4];
  auto fetch = [&]() {
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int w = w0 + E.tx * 4 + o;
      tpre[o] = xpre[o] = xppre[o] = T(0);
      if (h < H && w < W) {
        const int64_t i = E.gidx(h, w, E.ch);
        if (tv) tpre[o] = ldcg(a.TVG + i);
        xpre[o] = ldcg(a.in0 + i);
        xppre[o] = ldcg(a.in1 + i);
      }
    }
  };
  if (EP == 0) fetch();
  cp_wait<0>();
  __syncthreads();
  T acc[4];
  E.stencil(E.pa() + (size_t)E.ch * a.g.SH * E.swp(), E.wadj(), acc);
  if (EP == 1) fetch();
  double part = 0.0;
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const int q = E.tx * 4 + o;
    const int w = w0 + q;
    if (h < H && w < W) {
      const int64_t i = E.gidx(h, w, E.ch);
      T tg, xv, xpv;
      if (EP == 2) {
        E.opsm = true;
        tg = tv ? E.opv(0, E.ty, q, tpre, o) : T(0);
        xv = E.opv(1, E.ty, q, xpre, o);
        xpv = E.opv(2, E.ty, q, xppre, o);
      } else {
        tg = tpre[o];
        xv = xpre[o];
        xpv = xppre[o];
      }
      T gv = two * acc[o];
      if (tv) gv = gv + alpha * tg;
      a.G[i] = gv;
      part += (double)gv * (double)gv;
      const T xc = (xv + beta * (xv - xpv)) - gv / L;
      a.out0[i] = xc;
      a.out1[i] = xc + betaN * (xc - xv);
    }
  }
  E.tile_partial(a.s_t0, tile, part);
}

// the next extrapolation point of a backtracking retry: y'' = x_c + betaN (x_c - x) with
// x_c = (x + beta (x - x_prev)) - g / L   (step_b_kernel's expressions for out0 / out1)
template <typename T> struct SrcCandExtrap {
  const T* x; const T* xp; const T* g; T beta; T L; T betaN;
  __device__ T operator()(int64_t i) const {
    const T a = ldcg(x + i), b = ldcg(xp + i);
    const T xc = (a + beta * (a - b)) - ldcg(g + i) / L;
    return xc + betaN * (xc - a);
  }
};

// Backtracking retry (lower_solvers.py:170-177): CTAs [0, nTiles): the value at x_c = y - g / L with
// y = in0 + beta (in0 - in1) (lower_value form, x_c -> out0) + the restart-dot partial g.(x_c - in0);
// CTAs [nTiles, 2 nTiles) (launched only with the in-kernel decision sums): the speculative stage A at
// the retry's next extrapolation point (sums set: sflag & 2), so an accepted retry needs no separate
// stage-A launch.
template <typename T, bool FAST>
__global__ void __launch_bounds__(384, 2) step_c_kernel(const __grid_constant__ ConvArgs<T> a,
                                                            const __grid_constant__ StepW wt,
                                                            const __grid_constant__ StepTail tl) {
  Conv<T, FAST, 4, 0, false, true> E(a);   // wt: forward taps
  E.opsm = true;
  E.pw = wt.w;
  const bool tv = a.alpha != 0.0;
  const int nT = a.g.nTiles;
  const bool isC = (int)blockIdx.x < nT;
  const int tile = isC ? (int)blockIdx.x : (int)blockIdx.x - nT;
  E.tb0 = tile;       // the stage loops run this one tile
  E.tbs = nT;
  if (isC) {
    E.stageC(SrcCand<T>{a.in0, a.in1, a.G, T(a.sbeta), T(a.sL)}, a.RC, tv, a.TV2C, a.out0, a.G, a.in0, &a.s_t1,
             &a.s_fitc, &a.s_tvc);
    if (tl.on) tail_fold(E, a, tl, true, tile, nullptr, nullptr);
  } else {
    const SumDev* sf = (a.sflag & 2) ? &a.s_fit2 : &a.s_fit;
    const SumDev* st = (a.sflag & 2) ? &a.s_tv2 : &a.s_tv;
    E.stageA(SrcCandExtrap<T>{a.in0, a.in1, a.G, T(a.sbeta), T(a.sL), T(a.sbetaN)}, a.R, a.ydat, tv, a.TV2, a.TVG,
             sf, st);
    if (tl.on) tail_fold(E, a, tl, false, tile, sf, st);
  }
}

template <typename T, bool FAST>
__global__ void __launch_bounds__(384, 2) step_a_kernel(const __grid_constant__ ConvArgs<T> a,
                                                            const __grid_constant__ StepW wt,
                                                            const __grid_constant__ StepTail tl) {
  // value + TV gradient terms at a point (stage A): sflag 0: y = in0 (the
  // materialised y'); 1: y = in0 + beta (in0 - in1).  Sums into s_fit/s_tv
  // (sflag & 2: the second set s_fit2/s_tv2)
  Conv<T, FAST, 4, 0, false, true> E(a);   // wt: forward taps
  E.opsm = true;
  E.pw = wt.w;
  const bool tv = a.alpha != 0.0;
  const SumDev* sf = (a.sflag & 2) ? &a.s_fit2 : &a.s_fit;
  const SumDev* st = (a.sflag & 2) ? &a.s_tv2 : &a.s_tv;
  if (a.sflag & 1)
    E.stageA(SrcExtrap<T>{a.in0, a.in1, T(a.sbeta)}, a.R, a.ydat, tv, a.TV2, a.TVG, sf, st);
  else
    E.stageA(SrcLin<T>{a.in0}, a.R, a.ydat, tv, a.TV2, a.TVG, sf, st);
  if (tl.on) tail_fold(E, a, tl, false, (int)blockIdx.x, sf, st);   // one tile per CTA
}

// candidate value (as step_c, sflag 0) and speculative stage A at y' = out1
// (as step_a, sflag 0 / 2 in sL > 0 ? set 2 : set 1) in ONE launch of 2 x nTiles
// CTAs: the two independent passes share the waves (one tail instead of two).
// Both halves run ONE code path up to the end of the stencil (epilogue operands
// and the tile box as asynchronous copies, then the forward taps), so the
// kernel carries a single copy of the unrolled stencil (instruction-cache
// footprint); the epilogues are stageC's / stageA's (tileC / tileA on the
// precomputed accumulators: the same arithmetic).
template <typename T, bool FAST>
__global__ void __launch_bounds__(384, 2) step_ca_kernel(const __grid_constant__ ConvArgs<T> a,
                                                            const __grid_constant__ StepW wt,
                                                            const __grid_constant__ StepTail tl) {
  Conv<T, FAST, 4, 0, false, true> E(a);   // wt: forward taps
  E.pw = wt.w;
  const bool tv = a.alpha != 0.0;
  const int nT = a.g.nTiles;
  const bool isC = (int)blockIdx.x < nT;
  const int tile = isC ? (int)blockIdx.x : (int)blockIdx.x - nT;
  int h0, w0;
  E.tile_origin(tile, h0, w0);
  if (isC) {
    const T* const ops[3] = {a.ydat, a.G, a.in1};
    E.template stage_own_n<3>(h0, w0, ops, 0);
  } else {
    E.stage_own(h0, w0, a.ydat, 0);
  }
  E.load_async(h0, w0, isC ? a.in0 : a.out1, E.pa());
  cp_async_wait_all();
  __syncthreads();
  T acc[4];
  E.stencil(E.pa() + (size_t)E.ch * a.g.SH * E.swp(), E.wfwd(), acc);
  const T z[4] = {T(0), T(0), T(0), T(0)};
  E.opsm = true;
  const int koff = (int)(a.g.Ng / a.g.leafL);
  if (isC) {
    const double part = E.tileC(E.pa(), h0, w0, z, z, z, a.RC, tv, a.TV2C, nullptr, true, true, acc);
    E.tile_partial(a.s_t1, tile, part);
    E.tile_leaves(h0, w0, tv ? 3 : 1, &a.s_fitc, &a.s_tvc, koff);
    if (tl.on) tail_fold(E, a, tl, true, tile, nullptr, nullptr);
  } else {
    const SumDev* sf = (a.sflag & 2) ? &a.s_fit2 : &a.s_fit;
    const SumDev* st = (a.sflag & 2) ? &a.s_tv2 : &a.s_tv;
    E.tileA(E.pa(), E.pa(), 0, h0, w0, z, a.R, tv, a.TV2, a.TVG, true, acc);
    E.tile_leaves(h0, w0, tv ? 3 : 1, sf, st, koff);
    if (tl.on) tail_fold(E, a, tl, false, tile, sf, st);
  }
}

// the deterministic sums of one decision point -> scal[0..k), CTA 0
template <typename T>
__global__ void __launch_bounds__(512, 1) step_reduce_kernel(const __grid_constant__ ConvArgs<T> a) {
  ConvOps<T, false, 4> E(a);
  double o[6] = {0, 0, 0, 0, 0, 0};
  const int par = a.sflag & 1;
  const SumDev* sfit = par ? &a.s_fit2 : &a.s_fit;
  const SumDev* stv = par ? &a.s_tv2 : &a.s_tv;
  if ((a.sflag >> 1) == 0) E.reduce({sfit, stv, &a.s_t0, &a.s_t1, &a.s_fitc, &a.s_tvc}, o);
  else E.reduce({&a.s_fitc, &a.s_tvc, &a.s_t1}, o);
  if (blockIdx.x == 0 && threadIdx.x < 6) {
    a.scal[threadIdx.x] = o[threadIdx.x];
    if (a.hscal) a.hscal[threadIdx.x] = o[threadIdx.x];
  }
  if (a.hflag && blockIdx.x == 0) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();   // the results are visible to the host before the flag
      *a.hflag = a.hseq;
    }
  }
}

// converged: x~ = x + beta (x - x_prev)   (lower_solvers.py:200-201)
template <typename T>
__global__ void step_extrap_kernel(const T* x, const T* xp, T beta, T* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T xv = x[i], xpv = xp[i];
    out[i] = xv + beta * (xv - xpv);
  }
}

StepKernels step_kernels(int fast) {
  StepKernels k;
  const char* ev = getenv("ADP_SB");   // stage-B epilogue operand variant (see step_b_kernel)
  const int ep = ev ? atoi(ev) : 2;
  k.b_ep = ep;
  if (ep == 1) k.b = fast ? (const void*)step_b_kernel<double, true, 1> : (const void*)step_b_kernel<double, false, 1>;
  else if (ep == 2) k.b = fast ? (const void*)step_b_kernel<double, true, 2> : (const void*)step_b_kernel<double, false, 2>;
  else k.b = fast ? (const void*)step_b_kernel<double, true, 0> : (const void*)step_b_kernel<double, false, 0>;
  k.c = fast ? (const void*)step_c_kernel<double, true> : (const void*)step_c_kernel<double, false>;
  k.a = fast ? (const void*)step_a_kernel<double, true> : (const void*)step_a_kernel<double, false>;
  k.red = (const void*)step_reduce_kernel<double>;
  k.ca = fast ? (const void*)step_ca_kernel<double, true> : (const void*)step_ca_kernel<double, false>;
  k.extrap = (const void*)step_extrap_kernel<double>;
  return k;
}

}  // namespace adp
