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

// Programmatic dependent launch (see step_launch): let the next stage kernel's CTAs become resident,
// then wait until the previous grid has completed and its writes are visible.  Every stage kernel
// calls this before its first global-memory access.
__device__ __forceinline__ void pdl_sync() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Overlap of the candidate launch with the stage-B launch before it.  Stage B's CTAs signal
// launch_dependents at their start, so the candidate launch's first CTAs become resident while stage
// B's last wave (512 tiles on 296 CTA slots at c3: a quarter of the slots idle) still runs.  Instead
// of waiting for the whole stage-B grid (griddepcontrol.wait) they wait for the stage-B tiles they
// read: every stage-B CTA publishes its tile's sequence number with a release store after its last
// global write, a candidate / stage-A CTA acquires the flags of its tile's 3 x 3 neighbourhood (the
// halo of the box it loads -- also every stage-B tile that reads the R tile a stage-A CTA overwrites),
// a reducer the flags of its tile rows (the g.g tile partials).  Dependents are only scheduled once
// every stage-B CTA has started, so a waiting CTA never holds a slot a stage-B CTA needs.
__device__ __forceinline__ void tile_done(unsigned int* flag, int tile, unsigned int seq) {
  __syncthreads();   // the CTA's global writes before thread 0's release (cumulative)
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag + tile), "r"(seq) : "memory");
}
__device__ __forceinline__ void tile_wait_one(const unsigned int* flag, int tile, unsigned int seq) {
  unsigned int v;
  for (unsigned spins = 0;; ++spins) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag + tile) : "memory");
    if ((int)(v - seq) >= 0 || spins > (1u << 24)) break;   // (gives up after seconds: cannot happen for a launched grid)
    __nanosleep(64);
  }
}
// threads 0..8: the 3 x 3 tile neighbourhood of `tile`; the barrier orders every later load of the CTA
__device__ __forceinline__ void tile_wait_3x3(const unsigned int* flag, unsigned int seq, int tile, int tilesW,
                                              int tilesH, int trow) {
  if (threadIdx.x < 9) {
    const int dr = (int)threadIdx.x / 3 - 1, dc = (int)threadIdx.x % 3 - 1;
    const int r = trow + dr, c = tile - trow * tilesW + dc;
    if (r >= 0 && r < tilesH && c >= 0 && c < tilesW) tile_wait_one(flag, r * tilesW + c, seq);
  }
  __syncthreads();
}

// polls before a reducer gives up on a unit (>= 64 ns each: about two seconds)
constexpr unsigned kPollMax = 1u << 25;

// A leaf unit that may still be unwritten: the candidate half's leaves and tile partials are
// pre-set to an all-ones NaN pattern (never produced by the arithmetic: the hardware's NaN results
// are canonical), each is one 8-byte store, so reading anything else means reading the unit.  No
// fence, ticket or barrier on the producers' side.
__device__ __forceinline__ double ld_unit(const double* p, bool poll) {
  unsigned long long b;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
  if (poll) {
    for (unsigned spins = 0; b == ~0ull; ++spins) {
      if (spins > kPollMax) {   // never written (cannot happen for a completed producer grid): fail, do not hang
        b = 0x7ff8000000000000ull;
        break;
      }
      __nanosleep(100);
      asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
    }
  }
  return __longlong_as_double((long long)b);
}

// Perfect-tree folds of K runs of units read from L2 (n[i] <= 4 T units, T the largest power of two
// <= blockDim): reduce_k's register path -- chunks of <= 4 contiguous units per folding thread, zero
// padding to the next power of two, xor-shuffles, then the warp partials.  out valid in every thread.
// Runs i < NP are polled (ld_unit) and reset to the unwritten pattern once read.
template <int K, int NP>
__device__ __forceinline__ void fold_many(double* const (&src)[K], const int (&n)[K], double (&out)[K],
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
      const bool act = m < chunk && e < n[i] && (int)threadIdx.x < T;
      v[m] = act ? ld_unit(src[i] + e, i < NP) : 0.0;
      if (i < NP && act) src[i][e] = __longlong_as_double(-1LL);
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

// One warp folds one aligned run of <= 32 units of a sum (a subtree of the perfect pairwise tree:
// xor-shuffles 1..16, zero beyond n) -- four such tasks in flight per warp so the L2 round trips
// overlap; polled units (see ld_unit) are waited for and reset.  Lane 0 returns the subtree root.
struct WarpTask {
  double* p;   // first unit of the 32-run (nullptr: no task)
  int n;       // units in the run (<= 32)
};
template <bool POLL>
__device__ __forceinline__ void warp_fold4(const WarpTask (&t)[4], double (&out)[4]) {
  const int lane = threadIdx.x & 31;
  unsigned long long b[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    b[u] = 0ull;
    if (t[u].p && lane < t[u].n) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(b[u]) : "l"(t[u].p + lane) : "memory");
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (POLL && t[u].p && lane < t[u].n) {
      for (unsigned spins = 0; b[u] == ~0ull; ++spins) {
        if (spins > kPollMax) {   // see ld_unit: a NaN sum makes the host report a diverged solve
          b[u] = 0x7ff8000000000000ull;
          break;
        }
        __nanosleep(64);
        asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(b[u]) : "l"(t[u].p + lane) : "memory");
      }
      t[u].p[lane] = __longlong_as_double(-1LL);   // unwritten again for the next launch
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) out[u] = __longlong_as_double((long long)b[u]);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int u = 0; u < 4; ++u) out[u] = out[u] + __shfl_xor_sync(kFull, out[u], o);
}

// Reducer CTA `rid` of a candidate-value launch (see step_tail.h): folds the tile rows
// [rid * gpr, (rid + 1) * gpr) of the decision sums into sub-values -- the candidate half's leaves
// and tile partials are polled as they arrive -- takes a ticket, and the last reducer folds the
// sub-values and publishes the sums to the host.  (A backtracking retry re-runs the same launch: the
// three sums at the extrapolation point are folded again, unchanged.)
// Runs of a group, in this order: polled leaf runs (fitc, tvc, tvc'), plain leaf runs (fit, tv, tv'),
// polled tile run (t1), plain tile run (t0).
// (inlined: a real call in the stage kernels costs the hot path its register allocation -- measured)
template <typename T>
__device__ __forceinline__ void tail_reduce(double* red, const ConvArgs<T>& a, const StepTail& tl, int rid) {
  __shared__ int s_last;
  const int GL = tl.GL, tW = tl.tW, nG = tl.nG;
  const int koff = (int)(a.g.Ng / a.g.leafL);
  const SumDev* sf = tl.setR ? &a.s_fit2 : &a.s_fit;
  const SumDev* st = tl.setR ? &a.s_tv2 : &a.s_tv;
  const int g0 = rid * tl.gpr, ng = min(nG, g0 + tl.gpr) - g0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int segL = (GL + 31) >> 5, segT = (tW + 31) >> 5;     // 32-unit tasks per leaf / tile run
  constexpr int nrl = 6, nrt = 2;                              // leaf / tile runs per group
  double* partL = red;                                         // [ng][nrl][segL]
  double* partT = red + (size_t)tl.gpr * 6 * segL;             // [ng][nrt][segT]
  auto leaf_run = [&](int gi, int k) -> double* {
    const size_t lo = (size_t)(g0 + gi) * GL;
    switch (k) {
      case 0: return a.s_fitc.leaf_vals + lo;
      case 1: return a.s_tvc.leaf_vals + lo;
      case 2: return a.s_tvc.leaf_vals + koff + lo;
      case 3: return sf->leaf_vals + lo;
      case 4: return st->leaf_vals + lo;
      default: return st->leaf_vals + koff + lo;
    }
  };
  // polled tasks first (they may wait), the plain ones behind them
  const int ntl = ng * nrl * segL;
  for (int base = warp; base < ntl; base += 4 * nw) {
    WarpTask tp[4], tq[4];
    int idp[4], idq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int id = base + u * nw;
      tp[u].p = tq[u].p = nullptr;
      tp[u].n = tq[u].n = 0;
      idp[u] = idq[u] = -1;
      if (id < ntl) {
        const int gi = id / (nrl * segL), rem = id - gi * (nrl * segL), k = rem / segL, sg = rem - k * segL;
        WarpTask w;
        w.p = leaf_run(gi, k) + 32 * sg;
        w.n = min(32, GL - 32 * sg);
        if (k < 3) { tp[u] = w; idp[u] = id; } else { tq[u] = w; idq[u] = id; }
      }
    }
    double op[4], oq[4];
    warp_fold4<true>(tp, op);
    warp_fold4<false>(tq, oq);
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (idp[u] >= 0) partL[idp[u]] = op[u];
        if (idq[u] >= 0) partL[idq[u]] = oq[u];
      }
    }
  }
  const int ntt = ng * nrt * segT;
  for (int base = warp; base < ntt; base += 4 * nw) {
    WarpTask tp[4], tq[4];
    int idp[4], idq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int id = base + u * nw;
      tp[u].p = tq[u].p = nullptr;
      tp[u].n = tq[u].n = 0;
      idp[u] = idq[u] = -1;
      if (id < ntt) {
        const int gi = id / (nrt * segT), rem = id - gi * (nrt * segT), k = rem / segT, sg = rem - k * segT;
        WarpTask w;
        w.p = (k == 0 ? a.s_t1.leaf_vals : a.s_t0.leaf_vals) + (size_t)(g0 + gi) * tW + 32 * sg;
        w.n = min(32, tW - 32 * sg);
        if (k == 0) { tp[u] = w; idp[u] = id; } else { tq[u] = w; idq[u] = id; }
      }
    }
    double op[4], oq[4];
    warp_fold4<true>(tp, op);
    warp_fold4<false>(tq, oq);
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (idp[u] >= 0) partT[idp[u]] = op[u];
        if (idq[u] >= 0) partT[idq[u]] = oq[u];
      }
    }
  }
  __syncthreads();
  // one thread per run: the perfect tree over its 32-unit subtree roots -> sub-value
  for (int j = threadIdx.x; j < ng * (nrl + nrt); j += blockDim.x) {
    const bool leaf = j < ng * nrl;
    const int jj = leaf ? j : j - ng * nrl;
    const int per = leaf ? nrl : nrt, seg = leaf ? segL : segT;
    const int gi = jj / per, k = jj - gi * per;
    const double* c = (leaf ? partL : partT) + (size_t)jj * seg;
    const double v = seg == 1 ? c[0] : fold_pow2(c, seg);
    const int grp = g0 + gi;
    int o;
    if (leaf) o = k == 0 ? tl.o_fitc() + grp : k == 1 ? tl.o_tvc() + grp : k == 2 ? tl.o_tvc() + nG + grp
                  : k == 3 ? tl.o_fit() + grp : k == 4 ? tl.o_tv() + grp : tl.o_tv() + nG + grp;
    else o = k == 0 ? tl.o_t1() + grp : tl.o_t0() + grp;
    tl.sub[o] = v;
  }
  __threadfence();
  // ticket among the reducers: thread 0 wrote this reducer's sub-values; its fence orders them
  // before the ticket, the last reducer reads them from L2 after its own fence + barrier
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(tl.cnt, 1u) == (unsigned)tl.nR - 1;
    __threadfence();
  }
  __syncthreads();
  if (!s_last) return;
  double* src[6] = {tl.sub + tl.o_fit(),  tl.sub + tl.o_tv(),   tl.sub + tl.o_t0(),
                    tl.sub + tl.o_t1(),   tl.sub + tl.o_fitc(), tl.sub + tl.o_tvc()};
  const int n[6] = {nG, 2 * nG, nG, nG, nG, 2 * nG};
  double o[6];
  fold_many<6, 0>(src, n, o, red);
  if (threadIdx.x == 0) {
    *tl.cnt = 0;
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
// point y' = x_c + betaN (x_c - x) -> out1.  wt: flipped taps.  The epilogue
// operands (tvg, x, x_prev) are staged in the term buffers by asynchronous copies
// issued with the tile box (two CTAs per SM; measured against operands held in
// registers across the stencil or loaded after it, three CTAs per SM: c3 4.99 vs
// 4.86 / 4.83 Gpx-it/s).
template <typename T, bool FAST, int KD, int KU, class WT>
__global__ void __launch_bounds__(384, 2) step_b_kernel(const __grid_constant__ ConvArgs<T> a,
                                                         const __grid_constant__ WT wt) {
  Conv<T, FAST, 4, 0, false, true, KD, KU> E(a);
  E.pw = wt.w;
  const bool tv = a.alpha != 0.0;
  const T two = T(2), alpha = T(a.alpha), beta = T(a.sbeta), L = T(a.sL), betaN = T(a.sbetaN);
  const int H = a.g.H, W = a.g.W;
  const int tile = blockIdx.x;
  int h0, w0;
  E.tile_origin(tile, h0, w0);
  if (a.tflag && (a.sflag & 1)) {
    // this launch follows a candidate launch whose speculative stage A is its input: overlap that
    // launch's last wave (one CTA slot per SM idle at c3), waiting for the stage-A tiles whose R this
    // tile's box reads -- the same tiles read the y' tile this CTA overwrites -- instead of the grid
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    tile_wait_3x3(a.tflag + a.g.nTiles, (unsigned)a.hseq, tile, a.g.tilesW, a.g.tilesH, E.tile_row(tile));
  } else {
    pdl_sync();
  }
  if (tv) {
    const T* const ops[3] = {a.TVG, a.in0, a.in1};
    E.template stage_own_n<3>(h0, w0, ops, 0);
  } else {
    const T* const ops[2] = {a.in0, a.in1};
    E.template stage_own_n<2>(h0, w0, ops, 1);
  }
  E.load_async(h0, w0, a.R, E.pa());
  cp_commit();
  const int h = h0 + E.ty;
  cp_wait<0>();
  __syncthreads();
  T acc[4];
  E.stencil(E.pa() + (size_t)E.ch * a.g.SH * E.swp(), E.wadj(), acc);
  const T z[4] = {T(0), T(0), T(0), T(0)};
  E.opsm = true;
  double part = 0.0;
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const int q = E.tx * 4 + o;
    const int w = w0 + q;
    if (h < H && w < W) {
      const int64_t i = E.gidx(h, w, E.ch);
      const T tg = tv ? E.opv(0, E.ty, q, z, o) : T(0);
      const T xv = E.opv(1, E.ty, q, z, o);
      const T xpv = E.opv(2, E.ty, q, z, o);
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
  if (a.tflag) tile_done(a.tflag, tile, a.tseq);
}

// Backtracking retry without the in-kernel decision sums (ADP_TAIL=0 or a geometry the reducers do not
// cover; lower_solvers.py:170-177): the value at x_c = y - g / L with y = in0 + beta (in0 - in1)
// (lower_value form, x_c -> out0) + the restart-dot partial g.(x_c - in0); step_reduce_kernel follows.
// (With the in-kernel sums a retry is step_cand_kernel + the regular step_ca_kernel launch.)
template <typename T, bool FAST, int KD, int KU, class WT>
__global__ void __launch_bounds__(384, 2) step_c_kernel(const __grid_constant__ ConvArgs<T> a,
                                                            const __grid_constant__ WT wt) {
  Conv<T, FAST, 4, 0, false, true, KD, KU> E(a);   // wt: forward taps
  E.opsm = true;
  E.pw = wt.w;
  const bool tv = a.alpha != 0.0;
  pdl_sync();
  E.stageC(SrcCand<T>{a.in0, a.in1, a.G, T(a.sbeta), T(a.sL)}, a.RC, tv, a.TV2C, a.out0, a.G, a.in0, &a.s_t1,
           &a.s_fitc, &a.s_tvc);
}

template <typename T, bool FAST, int KD, int KU, class WT>
__global__ void __launch_bounds__(384, 2) step_a_kernel(const __grid_constant__ ConvArgs<T> a,
                                                            const __grid_constant__ WT wt) {
  // value + TV gradient terms at a point (stage A): sflag 0: y = in0 (the
  // materialised y'); 1: y = in0 + beta (in0 - in1).  Sums into s_fit/s_tv
  // (sflag & 2: the second set s_fit2/s_tv2)
  Conv<T, FAST, 4, 0, false, true, KD, KU> E(a);   // wt: forward taps
  E.opsm = true;
  E.pw = wt.w;
  const bool tv = a.alpha != 0.0;
  const SumDev* sf = (a.sflag & 2) ? &a.s_fit2 : &a.s_fit;
  const SumDev* st = (a.sflag & 2) ? &a.s_tv2 : &a.s_tv;
  pdl_sync();
  if (a.sflag & 1)
    E.stageA(SrcExtrap<T>{a.in0, a.in1, T(a.sbeta)}, a.R, a.ydat, tv, a.TV2, a.TVG, sf, st);
  else
    E.stageA(SrcLin<T>{a.in0}, a.R, a.ydat, tv, a.TV2, a.TVG, sf, st);
}

// candidate value (as step_c, sflag 0) and speculative stage A at y' = out1
// (as step_a, sflag 0 / 2 in sL > 0 ? set 2 : set 1) in ONE launch of 2 x nTiles
// CTAs (+ the reducer CTAs of step_tail.h between the halves): the two independent
// passes share the waves (one tail instead of two).
// Both halves run ONE code path up to the end of the stencil (epilogue operands
// and the tile box as asynchronous copies, then the forward taps), so the
// kernel carries a single copy of the unrolled stencil (instruction-cache
// footprint); the epilogues are stageC's / stageA's (tileC / tileA on the
// precomputed accumulators: the same arithmetic).
template <typename T, bool FAST, int KD, int KU, class WT>
__global__ void __launch_bounds__(384, 2) step_ca_kernel(const __grid_constant__ ConvArgs<T> a,
                                                            const __grid_constant__ WT wt,
                                                            const __grid_constant__ StepTail tl) {
  Conv<T, FAST, 4, 0, false, true, KD, KU> E(a);   // wt: forward taps
  E.pw = wt.w;
  const bool tv = a.alpha != 0.0;
  const int nT = a.g.nTiles, nR = tl.on ? tl.nR : 0;
  const int b = (int)blockIdx.x;
  const bool isC = b < nT;
  const bool ovl = tl.ovl && a.tflag;
  if (!isC && b < nT + nR) {   // reducer CTAs sit between the two halves (step_tail.h)
    if (ovl) {
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      const int rid = b - nT, t0 = rid * tl.gpr * tl.tW, t1 = min(nT, t0 + tl.gpr * tl.tW);
      for (int t = t0 + (int)threadIdx.x; t < t1; t += blockDim.x) tile_wait_one(a.tflag, t, a.tseq);
      __syncthreads();
    } else {
      pdl_sync();
    }
    tail_reduce(E.tm(), a, tl, b - nT);
    return;
  }
  const int tile = isC ? b : b - nT - nR;
  int h0, w0;
  E.tile_origin(tile, h0, w0);
  if (ovl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    tile_wait_3x3(a.tflag, a.tseq, tile, a.g.tilesW, a.g.tilesH, E.tile_row(tile));
  } else {
    pdl_sync();
  }
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
  } else {
    const SumDev* sf = (a.sflag & 2) ? &a.s_fit2 : &a.s_fit;
    const SumDev* st = (a.sflag & 2) ? &a.s_tv2 : &a.s_tv;
    E.tileA(E.pa(), E.pa(), 0, h0, w0, z, a.R, tv, a.TV2, a.TVG, true, acc);
    E.tile_leaves(h0, w0, tv ? 3 : 1, sf, st, koff);
    if (a.tflag && tl.aseq) tile_done(a.tflag + nT, tile, tl.aseq);
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

// backtracking retry (lower_solvers.py:170-177), elementwise: the candidate at the doubled L,
// x_c = (x + beta (x - x_prev)) - g / L -> out0, and its next extrapolation point
// y'' = x_c + betaN (x_c - x) -> out1 (step_b_kernel's expressions); the candidate-value kernel then
// runs on them exactly as for the first candidate.
template <typename T>
__global__ void step_cand_kernel(const T* x, const T* xp, const T* g, T beta, T L, T betaN, T* out0, T* out1,
                                 int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T xv = ldcg(x + i), xpv = ldcg(xp + i), gv = ldcg(g + i);
    const T xc = (xv + beta * (xv - xpv)) - gv / L;
    out0[i] = xc;
    out1[i] = xc + betaN * (xc - xv);
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

template <int KD, int KU, class WT>
static void pick(StepKernels& k, int fast) {
  k.b = fast ? (const void*)step_b_kernel<double, true, KD, KU, WT> : (const void*)step_b_kernel<double, false, KD, KU, WT>;
  k.ca = fast ? (const void*)step_ca_kernel<double, true, KD, KU, WT>
              : (const void*)step_ca_kernel<double, false, KD, KU, WT>;
  k.a = fast ? (const void*)step_a_kernel<double, true, KD, KU, WT> : (const void*)step_a_kernel<double, false, KD, KU, WT>;
  k.c = fast ? (const void*)step_c_kernel<double, true, KD, KU, WT> : (const void*)step_c_kernel<double, false, KD, KU, WT>;
}

StepKernels step_kernels(int fast, int ksz) {
  StepKernels k;
  k.b_ep = 2;
  // instances that carry one stencil size only: 15 x 15 (c3, c4) with the row loop unrolled 5 rows at a
  // time (ADP_SU=15: straight-line code, whose instruction footprint costs the candidate kernel 9 us per
  // launch; ADP_SU=0: the generic multi-stencil instances) and 31 x 31 (c5: one row per iteration, the
  // large tap block); everything else runs the generic instances
  const char* ev = getenv("ADP_SU");
  const int su = ev ? atoi(ev) : 5;
  if (ksz == 15 && su == 15) pick<15, 15, StepW>(k, fast);
  else if (ksz == 15 && su != 0) pick<15, 5, StepW>(k, fast);
  else if (ksz == 31) pick<31, 1, StepWL>(k, fast);
  else pick<0, 0, StepW>(k, fast);
  k.red = (const void*)step_reduce_kernel<double>;
  k.extrap = (const void*)step_extrap_kernel<double>;
  k.cand = (const void*)step_cand_kernel<double>;
  return k;
}

}  // namespace adp
