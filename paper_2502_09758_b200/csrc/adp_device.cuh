// Device-side building blocks shared by every engine kernel:
//   * grid-wide barrier for cooperative persistent kernels,
//   * deterministic reductions (NumPy pairwise leaves, fixed CTA trees,
//     host-built tree programs evaluated in shared memory),
//   * the multiply-add used by the stencils (strict = separate mul/add in
//     the reference's order; fast = FMA).
//
// The whole library is compiled with --fmad=false so that plain `a*b + c`
// never contracts: strict mode reproduces scipy.ndimage / NumPy rounding
// exactly; fast mode asks for fma() explicitly.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "adp_types.h"

namespace adp {

constexpr double kDblEps = 2.220446049250313e-16;   // DBL_EPSILON (ndimage tap skip)
constexpr unsigned kFull = 0xffffffffu;

template <bool FAST, typename T>
__device__ __forceinline__ T madd(T acc, T a, T b) {
  if constexpr (FAST) {
    return fma(a, b, acc);
  } else {
    return acc + a * b;
  }
}

template <typename T> __device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

// ---------------------------------------------------------------------------
// Grid barrier (all CTAs co-resident: cooperative launch).  `counter` is
// zeroed by the host before each launch; targets grow monotonically.
struct GridBarrier {
  unsigned int* counter;
  unsigned int nblocks;
  unsigned int target;

  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      target += nblocks;
      __threadfence();
      atomicAdd(counter, 1u);
      unsigned int v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        if ((int)(v - target) >= 0) break;
      }
      __threadfence();
    }
    __syncthreads();
  }
};

// ---------------------------------------------------------------------------
// Block-level deterministic sum of one double per thread (fixed pattern).
// `red` must hold >= 32 doubles.  Result valid in all threads.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  double r = red[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? red[lane] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(kFull, t, o));
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  double r = red[32];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// NumPy pairwise leaf (n <= 128) computed by one warp.  Restates
// pairwise_sum's block branch: r[k] = a[k]; r[k] += a[i+k] for i = 8, 16,
// ... < n - n%8; res = ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); res += tail.
// n < 8: res = 0.0 + a[0] + ... sequentially.  Result valid in lane 0.
template <class Src>
__device__ __forceinline__ double np_leaf_warp(const Src& src, int64_t s, int n) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
  if (n < 8) {
    if (lane == 0) {
      for (int k = 0; k < n; ++k) t = t + src(s + k);
    }
    return t;
  }
  const int nfull = n - (n % 8);
  double acc = 0.0;
  if (lane < 8) {
    acc = src(s + lane);
#pragma unroll 4
    for (int i = 8; i < nfull; i += 8) acc = acc + src(s + i + lane);
  }
  t = acc + __shfl_down_sync(kFull, acc, 1);
  t = t + __shfl_down_sync(kFull, t, 2);
  t = t + __shfl_down_sync(kFull, t, 4);
  if (lane == 0) {
    for (int i = nfull; i < n; ++i) t = t + src(s + i);
  }
  return t;
}

// All leaves of an element sum, distributed over every warp of the grid.
template <class Src>
__device__ void np_leaves(const SumDev& s, const Src& src) {
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + (threadIdx.x >> 5);
  const int nw = gridDim.x * wpb;
  for (int l = gw; l < s.nLeaves; l += nw) {
    const int64_t a = s.leaf_start[l];
    const int n = (int)(s.leaf_start[l + 1] - a);
    double v = np_leaf_warp(src, a, n);
    if ((threadIdx.x & 31) == 0) s.leaf_vals[l] = v;
  }
}

// ---------------------------------------------------------------------------
// Tree program evaluation in shared memory.  sv[0..nL) must hold the leaf
// values; returns the root (valid in all threads).  Ends with a barrier.
__device__ __forceinline__ double eval_prog(const int* __restrict__ prog, double* sv) {
  const int nL = prog[0], nI = prog[1], nLev = prog[2];
  const int* lev = prog + 3;
  const int* left = lev + nLev + 1;
  const int* right = left + nI;
  for (int lv = 0; lv < nLev; ++lv) {
    const int a = lev[lv], b = lev[lv + 1];
    for (int k = a + threadIdx.x; k < b; k += blockDim.x) sv[nL + k] = sv[left[k]] + sv[right[k]];
    __syncthreads();
  }
  const double r = nI ? sv[nL + nI - 1] : sv[0];
  __syncthreads();
  return r;
}

// Evaluate a single-level sum (nSub == 1) redundantly in this CTA.
__device__ __forceinline__ double sum_single(const SumDev& s, double* sv) {
  if (s.nLeaves == 0) return 0.0;
  for (int k = threadIdx.x; k < s.nLeaves; k += blockDim.x) sv[k] = ldcg(s.leaf_vals + k);
  __syncthreads();
  return eval_prog(s.progs + s.top_prog, sv);
}

// Two-level sums: phase 1 (subtrees, distributed), grid barrier, phase 2 (top).
__device__ __forceinline__ void sum_phase1(const SumDev& s, double* sv) {
  if (s.nSub <= 1) return;
  for (int t = blockIdx.x; t < s.nSub; t += gridDim.x) {
    const int l0 = s.sub_leaf[t], l1 = s.sub_leaf[t + 1];
    for (int k = threadIdx.x; k < l1 - l0; k += blockDim.x) sv[k] = ldcg(s.leaf_vals + l0 + k);
    __syncthreads();
    const double r = eval_prog(s.progs + s.sub_prog[t], sv);
    if (threadIdx.x == 0) s.sub_vals[t] = r;
  }
}

__device__ __forceinline__ double sum_phase2(const SumDev& s, double* sv) {
  if (s.nSub <= 1) return sum_single(s, sv);
  for (int k = threadIdx.x; k < s.nSub; k += blockDim.x) sv[k] = ldcg(s.sub_vals + k);
  __syncthreads();
  return eval_prog(s.progs + s.top_prog, sv);
}

// Reduce k sums: phase 1 for all, one barrier if any is two-level, then
// phase 2 for all.  out[i] valid in every thread of every CTA.
static __device__ __noinline__ void reduce_list(const SumDev* const* ss, int k, double* out, double* sv,
                                         GridBarrier& gb) {
  bool two = false;
  for (int i = 0; i < k; ++i) {
    if (ss[i]->nSub > 1) {
      two = true;
      sum_phase1(*ss[i], sv);
    }
  }
  if (two) gb.sync();
  for (int i = 0; i < k; ++i) out[i] = sum_phase2(*ss[i], sv);
}

// Tile partial (ddot-type): per-thread accumulation in a fixed order then
// block_sum; thread 0 stores the partial for `tile`.
__device__ __forceinline__ void store_tile_partial(const SumDev& s, int tile, double v, double* red) {
  const double t = block_sum(v, red);
  if (threadIdx.x == 0) s.leaf_vals[tile] = t;
}

}  // namespace adp
