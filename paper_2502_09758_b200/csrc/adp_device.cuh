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

// Loads of data produced earlier in the same (persistent) kernel.  Every
// grid barrier ends with a GPU-scope fence that invalidates the SM's L1
// (CCTL.IVALL), so plain weak loads observe the other CTAs' writes.
template <typename T> __device__ __forceinline__ T ldcg(const T* p) { return *p; }

// ---------------------------------------------------------------------------
// Grid barrier (all CTAs co-resident: cooperative launch).  `counter` is
// zeroed by the host before each launch; targets grow monotonically.
struct GridBarrier {
  unsigned int* counter;
  unsigned int nblocks;
  unsigned int target;

  // bar.sync orders the CTA's writes before thread 0's release-add (release
  // is cumulative); thread 0's gpu-scope acquire (which also invalidates the
  // SM's L1) then bar.sync order every later load of the CTA after all
  // arrivals.  Measured 1.27 us per barrier on 148 CTAs vs 1.41 us for
  // fence + atomicAdd + fence (tools/micro/barbench.cu).
  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      target += nblocks;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
      unsigned int v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        if ((int)(v - target) >= 0) break;
      }
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

// Regular layout (all leaves of length L, L % 8 == 0): one thread per
// accumulator chain r[k] (8 per leaf, 4 leaves per warp), then the fixed
// combine ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by xor-shuffles inside each
// 8-lane group (addition is commutative, so pairing order is irrelevant).
template <class Src>
__device__ void np_leaves_regular(const SumDev& s, const Src& src) {
  const int L = s.leaf_len;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t total = (int64_t)s.nLeaves * 8;
  const int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t g0 = 0; g0 < total; g0 += nthreads) {
    const int64_t g = g0 + base;       // warp-uniform loop trip count (total % 8 == 0)
    const bool act = g < total;
    const int64_t leaf = g >> 3;
    const int k = (int)(g & 7);
    double acc = 0.0;
    if (act) {
      // L <= 128: issue all (<= 16) loads of the chain, then add in order
      const int64_t e0 = leaf * L + k;
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

// All leaves of an element sum, distributed over every warp of the grid.
template <class Src>
__device__ void np_leaves(const SumDev& s, const Src& src) {
  if (s.regular) {
    np_leaves_regular(s, src);
    return;
  }
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

// 8-byte asynchronous global -> shared copy (LDGSTS); valid == false
// zero-fills the destination.
__device__ __forceinline__ void cp_async8(double* dst_smem, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
// 16-byte variant: `bytes` (0, 8 or 16) valid source bytes, the rest zero-filled
__device__ __forceinline__ void cp_async16(double* dst_smem, const double* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
// element-size asynchronous copy (4 or 8 bytes), zero-fill when !valid
template <typename T>
__device__ __forceinline__ void cp_async_el(T* dst_smem, const T* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  if (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Perfect binary tree over c[0..chunk), chunk a power of two (registers for
// chunk <= 16; 16-blocks combined by a binary counter beyond).
__device__ __forceinline__ double fold8(const double* c) {
  return ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[5]) + (c[6] + c[7]));
}
__device__ __forceinline__ double fold_small(const double* c, int chunk) {   // chunk <= 16
  switch (chunk) {
    case 1: return c[0];
    case 2: return c[0] + c[1];
    case 4: return (c[0] + c[1]) + (c[2] + c[3]);
    case 8: return fold8(c);
    default: return fold8(c) + fold8(c + 8);
  }
}
__device__ __forceinline__ double fold_pow2(const double* c, int chunk) {
  if (chunk <= 16) return fold_small(c, chunk);
  double st[12];
  double root = 0.0;
  for (int b = 0; b < chunk / 16; ++b) {
    double v = fold8(c + 16 * b) + fold8(c + 16 * b + 8);
#pragma unroll
    for (int lv = 0; lv < 12; ++lv) {
      if ((b >> lv) & 1) {
        v = st[lv] + v;
      } else {
        st[lv] = v;
        break;
      }
    }
    root = v;
  }
  return root;
}

// Perfect binary tree over vals[0..n), zero-padded to the next power of two,
// evaluated by one CTA (blockDim a power of two): values staged in shared
// memory, each thread folds a contiguous power-of-two chunk with a binary
// counter (exact perfect-tree order), then xor-shuffles across lanes and
// warps.  Result valid in every thread.
__device__ __forceinline__ double tree_reduce_cta(const double* __restrict__ vals, int n, double* sv, double* red) {
  int P = 1;
  while (P < n) P <<= 1;
  const int BD = blockDim.x;
  const int T = 1 << (31 - __clz(BD));          // folding threads: largest power of two <= blockDim
  const int chunk = P > T ? P / T : 1;
  for (int e = threadIdx.x; e < P; e += BD) cp_async8(sv + e, vals + (e < n ? e : 0), e < n);
  cp_async_wait_all();
  __syncthreads();
  double root = 0.0;
  if (threadIdx.x * chunk < P) root = fold_pow2(sv + threadIdx.x * chunk, chunk);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) root = root + __shfl_xor_sync(kFull, root, o);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = BD >> 5;
  if (lane == 0) red[warp] = root;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) t = t + __shfl_xor_sync(kFull, t, o);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}

// Evaluate a single-level sum (nSub == 1) redundantly in this CTA.  The
// slow paths below (program trees, two-level sums, oversized batches) are
// kept out of line: one copy of their code per kernel instead of one per
// call site keeps the hot loop's instruction footprint small.
static __device__ __noinline__ double sum_single(const SumDev& s, double* sv) {
  if (s.nLeaves == 0) return 0.0;
  if (s.regular) return tree_reduce_cta(s.leaf_vals, s.nLeaves, sv, sv + kTreeStage);
  for (int k = threadIdx.x; k < s.nLeaves; k += blockDim.x) sv[k] = ldcg(s.leaf_vals + k);
  __syncthreads();
  return eval_prog(s.progs + s.top_prog, sv);
}

// Two-level sums: phase 1 (subtrees, distributed), grid barrier, phase 2 (top).
// Subtree t of this sum goes to CTA (off + t) mod grid, so the subtrees of
// the several sums reduced together spread over different CTAs.
// Only subtrees [sub_own0, sub_own1) are evaluated (a row slab's own ones).
static __device__ __noinline__ void sum_phase1(const SumDev& s, double* sv, int off) {
  if (s.nSub <= 1) return;
  const int G = gridDim.x;
  const int u0 = ((int)blockIdx.x - off % G + G) % G;
  const int n0 = s.sub_own1 - s.sub_own0, n = n0 + (s.sub_own3 - s.sub_own2);
  if (s.regular) {
    for (int u = u0; u < n; u += G) {
      const int t = u < n0 ? s.sub_own0 + u : s.sub_own2 + (u - n0);
      const int a = t * s.sub_size;
      const double r = tree_reduce_cta(s.leaf_vals + a, min(s.sub_size, s.nLeaves - a), sv, sv + kTreeStage);
      if (threadIdx.x == 0) s.sub_vals[t] = r;
    }
    return;
  }
  for (int u = u0; u < n; u += G) {
    const int t = u < n0 ? s.sub_own0 + u : s.sub_own2 + (u - n0);
    const int l0 = s.sub_leaf[t], l1 = s.sub_leaf[t + 1];
    for (int k = threadIdx.x; k < l1 - l0; k += blockDim.x) sv[k] = ldcg(s.leaf_vals + l0 + k);
    __syncthreads();
    const double r = eval_prog(s.progs + s.sub_prog[t], sv);
    if (threadIdx.x == 0) s.sub_vals[t] = r;
  }
}

static __device__ __noinline__ double sum_phase2(const SumDev& s, double* sv) {
  if (s.nSub <= 1) return sum_single(s, sv);
  if (s.regular) return tree_reduce_cta(s.sub_vals, s.nSub, sv, sv + kTreeStage);
  for (int k = threadIdx.x; k < s.nSub; k += blockDim.x) sv[k] = ldcg(s.sub_vals + k);
  __syncthreads();
  return eval_prog(s.progs + s.top_prog, sv);
}

static __device__ __noinline__ double fold_pow2_big(const double* c, int chunk) { return fold_pow2(c, chunk); }

// Reduce k (<= 8) sums: phase 1 (distributed subtrees) for two-level sums and
// one grid barrier if there are any; then every regular sum (its leaves, or
// its subtree roots) is folded in ONE batched CTA pass — all loads in
// flight together (16-byte async copies), per-thread perfect-tree chunks,
// xor-shuffles across lanes, then every warp folds the warp partials itself
// (no broadcast round).  Irregular (program) sums fall back to the
// level-by-level evaluator.  out[i] valid in every thread of every CTA.
// Out of line and loop-based on purpose: it is called from every decision
// point of the persistent kernels, and a straight-line copy per call site
// (~5k instructions each) made instruction fetch its dominant cost.
static __device__ __noinline__ void reduce_list(const SumDev* const* ss, int k, double* out, double* sv,
                                         GridBarrier& gb, unsigned long long* tr) {
  const bool stamp = tr && blockIdx.x == 0 && threadIdx.x == 0;
  long long c0 = stamp ? clock64() : 0;
  auto lap = [&](int slot) {
    if (stamp) {
      const long long c = clock64();
      tr[slot] += (unsigned long long)(c - c0);
      c0 = c;
    }
  };
  bool two = false, irregular = false;
  int total = 0, off = 0;
#pragma unroll 1
  for (int i = 0; i < k; ++i) {
    const SumDev& s = *ss[i];
    if (s.nSub > 1) {
      two = true;
      sum_phase1(s, sv, off);
      off += s.nSub;
    }
    if (s.regular) {
      const int n = s.nSub > 1 ? s.nSub : s.nLeaves;
      const int P = n <= 1 ? 1 : 1 << (32 - __clz(n - 1));
      total += (P + 1) & ~1;   // keep every base 16-byte aligned
    } else {
      irregular = true;
    }
  }
  if (two) gb.sync();
  lap(0);
  if (total > kTreeStage) {
#pragma unroll 1
    for (int i = 0; i < k; ++i) out[i] = sum_phase2(*ss[i], sv);
    return;
  }
  const int BD = blockDim.x;
  const int T = 1 << (31 - __clz(BD));          // folding threads (power of two)
  // stage all regular sums with asynchronous copies: every element of every
  // sum is in flight at once (zero-filled past n), one wait for all
  int base = 0;
#pragma unroll 1
  for (int i = 0; i < k; ++i) {
    const SumDev& s = *ss[i];
    if (!s.regular) continue;
    const int n = s.nSub > 1 ? s.nSub : s.nLeaves;
    const int P = n <= 1 ? 1 : 1 << (32 - __clz(n - 1));
    const double* src = s.nSub > 1 ? s.sub_vals : s.leaf_vals;
    if (P == 1) {
      if (threadIdx.x == 0) cp_async8(sv + base, src, n > 0);
    } else {
      // pairs: base and P are even, sources 256-byte aligned
#pragma unroll 1
      for (int e = 2 * threadIdx.x; e < P; e += 2 * BD)
        cp_async16(sv + base + e, src + (e < n ? e : 0), min(max(n - e, 0), 2) * 8);
    }
    base += (P + 1) & ~1;
  }
  lap(1);
  cp_async_wait_all();
  __syncthreads();
  lap(2);
  double* red = sv + kTreeStage;   // 8 x 32 warp partials
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = BD >> 5;
  base = 0;
#pragma unroll 1
  for (int i = 0; i < k; ++i) {
    const SumDev& s = *ss[i];
    if (!s.regular) continue;
    const int n = s.nSub > 1 ? s.nSub : s.nLeaves;
    const int P = n <= 1 ? 1 : 1 << (32 - __clz(n - 1));
    const int chunk = P > T ? P / T : 1;
    const double* c = sv + base + threadIdx.x * chunk;
    double root = 0.0;
    if (threadIdx.x * chunk < P) root = chunk <= 16 ? fold_small(c, chunk) : fold_pow2_big(c, chunk);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) root = root + __shfl_xor_sync(kFull, root, o);
    if (lane == 0) red[i * 32 + warp] = root;
    base += (P + 1) & ~1;
  }
  __syncthreads();
  lap(3);
  // every warp folds the warp partials (identical order in all warps)
#pragma unroll 1
  for (int i = 0; i < k; ++i) {
    if (!ss[i]->regular) continue;
    double t = lane < nw ? red[i * 32 + lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) t = t + __shfl_xor_sync(kFull, t, o);
    out[i] = t;
  }
  __syncthreads();   // red / staging are reused by the caller's next shared-memory phase
  if (irregular) {
#pragma unroll 1
    for (int i = 0; i < k; ++i)
      if (!ss[i]->regular) out[i] = sum_phase2(*ss[i], sv);
  }
  lap(4);
  if (stamp) tr[7] += 1;
}

// Hot-path form of reduce_list for K sums known at the call site: when every
// sum is a regular single-level tree and the batch fits the staging area,
// all descriptor reads, copies, folds and shuffles of the K sums are
// independent (unrolled) so their latencies overlap; otherwise the generic
// out-of-line routine runs.  Same tree order, same results.
// OWN: give the out-of-line fallback its own stack copies (see below); used by
// the register-rich c2 kernel, while the 168-register RW = 4 kernels keep the
// shared arrays (the copies cost them spills).
template <int K, bool OWN = false>
__device__ __forceinline__ void reduce_k(const SumDev* const (&ss)[K], double* out, double* sv, GridBarrier& gb,
                                         unsigned long long* tr) {
  const bool stamp = tr && blockIdx.x == 0 && threadIdx.x == 0;
  long long c0 = stamp ? clock64() : 0;
  auto lap = [&](int slot) {
    if (stamp) {
      const long long c = clock64();
      tr[slot] += (unsigned long long)(c - c0);
      c0 = c;
    }
  };
  int n[K], P[K];
  const double* src[K];
  bool fast = true, two = false;
  int total = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const SumDev& s = *ss[i];
    fast = fast && s.regular;
    two = two || s.nSub > 1;
    n[i] = s.nSub > 1 ? s.nSub : s.nLeaves;
    P[i] = n[i] <= 1 ? 1 : 1 << (32 - __clz(n[i] - 1));
    src[i] = s.nSub > 1 ? s.sub_vals : s.leaf_vals;
    total += (P[i] + 1) & ~1;
  }
  if ((!fast || total > kTreeStage) && !OWN) {
    reduce_list(ss, K, out, sv, gb, tr);
    return;
  }
  if (!fast || total > kTreeStage) {
    // the out-of-line routine takes addresses: give it its own copies so the
    // caller's descriptor and result arrays stay in registers on the fast
    // path (a stack copy is re-read from L2 after the grid barrier's acquire)
    const SumDev* tss[K];
    double tout[K];
#pragma unroll
    for (int i = 0; i < K; ++i) tss[i] = ss[i];
    reduce_list(tss, K, tout, sv, gb, tr);
#pragma unroll
    for (int i = 0; i < K; ++i) out[i] = tout[i];
    return;
  }
  if (two) {
    // phase 1: subtrees of the two-level sums, spread over the CTAs
    int off = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (ss[i]->nSub > 1) {
        sum_phase1(*ss[i], sv, off);
        off += ss[i]->nSub;
      }
    }
    gb.sync();
    lap(0);
  }
  const int BD = blockDim.x;
  const int lgT = 31 - __clz(BD);
  const int T = 1 << lgT;
  bool small = true;
#pragma unroll
  for (int i = 0; i < K; ++i) small = small && P[i] <= 4 * T;
  double root[K];
  if (small) {
    // every folding thread's chunk (<= 4 contiguous units) goes straight
    // from L2 into registers: the loads of all K sums are in flight at once,
    // no shared-memory staging; zero padding past n, perfect-tree fold
    double v[K][4];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int chunk = P[i] > T ? P[i] >> lgT : 1;
      const int e0 = threadIdx.x * chunk;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int e = e0 + m;
        v[i][m] = (m < chunk && e < n[i] && (int)threadIdx.x < T) ? ldcg(src[i] + e) : 0.0;
      }
    }
    lap(1);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int chunk = P[i] > T ? P[i] >> lgT : 1;
      root[i] = chunk == 1 ? v[i][0] : chunk == 2 ? v[i][0] + v[i][1] : (v[i][0] + v[i][1]) + (v[i][2] + v[i][3]);
    }
    lap(2);
  } else {
    int base = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (P[i] == 1) {
        if (threadIdx.x == 0) cp_async8(sv + base, src[i], n[i] > 0);
      } else {
        for (int e = 2 * threadIdx.x; e < P[i]; e += 2 * BD)
          cp_async16(sv + base + e, src[i] + (e < n[i] ? e : 0), min(max(n[i] - e, 0), 2) * 8);
      }
      base += (P[i] + 1) & ~1;
    }
    lap(1);
    cp_async_wait_all();
    __syncthreads();
    lap(2);
    base = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int chunk = P[i] > T ? P[i] >> lgT : 1;
      root[i] = 0.0;
      if (threadIdx.x * chunk < P[i])
        root[i] = chunk <= 16 ? fold_small(sv + base + threadIdx.x * chunk, chunk)
                              : fold_pow2_big(sv + base + threadIdx.x * chunk, chunk);
      base += (P[i] + 1) & ~1;
    }
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < K; ++i) root[i] = root[i] + __shfl_xor_sync(kFull, root[i], o);
  double* red = sv + kTreeStage;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = BD >> 5;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) red[i * 32 + warp] = root[i];
  }
  __syncthreads();
  lap(3);
#pragma unroll
  for (int i = 0; i < K; ++i) root[i] = lane < nw ? red[i * 32 + lane] : 0.0;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < K; ++i) root[i] = root[i] + __shfl_xor_sync(kFull, root[i], o);
#pragma unroll
  for (int i = 0; i < K; ++i) out[i] = root[i];
  __syncthreads();
  lap(4);
  if (stamp) tr[7] += 1;
}

// Tile partial (ddot-type): per-thread accumulation in a fixed order then
// block_sum; thread 0 stores the partial for `tile`.
// Same tree as block_sum (xor-shuffles 16..1, then warp 0 over the warp
// partials), but only thread 0 needs the result: no broadcast round, two
// CTA barriers instead of four.
__device__ __forceinline__ void store_tile_partial(const SumDev& s, int tile, double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  __syncthreads();   // every warp is past earlier reads of red
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
    if (lane == 0) s.leaf_vals[tile] = t;
  }
}

}  // namespace adp
