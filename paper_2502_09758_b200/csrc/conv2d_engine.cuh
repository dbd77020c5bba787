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
//     Threads are channel-parallel: thread = (channel, row, RW-column group).
//     Loaders walk tile rows warp by warp (coalesced, no integer division),
//     with 8 loads in flight per lane.  Shared memory is addressed through
//     byte offsets from the dynamic window (LDS/STS, never generic).
//   * Strict mode reproduces scipy.ndimage.correlate bit for bit: taps in
//     row-major order, acc = 0.0 then acc + x*w (no FMA), taps with
//     |w| <= DBL_EPSILON skipped.  Fast mode uses FMA.
//   * Element sums the reference takes with np.sum use NumPy's pairwise
//     tree (bitwise).  When the layout is regular and leaf-aligned with the
//     tiles, each tile computes its leaves from shared memory ("fused");
//     otherwise the terms go to global memory and a leaf pass follows.
//     ddot-type sums (norms, vdot) use fixed per-tile trees.
#pragma once
#include "adp_device.cuh"
#include "conv2d_args.h"

namespace adp {

__device__ __forceinline__ unsigned char* dsm() {
  extern __shared__ __align__(16) unsigned char adp_dyn_smem[];
  return adp_dyn_smem;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// sub-phase SM-cycle stamps (CTA 0, thread 0), accumulated over calls:
// trace[1024 + k] += t_{k+1} - t_k, trace[1023 + 64] counts calls
#define ADP_SUB(k)                                                                  \
  do {                                                                              \
    if (a.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0) sub_t[k] = clock64(); \
  } while (0)
#define ADP_SUB_FLUSH(n)                                                            \
  do {                                                                              \
    if (a.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0) {                      \
      for (int k_ = 0; k_ + 1 < (n); ++k_)                                          \
        a.trace[1152 + (threadIdx.x >> 5) * 8 + k_] += (unsigned long long)(sub_t[k_ + 1] - sub_t[k_]); \
      if (threadIdx.x == 0) a.trace[1024 + 63] += 1;                                \
    }                                                                               \
  } while (0)

// ---------------------------------------------------------------------------
// value sources used by the tile loaders (each computes exactly the
// reference expression for one element)
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

// ---------------------------------------------------------------------------
// KS > 0: the stencil size is a compile-time constant (the latency-bound c2
// solve kernel is instantiated with KS = 9 so it carries no other stencil
// variant); KS = 0: runtime dispatch over the unrolled sizes + generic loop.
// PW: the stencil taps come from a kernel-parameter array (constant bank 0,
// the host-stepped stage kernels: StepW) instead of shared memory; warps are
// channel-uniform (tpc % 32 == 0, host check), so the channel index is moved
// to a uniform register and every tap is an LDCU into the uniform register
// file feeding DMUL's second operand: no shared-memory wavefronts or vector
// registers for the weights, no per-CTA weight staging.
// KD > 0 (host-stepped stage kernels): the kernel serves KD x KD stencils only (any channel count),
// so it carries one stencil variant; KU: rows of that stencil unrolled per loop iteration (KD % KU == 0;
// KU == KD: straight-line code) -- the instruction footprint of the hot path against the instruction caches.
template <typename T, bool FAST, int RW, int KS = 0, bool TMA = false, bool PW = false, int KD = 0, int KU = 0>
struct Conv {
  static_assert((RW & (RW - 1)) == 0, "RW must be a power of two");
  static constexpr int kShift = RW == 1 ? 0 : RW == 2 ? 1 : RW == 4 ? 2 : 3;
  static constexpr int kB = 8;   // loads in flight per lane in the tile loaders

  const ConvArgs<T>& a;
  int ch, ty, tx;                // this thread's channel, tile row, column group
  int tb0, tbs;                  // stageA / stageC tile walk: first tile, stride (default: the grid)
  bool opsm = false;             // stageA / stageC (fused, float64): epilogue operands staged in the term
                                 // buffers by asynchronous copies instead of registers held across the stencil
  const T* pw = nullptr;         // PW: the launch's tap set in parameter space ([c][i][j], forward or flipped)
  int chu = 0;                   // PW: ch in a uniform register

  __device__ __forceinline__ int nC() const { return KS > 0 ? 1 : a.g.C; }
  // plane column of box column `col` (box column 0 = image column w0 - rw - 1):
  // skewed (one pad per RW elements) for LDS-fed boxes; dense and shifted by
  // one for TMA boxes (the TMA box starts at w0 - rw - 2 so the RW = 2 windows
  // start on 16-byte boundaries: LDS.128 window loads, conflict-free)
  __device__ static __forceinline__ int sk(int col) { return TMA ? col + 1 : RW == 1 ? col : col + (col >> kShift); }
  __device__ static __forceinline__ int skr(int m) { return TMA ? m : RW == 1 ? m : m + (m >> kShift); }
  __device__ __forceinline__ int swp() const { return TMA ? a.g.SWPt : a.g.SWP; }

  __device__ explicit Conv(const ConvArgs<T>& a_) : a(a_), tb0(blockIdx.x), tbs(gridDim.x) {
    const int tpr = a.g.TW / RW;
    // KS > 0 instances serve single-channel images only (host check), so the
    // channel index and count are compile-time
    ch = KS > 0 ? 0 : (int)(threadIdx.x / a.g.tpc);
    if constexpr (PW) chu = __reduce_max_sync(0xffffffffu, ch);
    const int r = threadIdx.x - ch * a.g.tpc;
    ty = r / tpr;
    tx = r - ty * tpr;
  }

  // ---- shared-memory views (byte offsets from the dynamic window)
  // dynamic shared-memory base; TMA kernels shift it to the next 128-byte
  // boundary (TMA destinations; the host adds 128 bytes to the allocation)
  __device__ __forceinline__ unsigned char* sbase() const {
    if constexpr (TMA) {
      unsigned char* b = dsm();
      const unsigned o = (unsigned)__cvta_generic_to_shared(b);
      return b + ((128u - (o & 127u)) & 127u);
    } else {
      return dsm();
    }
  }
  __device__ __forceinline__ double* red() const { return reinterpret_cast<double*>(sbase()); }
  __device__ __forceinline__ T* ws() const { return reinterpret_cast<T*>(sbase() + a.g.o_ws); }
  __device__ __forceinline__ T* wf() const { return reinterpret_cast<T*>(sbase() + a.g.o_wf); }
  __device__ __forceinline__ T* pa() const { return reinterpret_cast<T*>(sbase() + a.g.o_pa); }
  __device__ __forceinline__ T* pa2() const { return reinterpret_cast<T*>(sbase() + a.g.o_pa2); }
  __device__ __forceinline__ double* tm() const { return reinterpret_cast<double*>(sbase() + a.g.o_tm); }
  __device__ __forceinline__ double* sv() const { return reinterpret_cast<double*>(sbase() + a.g.o_sv); }
  __device__ __forceinline__ T* plane(int c) const { return pa() + (size_t)c * a.g.SH * swp(); }
  // this thread's channel taps: forward (correlation) and flipped (adjoint);
  // PW kernels carry exactly one of the two sets, chosen by the host
  // (PW: channel blocks padded to an even tap count, so tap pairs are 16-byte aligned)
  __device__ __forceinline__ const T* wfwd() const {
    if constexpr (PW) return pw + chu * ((a.g.kh * a.g.kw + 1) & ~1);
    else return ws() + ch * a.g.kh * a.g.kw;
  }
  __device__ __forceinline__ const T* wadj() const {
    if constexpr (PW) return pw + chu * ((a.g.kh * a.g.kw + 1) & ~1);
    else return wf() + ch * a.g.kh * a.g.kw;
  }

  // ---- weights: ws[c][i][j] = kern[i][j][c] (|w| <= eps -> 0), wf flipped
  __device__ void load_weights(const T* kern) {
    const int kh = a.g.kh, kw = a.g.kw, C = nC(), nk = kh * kw * C;
    T* s = ws();
    T* f = wf();
    for (int e = threadIdx.x; e < nk; e += blockDim.x) {
      const int c = e % C, ij = e / C, i = ij / kw, j = ij % kw;
      T w = kern[e];
      if (!(fabs((double)w) > kDblEps)) w = T(0);  // ndimage: only |w| > DBL_EPSILON taps
      s[(c * kh + i) * kw + j] = w;
      f[(c * kh + (kh - 1 - i)) * kw + (kw - 1 - j)] = w;
    }
    __syncthreads();
  }
  // squared flipped taps (gram_diag: correlate(ones, flipped**2), operators.py:120-122)
  __device__ void load_weights_sq(const T* kern) {
    const int kh = a.g.kh, kw = a.g.kw, C = nC(), nk = kh * kw * C;
    T* f = wf();
    __syncthreads();
    for (int e = threadIdx.x; e < nk; e += blockDim.x) {
      const int c = e % C, ij = e / C, i = ij / kw, j = ij % kw;
      T w = kern[e];
      w = w * w;
      if (!(fabs((double)w) > kDblEps)) w = T(0);
      f[(c * kh + (kh - 1 - i)) * kw + (kw - 1 - j)] = w;
    }
    __syncthreads();
  }

  // n / d for n < 2^16 with m = ceil(2^32 / d); m == 0 encodes d == 1
  __device__ static __forceinline__ int mdiv(int n, unsigned m) { return m ? (int)__umulhi((unsigned)n, m) : n; }
  __device__ __forceinline__ int tile_row(int tile) const { return mdiv(tile, a.g.magicTW); }
  __device__ __forceinline__ void tile_origin(int tile, int& h0, int& w0) const {
    const int tr = tile_row(tile);
    h0 = tr * a.g.TH;
    w0 = (tile - tr * a.g.tilesW) * a.g.TW;
  }
  __device__ __forceinline__ int64_t gidx(int h, int w, int c) const {
    return ((int64_t)h * a.g.W + w) * nC() + c;
  }

  // ---- load tile + (r+1) halo of all channels into the planes.  One warp
  // per tile row (a contiguous run of global memory), lanes over elements,
  // kB loads per lane in flight before any store.
  // element k of the flattened (row, interleaved column) tile box -> global
  // index (or -1 when outside the image) and plane offset
  __device__ __forceinline__ void box_elem(int k, int gh0, int gw0, int64_t& gi, int& off) const {
    const int C = nC(), rowE = (a.g.TW + 2 * a.g.rw + 2) * C;
    const int sr = (int)(((unsigned long long)k * a.g.magicRow) >> 32);
    const int e = k - sr * rowE;
    const int px = (int)(((unsigned long long)e * a.g.magicC) >> 20);
    const int c = e - px * C;
    const int gh = gh0 + sr, gw = gw0 + px;
    off = c * a.g.SH * swp() + sr * swp() + sk(px);
    gi = (gh >= 0 && gh < a.g.H && gw >= 0 && gw < a.g.W) ? ((int64_t)gh * a.g.W + gw) * C + c : -1;
  }

  // Tile-box loader: warps own rows (each a contiguous run of global
  // memory), lanes walk the row's interleaved elements; two rows per warp
  // in flight, predicated (branch-free) loads, geometry in registers.
  static constexpr int kJ = 8;   // lane steps per row handled per pass (rows longer than 256 loop)
  template <class Src>
  __device__ void load_full(int h0, int w0, const Src& src, T* dst_region = nullptr) const {
    const int C = nC(), H = a.g.H, W = a.g.W, SH = a.g.SH, SWP = swp();
    const unsigned mC = a.g.magicC;
    const int rowE = (a.g.TW + 2 * a.g.rw + 2) * C, planeSz = SH * SWP;
    const int gh0 = h0 - a.g.rh - 1, gw0 = w0 - a.g.rw - 1;
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    T* dst = dst_region ? dst_region : pa();
    if (C == 1) {
      // single channel: element = pixel, no de-interleave
      for (int e0 = 0; e0 < rowE; e0 += 32 * kJ) {
        for (int sr0 = threadIdx.x >> 5; sr0 < SH; sr0 += 2 * nw) {
          T v[2][kJ];
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int sr = sr0 + rr * nw;
            const int gh = gh0 + sr;
            const bool rowok = sr < SH && gh >= 0 && gh < H;
            const int64_t rowbase = (int64_t)gh * W + gw0;
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
              const int e = e0 + lane + 32 * j;
              const bool ok = rowok && e < rowE && (unsigned)(gw0 + e) < (unsigned)W;
              v[rr][j] = ok ? src(rowbase + e) : T(0);
            }
          }
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int sr = sr0 + rr * nw;
            if (sr < SH) {
              T* drow = dst + sr * SWP;
#pragma unroll
              for (int j = 0; j < kJ; ++j) {
                const int e = e0 + lane + 32 * j;
                if (e < rowE) drow[sk(e)] = v[rr][j];
              }
            }
          }
        }
      }
      return;
    }
    for (int e0 = 0; e0 < rowE; e0 += 32 * kJ) {
      for (int sr0 = threadIdx.x >> 5; sr0 < SH; sr0 += 2 * nw) {
        T v[2][kJ];
        int off[2][kJ];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int sr = sr0 + rr * nw;
          const int gh = gh0 + sr;
          const bool rowok = sr < SH && gh >= 0 && gh < H;
          const int64_t rowbase = ((int64_t)gh * W + gw0) * C;
#pragma unroll
          for (int j = 0; j < kJ; ++j) {
            const int e = e0 + lane + 32 * j;
            const int px = (int)(((unsigned long long)(unsigned)e * mC) >> 20);
            const int c = e - px * C;
            const int gw = gw0 + px;
            const bool ok = rowok && e < rowE && (unsigned)gw < (unsigned)W;
            off[rr][j] = (sr < SH && e < rowE) ? c * planeSz + sr * SWP + sk(px) : -1;
            v[rr][j] = ok ? src(rowbase + e) : T(0);
          }
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
          for (int j = 0; j < kJ; ++j)
            if (off[rr][j] >= 0) dst[off[rr][j]] = v[rr][j];
      }
    }
  }
  // plain copies: asynchronous global -> shared (LDGSTS), zero fill outside;
  // the caller's __syncthreads() after cp_async_wait_all() publishes them
  __device__ void load_copy(int h0, int w0, const T* x) const {
    const int total = a.g.SH * (a.g.TW + 2 * a.g.rw + 2) * nC();
    const int gh0 = h0 - a.g.rh - 1, gw0 = w0 - a.g.rw - 1;
    T* dst = pa();
    for (int k = threadIdx.x; k < total; k += blockDim.x) {
      int64_t gi;
      int off;
      box_elem(k, gh0, gw0, gi, off);
      const unsigned d = (unsigned)__cvta_generic_to_shared(dst + off);
      const T* s = x + (gi >= 0 ? gi : 0);
      if (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(s), "r"(gi >= 0 ? 8 : 0) : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(s), "r"(gi >= 0 ? 4 : 0) : "memory");
    }
    cp_async_wait_all();
  }

  // Asynchronous copy (LDGSTS) of the tile box of a plain array into a plane
  // region, zero-filled outside the image: warps own box rows (contiguous in
  // global memory), lanes walk the row's interleaved elements.  The caller
  // commits the group and waits before the barrier that publishes it.
  __device__ void load_async(int h0, int w0, const T* x, T* dst) const {
    const int C = nC(), H = a.g.H, W = a.g.W, SH = a.g.SH, SWP = swp();
    const unsigned mC = a.g.magicC;
    const int rowE = (a.g.TW + 2 * a.g.rw + 2) * C, planeSz = SH * SWP;
    const int gh0 = h0 - a.g.rh - 1, gw0 = w0 - a.g.rw - 1;
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const unsigned sdst = (unsigned)__cvta_generic_to_shared(dst);
    for (int e0 = 0; e0 < rowE; e0 += 32 * kJ) {
      // the lane's (up to kJ) elements of a box row: their plane offsets and column validity are
      // the same for every row, so the de-interleave arithmetic runs once per pass, not per element
      unsigned soff[kJ];
      unsigned inb = 0, okc = 0;
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int e = e0 + lane + 32 * j;
        const int px = C == 1 ? e : (int)(((unsigned long long)(unsigned)e * mC) >> 20);
        const int c = e - px * C;
        soff[j] = (unsigned)((c * planeSz + sk(px)) * (int)sizeof(T));
        if (e < rowE) inb |= 1u << j;
        if (e < rowE && (unsigned)(gw0 + px) < (unsigned)W) okc |= 1u << j;
      }
      for (int sr = threadIdx.x >> 5; sr < SH; sr += nw) {
        const int gh = gh0 + sr;
        const bool rowok = gh >= 0 && gh < H;
        const T* grow = x + ((int64_t)(rowok ? gh : 0) * W + gw0) * C + (e0 + lane);
        const unsigned srow = sdst + (unsigned)(sr * SWP * (int)sizeof(T));
        const unsigned okr = rowok ? okc : 0u;
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
          if ((inb >> j) & 1u) {
            const bool ok = (okr >> j) & 1u;
            const T* src = ok ? grow + 32 * j : x;
            if (sizeof(T) == 8)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(srow + soff[j]), "l"(src),
                           "r"(ok ? 8 : 0)
                           : "memory");
            else
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(srow + soff[j]), "l"(src),
                           "r"(ok ? 4 : 0)
                           : "memory");
          }
        }
      }
    }
  }
  __device__ __forceinline__ T* qs() const { return reinterpret_cast<T*>(sbase() + a.g.o_q); }

  // window of NW box elements starting one past the row base: scalar loads
  // on the skewed layout; 16-byte loads on the (aligned) dense TMA layout
  template <int NW>
  __device__ __forceinline__ void load_win(const T* row, T (&win)[NW]) const {
    if constexpr (TMA && sizeof(T) == 8 && NW % 2 == 0 && RW % 2 == 0) {
      const double2* r2 = reinterpret_cast<const double2*>(row + 1);
#pragma unroll
      for (int m = 0; m < NW / 2; ++m) {
        const double2 v = r2[m];
        win[2 * m] = v.x;
        win[2 * m + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int m = 0; m < NW; ++m) win[m] = row[skr(1 + m)];
    }
  }

  // ---- TMA tile boxes (KS = 9 single-channel kernel): one 2-D tensor copy
  // per box (cp.async.bulk.tensor, zero fill outside the image), completion on
  // an mbarrier.  Thread 0 issues; every thread waits on the barrier's phase.
  __device__ __forceinline__ static unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
  }
  __device__ __forceinline__ void tma_box(const CUtensorMap* tm, int h0, int w0, T* dst, unsigned long long* mbar) const {
    if (threadIdx.x == 0) {
      const unsigned bar = smem_u32(mbar);
      const unsigned bytes = (unsigned)(a.g.SH * a.g.SWPt * sizeof(T));
      // generic-proxy writes (other CTAs' global stores before the grid barrier, this
      // CTA's earlier reads of dst) ordered before the async-proxy copy
      asm volatile("fence.proxy.async;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(dst)),
          "l"(tm), "r"(w0 - a.g.rw - 2), "r"(h0 - a.g.rh - 1), "r"(bar)
          : "memory");
    }
  }
  __device__ __forceinline__ static void tma_wait(unsigned long long* mbar, unsigned phase) {
    const unsigned bar = smem_u32(mbar);
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar), "r"(phase)
          : "memory");
    }
  }

  // ---- register-blocked correlation: RW consecutive outputs (row ty, cols
  // tx*RW..) of the thread's channel plane with stencil w (kh x kw).  Per
  // output the taps are accumulated in row-major order starting from 0.
  // Compile-time K x K form (the benchmark stencils): fully unrolled, so the
  // window and tap loads of a row are issued together with immediate
  // offsets and their latency overlaps the multiply-add chains.  Same tap
  // order as the generic loop.
  template <int K>
  __device__ __forceinline__ void stencil_k(const T* __restrict__ pl, const T* __restrict__ w, T (&acc)[RW]) const {
    const int SWP = swp();
    const T* base = pl + (ty + 1) * SWP + sk(tx * RW);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const T* row = base + i * SWP;
      T win[K + RW - 1];
      load_win<K + RW - 1>(row, win);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const T wt = w[i * K + j];
#pragma unroll
        for (int o = 0; o < RW; ++o) acc[o] = madd<FAST>(acc[o], win[o + j], wt);
      }
    }
  }

  // PW form of stencil_k: the taps are read from parameter space as 16-byte pairs (flattened
  // row-major tap index t: pair t >> 1; the channel blocks are padded to an even tap count), half
  // the uniform loads of the scalar form.  Same tap order.
  template <int K>
  __device__ __forceinline__ void stencil_kp(const T* __restrict__ pl, const T* __restrict__ w, T (&acc)[RW]) const {
    static_assert(sizeof(T) == 8, "parameter-space taps: float64 only");
    const int SWP = swp();
    const T* base = pl + (ty + 1) * SWP + sk(tx * RW);
    const double2* w2 = reinterpret_cast<const double2*>(w);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const T* row = base + i * SWP;
      T win[K + RW - 1];
      load_win<K + RW - 1>(row, win);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int t = i * K + j;
        const double2 wp = w2[t >> 1];
        const T wt = (t & 1) ? wp.y : wp.x;
#pragma unroll
        for (int o = 0; o < RW; ++o) acc[o] = madd<FAST>(acc[o], win[o + j], wt);
      }
    }
  }

  // K x K taps with the row loop unrolled U rows at a time (K % U == 0), taps from parameter space
  // (scalar uniform loads, row index in a uniform register).  Same tap order as stencil_k.
  template <int K, int U>
  __device__ __forceinline__ void stencil_ku(const T* __restrict__ pl, const T* __restrict__ w, T (&acc)[RW]) const {
    static_assert(K % U == 0, "row unroll must divide the stencil height");
    const int SWP = swp();
    const T* base = pl + (ty + 1) * SWP + sk(tx * RW);
#pragma unroll 1
    for (int i0 = 0; i0 < K; i0 += U) {
#pragma unroll
      for (int ii = 0; ii < U; ++ii) {
        const T* row = base + (i0 + ii) * SWP;
        const T* wr = w + (i0 + ii) * K;
        T win[K + RW - 1];
        load_win<K + RW - 1>(row, win);
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const T wt = wr[j];
#pragma unroll
          for (int o = 0; o < RW; ++o) acc[o] = madd<FAST>(acc[o], win[o + j], wt);
        }
      }
    }
  }

  // Two planes through the same compile-time K x K taps (the fused candidate
  // stage): each tap is loaded once for both accumulations; per output the
  // order is exactly stencil_k's.
  template <int K>
  __device__ __forceinline__ void stencil_k2(const T* __restrict__ pl1, const T* __restrict__ pl2,
                                             const T* __restrict__ w, T (&acc1)[RW], T (&acc2)[RW]) const {
    const int SWP = swp();
    const int b = (ty + 1) * SWP + sk(tx * RW);
#pragma unroll
    for (int o = 0; o < RW; ++o) acc1[o] = acc2[o] = T(0);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const T* row1 = pl1 + b + i * SWP;
      const T* row2 = pl2 + b + i * SWP;
      T win1[K + RW - 1], win2[K + RW - 1];
      load_win<K + RW - 1>(row1, win1);
      load_win<K + RW - 1>(row2, win2);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const T wt = w[i * K + j];
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          acc1[o] = madd<FAST>(acc1[o], win1[o + j], wt);
          acc2[o] = madd<FAST>(acc2[o], win2[o + j], wt);
        }
      }
    }
  }
  // forward taps over two regions; the compile-time-K kernels share the tap loads
  __device__ __forceinline__ void stencil_fwd_pair(const T* pr1, const T* pr2, T (&acc1)[RW], T (&acc2)[RW]) const {
    const size_t co = (size_t)ch * a.g.SH * swp();
    const T* w = wfwd();
    if constexpr (KS > 0) {
      stencil_k2<KS>(pr1 + co, pr2 + co, w, acc1, acc2);
    } else {
      stencil(pr1 + co, w, acc1);
      stencil(pr2 + co, w, acc2);
    }
  }

  // Large K (c5: 31): rows stay a runtime loop (code size), each row fully
  // unrolled so its window and taps are loaded together.
  template <int K>
  __device__ __forceinline__ void stencil_kr(const T* __restrict__ pl, const T* __restrict__ w, T (&acc)[RW]) const {
    const int SWP = swp();
    const T* base = pl + (ty + 1) * SWP + sk(tx * RW);
#pragma unroll 1
    for (int i = 0; i < K; ++i) {
      const T* row = base + i * SWP;
      const T* wr = w + i * K;
      T win[K + RW - 1];
#pragma unroll
      for (int m = 0; m < K + RW - 1; ++m) win[m] = row[skr(1 + m)];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const T wt = wr[j];
#pragma unroll
        for (int o = 0; o < RW; ++o) acc[o] = madd<FAST>(acc[o], win[o + j], wt);
      }
    }
  }

  __device__ __forceinline__ void stencil(const T* __restrict__ pl, const T* __restrict__ w, T (&acc)[RW]) const {
#pragma unroll
    for (int o = 0; o < RW; ++o) acc[o] = T(0);
    if constexpr (KS > 0) {
      stencil_k<KS>(pl, w, acc);
      return;
    }
    if constexpr (KD > 0) {   // the host selected this instance for KD x KD stencils
      if constexpr (KU > 0 && KU < KD) stencil_ku<KD, KU>(pl, w, acc);
      else if constexpr (PW) stencil_kp<KD>(pl, w, acc);
      else stencil_k<KD>(pl, w, acc);
      return;
    }
    const int kh = a.g.kh, kw = a.g.kw, SWP = swp();
    if (kh == 9 && kw == 9) {
      if constexpr (PW) stencil_kp<9>(pl, w, acc);
      else stencil_k<9>(pl, w, acc);
      return;
    }
    if (kh == 15 && kw == 15) {
      if constexpr (PW) stencil_kp<15>(pl, w, acc);
      else stencil_k<15>(pl, w, acc);
      return;
    }
    if (kh == 31 && kw == 31) {
      stencil_kr<31>(pl, w, acc);
      return;
    }
    // phys(tx*RW + m) = sk(tx*RW) + skr(m); separable because tx*RW and the
    // j-block starts are multiples of RW
    const T* base = pl + (ty + 1) * SWP + sk(tx * RW);
    for (int i = 0; i < kh; ++i) {
      const T* row = base + i * SWP;
      const T* wr = w + i * kw;
      T win[RW];
#pragma unroll
      for (int q = 0; q < RW - 1; ++q) win[q] = row[skr(1 + q)];
      int j = 0;
      for (; j + RW <= kw; j += RW) {
        const T* rj = row + skr(j);
#pragma unroll
        for (int jj = 0; jj < RW; ++jj) {
          const int q = jj + RW - 1;
          win[(jj + RW - 1) % RW] = rj[skr(1 + q)];
          const T wt = wr[j + jj];
#pragma unroll
          for (int o = 0; o < RW; ++o) acc[o] = madd<FAST>(acc[o], win[(o + jj) % RW], wt);
        }
      }
      if (j < kw) {
        const T* rj = row + skr(j);
#pragma unroll
        for (int jj = 0; jj < RW - 1; ++jj) {
          if (j + jj < kw) {
            const int q = jj + RW - 1;
            win[(jj + RW - 1) % RW] = rj[skr(1 + q)];
            const T wt = wr[j + jj];
#pragma unroll
            for (int o = 0; o < RW; ++o) acc[o] = madd<FAST>(acc[o], win[(o + jj) % RW], wt);
          }
        }
      }
    }
  }
  __device__ __forceinline__ void stencil_fwd(T (&acc)[RW]) const {
    stencil(plane(ch), wfwd(), acc);
  }
  __device__ __forceinline__ void stencil_adj(T (&acc)[RW]) const {
    stencil(plane(ch), wadj(), acc);
  }

  // plane value of this thread's channel at tile pixel (r, q)
  __device__ __forceinline__ T fp(int r, int q) const {
    return plane(ch)[(r + a.g.rh + 1) * swp() + sk(q + a.g.rw + 1)];
  }

  // TV edges are those of the GLOBAL image (a row slab sees its global row
  // index h + row0); the zero padding of the stencils is that of the local
  // array, whose outer rows are either global edges or ghost rows.
  __device__ __forceinline__ bool has_below(int h) const { return h + a.g.row0 < a.g.Hg - 1; }
  __device__ __forceinline__ bool has_above(int h) const { return h + a.g.row0 >= 1; }
  // sums cover owned rows only, indexed globally (tiles are TH-aligned, so a
  // tile is wholly owned or not)
  __device__ __forceinline__ bool tile_owned(int h0) const { return h0 >= a.g.own0 && h0 < a.g.own1; }
  __device__ __forceinline__ void tile_partial(const SumDev& s, int tile, double part) const {
    if (tile_owned(tile_row(tile) * a.g.TH)) store_tile_partial(s, tile + a.g.tileOff, part, red());
  }

  // ---- fused NumPy-pairwise leaves of up to 3 term buffers (tm[k], each
  // TH x (TW*C) doubles, interleaved like the image) -> leaf_vals.  Leaf
  // index of (tile row r, segment s): (h*W*C + w0*C)/L + s; buffer k goes to
  // sums[k] with a leaf offset koff[k].
  // Optional second sum set (s0b, s1b) from term buffers 3.. (the fused
  // candidate stage): both sets folded in one pass.
  __device__ void tile_leaves(int h0, int w0, int nbuf, const SumDev* s0, const SumDev* s1, int koff2, int b0 = 0,
                              const SumDev* s0b = nullptr, const SumDev* s1b = nullptr) {
    if (!tile_owned(h0)) return;   // CTA-uniform
    __syncthreads();
    // fused layouts have TW | W, so every tile row holds segs whole leaves
    const int C = nC(), L = a.g.leafL;
    const int rows = min(a.g.TH, a.g.H - h0);
    const int segs = a.g.segs;
    const int per_buf = rows * segs * 8;
    const int tmE = a.g.TH * a.g.TW * C;
    const int nb = s0b ? 2 * nbuf : nbuf;    // <= 6 buffers
    const int total = per_buf * nb;
    const int64_t lbase = (int64_t)(h0 + a.g.row0) * a.g.rowL + (int64_t)mdiv(w0, a.g.magicTWpx) * segs;
    for (int g0 = 0; g0 < total; g0 += blockDim.x) {      // total % 8 == 0, blockDim % 32 == 0
      const int gch = g0 + threadIdx.x;
      const bool act = gch < total;
      double acc = 0.0;
      int buf = 0, k = 0, r = 0, s = 0;
      if (act) {
        buf = (gch >= per_buf) + (gch >= 2 * per_buf) + (gch >= 3 * per_buf) + (gch >= 4 * per_buf) +
              (gch >= 5 * per_buf);
        const int rem = gch - buf * per_buf;
        const int leaf_l = rem >> 3;
        k = rem & 7;
        r = mdiv(leaf_l, a.g.magicSegs);
        s = leaf_l - r * segs;
        const int setb = buf >= nbuf, lb = buf - setb * nbuf;
        const double* t = tm() + (size_t)(setb ? 3 + lb : b0 + lb) * tmE + (size_t)r * a.g.TW * C + s * L + k;
        acc = t[0];
        for (int i = 8; i < L; i += 8) acc = acc + t[i];
      }
      acc = acc + __shfl_xor_sync(kFull, acc, 1);
      acc = acc + __shfl_xor_sync(kFull, acc, 2);
      acc = acc + __shfl_xor_sync(kFull, acc, 4);
      if (act && k == 0) {
        const int setb = buf >= nbuf, lb = buf - setb * nbuf;
        const int64_t li = lbase + (int64_t)r * a.g.rowL + s + (lb == 2 ? koff2 : 0);
        const SumDev* sd = setb ? (lb == 0 ? s0b : s1b) : (lb == 0 ? s0 : s1);
        sd->leaf_vals[li] = acc;
      }
    }
  }
  __device__ __forceinline__ void put_term(int buf, int r, int q, double v) const {
    tm()[(size_t)buf * a.g.TH * a.g.TW * nC() + ((size_t)r * a.g.TW + q) * nC() + ch] = v;
  }
  // opsm: the operand staged in term buffer `buf` for own pixel (r, q), read before that slot's term
  // is written (same thread); else the prefetched register
  __device__ __forceinline__ T opv(int buf, int r, int q, const T (&pre)[RW], int o) const {
    if constexpr (sizeof(T) == 8) {
      if (opsm) return (T)tm()[(size_t)buf * a.g.TH * a.g.TW * nC() + ((size_t)r * a.g.TW + q) * nC() + ch];
    }
    return pre[o];
  }
  // asynchronous copies of the tile's own pixels of NB arrays into term buffers buf0.. (rows of TW * C
  // contiguous doubles, 16-byte copies; rows outside the image zero-filled).  One index computation
  // (a single integer division per thread) serves all NB arrays.
  template <int NB>
  __device__ void stage_own_n(int h0, int w0, const T* const (&src)[NB], int buf0) const {
    if constexpr (sizeof(T) == 8) {
      const int C = nC(), H = a.g.H, W = a.g.W, TH = a.g.TH;
      const int rowE = a.g.TW * C, pairs = rowE >> 1;
      const int BD = blockDim.x;
      const int dr = BD / pairs, de = BD - dr * pairs;
      int r = threadIdx.x / pairs, p = threadIdx.x - r * pairs;
      const unsigned bufB = (unsigned)(TH * rowE * 8);
      const unsigned d0 = (unsigned)__cvta_generic_to_shared(tm()) + (unsigned)buf0 * bufB;
      while (r < TH) {
        const int h = h0 + r, e = 2 * p;
        const int64_t gi = ((int64_t)h * W + w0) * C + e;
        const int valid = (h < H && w0 * C + e < W * C) ? 16 : 0;
        const unsigned d = d0 + (unsigned)((r * rowE + e) * 8);
#pragma unroll
        for (int b = 0; b < NB; ++b)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d + b * bufB),
                       "l"(valid ? (const double*)src[b] + gi : (const double*)src[b]), "r"(valid)
                       : "memory");
        r += dr;
        p += de;
        if (p >= pairs) {
          p -= pairs;
          ++r;
        }
      }
    }
  }
  __device__ void stage_own(int h0, int w0, const T* src, int buf) const {
    const T* const one[1] = {src};
    stage_own_n<1>(h0, w0, one, buf);
  }

  // =========================================================================
  // Stage A: r = B y - ydat (write R); TV at y: root terms, grad -> TVG
  // (lower_value_and_grad, lower_solvers.py:50-63; SmoothedTV.value_and_grad,
  // regularizers.py:167-175).  `tv` false when alpha == 0.  Fused mode: the
  // fit / TV leaves go straight to s_fit / s_tv.
  //
  // tileA / tileC compute one tile from a loaded plane region `pr` (channel
  // planes of y resp. xc) into term buffers tb.. (tb = 0 or 3); tileA's TV
  // pass publishes neighbour values through the region `qr` (free by then).
  __device__ __forceinline__ T fpr(const T* pr, int r, int q) const {
    return pr[(size_t)ch * a.g.SH * swp() + (r + a.g.rh + 1) * swp() + sk(q + a.g.rw + 1)];
  }
  __device__ __forceinline__ void tileA(const T* pr, T* qr, int tb, int h0, int w0, const T (&ypre)[RW], T* Rout,
                                        bool tv, T* TV2out, T* TVGout, bool fused, const T* pre_acc = nullptr) {
    const T nu = T(a.nu), nu2 = nu * nu;
    const int H = a.g.H, W = a.g.W, TH = a.g.TH, TW = a.g.TW, C = nC();
    const int64_t N = a.g.N;
    const int h = h0 + ty;
    T acc[RW];
    if (pre_acc) {
#pragma unroll
      for (int o = 0; o < RW; ++o) acc[o] = pre_acc[o];
    } else {
      stencil(pr + (size_t)ch * a.g.SH * swp(), wfwd(), acc);
    }
#pragma unroll
    for (int o = 0; o < RW; ++o) {
      const int q = tx * RW + o;
      const int w = w0 + q;
      if (h < H && w < W) {
        const int64_t i = gidx(h, w, ch);
        const T r = acc[o] - opv(tb + 0, ty, q, ypre, o);
        Rout[i] = r;
        if (fused) put_term(tb + 0, ty, q, (double)(r * r));
      }
    }
    if (!tv) return;
    // q = d / sqrt(d^2 + nu^2) for the own pixels (registers), the row
    // above the tile (ty == 0) and the column left of it (tx == 0)
    T q0[RW], q1[RW], q0u[RW], q1l = T(0);
#pragma unroll
    for (int o = 0; o < RW; ++o) {
      const int q = tx * RW + o;
      const int w = w0 + q;
      const T yc = fpr(pr, ty, q);
      const T d0 = has_below(h) ? fpr(pr, ty + 1, q) - yc : T(0);
      const T d1 = (w < W - 1) ? fpr(pr, ty, q + 1) - yc : T(0);
      const T rt0 = sqrt(d0 * d0 + nu2), rt1 = sqrt(d1 * d1 + nu2);
      q0[o] = d0 / rt0;
      q1[o] = d1 / rt1;
      if (h < H && w < W) {
        if (fused) {
          put_term(tb + 1, ty, q, (double)rt0);
          put_term(tb + 2, ty, q, (double)rt1);
        } else {
          const int64_t i = gidx(h, w, ch);
          TV2out[i] = rt0;
          TV2out[N + i] = rt1;
        }
      }
      q0u[o] = T(0);
      if (ty == 0 && has_above(h0)) {     // edge (h0-1) -> (h0): h0 - 1 < H - 1 always
        const T du = yc - fpr(pr, -1, q);
        q0u[o] = du / sqrt(du * du + nu2);
      }
    }
    if (tx == 0 && w0 >= 1) {
      const T dl = fpr(pr, ty, 0) - fpr(pr, ty, -1);
      q1l = dl / sqrt(dl * dl + nu2);
    }
    // publish neighbour values through the (now free) region qr
    __syncthreads();
    T* Q0 = qr;                                      // [C][TH+1][TW]  (row r at r+1)
    T* Q1 = Q0 + (size_t)C * (TH + 1) * TW;          // [C][TH][TW+1]  (col q at q+1)
#pragma unroll
    for (int o = 0; o < RW; ++o) {
      const int q = tx * RW + o;
      Q0[((size_t)ch * (TH + 1) + ty + 1) * TW + q] = q0[o];
      if (ty == 0) Q0[((size_t)ch * (TH + 1)) * TW + q] = q0u[o];
      Q1[((size_t)ch * TH + ty) * (TW + 1) + q + 1] = q1[o];
    }
    if (tx == 0) Q1[((size_t)ch * TH + ty) * (TW + 1)] = q1l;
    __syncthreads();
#pragma unroll
    for (int o = 0; o < RW; ++o) {
      const int q = tx * RW + o;
      const int w = w0 + q;
      if (h < H && w < W) {
        // image_forward_diff_adjoint (regularizers.py:61-67), per-pixel order
        T t = T(0);
        if (has_above(h)) t = t + Q0[((size_t)ch * (TH + 1) + ty) * TW + q];
        if (has_below(h)) t = t - q0[o];
        if (w >= 1) t = t + (o > 0 ? q1[o > 0 ? o - 1 : 0] : Q1[((size_t)ch * TH + ty) * (TW + 1) + q]);
        if (w <= W - 2) t = t - q1[o];
        TVGout[gidx(h, w, ch)] = t;
      }
    }
  }

  template <class Src>
  __device__ void stageA(const Src& src, T* Rout, const T* ydat, bool tv, T* TV2out, T* TVGout,
                         const SumDev* sfit, const SumDev* stv) {
    const int H = a.g.H, W = a.g.W;
    const bool fused = a.g.fused && sfit;
    for (int tile = tb0; tile < a.g.nTiles; tile += tbs) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      const int h = h0 + ty;
      T ypre[RW];   // epilogue operands: issued before the tile box so both share one round trip
      if (opsm && fused) {
        stage_own(h0, w0, ydat, 0);
#pragma unroll
        for (int o = 0; o < RW; ++o) ypre[o] = T(0);
      } else {
#pragma unroll
        for (int o = 0; o < RW; ++o) {
          const int w = w0 + tx * RW + o;
          ypre[o] = (h < H && w < W) ? ydat[gidx(h, w, ch)] : T(0);
        }
      }
      load_full(h0, w0, src);
      if (opsm && fused) cp_async_wait_all();
      __syncthreads();
      tileA(pa(), pa(), 0, h0, w0, ypre, Rout, tv, TV2out, TVGout, fused);
      if (fused) tile_leaves(h0, w0, tv ? 3 : 1, sfit, stv, (int)(a.g.Ng / a.g.leafL));
    }
  }

  // Stage B: g = 2 * B^T r (+ alpha * tvg); tile partial of g.g -> sgg.
  // Optionally the first backtracking candidate xc = y - g / L for the own
  // pixels (y = x + beta (x - x_prev)), written to Xc.
  __device__ void stageB(const T* Rin, bool tv, const T* TVGin, T* Gout, const SumDev* sgg, const T* Xs = nullptr,
                         const T* XPs = nullptr, T beta = T(0), T L = T(1), T* Xc = nullptr) {
    const T two = T(2), alpha = T(a.alpha);
    const int H = a.g.H, W = a.g.W;
    long long sub_t[8];
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      ADP_SUB(0);
      __syncthreads();
      const int h = h0 + ty;
      T tpre[RW], xpre[RW], xppre[RW];   // epilogue operands, in flight with the tile box
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        tpre[o] = xpre[o] = xppre[o] = T(0);
        if (h < H && w < W) {
          const int64_t i = gidx(h, w, ch);
          if (tv) tpre[o] = ldcg(TVGin + i);
          if (Xc) {
            xpre[o] = ldcg(Xs + i);
            xppre[o] = ldcg(XPs + i);
          }
        }
      }
      load_full(h0, w0, SrcLin<T>{Rin});
      ADP_SUB(1);
      __syncthreads();
      ADP_SUB(2);
      double part = 0.0;
      T acc[RW];
      stencil_adj(acc);
      ADP_SUB(3);
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        if (h < H && w < W) {
          const int64_t i = gidx(h, w, ch);
          T gv = two * acc[o];
          if (tv) gv = gv + alpha * tpre[o];
          Gout[i] = gv;
          part += (double)gv * (double)gv;
          if (Xc) Xc[i] = (xpre[o] + beta * (xpre[o] - xppre[o])) - gv / L;
        }
      }
      ADP_SUB(4);
      if (sgg) tile_partial(*sgg, tile, part);
      ADP_SUB(5);
      ADP_SUB_FLUSH(6);
    }
  }

  // Stage B, pipelined (RW = 4 plans with two plane regions and the Q
  // scratch): the R tile boxes alternate between the two regions, the copy
  // of tile k+1 in flight while tile k is computed; besides g and the first
  // candidate xc = y - g / L it writes the next extrapolation point
  // y' = xc + betaN (xc - x) to Yn (SrcExtrap's expression, exact), which
  // stageCA_pipe then copies as a plain box.
  __device__ void stageB_pipe(const T* Rin, bool tv, const T* TVGin, T* Gout, const SumDev* sgg, const T* Xs,
                              const T* XPs, T beta, T L, T* Xc, T betaN, T* Yn) {
    const T two = T(2), alpha = T(a.alpha);
    const int H = a.g.H, W = a.g.W;
    const size_t co = (size_t)ch * a.g.SH * swp();
    int tile = blockIdx.x;
    if (tile < a.g.nTiles) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      load_async(h0, w0, Rin, pa());
    }
    cp_commit();
    for (int k = 0; tile < a.g.nTiles; tile += gridDim.x, ++k) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      const T* cur = (k & 1) ? pa2() : pa();
      const int nt = tile + gridDim.x;
      if (nt < a.g.nTiles) {
        int h1, w1;
        tile_origin(nt, h1, w1);
        load_async(h1, w1, Rin, (k & 1) ? pa() : pa2());
      }
      cp_commit();
      const int h = h0 + ty;
      T tpre[RW], xpre[RW], xppre[RW];
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        tpre[o] = xpre[o] = xppre[o] = T(0);
        if (h < H && w < W) {
          const int64_t i = gidx(h, w, ch);
          if (tv) tpre[o] = ldcg(TVGin + i);
          xpre[o] = ldcg(Xs + i);
          xppre[o] = ldcg(XPs + i);
        }
      }
      cp_wait<1>();
      __syncthreads();
      double part = 0.0;
      T acc[RW];
      stencil(cur + co, wadj(), acc);
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        if (h < H && w < W) {
          const int64_t i = gidx(h, w, ch);
          T gv = two * acc[o];
          if (tv) gv = gv + alpha * tpre[o];
          Gout[i] = gv;
          part += (double)gv * (double)gv;
          const T xc = (xpre[o] + beta * (xpre[o] - xppre[o])) - gv / L;
          Xc[i] = xc;
          Yn[i] = xc + betaN * (xc - xpre[o]);
        }
      }
      if (sgg) tile_partial(*sgg, tile, part);
      __syncthreads();   // every warp is done with `cur` before it receives tile k+2
    }
  }

  // Stage CA, pipelined (see stageCA): the candidate's box (Xc) and the next
  // extrapolation point's box (Yn, written by stageB_pipe) are plain
  // asynchronous copies: Yn(k) lands during the candidate pass of tile k and
  // Xc(k+1) during its speculative stage-A pass; tileA publishes its TV
  // neighbour values through the Q scratch (the first region is receiving
  // the next box).  Same arithmetic and leaves as stageCA.
  __device__ void stageCA_pipe(const T* Xc, const T* Yn, const T* Xold, const T* Gin, bool tv, T* Rout, T* TVGout,
                               const SumDev* sdot, const SumDev* sfitc, const SumDev* stvc, const SumDev* sfit2,
                               const SumDev* stv2) {
    int tile = blockIdx.x;
    if (tile < a.g.nTiles) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      load_async(h0, w0, Xc, pa());
    }
    cp_commit();
    const int koff = (int)(a.g.Ng / a.g.leafL);
    for (; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      cp_wait<0>();
      __syncthreads();                       // Xc(k) landed; the second region is free
      load_async(h0, w0, Yn, pa2());
      cp_commit();
      T ypre[RW], gpre[RW], xopre[RW];
      prefetch_c(h0, w0, Gin, Xold, true, ypre, gpre, xopre);
      const double part = tileC(pa(), h0, w0, ypre, gpre, xopre, nullptr, tv, nullptr, nullptr, true, true);
      tile_partial(*sdot, tile, part);       // its barriers: every warp is done reading the first region
      tile_leaves(h0, w0, tv ? 3 : 1, sfitc, stvc, koff);
      __syncthreads();
      const int nt = tile + gridDim.x;
      if (nt < a.g.nTiles) {
        int h1, w1;
        tile_origin(nt, h1, w1);
        load_async(h1, w1, Xc, pa());
      }
      cp_commit();
      cp_wait<1>();
      __syncthreads();                       // Yn(k) landed
      tileA(pa2(), qs(), 3, h0, w0, ypre, Rout, tv, nullptr, TVGout, true);
      tile_leaves(h0, w0, tv ? 3 : 1, sfit2, stv2, koff, 3);
      __syncthreads();                       // the second region is read before Yn(k+1) is issued
    }
  }

  // Stage B / CA with TMA tile boxes (KS = 9, single channel): R, and then
  // the candidate x_c and the next extrapolation point y' (materialised here
  // in Yn, SrcExtrap's exact expression) arrive as 2-D tensor copies on the
  // mbarriers; the arithmetic is stageB / stageCA's.
  __device__ void stageB_tma(const CUtensorMap* tmR, bool tv, const T* TVGin, T* Gout, const SumDev* sgg,
                             const T* Xs, const T* XPs, T beta, T L, T* Xc, T betaN, T* Yn,
                             unsigned long long* mbar, unsigned& ph) {
    const T two = T(2), alpha = T(a.alpha);
    const int H = a.g.H, W = a.g.W;
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      tma_box(tmR, h0, w0, pa(), mbar);
      const int h = h0 + ty;
      T tpre[RW], xpre[RW], xppre[RW];
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        tpre[o] = xpre[o] = xppre[o] = T(0);
        if (h < H && w < W) {
          const int64_t i = gidx(h, w, ch);
          if (tv) tpre[o] = ldcg(TVGin + i);
          xpre[o] = ldcg(Xs + i);
          xppre[o] = ldcg(XPs + i);
        }
      }
      tma_wait(mbar, ph);
      ph ^= 1u;
      double part = 0.0;
      T acc[RW];
      stencil_adj(acc);
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        if (h < H && w < W) {
          const int64_t i = gidx(h, w, ch);
          T gv = two * acc[o];
          if (tv) gv = gv + alpha * tpre[o];
          Gout[i] = gv;
          part += (double)gv * (double)gv;
          const T xc = (xpre[o] + beta * (xpre[o] - xppre[o])) - gv / L;
          Xc[i] = xc;
          Yn[i] = xc + betaN * (xc - xpre[o]);
        }
      }
      if (sgg) tile_partial(*sgg, tile, part);
    }
  }

  __device__ void stageCA_tma(const CUtensorMap* tmXc, const CUtensorMap* tmYn, const T* Xold, const T* Gin, bool tv,
                              T* Rout, T* TVGout, const SumDev* sdot, const SumDev* sfitc, const SumDev* stvc,
                              const SumDev* sfit2, const SumDev* stv2, unsigned long long* mbar, unsigned* ph) {
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      tma_box(tmXc, h0, w0, pa(), mbar);
      tma_box(tmYn, h0, w0, pa2(), mbar + 1);
      T ypre[RW], gpre[RW], xopre[RW];
      prefetch_c(h0, w0, Gin, Xold, true, ypre, gpre, xopre);
      tma_wait(mbar, ph[0]);
      tma_wait(mbar + 1, ph[1]);
      ph[0] ^= 1u;
      ph[1] ^= 1u;
      T acc1[RW], acc2[RW];
      stencil_fwd_pair(pa(), pa2(), acc1, acc2);
      const double part = tileC(pa(), h0, w0, ypre, gpre, xopre, nullptr, tv, nullptr, nullptr, true, true, acc1);
      tileA(pa2(), pa(), 3, h0, w0, ypre, Rout, tv, nullptr, TVGout, true, acc2);   // syncs before reusing pa()
      tile_partial(*sdot, tile, part);
      tile_leaves(h0, w0, tv ? 3 : 1, sfitc, stvc, (int)(a.g.Ng / a.g.leafL), 0, sfit2, stv2);
    }
  }

  // Stage C (value at a candidate): xc = src; rc = B xc - y; TV terms
  // sqrt(d^2+nu^2) - nu (tv_value, regularizers.py:70-72); optional tile
  // partial of g.(xc - xold); xc written to Xout (if non-null).  Fused:
  // leaves to sfitc / stvc; otherwise rc -> RCout and TV terms -> TV2Cout.
  __device__ __forceinline__ double tileC(const T* pr, int h0, int w0, const T (&ypre)[RW], const T (&gpre)[RW],
                                          const T (&xopre)[RW], T* RCout, bool tv, T* TV2Cout, T* Xout, bool dot,
                                          bool fused, const T* pre_acc = nullptr) {
    const T nu = T(a.nu), nu2 = nu * nu;
    const int H = a.g.H, W = a.g.W;
    const int64_t N = a.g.N;
    const int h = h0 + ty;
    double part = 0.0;
    T acc[RW];
    if (pre_acc) {
#pragma unroll
      for (int o = 0; o < RW; ++o) acc[o] = pre_acc[o];
    } else {
      stencil(pr + (size_t)ch * a.g.SH * swp(), wfwd(), acc);
    }
#pragma unroll
    for (int o = 0; o < RW; ++o) {
      const int q = tx * RW + o;
      const int w = w0 + q;
      if (h < H && w < W) {
        const int64_t i = gidx(h, w, ch);
        const T yv = opv(0, ty, q, ypre, o), gv = opv(1, ty, q, gpre, o), xov = opv(2, ty, q, xopre, o);
        const T rc = acc[o] - yv;
        const T xc = fpr(pr, ty, q);
        if (fused) put_term(0, ty, q, (double)(rc * rc));
        else RCout[i] = rc;
        if (tv) {
          const T d0 = has_below(h) ? fpr(pr, ty + 1, q) - xc : T(0);
          const T d1 = (w < W - 1) ? fpr(pr, ty, q + 1) - xc : T(0);
          const T t0 = sqrt(d0 * d0 + nu2) - nu;
          const T t1 = sqrt(d1 * d1 + nu2) - nu;
          if (fused) {
            put_term(1, ty, q, (double)t0);
            put_term(2, ty, q, (double)t1);
          } else {
            TV2Cout[i] = t0;
            TV2Cout[N + i] = t1;
          }
        }
        if (Xout) Xout[i] = xc;
        if (dot) part += (double)gv * (double)(xc - xov);
      }
    }
    return part;
  }

  __device__ __forceinline__ void prefetch_c(int h0, int w0, const T* Gin, const T* Xold, bool dot, T (&ypre)[RW],
                                             T (&gpre)[RW], T (&xopre)[RW]) const {
    const int H = a.g.H, W = a.g.W;
    const int h = h0 + ty;
#pragma unroll
    for (int o = 0; o < RW; ++o) {
      const int w = w0 + tx * RW + o;
      ypre[o] = gpre[o] = xopre[o] = T(0);
      if (h < H && w < W) {
        const int64_t i = gidx(h, w, ch);
        ypre[o] = a.ydat[i];
        if (dot) {
          gpre[o] = ldcg(Gin + i);
          xopre[o] = ldcg(Xold + i);
        }
      }
    }
  }

  template <class Src>
  __device__ void stageC(const Src& src, T* RCout, bool tv, T* TV2Cout, T* Xout, const T* Gin, const T* Xold,
                         const SumDev* sdot, const SumDev* sfitc, const SumDev* stvc) {
    const bool fused = a.g.fused && sfitc;
    for (int tile = tb0; tile < a.g.nTiles; tile += tbs) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      T ypre[RW], gpre[RW], xopre[RW];   // epilogue operands, in flight with the tile box
      const bool st = opsm && fused && sdot != nullptr;
      if (st) {
        stage_own(h0, w0, a.ydat, 0);
        stage_own(h0, w0, Gin, 1);
        stage_own(h0, w0, Xold, 2);
#pragma unroll
        for (int o = 0; o < RW; ++o) ypre[o] = gpre[o] = xopre[o] = T(0);
      } else {
        prefetch_c(h0, w0, Gin, Xold, sdot != nullptr, ypre, gpre, xopre);
      }
      load_full(h0, w0, src);
      if (st) cp_async_wait_all();
      __syncthreads();
      const bool keep = opsm;
      opsm = st;
      const double part = tileC(pa(), h0, w0, ypre, gpre, xopre, RCout, tv, TV2Cout, Xout, sdot != nullptr, fused);
      opsm = keep;
      if (sdot) tile_partial(*sdot, tile, part);
      if (fused) tile_leaves(h0, w0, tv ? 3 : 1, sfitc, stvc, (int)(a.g.Ng / a.g.leafL));
    }
  }

  // Fused candidate value + speculative next value/grad (fused layouts with
  // room for two plane regions, a.g.fuseCA): per tile, plane region 1 holds
  // the first candidate xc (stage C of iteration t, leaves -> sfitc/stvc,
  // restart dot -> sdot) and region 2 the next extrapolation point
  // y' = xc + beta' (xc - x) (stage A of iteration t + 1 assuming the
  // candidate is accepted without restart; leaves -> sfit2/stv2, terms in
  // buffers 3..5).  One tile load round trip and no grid barrier between them.
  __device__ void stageCA(const T* Xc, const T* Xold, T betaN, const T* Gin, bool tv, T* Rout, T* TVGout,
                          const SumDev* sdot, const SumDev* sfitc, const SumDev* stvc, const SumDev* sfit2,
                          const SumDev* stv2) {
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      T ypre[RW], gpre[RW], xopre[RW];
      prefetch_c(h0, w0, Gin, Xold, true, ypre, gpre, xopre);
      load_full(h0, w0, SrcLin<T>{Xc}, pa());
      load_full(h0, w0, SrcExtrap<T>{Xc, Xold, betaN}, pa2());
      __syncthreads();
      if constexpr (KS > 0) {
        // compile-time K (c2): shared tap loads, both leaf sets in one pass
        T acc1[RW], acc2[RW];
        stencil_fwd_pair(pa(), pa2(), acc1, acc2);
        const double part = tileC(pa(), h0, w0, ypre, gpre, xopre, nullptr, tv, nullptr, nullptr, true, true, acc1);
        tileA(pa2(), pa(), 3, h0, w0, ypre, Rout, tv, nullptr, TVGout, true, acc2);   // syncs before reusing pa()
        tile_partial(*sdot, tile, part);
        tile_leaves(h0, w0, tv ? 3 : 1, sfitc, stvc, (int)(a.g.Ng / a.g.leafL), 0, sfit2, stv2);
      } else {
        // generic sizes: one stencil at a time (register pressure at RW = 4)
        const double part = tileC(pa(), h0, w0, ypre, gpre, xopre, nullptr, tv, nullptr, nullptr, true, true);
        tileA(pa2(), pa(), 3, h0, w0, ypre, Rout, tv, nullptr, TVGout, true);
        tile_partial(*sdot, tile, part);
        tile_leaves(h0, w0, tv ? 3 : 1, sfitc, stvc, (int)(a.g.Ng / a.g.leafL));
        tile_leaves(h0, w0, tv ? 3 : 1, sfit2, stv2, (int)(a.g.Ng / a.g.leafL), 3);
      }
    }
  }

  // Light candidate (non-adaptive step): xc = src per own pixel, dot partial.
  template <class Src>
  __device__ void stageCLight(const Src& src, T* Xout, const T* Gin, const T* Xold, const SumDev* sdot) {
    foreach_pixel_sum([&](int64_t i, int, int, int) {
      const T xc = src(i);
      Xout[i] = xc;
      return (double)ldcg(Gin + i) * (double)(xc - ldcg(Xold + i));
    }, *sdot);
  }

  // Plain correlation pass: out = scale * (B src - sub) (or B^T with flipped
  // taps), optional tile partial of out.out.
  template <class Src>
  __device__ void stage_corr(const Src& src, bool flipped, T* Out, const T* sub, T scale, const SumDev* ssq) {
    const int H = a.g.H, W = a.g.W;
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      __syncthreads();
      load_full(h0, w0, src);
      __syncthreads();
      const int h = h0 + ty;
      double part = 0.0;
      T acc[RW];
      if (flipped) stencil_adj(acc);
      else stencil_fwd(acc);
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        if (h < H && w < W) {
          const int64_t i = gidx(h, w, ch);
          T v = acc[o];
          if (sub) v = v - sub[i];
          v = scale * v;
          Out[i] = v;
          part += (double)v * (double)v;
        }
      }
      if (ssq) tile_partial(*ssq, tile, part);
    }
  }

  // Elementwise over own pixels of every tile (grid-stride by tiles).
  template <class F>
  __device__ void foreach_pixel(const F& f) {
    const int H = a.g.H, W = a.g.W;
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      const int h = h0 + ty;
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        if (h < H && w < W) f(gidx(h, w, ch), h, w, ch);
      }
    }
  }
  // Same, with a per-tile partial accumulated from f's return value.
  template <class F>
  __device__ void foreach_pixel_sum(const F& f, const SumDev& s) {
    const int H = a.g.H, W = a.g.W;
    for (int tile = blockIdx.x; tile < a.g.nTiles; tile += gridDim.x) {
      int h0, w0;
      tile_origin(tile, h0, w0);
      const int h = h0 + ty;
      double part = 0.0;
#pragma unroll
      for (int o = 0; o < RW; ++o) {
        const int w = w0 + tx * RW + o;
        if (h < H && w < W) part += f(gidx(h, w, ch), h, w, ch);
      }
      tile_partial(s, tile, part);
    }
  }
};

}  // namespace adp
