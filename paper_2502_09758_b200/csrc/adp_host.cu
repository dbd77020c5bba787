// Host runtime of the B200 MAID engine: plan creation (tile geometry,
// workspace, deterministic-sum programs), cooperative launches and the
// extern "C" ABI declared in include/adp_b200.h.
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "adp_plan.h"
#include "conv2d_args.h"
#include "dense1d_args.h"

namespace adp {

static thread_local std::string g_err;
static int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}
int dense_fail(int code, const char* m) { return fail(code, m); }
#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) return fail(ADP_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// Tree programs.
//   numpy rule (np == true): leaf if n <= 128, else split at
//     n2 = n/2 - (n/2) % 8       (numpy pairwise_sum, PW_BLOCKSIZE = 128)
//   binary rule: leaf if n <= 1, else split at n/2.
static bool is_leaf(bool np, int64_t n) { return np ? n <= 128 : n <= 1; }
static int64_t split_at(bool np, int64_t n) {
  if (np) {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return n2;
  }
  return n / 2;
}

struct LeafCounter {
  bool np;
  std::map<int64_t, int64_t> memo;
  int64_t operator()(int64_t n) {
    if (is_leaf(np, n)) return 1;
    auto it = memo.find(n);
    if (it != memo.end()) return it->second;
    const int64_t a = split_at(np, n);
    const int64_t v = (*this)(a) + (*this)(n - a);
    memo[n] = v;
    return v;
  }
};

// Program over the tree of size n whose terminal nodes are given by term().
static std::vector<int> make_prog(int64_t n, bool np, const std::function<bool(int64_t)>& term) {
  struct Inner { int l, r, h; };
  std::vector<Inner> inner;     // temp ids: leaves >= 0, inner -> -(k+1)
  int nL = 0;
  std::function<std::pair<int, int>(int64_t)> rec = [&](int64_t m) -> std::pair<int, int> {
    if (term(m)) return {nL++, 0};
    const int64_t a = split_at(np, m);
    auto L = rec(a);
    auto R = rec(m - a);
    const int h = 1 + std::max(L.second, R.second);
    inner.push_back({L.first, R.first, h});
    return {-(int)inner.size(), h};
  };
  rec(n);
  const int nI = (int)inner.size();
  std::vector<int> order(nI);
  for (int k = 0; k < nI; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return inner[x].h < inner[y].h; });
  std::vector<int> rank(nI);
  for (int k = 0; k < nI; ++k) rank[order[k]] = k;
  auto fin = [&](int t) { return t >= 0 ? t : nL + rank[-t - 1]; };
  int nLev = nI ? inner[order[nI - 1]].h : 0;
  std::vector<int> prog;
  prog.push_back(nL);
  prog.push_back(nI);
  prog.push_back(nLev);
  // level starts (heights 1..nLev)
  std::vector<int> lev(nLev + 1, 0);
  {
    int k = 0;
    for (int h = 1; h <= nLev; ++h) {
      lev[h - 1] = k;
      while (k < nI && inner[order[k]].h == h) ++k;
    }
    lev[nLev] = nI;
  }
  for (int v : lev) prog.push_back(v);
  for (int k = 0; k < nI; ++k) prog.push_back(fin(inner[order[k]].l));
  for (int k = 0; k < nI; ++k) prog.push_back(fin(inner[order[k]].r));
  return prog;
}

int ProgPool::add(const std::string& key, const std::vector<int>& prog) {
  for (auto& kv : memo)
    if (kv.first == key) return kv.second;
  const int off = (int)words.size();
  words.insert(words.end(), prog.begin(), prog.end());
  memo.push_back({key, off});
  return off;
}

void build_sum(SumHost& s, int64_t n, bool np, ProgPool& pool, bool allow_regular) {
  s.n = n;
  s.np = np;
  LeafCounter cnt{np, {}};
  s.leaf_start.clear();
  s.sub_leaf.clear();
  s.sub_prog.clear();
  if (n <= 0) {
    s.nLeaves = 0;
    s.nSub = 1;
    s.leaf_start.push_back(0);
    s.sub_leaf = {0, 0};
    s.top_prog = pool.add("empty", {0, 0, 0, 0});
    s.sub_prog = {s.top_prog};
    return;
  }
  if (np) {
    std::function<void(int64_t, int64_t)> rec = [&](int64_t off, int64_t m) {
      if (is_leaf(true, m)) {
        s.leaf_start.push_back(off);
        return;
      }
      const int64_t a = split_at(true, m);
      rec(off, a);
      rec(off + a, m - a);
    };
    rec(0, n);
    s.leaf_start.push_back(n);
  }
  s.nLeaves = (int)cnt(n);
  // regular: perfect tree (element sums: equal leaves, L % 8 == 0, pow2 count;
  // tile sums: always, zero-padded) -> register/shuffle evaluation on device
  s.regular = 0;
  s.leaf_len = 0;
  if (np) {
    const int64_t L = s.leaf_start[1] - s.leaf_start[0];
    bool eq = (L % 8 == 0);
    for (size_t i = 1; eq && i + 1 < s.leaf_start.size(); ++i) eq = (s.leaf_start[i + 1] - s.leaf_start[i]) == L;
    const bool pow2 = (s.nLeaves & (s.nLeaves - 1)) == 0;
    if (allow_regular && eq && pow2) { s.regular = 1; s.leaf_len = (int)L; }
  } else {
    s.regular = allow_regular ? 1 : 0;
  }
  if (s.regular) {
    int64_t P = 1;
    while (P < s.nLeaves) P <<= 1;
    s.sub_size = 2048;
    s.nSub = P <= 4096 ? 1 : (int)((s.nLeaves + 2047) / 2048);
    s.sub_leaf.clear();
    s.sub_prog.clear();
    for (int t = 0; t <= s.nSub; ++t) s.sub_leaf.push_back(std::min<int64_t>((int64_t)t * 2048, s.nLeaves));
    for (int t = 0; t < s.nSub; ++t) s.sub_prog.push_back(0);
    if (s.nSub == 1) s.sub_leaf = {0, s.nLeaves};
    s.top_prog = 0;
    return;
  }
  const std::string tag = np ? "np" : "bin";
  auto leafterm = [&](int64_t m) { return is_leaf(np, m); };
  if (s.nLeaves <= kMaxProgLeaves) {
    s.nSub = 1;
    s.top_prog = pool.add(tag + ":" + std::to_string(n), make_prog(n, np, leafterm));
    s.sub_leaf = {0, s.nLeaves};
    s.sub_prog = {s.top_prog};
    return;
  }
  // cut into maximal subtrees with <= kMaxProgLeaves leaves
  auto cutterm = [&](int64_t m) { return cnt(m) <= kMaxProgLeaves; };
  int64_t lacc = 0;
  std::function<void(int64_t)> rec = [&](int64_t m) {
    if (cutterm(m)) {
      s.sub_leaf.push_back((int)lacc);
      s.sub_prog.push_back(pool.add(tag + ":" + std::to_string(m), make_prog(m, np, leafterm)));
      lacc += cnt(m);
      return;
    }
    const int64_t a = split_at(np, m);
    rec(a);
    rec(m - a);
  };
  rec(n);
  s.sub_leaf.push_back((int)lacc);
  s.nSub = (int)s.sub_prog.size();
  s.top_prog = pool.add(tag + ":top:" + std::to_string(n), make_prog(n, np, cutterm));
}

// ---------------------------------------------------------------------------
static int device_props(int& sms, size_t& smem_optin) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int v = 0;
  CK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  smem_optin = (size_t)v;
  return ADP_OK;
}

static constexpr int kRW = 4;

// Tile choice.  When the NumPy-pairwise layout of N elements is regular
// (equal leaves of L elements, power-of-two count) and a tile row can hold
// whole leaves (W*C % L == 0), the tile width is a multiple of L/C-aligned
// element runs so every tile computes its own leaves ("fused").
static void choose_tiles(const adp_plan_desc& d, int leafL, int& TH, int& TW, int& fused) {
  const int64_t px = (int64_t)d.H * d.W;
  fused = 0;
  if (d.tile_w > 0 && d.tile_h > 0) {
    TH = d.tile_h;
    TW = d.tile_w;
  } else {
    TW = 64;
    if (d.W <= 32) TW = 32;
    TH = px >= (1 << 20) ? 16 : 8;
    if (d.kh >= 25) TH = 8;
    if (leafL > 0 && ((int64_t)d.W * d.C) % leafL == 0) {
      // smallest width (multiple of 32 px) holding whole leaves, >= 64 px if the image allows
      for (int tw = 32; tw <= 512; tw += 32) {
        if (((int64_t)tw * d.C) % leafL == 0 && (tw >= 64 || tw >= d.W)) {
          TW = tw;
          break;
        }
      }
      TH = std::max(1, 512 / TW);    // 128 threads at RW = 4
      if (px >= (1 << 20) && d.kh < 25 && TW <= 64) TH = 16;
    }
  }
  if (leafL > 0 && ((int64_t)d.W * d.C) % leafL == 0 && ((int64_t)TW * d.C) % leafL == 0) fused = 1;
}

// Dynamic shared-memory layout (byte offsets; see ConvGeom).
static size_t conv_smem(ConvGeom& g, int esize, size_t cap = 0) {
  const size_t nk = (size_t)g.kh * g.kw * g.C;
  size_t off = 64 * sizeof(double);                  // red
  g.o_ws = (int)off;
  off += (nk * esize + 15) & ~size_t(15);
  g.o_wf = (int)off;
  off += (nk * esize + 15) & ~size_t(15);
  off = (off + 127) & ~size_t(127);
  const size_t R0 = off;
  g.QP = 0;   // TV Q values are staged through registers into the plane region
  const size_t pa = ((size_t)g.C * g.SH * g.SWP * esize + 127) & ~size_t(127);   // 128 B: TMA destinations
  const size_t tm = g.fused ? (size_t)3 * g.TH * g.TW * g.C * sizeof(double) : 0;
  const int np = g.fuseCA ? 2 : 1;   // fuseCA: two plane regions, six term buffers
  g.o_pa = (int)R0;
  g.o_pa2 = (int)(R0 + pa);
  g.o_pq = (int)R0;
  g.o_tm = (int)(R0 + np * pa);
  g.o_sv = (int)R0;
  const size_t region = std::max(np * (pa + tm), (size_t)(kTreeStage + 512) * sizeof(double));
  g.o_q = 0;
  if (g.fuseCA && g.rwb == 4) {
    // TV neighbour scratch of the pipelined stages: [C][TH+1][TW] + [C][TH][TW+1]
    const size_t q = ((size_t)g.C * ((g.TH + 1) * g.TW + g.TH * (g.TW + 1)) * esize + 15) & ~size_t(15);
    const char* ev = getenv("ADP_PIPE");    // ADP_PIPE=0: the unpipelined stages (A/B)
    if (!(ev && atoi(ev) == 0) && R0 + region + q + 2048 <= cap) {
      g.o_q = (int)(R0 + region);
      return R0 + region + q;
    }
  }
  return R0 + region;
}

template <typename T>
static void fill_sum(SumDev& sd, const SumHost& sh, const int* d_progs, const int64_t* d_leaf, int* d_subleaf,
                     int* d_subprog, double* leaf_vals, double* sub_vals) {
  sd.nLeaves = sh.nLeaves;
  sd.nSub = sh.nSub;
  sd.sub_own0 = 0;
  sd.sub_own1 = sh.nSub;
  sd.sub_own2 = sd.sub_own3 = 0;
  sd.regular = sh.regular;
  sd.sub_size = sh.sub_size;
  sd.leaf_len = sh.leaf_len;
  sd.top_prog = sh.top_prog;
  sd.leaf_start = d_leaf;
  sd.sub_leaf = d_subleaf;
  sd.sub_prog = d_subprog;
  sd.progs = d_progs;
  sd.leaf_vals = leaf_vals;
  sd.sub_vals = sub_vals;
}

static int setup_kernel(PlanImpl& P, KernelInfo& k, const void* fn, int threads, size_t smem, int max_grid) {
  k.fn = fn;
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, fn));
  const size_t dyn_max = P.smem_optin - fa.sharedSizeBytes;   // static smem (argument copy) counts too
  if (smem > dyn_max) return fail(ADP_ERR_UNSUPPORTED, "tile + halo exceeds shared memory; use a smaller tile");
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max));
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem));
  if (nb <= 0) return fail(ADP_ERR_UNSUPPORTED, "kernel does not fit on an SM (smem/registers)");
  k.grid = std::max(1, std::min(max_grid, nb * P.sm_count));
  return ADP_OK;
}

// 2-D TMA descriptors (W inner, H outer; float64) of the plan's workspace
// images X[0..2], R, P[0]: box (SWPt, SH), zero fill outside the image.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static int build_tmaps(PlanImpl& P) {
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return ADP_ERR_UNSUPPORTED;
    enc = (EncodeTiledFn)fn;
  }
  const ConvGeom& g = P.g;
  if (g.SWPt > 256 || g.SH > 256 || ((size_t)g.W * 8) % 16) return ADP_ERR_UNSUPPORTED;
  const int idx[5] = {0, 1, 2, 3, 10};   // X[0..2], R, P[0] (ws indices, conv_base)
  for (int k = 0; k < 5; ++k) {
    cuuint64_t dims[2] = {(cuuint64_t)g.W, (cuuint64_t)g.H};
    cuuint64_t strides[1] = {(cuuint64_t)g.W * sizeof(double)};
    cuuint32_t box[2] = {(cuuint32_t)g.SWPt, (cuuint32_t)g.SH};
    cuuint32_t es[2] = {1, 1};
    if (enc(&P.tm[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P.ws[idx[k]], dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return ADP_ERR_UNSUPPORTED;
  }
  return ADP_OK;
}

static int conv_plan_init(PlanImpl& P) {
  const adp_plan_desc& d = P.d;
  size_t smem_optin = 0;
  if (int e = device_props(P.sm_count, smem_optin)) return e;
  P.smem_optin = smem_optin;
  ConvGeom& g = P.g;
  g.H = d.H; g.W = d.W; g.C = d.C; g.kh = d.kh; g.kw = d.kw;
  g.rh = d.kh / 2; g.rw = d.kw / 2;
  // row slab: sums, tiles and heuristics follow the GLOBAL image
  const bool slab = d.Hg > 0;
  if (slab && (d.row0 < 0 || d.row0 + d.H > d.Hg || d.own0 < 0 || d.own0 >= d.own1 || d.own1 > d.H))
    return fail(ADP_ERR_ARG, "bad row-slab geometry");
  g.row0 = slab ? d.row0 : 0;
  g.Hg = slab ? d.Hg : d.H;
  g.own0 = slab ? d.own0 : 0;
  g.own1 = slab ? d.own1 : d.H;
  g.Ng = (int64_t)g.Hg * d.W * d.C;
  adp_plan_desc dg = d;
  dg.H = g.Hg;
  {
    ProgPool tmp;
    SumHost s;
    build_sum(s, g.Ng, true, tmp);
    g.leafL = s.regular ? s.leaf_len : 0;
  }
  choose_tiles(dg, g.leafL, g.TH, g.TW, g.fused);
  // register blocking: small single-channel problems are latency-bound with
  // one warp per SM sub-partition at RW = 4; RW = 2 gives 2x the warps on the
  // same tile (c2 512x512x1: 41 us/iter vs 51 at RW = 4; RW = 1 measured 43,
  // the extra warps do not pay for the lost window reuse).  ADP_RW overrides.
  {
    const int64_t px_per_sm = (int64_t)g.Hg * d.W / std::max(1, P.sm_count);
    int rwb = (d.C == 1 && px_per_sm < 8192) ? 2 : 4;
    if (d.rw == 1 || d.rw == 2 || d.rw == 4) rwb = d.rw;
    if (const char* ev = getenv("ADP_RW")) {
      const int v = atoi(ev);
      if (v == 1 || v == 2 || v == 4) rwb = v;
    }
    if (P.d.dtype == ADP_DTYPE_F32) rwb = 4;
    g.rwb = rwb;
  }
  const int kRWp = g.rwb;
  if (g.TW % 4) return fail(ADP_ERR_ARG, "tile width must be a multiple of 4");
  if (d.tile_h <= 0)
    while (g.TH > 1 && g.TH * (g.TW / kRWp) * g.C > 512) g.TH /= 2;   // channel-parallel CTA <= 512 threads
  g.tpc = g.TH * g.TW / kRWp;
  g.threads = g.tpc * g.C;
  g.magicC = (unsigned)((1u << 20) + g.C - 1) / (unsigned)g.C;
  if (g.tpc % 32 || g.threads > 512)
    return fail(ADP_ERR_ARG, "tile must map to 32-thread multiples per channel and <= 512 threads");
  g.tilesH = (g.H + g.TH - 1) / g.TH;
  g.tilesW = (g.W + g.TW - 1) / g.TW;
  g.nTiles = g.tilesH * g.tilesW;
  g.SH = g.TH + 2 * g.rh + 2;
  const int SWL = g.TW + 2 * g.rw + 2;
  g.SWP = kRWp == 1 ? SWL + 1 : SWL + SWL / kRWp + 1;
  g.SWPt = (SWL + 2 + 1) & ~1;   // dense TMA box: one extra column on each side, even pitch
  {
    const unsigned long long rowE = (unsigned long long)SWL * g.C;
    g.magicRow = (unsigned)(((1ull << 32) + rowE - 1) / rowE);
  }
  g.YSH = g.TH + 2;
  g.YSWP = (g.TW + 2) + (g.TW + 2) / kRWp + 1;
  g.N = (int64_t)g.H * g.W * g.C;
  g.tileOff = (g.row0 / g.TH) * g.tilesW;
  // division-free device indexing (exact for numerators < 2^16)
  auto magic = [](int d) { return d <= 1 ? 0u : (unsigned)(((1ull << 32) + d - 1) / d); };   // 0: d == 1
  g.magicTW = magic(g.tilesW);
  g.magicTWpx = magic(g.TW);
  g.segs = g.fused ? g.TW * g.C / g.leafL : 1;
  g.magicSegs = magic(g.segs);
  g.rowL = g.fused ? (int64_t)g.W * g.C / g.leafL : 0;
  if ((int64_t)g.tilesH * g.tilesW >= 65536 || g.W >= 65536)
    return fail(ADP_ERR_UNSUPPORTED, "more than 65535 tiles or columns per plan");
  if (slab) {
    if (!g.fused) return fail(ADP_ERR_UNSUPPORTED, "row slabs need the fused (tile-aligned pairwise) sum layout");
    const bool bottom = g.row0 + g.H == g.Hg && g.own1 == g.H;
    if (g.row0 % g.TH || g.own0 % g.TH || (g.own1 % g.TH && !bottom))
      return fail(ADP_ERR_ARG, "row slab bounds must be multiples of the tile height");
  }
  // fused candidate + speculative next stage when two plane regions fit
  // (leaves of 8 KB static smem headroom); ADP_FUSECA=0 disables
  g.fuseCA = 0;
  if (g.fused && !slab) {
    g.fuseCA = 1;
    const char* ev = getenv("ADP_FUSECA");
    if ((ev && atoi(ev) == 0) || conv_smem(g, P.esize) + 8192 > smem_optin) g.fuseCA = 0;
  }
  P.smem = conv_smem(g, P.esize, smem_optin);
  if (P.smem > smem_optin) return fail(ADP_ERR_UNSUPPORTED, "tile + halo exceeds shared memory; use a smaller tile");
  if (P.probe_only) return ADP_OK;   // adp_plan_probe: geometry only, no device memory

  // workspace: 18 N-arrays + 2 arrays of 2N
  const int64_t N = g.N;
  const size_t es = (size_t)P.esize;
  std::vector<size_t> sizes;
  for (int k = 0; k < 18; ++k) sizes.push_back((size_t)N * es);
  sizes.push_back((size_t)2 * N * es);
  sizes.push_back((size_t)2 * N * es);
  // sums
  ProgPool pool;
  SumHost sN, s2N, sT;
  const int nTilesG = ((g.Hg + g.TH - 1) / g.TH) * g.tilesW;
  build_sum(sN, g.Ng, true, pool);
  build_sum(s2N, 2 * g.Ng, true, pool);
  build_sum(sT, nTilesG, false, pool);
  // kgc partial groups
  {
    // kernel_gram_correlation groups: (tile row of 16 GLOBAL rows, column
    // block); the count depends on the geometry only (identical on every rank)
    const int thH = (g.Hg + 15) / 16, thW = (g.W + 15) / 16;
    P.kgc_cblocks = std::max(1, std::min(thW, (296 + thH - 1) / thH));
    P.kgc_groups = thH * P.kgc_cblocks;
  }
  const size_t nk = (size_t)g.kh * g.kw * g.C;
  // layout the device block
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  std::vector<size_t> wofs;
  for (size_t b : sizes) wofs.push_back(take(b));
  const size_t o_progs = take(pool.words.size() * sizeof(int));
  const size_t o_leafN = take(sN.leaf_start.size() * sizeof(int64_t));
  const size_t o_leaf2N = take(s2N.leaf_start.size() * sizeof(int64_t));
  const SumHost* shs[3] = {&sN, &s2N, &sT};
  size_t o_sl[3], o_sp[3];
  for (int k = 0; k < 3; ++k) {
    o_sl[k] = take(shs[k]->sub_leaf.size() * sizeof(int));
    o_sp[k] = take(shs[k]->sub_prog.size() * sizeof(int));
  }
  const int tileLeaves = std::max(sT.nLeaves, 4 * P.sm_count * 32);
  size_t o_lv[9], o_sv[9];
  const int nLeavesOf[9] = {sN.nLeaves, s2N.nLeaves, sN.nLeaves, s2N.nLeaves, tileLeaves, tileLeaves, tileLeaves,
                            sN.nLeaves, s2N.nLeaves};
  const int nSubOf[9] = {sN.nSub, s2N.nSub, sN.nSub, s2N.nSub, sT.nSub, sT.nSub, sT.nSub, sN.nSub, s2N.nSub};
  for (int k = 0; k < 9; ++k) {
    o_lv[k] = take((size_t)nLeavesOf[k] * sizeof(double));
    o_sv[k] = take((size_t)nSubOf[k] * sizeof(double));
  }
  const size_t o_bar = take(256);
  const size_t o_sres = take(sizeof(SolveOut));
  const size_t o_cres = take(sizeof(CGOut));
  const size_t o_scal = take(64 * sizeof(double));
  const size_t o_kgc = take((size_t)P.kgc_groups * nk * sizeof(double));
  P.dbytes = off;
  CK(cudaMalloc(&P.dmem, off));
  char* base = (char*)P.dmem;
  P.nws = (int)sizes.size();
  for (int k = 0; k < P.nws; ++k) P.ws[k] = base + wofs[k];
  P.d_progs = (int*)(base + o_progs);
  P.d_leaf_N = (int64_t*)(base + o_leafN);
  P.d_leaf_2N = (int64_t*)(base + o_leaf2N);
  CK(cudaMemcpy(P.d_progs, pool.words.data(), pool.words.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(P.d_leaf_N, sN.leaf_start.data(), sN.leaf_start.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(P.d_leaf_2N, s2N.leaf_start.data(), s2N.leaf_start.size() * sizeof(int64_t),
                cudaMemcpyHostToDevice));
  for (int k = 0; k < 3; ++k) {
    P.d_sub[2 * k] = (int*)(base + o_sl[k]);
    P.d_sub[2 * k + 1] = (int*)(base + o_sp[k]);
    CK(cudaMemcpy(P.d_sub[2 * k], shs[k]->sub_leaf.data(), shs[k]->sub_leaf.size() * sizeof(int),
                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(P.d_sub[2 * k + 1], shs[k]->sub_prog.data(), shs[k]->sub_prog.size() * sizeof(int),
                  cudaMemcpyHostToDevice));
  }
  SumDev* sds[9] = {&P.s_fit, &P.s_tv, &P.s_fitc, &P.s_tvc, &P.s_t0, &P.s_t1, &P.s_t2, &P.s_fit2, &P.s_tv2};
  const int which[9] = {0, 1, 0, 1, 2, 2, 2, 0, 1};
  for (int k = 0; k < 9; ++k) {
    const SumHost& sh = *shs[which[k]];
    const int64_t* dl = which[k] == 0 ? P.d_leaf_N : which[k] == 1 ? P.d_leaf_2N : nullptr;
    fill_sum<double>(*sds[k], sh, P.d_progs, dl, P.d_sub[2 * which[k]], P.d_sub[2 * which[k] + 1],
                     (double*)(base + o_lv[k]), (double*)(base + o_sv[k]));
  }
  // units each sum contributes: leaves, or subtree roots when two-level; a
  // slab fills only the ranges of its owned rows / tiles
  {
    const int64_t rowL = g.fused ? (int64_t)g.W * g.C / g.leafL : 0;
    const int64_t NL = g.fused ? g.Ng / g.leafL : 0;
    const int64_t l0 = (g.row0 + g.own0) * rowL, l1 = (g.row0 + g.own1) * rowL;
    const int64_t t0 = g.tileOff + (int64_t)(g.own0 / g.TH) * g.tilesW;
    const int64_t t1 = g.tileOff + (int64_t)((g.own1 + g.TH - 1) / g.TH) * g.tilesW;
    const int64_t rng[7][4] = {{l0, l1, 0, 0}, {l0, l1, l0 + NL, l1 + NL}, {l0, l1, 0, 0}, {l0, l1, l0 + NL, l1 + NL},
                               {t0, t1, 0, 0}, {t0, t1, 0, 0}, {t0, t1, 0, 0}};
    for (int k = 0; k < 7; ++k) {
      SumDev& sd = *sds[k];
      P.units_n[k] = sd.nSub > 1 ? sd.nSub : sd.nLeaves;
      for (int j = 0; j < 4; ++j) P.units_own[k][j] = slab ? rng[k][j] : (j == 1 ? P.units_n[k] : 0);
      if (slab && sd.nSub > 1) {
        for (int j = 0; j < 4; ++j) {
          const int64_t v = rng[k][j];
          const bool end = (j & 1) && v == (int64_t)sd.nLeaves;
          if (v % sd.sub_size && !end) return fail(ADP_ERR_UNSUPPORTED, "row slab is not aligned to the sum's subtrees");
          P.units_own[k][j] = (v + sd.sub_size - 1) / sd.sub_size;
        }
        sd.sub_own0 = (int)P.units_own[k][0];
        sd.sub_own1 = (int)P.units_own[k][1];
        sd.sub_own2 = (int)P.units_own[k][2];
        sd.sub_own3 = (int)P.units_own[k][3];
      }
    }
  }
  P.d_bar = (unsigned int*)(base + o_bar);
  P.d_sres = (SolveOut*)(base + o_sres);
  P.d_cres = (CGOut*)(base + o_cres);
  P.d_scal = (double*)(base + o_scal);
  P.d_kgc_part = (double*)(base + o_kgc);
  CK(cudaMallocHost(&P.h_sres, sizeof(SolveOut)));
  CK(cudaMallocHost(&P.h_cres, sizeof(CGOut)));
  CK(cudaMallocHost(&P.h_scal, 64 * sizeof(double)));

  ConvKernelSet ks = conv_kernels(P.d.dtype, P.d.mode, P.g.rwb);
  {
    const char* ev = getenv("ADP_K9");
    if (g.C == 1 && g.kh == 9 && g.kw == 9 && g.rwb == 2 && g.threads <= kSolveKSThreads &&
        P.d.dtype == ADP_DTYPE_F64 && !(ev && atoi(ev) == 0)) {
      ks.solve = conv_solve_k9(P.d.mode == ADP_MODE_FAST);
      // TMA tile boxes for the c2 kernel (ADP_TMA=0: the LDS-fed loaders)
      const char* et = getenv("ADP_TMA");
      if (!(et && atoi(et) == 0) && !slab && (size_t)g.SH * g.SWPt <= (size_t)g.SH * g.SWP &&
          P.smem + 128 <= smem_optin && build_tmaps(P) == ADP_OK) {
        P.tma = 1;
        P.smem += 128;   // the kernel aligns its dynamic shared-memory base to 128 bytes
        ks.solve = conv_solve_k9_tma(P.d.mode == ADP_MODE_FAST);
      }
    }
    else if (g.rwb == 4 && g.threads <= kSolveT384 && !(getenv("ADP_T384") && atoi(getenv("ADP_T384")) == 0))
      ks.solve = conv_solve_t384(P.d.dtype, P.d.mode == ADP_MODE_FAST);
  }
  // host-stepped high-occupancy solve (conv2d_step.cu): float64 RW = 4 plans
  // with fused leaves, not slabs; ADP_STEP=0 disables, =1 enables for every
  // eligible plan, default: images of >= 2^18 elements (c3-c5)
  {
    const char* ev = getenv("ADP_STEP");
    const int want = ev ? atoi(ev) : -1;
    if (want != 0 && P.d.dtype == ADP_DTYPE_F64 && g.rwb == 4 && g.fused && !slab &&
        g.threads <= 384 && (want == 1 || g.N >= (1 << 18)) &&
        ((g.kh * g.kw + 1) & ~1) * g.C <= ((g.kh == 31 && g.kw == 31) ? kStepWMax : kStepWSmall) &&
        g.tpc % 32 == 0) {   // taps as kernel parameters (the 31 x 31 instances take the large block); channel-uniform warps
      const size_t es = (size_t)P.esize;
      const size_t pa = ((size_t)g.C * g.SH * g.SWP * es + 127) & ~size_t(127);
      const size_t tm = (size_t)3 * g.TH * g.TW * g.C * sizeof(double);
      P.step_o_tm = g.o_pa + (int)pa;
      P.step_smem = (size_t)P.step_o_tm + tm;
      StepKernels sk = step_kernels(P.d.mode == ADP_MODE_FAST, g.kh == g.kw ? g.kh : 0);
      P.k_extrap = sk.extrap;
      P.k_cand = sk.cand;
      P.step_smem_b = sk.b_ep == 2 ? P.step_smem : (size_t)g.o_pa + pa;   // stage B: no term buffers (three CTAs per SM)
      if (setup_kernel(P, P.k_sb, sk.b, g.threads, P.step_smem_b, g.nTiles) == ADP_OK &&
          setup_kernel(P, P.k_sca, sk.ca, g.threads, P.step_smem, 2 * g.nTiles) == ADP_OK &&
          setup_kernel(P, P.k_sc, sk.c, g.threads, P.step_smem, g.nTiles) == ADP_OK &&
          setup_kernel(P, P.k_sa, sk.a, g.threads, P.step_smem, g.nTiles) == ADP_OK &&
          setup_kernel(P, P.k_sred, sk.red, g.threads, P.smem, g.nTiles) == ADP_OK) {
        CK(cudaMallocHost(&P.h_kern, (size_t)g.kh * g.kw * g.C * sizeof(double)));
        P.step = 1;
        P.pdl = !(getenv("ADP_PDL") && atoi(getenv("ADP_PDL")) == 0);
        // in-kernel decision sums (step_tail.h): whole tiles, tile rows = power-of-two runs of the
        // perfect sum trees, every fold within one register pass (<= 1024 units); ADP_TAIL=0 disables
        auto pow2 = [](int64_t v) { return v > 0 && (v & (v - 1)) == 0; };
        const int64_t GL = (int64_t)g.TH * g.rowL;
        const char* et = getenv("ADP_TAIL");
        if (!(et && atoi(et) == 0) && g.H % g.TH == 0 && g.W % g.TW == 0 && pow2(GL) && GL <= 1024 &&
            pow2(g.tilesW) && g.tilesW <= 1024 && pow2(g.tilesH) && 2 * g.tilesH <= 1024 && P.s_fit.regular &&
            P.s_tv.regular && P.s_t0.regular && (int64_t)P.s_fit.nLeaves == GL * g.tilesH &&
            (int64_t)P.s_tv.nLeaves == 2 * GL * g.tilesH && g.threads >= 64) {
          const size_t nsub = (size_t)11 * g.tilesH * sizeof(double);
          const size_t ncnt = 64;
          const size_t nflag = (size_t)2 * g.nTiles * sizeof(unsigned int);   // stage-B tiles, stage-A tiles
          CK(cudaMalloc(&P.d_tail, nsub + ncnt + nflag));
          CK(cudaMemset(P.d_tail, 0, nsub + ncnt + nflag));
          P.tail.sub = (double*)P.d_tail;
          P.tail.cnt = (unsigned int*)((char*)P.d_tail + nsub);
          // the candidate launch overlaps the stage-B launch's last wave (per-tile completion flags,
          // conv2d_step.cu); needs programmatic dependent launch; ADP_OVL=0: off
          const char* eo = getenv("ADP_OVL");
          if (P.pdl && !(eo && atoi(eo) == 0)) P.d_tflag = (unsigned int*)((char*)P.d_tail + nsub + ncnt);
          // ADP_OVL=2: stage B also overlaps the candidate launch's last wave (stage-A tile flags); measured
          // and left off: the stage-A CTAs' release costs what the overlap gains (117.9 vs 117.8 us at c3)
          P.ovl_b = eo && atoi(eo) == 2;
          P.tail.on = 1;
          P.tail.nG = g.tilesH;
          P.tail.GL = (int)GL;
          P.tail.tW = g.tilesW;
          P.tail.gpr = std::min(g.tilesH, 8);   // tile rows per reducer CTA
          P.tail.nR = g.tilesH / P.tail.gpr;
        }
      }
    }
  }
  const int maxg = g.nTiles;
  if (int e = setup_kernel(P, P.k_solve, ks.solve, g.threads, P.smem, maxg)) return e;
  if (int e = setup_kernel(P, P.k_cg, ks.cg, g.threads, P.smem, maxg)) return e;
  if (int e = setup_kernel(P, P.k_misc, ks.misc, g.threads, P.smem, maxg)) return e;
  g.grid = P.k_solve.grid;
  P.k_misc.attr_set = true;
  return ADP_OK;
}

// ---------------------------------------------------------------------------
template <typename T>
static ConvArgs<T> conv_base(PlanImpl& P) {
  ConvArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.g = P.g;
  T** w = (T**)P.ws;
  a.X[0] = w[0]; a.X[1] = w[1]; a.X[2] = w[2];
  a.R = w[3]; a.RC = w[4]; a.G = w[5]; a.TVG = w[6];
  a.DIAG = w[7]; a.WV = w[8]; a.WH = w[9];
  a.P[0] = w[10]; a.P[1] = w[11]; a.BP = w[12]; a.HP = w[13]; a.CR = w[14]; a.CS = w[15];
  a.TV2 = w[18]; a.TV2C = w[19];
  a.s_fit = P.s_fit; a.s_tv = P.s_tv; a.s_fitc = P.s_fitc; a.s_tvc = P.s_tvc;
  a.s_t0 = P.s_t0; a.s_t1 = P.s_t1; a.s_t2 = P.s_t2;
  a.s_fit2 = P.s_fit2; a.s_tv2 = P.s_tv2;
  if (P.tma) std::memcpy(a.tm, P.tm, sizeof(a.tm));
  a.bar = P.d_bar;
  a.sres = P.d_sres;
  a.cres = P.d_cres;
  a.scal = P.d_scal;
  return a;
}

template <typename T>
static void set_lower(ConvArgs<T>& a, const adp_lower* lp) {
  a.kern = (const T*)lp->kernel;
  a.ydat = (const T*)lp->y;
  a.alpha = lp->alpha;
  a.nu = lp->nu;
  a.reg = lp->reg;
  a.regcurv = 8.0 / lp->nu;   // SmoothedTV.curvature (regularizers.py:148-156)
}

template <typename T>
static int launch_coop(PlanImpl& P, KernelInfo& k, ConvArgs<T>& a, cudaStream_t st) {
  if ((P.g.Hg != P.g.H || P.g.row0) && !(k.fn == P.k_misc.fn && a.mode >= CM_SLAB_ABC))
    return fail(ADP_ERR_UNSUPPORTED, "row-slab plans run adp_slab_step only");
  a.g.grid = k.grid;
  CK(cudaMemsetAsync(P.d_bar, 0, sizeof(unsigned int), st));
  void* args[] = {&a};
  CK(cudaLaunchCooperativeKernel(k.fn, dim3(k.grid), dim3(P.g.threads), args, P.smem, st));
  return ADP_OK;
}

static int fetch_scal(PlanImpl& P, int n, cudaStream_t st) {
  CK(cudaMemcpyAsync(P.h_scal, P.d_scal, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return ADP_OK;
}

template <typename T>
static int conv_misc(PlanImpl& P, int mode, const adp_lower* lp, const void* kernel, const void* in0,
                     const void* in1, void* out0, void* out1, const void* ydat, cudaStream_t st) {
  ConvArgs<T> a = conv_base<T>(P);
  if (lp) set_lower(a, lp);
  if (kernel) a.kern = (const T*)kernel;
  if (ydat) a.ydat = (const T*)ydat;
  a.mode = mode;
  a.in0 = (const T*)in0;
  a.in1 = (const T*)in1;
  a.out0 = (T*)out0;
  a.out1 = (T*)out1;
  return launch_coop(P, P.k_misc, a, st);
}

template <typename T>
static int conv_slab_step(PlanImpl& P, const adp_lower* lp, int op, const void* x, const void* xp, void* out,
                          double beta, double L, cudaStream_t st) {
  static const int modes[5] = {CM_SLAB_ABC, CM_SLAB_C, CM_SLAB_POWER, CM_SLAB_NORM0, CM_SLAB_GRAD};
  ConvArgs<T> a = conv_base<T>(P);
  if (lp) set_lower(a, lp);
  a.mode = modes[op];
  a.in0 = (const T*)x;
  a.in1 = (const T*)xp;
  a.out0 = (T*)out;
  a.sbeta = beta;
  a.sL = L;
  return launch_coop(P, P.k_misc, a, st);
}

template <typename T>
static int conv_kgc(PlanImpl& P, const void* xa, const void* va, const void* xb, const void* vb, void* out,
                    double scale, cudaStream_t st, double* part) {
  // part != null: row slab, partials of the owned groups into the caller's vector (no final sum)
  if ((P.g.Hg != P.g.H || P.g.row0) && !part) return fail(ADP_ERR_UNSUPPORTED, "row-slab plans: use adp_slab_mixed");
  ConvKernelSet ks = conv_kernels(P.d.dtype, P.d.mode, P.g.rwb);
  KgcArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.g = P.g;
  a.xa = (const T*)xa; a.va = (const T*)va; a.xb = (const T*)xb; a.vb = (const T*)vb;
  a.part = part ? part : P.d_kgc_part;
  a.ngroups = P.kgc_groups;
  a.cblocks = P.kgc_cblocks;
  a.out = (T*)out;
  a.scale = scale;
  const int KT = 16;
  const size_t smem = ((size_t)(KT + P.g.kh - 1) * (KT + P.g.kw - 1) + KT * KT) * sizeof(T);
  CK(cudaFuncSetAttribute(ks.kgc_part, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem_optin));
  void* args[] = {&a};
  CK(cudaLaunchKernel(ks.kgc_part, dim3(P.kgc_groups), dim3(256), args, smem, st));
  if (part) return ADP_OK;
  const int n = P.g.kh * P.g.kw * P.g.C;
  CK(cudaLaunchKernel(ks.kgc_final, dim3((n + 255) / 256), dim3(256), args, 0, st));
  return ADP_OK;
}

template <typename T>
static int conv_kgc_final(PlanImpl& P, const double* part, void* out, double scale, cudaStream_t st) {
  ConvKernelSet ks = conv_kernels(P.d.dtype, P.d.mode, P.g.rwb);
  KgcArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.g = P.g;
  a.part = const_cast<double*>(part);
  a.ngroups = P.kgc_groups;
  a.cblocks = P.kgc_cblocks;
  a.out = (T*)out;
  a.scale = scale;
  void* args[] = {&a};
  const int n = P.g.kh * P.g.kw * P.g.C;
  CK(cudaLaunchKernel(ks.kgc_final, dim3((n + 255) / 256), dim3(256), args, 0, st));
  return ADP_OK;
}

template <typename T>
static int conv_slab_cg(PlanImpl& P, const adp_lower* lp, int op, const void* in0, const void* in1, void* out0,
                        void* out1, double s, int flag, cudaStream_t st) {
  static const int modes[4] = {CM_SLAB_CG_DIAG, CM_SLAB_CG_INIT, CM_SLAB_CG_HV, CM_SLAB_CG_UPD};
  ConvArgs<T> a = conv_base<T>(P);
  set_lower(a, lp);
  a.mode = modes[op];
  a.in0 = (const T*)in0;
  a.in1 = (const T*)in1;
  a.out0 = (T*)out0;
  a.out1 = (T*)out1;
  a.sbeta = s;
  a.sL = s;
  a.sflag = flag;
  return launch_coop(P, P.k_misc, a, st);
}

}  // namespace adp

using namespace adp;

// ===========================================================================
// dense 1-D dispatch (adp_dense.cu)
namespace adp {
int dense_plan_init(PlanImpl& P);
int dense_call(PlanImpl& P, int op, const void* kernel, const adp_lower* lp, const void* a0, const void* a1,
               void* o0, void* o1, const void* ydat, double* scal, cudaStream_t st);
int dense_solve(PlanImpl& P, const adp_lower* lp, const void* x0, void* x_out, const adp_solve_args* args,
                adp_solve_result* res, cudaStream_t st);
int dense_cg(PlanImpl& P, const adp_lower* lp, const void* xt, const void* rhs, void* q, int warm,
             const void* precond, double tol, int max_iters, adp_cg_result* res, cudaStream_t st);
int dense_prox(PlanImpl& P, const adp_lower* lp, const void* x0, void* x_out, int n_iters, double step,
               cudaStream_t st);
void dense_plan_free(PlanImpl& P);
}  // namespace adp

#define DISPATCH_T(P, CALL)                          \
  ((P).d.dtype == ADP_DTYPE_F32 ? CALL<float> : CALL<double>)

extern "C" {

const char* adp_last_error(void) { return g_err.c_str(); }

int adp_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev));
  CK(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
  return ADP_OK;
}

int adp_plan_create(adp_plan** out, const adp_plan_desc* desc) {
  if (!out || !desc) return fail(ADP_ERR_ARG, "null argument");
  *out = nullptr;
  const adp_plan_desc& d = *desc;
  if (d.dtype != ADP_DTYPE_F64 && d.dtype != ADP_DTYPE_F32) return fail(ADP_ERR_ARG, "bad dtype");
  if (d.H < 1 || d.W < 1 || d.C < 1) return fail(ADP_ERR_ARG, "bad shape");
  if (d.layout == ADP_LAYOUT_DEPTHWISE2D) {
    if (d.kh < 1 || d.kw < 1 || d.kh % 2 == 0 || d.kw % 2 == 0)
      return fail(ADP_ERR_ARG, "depthwise2d kernel must have odd spatial size");
  } else if (d.layout == ADP_LAYOUT_DENSE1D) {
    if (d.H != 1 || d.C != 1 || d.kh != d.W || d.kw != d.W) return fail(ADP_ERR_ARG, "bad dense1d plan");
  } else {
    return fail(ADP_ERR_ARG, "unknown layout");
  }
  adp_plan* p = new adp_plan();
  p->impl.d = d;
  p->impl.esize = d.dtype == ADP_DTYPE_F32 ? 4 : 8;
  int e = d.layout == ADP_LAYOUT_DEPTHWISE2D ? conv_plan_init(p->impl) : dense_plan_init(p->impl);
  if (e) {
    adp_plan_destroy(p);
    return e;
  }
  *out = p;
  return ADP_OK;
}

void adp_plan_destroy(adp_plan* p) {
  if (!p) return;
  PlanImpl& P = p->impl;
  if (P.d.layout == ADP_LAYOUT_DENSE1D) dense_plan_free(P);
  if (P.dmem) cudaFree(P.dmem);
  if (P.d_zero) cudaFree(P.d_zero);
  if (P.d_tail) cudaFree(P.d_tail);
  if (P.h_sres) cudaFreeHost(P.h_sres);
  if (P.h_cres) cudaFreeHost(P.h_cres);
  if (P.h_scal) cudaFreeHost(P.h_scal);
  if (P.h_flag) cudaFreeHost(P.h_flag);
  if (P.h_kern) cudaFreeHost(P.h_kern);
  if (P.prof_ev[0]) cudaEventDestroy(P.prof_ev[0]);
  if (P.prof_ev[1]) cudaEventDestroy(P.prof_ev[1]);
  delete p;
}

size_t adp_plan_workspace_bytes(const adp_plan* p) { return p ? p->impl.dbytes : 0; }

#define STREAM(s) ((cudaStream_t)(s))
#define IS_DENSE(p) ((p)->impl.d.layout == ADP_LAYOUT_DENSE1D)

enum DenseOp { DO_APPLY, DO_ADJOINT, DO_GRAM, DO_VALUE, DO_VG, DO_GRAD, DO_HV, DO_HDIAG, DO_UPPER, DO_POWER, DO_MIXED,
               DO_DOT, DO_KGC };

int adp_apply(adp_plan* p, const void* kernel, const void* x, void* out, void* stream) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  if (IS_DENSE(p)) return dense_call(p->impl, DO_APPLY, kernel, nullptr, x, nullptr, out, nullptr, nullptr, nullptr, STREAM(stream));
  return DISPATCH_T(p->impl, conv_misc)(p->impl, CM_APPLY, nullptr, kernel, x, nullptr, out, nullptr, nullptr,
                                        STREAM(stream));
}

int adp_adjoint(adp_plan* p, const void* kernel, const void* y, void* out, void* stream) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  if (IS_DENSE(p)) return dense_call(p->impl, DO_ADJOINT, kernel, nullptr, y, nullptr, out, nullptr, nullptr, nullptr, STREAM(stream));
  return DISPATCH_T(p->impl, conv_misc)(p->impl, CM_ADJOINT, nullptr, kernel, y, nullptr, out, nullptr, nullptr,
                                        STREAM(stream));
}

int adp_gram_diag(adp_plan* p, const void* kernel, void* out, void* stream) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  if (IS_DENSE(p)) return dense_call(p->impl, DO_GRAM, kernel, nullptr, nullptr, nullptr, out, nullptr, nullptr, nullptr, STREAM(stream));
  return DISPATCH_T(p->impl, conv_misc)(p->impl, CM_GRAM_DIAG, nullptr, kernel, nullptr, nullptr, out, nullptr,
                                        nullptr, STREAM(stream));
}

int adp_op_norm_sq(adp_plan* p, const void* kernel, const void* v0, int32_t max_iters, double tol, double* lam,
                   int32_t* converged, int32_t* iters, void* stream) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  PlanImpl& P = p->impl;
  int e;
  if (IS_DENSE(p)) {
    double sc[3];
    adp_lower lp{};
    lp.kernel = kernel;
    lp.l1 = tol;
    lp.alpha = (double)max_iters;
    e = dense_call(P, DO_POWER, kernel, &lp, v0, nullptr, nullptr, nullptr, nullptr, sc, STREAM(stream));
    if (e) return e;
    *lam = sc[0]; *converged = (int)sc[1]; *iters = (int)sc[2];
    return ADP_OK;
  }
  auto run = [&](auto tag) -> int {
    using T = decltype(tag);
    ConvArgs<T> a = conv_base<T>(P);
    a.kern = (const T*)kernel;
    a.v0 = (const T*)v0;
    a.mode = CM_POWER;
    a.power_max_iters = max_iters;
    a.power_tol = tol;
    if (int e2 = launch_coop(P, P.k_misc, a, STREAM(stream))) return e2;
    if (int e2 = fetch_scal(P, 3, STREAM(stream))) return e2;
    *lam = P.h_scal[0];
    *converged = (int)P.h_scal[1];
    *iters = (int)P.h_scal[2];
    return ADP_OK;
  };
  return P.d.dtype == ADP_DTYPE_F32 ? run(float()) : run(double());
}

int adp_kgc(adp_plan* p, const void* x, const void* v, void* out, void* stream) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  if (IS_DENSE(p)) return dense_call(p->impl, DO_KGC, nullptr, nullptr, x, v, out, nullptr, nullptr, nullptr, STREAM(stream));
  return DISPATCH_T(p->impl, conv_kgc)(p->impl, x, v, nullptr, nullptr, out, 1.0, STREAM(stream), nullptr);
}

static int check_lower(adp_plan* p, const adp_lower* lp) {
  if (!p || !lp) return fail(ADP_ERR_ARG, "null argument");
  if (!IS_DENSE(p) && lp->reg != ADP_REG_TV) return fail(ADP_ERR_UNSUPPORTED, "depthwise2d path supports SmoothedTV");
  if (lp->reg == ADP_REG_TV && lp->alpha != 0.0 && !(lp->nu > 0.0))
    return fail(ADP_ERR_ARG, "gradient requested on the nonsmooth branch (nu = 0)");
  return ADP_OK;
}

int adp_lower_value(adp_plan* p, const adp_lower* lp, const void* x, double* value, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) return dense_call(P, DO_VALUE, lp->kernel, lp, x, nullptr, nullptr, nullptr, nullptr, value, STREAM(stream));
  if (int e = DISPATCH_T(P, conv_misc)(P, CM_VALUE, lp, nullptr, x, nullptr, nullptr, nullptr, nullptr, STREAM(stream)))
    return e;
  if (int e = fetch_scal(P, 1, STREAM(stream))) return e;
  *value = P.h_scal[0];
  return ADP_OK;
}

int adp_lower_value_and_grad(adp_plan* p, const adp_lower* lp, const void* x, double* value, void* g, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) return dense_call(P, DO_VG, lp->kernel, lp, x, nullptr, g, nullptr, nullptr, value, STREAM(stream));
  if (int e = DISPATCH_T(P, conv_misc)(P, CM_VALUE_GRAD, lp, nullptr, x, nullptr, g, nullptr, nullptr, STREAM(stream)))
    return e;
  if (int e = fetch_scal(P, 2, STREAM(stream))) return e;
  *value = P.h_scal[0];
  return ADP_OK;
}

int adp_lower_grad(adp_plan* p, const adp_lower* lp, const void* x, void* g, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) return dense_call(P, DO_GRAD, lp->kernel, lp, x, nullptr, g, nullptr, nullptr, nullptr, STREAM(stream));
  return DISPATCH_T(P, conv_misc)(P, CM_GRAD, lp, nullptr, x, nullptr, g, nullptr, nullptr, STREAM(stream));
}

int adp_lower_hess_vec(adp_plan* p, const adp_lower* lp, const void* x, const void* v, void* out, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) return dense_call(P, DO_HV, lp->kernel, lp, x, v, out, nullptr, nullptr, nullptr, STREAM(stream));
  return DISPATCH_T(P, conv_misc)(P, CM_HESS_VEC, lp, nullptr, x, v, out, nullptr, nullptr, STREAM(stream));
}

int adp_lower_hess_diag(adp_plan* p, const adp_lower* lp, const void* x, void* out, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) return dense_call(P, DO_HDIAG, lp->kernel, lp, x, nullptr, out, nullptr, nullptr, nullptr, STREAM(stream));
  return DISPATCH_T(P, conv_misc)(P, CM_HESS_DIAG, lp, nullptr, x, nullptr, out, nullptr, nullptr, STREAM(stream));
}

// ---------------------------------------------------------------------------
// Host-stepped solve_lower (adaptive AGD with restart on smoothed TV,
// lower_solvers.py:104-213) for plans with P.step: the persistent kernel's
// stages as one-tile-per-CTA kernels (conv2d_step.cu) and its scalar control
// flow here, expression for expression (conv_solve_kernel), so iterates,
// decisions and counters are identical to the single-launch solve.
static int step_launch(PlanImpl& P, KernelInfo& k, ConvArgs<double>& a, cudaStream_t st, bool coop, size_t smem,
                       int grid, const StepWL* wt = nullptr, const StepTail* tl = nullptr) {
  void* args[] = {&a, (void*)wt, (void*)tl};
  if (coop) {
    CK(cudaMemsetAsync(P.d_bar, 0, sizeof(unsigned int), st));
    CK(cudaLaunchCooperativeKernel(k.fn, dim3(grid), dim3(P.g.threads), args, smem, st));
  } else {
    // programmatic dependent launch: the stage kernel's CTAs may become resident while the previous
    // stage kernel drains (it signals at its start); they wait (griddepcontrol.wait) for that grid's
    // completion before touching its data, so only launch latency and index set-up overlap.  ADP_PDL=0: off
    const bool pdl = P.pdl;   // read at plan creation
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(P.g.threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelExC(&cfg, k.fn, args));
  }
  return ADP_OK;
}

static int conv_solve_step(PlanImpl& P, const adp_lower* lp, const void* x0, void* x_out, const adp_solve_args* sa,
                           adp_solve_result* res, cudaStream_t st) {
  using T = double;
  const ConvGeom& g = P.g;
  ConvArgs<T> base = conv_base<T>(P);
  set_lower(base, lp);
  // the stage kernels' taps as kernel parameters (StepW): forward [c][i][j] and flipped, ndimage's
  // |w| <= DBL_EPSILON taps zeroed (Conv::load_weights' rule)
  const int kk = g.kh * g.kw, nk = kk * g.C, kkp = (kk + 1) & ~1;   // channel blocks padded to even
  CK(cudaMemcpyAsync(P.h_kern, lp->kernel, (size_t)nk * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int e = 0; e < nk; ++e) {
    const int c = e % g.C, ij = e / g.C, i = ij / g.kw, j = ij % g.kw;
    double w = P.h_kern[e];
    if (!(fabs(w) > 2.220446049250313e-16)) w = 0.0;
    P.wfwd.w[c * kkp + i * g.kw + j] = w;
    P.wadj.w[c * kkp + (g.kh - 1 - i) * g.kw + (g.kw - 1 - j)] = w;
  }
  ConvArgs<T> sa_args = base;   // stage kernels: one plane region, term buffers right after it
  sa_args.g.o_tm = P.step_o_tm;
  sa_args.g.o_pa2 = P.step_o_tm;   // never addressed with one tile per CTA
  const double alpha = lp->alpha, nu = lp->nu;
  const double twoN = 2.0 * (double)g.N;
  const double tol = sa->eps * sa->mu;
  long long launches = 0, dom_n = 0;
  double dom_ms = 0.0;
  bool prof_now = false, prof_pending = false;
  // ---- step size / Lipschitz constant (solve_lower lines 135-140, L_of_b 90-96)
  double lip, lam = sa->norm_sq;
  int pit = 0, pconv = 1;
  if (sa->step_size > 0) {
    lip = 1.0 / sa->step_size;
  } else {
    if (!(sa->norm_sq >= 0.0)) {
      ConvArgs<T> a = base;
      a.v0 = (const T*)sa->v0;
      a.mode = CM_POWER;
      a.power_max_iters = sa->norm_max_iters;
      a.power_tol = sa->norm_tol;
      if (int e = launch_coop(P, P.k_misc, a, st)) return e;
      if (int e = fetch_scal(P, 3, st)) return e;
      lam = P.h_scal[0];
      pconv = (int)P.h_scal[1];
      pit = (int)P.h_scal[2];
      ++launches;
    }
    lip = 2.0 * lam + alpha * (8.0 / nu);
  }
  // ---- x = x_prev = x0 (or the injected state of a P2 lockstep step)
  T* X[3] = {(T*)P.ws[0], (T*)P.ws[1], (T*)P.ws[2]};
  T* Yn = (T*)P.ws[10];
  const size_t nbytes = (size_t)g.N * sizeof(T);
  CK(cudaMemcpyAsync(X[0], x0, nbytes, cudaMemcpyDeviceToDevice, st));
  if (sa->x_prev0) CK(cudaMemcpyAsync(X[1], sa->x_prev0, nbytes, cudaMemcpyDeviceToDevice, st));
  if (P.tail.on) {
    // the candidate half's sum units start unwritten (all-ones pattern, step_tail.h); the reducers
    // reset what they read, so this covers units left by other kernels of the plan
    CK(cudaMemsetAsync(P.s_fitc.leaf_vals, 0xFF, (size_t)P.s_fitc.nLeaves * sizeof(double), st));
    CK(cudaMemsetAsync(P.s_tvc.leaf_vals, 0xFF, (size_t)P.s_tvc.nLeaves * sizeof(double), st));
    CK(cudaMemsetAsync(P.s_t1.leaf_vals, 0xFF, (size_t)g.nTiles * sizeof(double), st));
  }
  int ix = 0, ixp = sa->x_prev0 ? 1 : 0, ic = sa->x_prev0 ? 2 : 1;
  double t_mom = sa->t_mom0 > 0.0 ? sa->t_mom0 : 1.0, lip_t = sa->lip_t0 > 0.0 ? sa->lip_t0 : lip;
  int status = ST_OK, fail_iter = -1, iters = sa->max_iters, converged = 0;
  double gn = 0.0, h_y = 0.0, beta = 0.0;
  long long vg = 0, vals = 0, restarts = 0;
  bool done = false, a_ready = false;
  unsigned int last_aseq = 0;   // != 0: the last launch queued is a candidate launch publishing its stage-A tiles
  int par = 0;
  const int nT = g.nTiles;
  if (P.profile && !P.prof_ev[0]) {
    CK(cudaEventCreate(&P.prof_ev[0]));
    CK(cudaEventCreate(&P.prof_ev[1]));
  }
  if (!P.h_flag) {
    CK(cudaHostAlloc(&P.h_flag, sizeof(int), cudaHostAllocMapped));
    *(volatile int*)P.h_flag = 0;
  }
  double* d_hscal = nullptr;
  int* d_hflag = nullptr;
  CK(cudaHostGetDevicePointer((void**)&d_hscal, P.h_scal, 0));
  CK(cudaHostGetDevicePointer((void**)&d_hflag, P.h_flag, 0));
  // the reduction writes its sums and then a sequence number into mapped pinned memory; the host
  // spins on the number (no stream synchronisation on the decision path), checking for errors
  auto wait_flag = [&](int seq) -> int {
    for (long long spin = 0; *(volatile int*)P.h_flag != seq; ++spin) {
      if ((spin & 0xfffff) == 0xfffff) {
        const cudaError_t q = cudaStreamQuery(st);
        if (q != cudaErrorNotReady && q != cudaSuccess) return fail(ADP_ERR_CUDA, cudaGetErrorString(q));
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return ADP_OK;
  };
  auto reduce = [&](int mode, int n) -> int {
    ConvArgs<T> a = base;
    a.sflag = mode;
    a.hscal = d_hscal;
    a.hflag = d_hflag;
    a.hseq = ++P.step_seq;
    if (int e = step_launch(P, P.k_sred, a, st, true, P.smem, P.k_sred.grid)) return e;
    ++launches;
    (void)n;
    return wait_flag(a.hseq);
  };
  for (int t = 0; t < sa->max_iters; ++t) {
    const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t_mom * t_mom));
    beta = (t_mom - 1.0) / t_next;
    t_mom = t_next;
    double L_try = lip_t;
    if (!a_ready) {   // stage A at y = x + beta (x - x_prev), sums set `par`
      ConvArgs<T> a = sa_args;
      a.in0 = X[ix]; a.in1 = X[ixp]; a.sbeta = beta; a.sflag = 1 | (par ? 2 : 0);
      last_aseq = 0;
      if (int e = step_launch(P, P.k_sa, a, st, false, P.step_smem, nT, &P.wfwd)) return e;
      ++launches;
    }
    const double t_next2 = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t_mom * t_mom));   // next momentum, no restart
    const double beta2 = (t_mom - 1.0) / t_next2;
    {   // stage B: g, first candidate, next extrapolation point
      ConvArgs<T> a = sa_args;
      a.in0 = X[ix]; a.in1 = X[ixp]; a.out0 = X[ic]; a.out1 = Yn;
      a.sbeta = beta; a.sL = L_try; a.sbetaN = beta2;
      a.tflag = P.d_tflag; a.tseq = ++P.tile_seq;
      // directly after a candidate launch whose speculative stage A is this launch's input: overlap it
      if (P.d_tflag && a_ready && last_aseq) { a.sflag = 1; a.hseq = (int)last_aseq; }
      last_aseq = 0;
      if (int e = step_launch(P, P.k_sb, a, st, false, P.step_smem_b, nT, &P.wadj)) return e;
      ++launches;
    }
    {   // candidate value + restart dot, and the speculative stage A at y' (valid iff the candidate is
        // accepted without retry or restart; the other sums set), in one launch
      ConvArgs<T> a = sa_args;
      a.in0 = X[ic]; a.in1 = X[ix]; a.out1 = Yn; a.sflag = par ? 0 : 2;
      if (prof_pending) {   // the sampled launch of an earlier iteration has completed (stream order)
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, P.prof_ev[0], P.prof_ev[1]) == cudaSuccess) {
          dom_ms += ms;
          ++dom_n;
          prof_pending = false;
        } else {
          (void)cudaGetLastError();   // not ready yet: keep the events for a later iteration
        }
      }
      StepTail tl = P.tail;
      tl.setR = par;   // (the speculative stage A writes the other (fit, tv) set)
      // overlap with the stage-B launch just queued (not for the sampled, event-bracketed launch)
      prof_now = P.profile && (t % P.profile == 0) && !prof_pending;   // sampled: every P.profile-th iteration
      tl.ovl = tl.on && P.d_tflag && !prof_now;
      a.tflag = P.d_tflag; a.tseq = P.tile_seq;
      if (tl.on && P.d_tflag && P.ovl_b && !prof_now) last_aseq = tl.aseq = ++P.a_seq ? P.a_seq : ++P.a_seq;
      if (tl.on) {   // reducer CTAs publish the six sums (step_tail.h)
        a.hscal = d_hscal;
        a.hflag = d_hflag;
        a.hseq = ++P.step_seq;
      }
      if (prof_now) CK(cudaEventRecord(P.prof_ev[0], st));
      if (int e = step_launch(P, P.k_sca, a, st, false, P.step_smem, 2 * nT + (tl.on ? tl.nR : 0), &P.wfwd, &tl))
        return e;
      if (prof_now) {
        CK(cudaEventRecord(P.prof_ev[1], st));
        prof_pending = true;
      }
      ++launches;
      if (tl.on) {
        if (int e = wait_flag(a.hseq)) return e;
      }
    }
    ++vg;
    ++vals;
    if (!P.tail.on) {
      if (int e = reduce(par, 6)) return e;
    }
    const double* o = P.h_scal;
    const double fit = o[0];
    h_y = fit + alpha * (o[1] - nu * twoN);
    gn = sqrt(o[2]);
    double dot = o[3];
    double fitc = o[4], tvc = o[5];
    if (!std::isfinite(gn)) { status = ST_DIVERGED; fail_iter = t; done = true; break; }
    if (gn <= tol) {
      // converged: return y (lower_solvers.py:200-201)
      const int64_t n = g.N;
      const T* xp = X[ix];
      const T* xpp = X[ixp];
      T bb = (T)beta;
      T* outp = (T*)x_out;
      int64_t nn = n;
      void* args[] = {(void*)&xp, (void*)&xpp, (void*)&bb, (void*)&outp, (void*)&nn};
      CK(cudaLaunchKernel(P.k_extrap, dim3(4 * P.sm_count), dim3(256), args, 0, st));
      ++launches;
      iters = t;
      converged = 1;
      done = true;
      break;
    }
    int k = 0;
    while (true) {   // _backtracked_step (lower_solvers.py:170-177)
      const double val = fitc + alpha * tvc;
      if (val <= h_y - 0.5 * gn * gn / L_try + 1e-15 * fabs(h_y)) break;
      L_try *= 2.0;
      if (++k >= 60) { status = ST_BT_FAIL; fail_iter = t; break; }
      if (P.tail.on) {
        // in-kernel sums: the retry's candidate and next extrapolation point are materialised
        // elementwise, then the candidate-value + speculative stage-A launch runs as for the first
        // candidate (its reducers fold all six sums again; the first three are unchanged)
        {
          const T* xp_ = X[ix]; const T* xpp_ = X[ixp]; const T* gp_ = (const T*)P.ws[5];
          T b_ = (T)beta, L_ = (T)L_try, bn_ = (T)beta2;
          T* o0 = X[ic]; T* o1 = Yn;
          int64_t nn = g.N;
          void* cargs[] = {(void*)&xp_, (void*)&xpp_, (void*)&gp_, (void*)&b_, (void*)&L_, (void*)&bn_,
                           (void*)&o0, (void*)&o1, (void*)&nn};
          CK(cudaLaunchKernel(P.k_cand, dim3(4 * P.sm_count), dim3(256), cargs, 0, st));
          ++launches;
        }
        ConvArgs<T> a = sa_args;
        a.in0 = X[ic]; a.in1 = X[ix]; a.out1 = Yn; a.sflag = par ? 0 : 2;
        StepTail tl = P.tail;
        tl.setR = par;
        a.tflag = P.d_tflag;
        if (P.d_tflag && P.ovl_b) last_aseq = tl.aseq = ++P.a_seq ? P.a_seq : ++P.a_seq;
        a.hscal = d_hscal;
        a.hflag = d_hflag;
        a.hseq = ++P.step_seq;
        if (int e = step_launch(P, P.k_sca, a, st, false, P.step_smem, 2 * nT + tl.nR, &P.wfwd, &tl)) return e;
        ++launches;
        ++vals;
        if (int e = wait_flag(a.hseq)) return e;
        fitc = P.h_scal[4]; tvc = P.h_scal[5]; dot = P.h_scal[3];
      } else {
        ConvArgs<T> a = sa_args;
        a.in0 = X[ix]; a.in1 = X[ixp]; a.out0 = X[ic]; a.sbeta = beta; a.sL = L_try; a.sflag = 1;
        if (int e = step_launch(P, P.k_sc, a, st, false, P.step_smem, nT, &P.wfwd)) return e;
        ++launches;
        ++vals;
        if (int e = reduce(2, 3)) return e;
        fitc = P.h_scal[0]; tvc = P.h_scal[1]; dot = P.h_scal[2];
      }
    }
    if (status != ST_OK) { done = true; break; }
    const double bstep = 1.0 / L_try;
    lip_t = fmax(1.0 / bstep * 0.9, lip * 1e-8);
    ixp = ix;
    ix = ic;
    const bool restart = dot > 0.0;
    if (restart) {
      t_mom = 1.0;
      ixp = ix;
      ++restarts;
    }
    for (int b = 0; b < 3; ++b)
      if (b != ix && b != ixp) { ic = b; break; }
    a_ready = (k == 0 || P.tail.on) && !restart;   // an accepted retry carried its own speculative stage A
    if (a_ready) par ^= 1;
  }
  if (!done) {
    // max_iters reached: g = lower_grad(p, x) (lower_solvers.py:212-213)
    ConvArgs<T> a = base;
    a.mode = CM_GRAD;
    a.in0 = X[ix];
    a.out0 = (T*)P.ws[5];
    if (int e = launch_coop(P, P.k_misc, a, st)) return e;
    ++launches;
    if (int e = fetch_scal(P, 2, st)) return e;
    gn = P.h_scal[1];
    CK(cudaMemcpyAsync(x_out, X[ix], nbytes, cudaMemcpyDeviceToDevice, st));
    iters = sa->max_iters;
    converged = gn <= tol;
  }
  CK(cudaStreamSynchronize(st));
  if (prof_pending) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, P.prof_ev[0], P.prof_ev[1]));
    dom_ms += ms;
    ++dom_n;
  }
  res->norm_sq = lam;
  res->lip = lip;
  res->grad_norm = gn;
  res->value = h_y;
  res->iters = iters;
  res->converged = converged;
  res->status = status;
  res->fail_iter = fail_iter;
  res->power_iters = pit;
  res->power_converged = pconv;
  res->vg_evals = vg;
  res->value_evals = vals;
  res->restarts = restarts;
  res->t_mom = t_mom;
  res->lip_t = lip_t;
  res->launches = launches;
  res->dominant_ms = dom_ms;
  res->dominant_launches = dom_n;
  return ADP_OK;
}

int adp_lower_solve(adp_plan* p, const adp_lower* lp, const void* x0, void* x_out, const adp_solve_args* sa,
                    adp_solve_result* res, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  if (!sa || !res) return fail(ADP_ERR_ARG, "null argument");
  if (!(sa->eps > 0)) return fail(ADP_ERR_ARG, "eps must be > 0");
  if (!(sa->mu > 0)) return fail(ADP_ERR_ARG, "mu must be > 0");
  if (sa->method < 0 || sa->method > 2) return fail(ADP_ERR_ARG, "unknown lower solver method");
  PlanImpl& P = p->impl;
  const bool injected = sa->x_prev0 || sa->t_mom0 > 0 || sa->lip_t0 > 0;
  if (IS_DENSE(p)) {
    if (injected) return fail(ADP_ERR_UNSUPPORTED, "injected AGD state: depthwise 2-D plans only");
    *res = adp_solve_result{};
    const int e = dense_solve(P, lp, x0, x_out, sa, res, STREAM(stream));
    res->launches = 1;
    return e;
  }
  *res = adp_solve_result{};
  if (P.step && sa->method == M_AGD && sa->adaptive && lp->alpha != 0.0 && !P.d_trace)
    return conv_solve_step(P, lp, x0, x_out, sa, res, STREAM(stream));
  auto run = [&](auto tag) -> int {
    using T = decltype(tag);
    ConvArgs<T> a = conv_base<T>(P);
    set_lower(a, lp);
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
    a.xprev0 = (const T*)sa->x_prev0;
    a.t_mom0 = sa->t_mom0;
    a.lip_t0 = sa->lip_t0;
    a.out = (T*)x_out;
    a.trace = P.d_trace;
    if (int e = launch_coop(P, P.k_solve, a, STREAM(stream))) return e;
    CK(cudaMemcpyAsync(P.h_sres, P.d_sres, sizeof(SolveOut), cudaMemcpyDeviceToHost, STREAM(stream)));
    CK(cudaStreamSynchronize(STREAM(stream)));
    const SolveOut& o = *P.h_sres;
    res->norm_sq = o.lam;
    res->lip = o.lip;
    res->grad_norm = o.grad_norm;
    res->value = o.value;
    res->iters = o.iters;
    res->converged = o.converged;
    res->status = o.status;
    res->fail_iter = o.fail_iter;
    res->power_iters = o.power_iters;
    res->power_converged = o.power_converged;
    res->vg_evals = o.vg_evals;
    res->value_evals = o.value_evals;
    res->restarts = o.restarts;
    res->t_mom = o.t_mom;
    res->lip_t = o.lip_t;
    res->launches = 1;
    res->dominant_ms = 0.0;
    res->dominant_launches = 0;
    return ADP_OK;
  };
  return P.d.dtype == ADP_DTYPE_F32 ? run(float()) : run(double());
}

int adp_lower_iter(adp_plan* p, const adp_lower* lp, const void* x, const void* x_prev, double t_mom, double lip_t,
                   const adp_solve_args* args, void* x_out, adp_solve_result* res, void* stream) {
  if (!args || !x_prev) return fail(ADP_ERR_ARG, "null argument");
  adp_solve_args a = *args;
  a.max_iters = 1;
  a.x_prev0 = x_prev;
  a.t_mom0 = t_mom;
  a.lip_t0 = lip_t;
  return adp_lower_solve(p, lp, x, x_out, &a, res, stream);
}

static int hess_cg_impl(adp_plan* p, const adp_lower* lp, const void* x_tilde, const void* rhs, void* q, int32_t warm,
                        const void* precond, double tol, int32_t max_iters, adp_cg_result* res, void* r_io,
                        const void* p_dir, double rs0, void* stream);

int adp_hess_cg(adp_plan* p, const adp_lower* lp, const void* x_tilde, const void* rhs, void* q, int32_t warm,
                const void* precond, double tol, int32_t max_iters, adp_cg_result* res, void* stream) {
  return hess_cg_impl(p, lp, x_tilde, rhs, q, warm, precond, tol, max_iters, res, nullptr, nullptr, 0.0, stream);
}

int adp_cg_iter(adp_plan* p, const adp_lower* lp, const void* x_tilde, void* q, void* r, const void* p_dir, double rs,
                adp_cg_result* res, void* stream) {
  if (!q || !r || !p_dir) return fail(ADP_ERR_ARG, "null argument");
  if (IS_DENSE(p)) return fail(ADP_ERR_UNSUPPORTED, "cg lockstep: depthwise 2-D plans only");
  // tol tiny: the step is taken; rhs is only used by the true-residual pass (r stands in for it)
  return hess_cg_impl(p, lp, x_tilde, r, q, 1, nullptr, 1e-300, 1, res, r, p_dir, rs, stream);
}

static int hess_cg_impl(adp_plan* p, const adp_lower* lp, const void* x_tilde, const void* rhs, void* q, int32_t warm,
                        const void* precond, double tol, int32_t max_iters, adp_cg_result* res, void* r_io,
                        const void* p_dir, double rs0, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  if (!res) return fail(ADP_ERR_ARG, "null argument");
  if (!(tol > 0)) return fail(ADP_ERR_ARG, "tol must be > 0");
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) return dense_cg(P, lp, x_tilde, rhs, q, warm, precond, tol, max_iters, res, STREAM(stream));
  auto run = [&](auto tag) -> int {
    using T = decltype(tag);
    ConvArgs<T> a = conv_base<T>(P);
    set_lower(a, lp);
    a.xt = (const T*)x_tilde;
    a.rhs = (const T*)rhs;
    a.Q = (T*)q;
    a.warm = warm;
    a.diag_in = (const T*)precond;
    a.tol = tol;
    a.max_iters = max_iters;
    a.cg_r = (T*)r_io;
    a.cg_p0 = (const T*)p_dir;
    a.cg_rs0 = rs0;
    if (int e = launch_coop(P, P.k_cg, a, STREAM(stream))) return e;
    CK(cudaMemcpyAsync(P.h_cres, P.d_cres, sizeof(CGOut), cudaMemcpyDeviceToHost, STREAM(stream)));
    CK(cudaStreamSynchronize(STREAM(stream)));
    const CGOut& o = *P.h_cres;
    res->residual = o.residual;
    res->curv = o.curv;
    res->iters = o.iters;
    res->converged = o.converged;
    res->status = o.status;
    res->hv = o.hv;
    res->rs = o.rs;
    return ADP_OK;
  };
  return P.d.dtype == ADP_DTYPE_F32 ? run(float()) : run(double());
}

int adp_mixed_T(adp_plan* p, const adp_lower* lp, const void* x_tilde, const void* q, void* out, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) return dense_call(P, DO_MIXED, lp->kernel, lp, x_tilde, q, out, nullptr, nullptr, nullptr, STREAM(stream));
  void* resid = P.ws[3];  // R
  void* bq = P.ws[12];    // BP
  if (int e = DISPATCH_T(P, conv_misc)(P, CM_MIXED_PREP, lp, nullptr, x_tilde, q, resid, bq, nullptr, STREAM(stream)))
    return e;
  return DISPATCH_T(P, conv_kgc)(P, x_tilde, bq, q, resid, out, 2.0, STREAM(stream), nullptr);
}

int adp_upper_terms(adp_plan* p, const void* A_kernel, const void* x, const void* y_delta, double* fit,
                    double* grad_norm, void* grad_out, void* stream) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) {
    double sc[2];
    if (int e = dense_call(P, DO_UPPER, A_kernel, nullptr, x, nullptr, grad_out, nullptr, y_delta, sc, STREAM(stream))) return e;
    *fit = sc[0];
    *grad_norm = sc[1];
    return ADP_OK;
  }
  if (int e = DISPATCH_T(P, conv_misc)(P, CM_UPPER, nullptr, A_kernel, x, nullptr, grad_out, nullptr, y_delta,
                                       STREAM(stream)))
    return e;
  if (int e = fetch_scal(P, 2, STREAM(stream))) return e;
  *fit = P.h_scal[0];
  *grad_norm = P.h_scal[1];
  return ADP_OK;
}

// Regularizer alone (SmoothedTV / SmoothedElasticNet methods): the lower
// machinery with the operator term removed (zero stencil / reg_only) and
// alpha = 1, which reproduces J's own value / gradient / Hessian exactly.
int adp_reg_op(adp_plan* p, const adp_lower* reg, int32_t op, const void* x, const void* v, void* out,
               double* value, void* stream) {
  if (!p || !reg) return fail(ADP_ERR_ARG, "null argument");
  PlanImpl& P = p->impl;
  adp_lower lp = *reg;
  lp.alpha = 1.0;
  if (IS_DENSE(p)) {
    if (lp.reg != ADP_REG_ELASTIC) return fail(ADP_ERR_UNSUPPORTED, "dense1d path supports SmoothedElasticNet");
    const int ops[5] = {DO_VALUE, DO_VG, DO_GRAD, DO_HV, DO_HDIAG};
    if (op < 0 || op > 4) return fail(ADP_ERR_ARG, "bad reg op");
    double sc[2] = {0, 0};
    if (int e = dense_call(P, 100 + ops[op], nullptr, &lp, x, v, out, nullptr, nullptr, sc, STREAM(stream))) return e;
    if (value) *value = sc[0];
    return ADP_OK;
  }
  if (lp.reg != ADP_REG_TV) return fail(ADP_ERR_UNSUPPORTED, "depthwise2d path supports SmoothedTV");
  if (!(lp.nu > 0.0) && op != 0) return fail(ADP_ERR_ARG, "gradient requested on the nonsmooth branch (nu = 0)");
  if (!P.d_zero) {
    CK(cudaMalloc(&P.d_zero, (size_t)(P.g.N + (int64_t)P.g.kh * P.g.kw * P.g.C) * P.esize));
    CK(cudaMemset(P.d_zero, 0, (size_t)(P.g.N + (int64_t)P.g.kh * P.g.kw * P.g.C) * P.esize));
  }
  lp.kernel = P.d_zero;
  lp.y = P.d_zero;
  auto run = [&](auto tag) -> int {
    using T = decltype(tag);
    ConvArgs<T> a = conv_base<T>(P);
    set_lower(a, &lp);
    const int modes[5] = {CM_VALUE, CM_VALUE_GRAD, CM_GRAD, CM_HESS_VEC, CM_HESS_DIAG};
    if (op < 0 || op > 4) return fail(ADP_ERR_ARG, "bad reg op");
    a.mode = modes[op];
    a.nofloor = 1;
    a.in0 = (const T*)x;
    a.in1 = (const T*)v;
    a.out0 = (T*)out;
    if (int e = launch_coop(P, P.k_misc, a, STREAM(stream))) return e;
    if (op <= 1) {
      if (int e = fetch_scal(P, 1, STREAM(stream))) return e;
      if (value) *value = P.h_scal[0];
    }
    return ADP_OK;
  };
  return P.d.dtype == ADP_DTYPE_F32 ? run(float()) : run(double());
}

int adp_dot(adp_plan* p, const void* a, const void* b, double* out, void* stream) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  PlanImpl& P = p->impl;
  if (IS_DENSE(p)) return dense_call(P, DO_DOT, nullptr, nullptr, a, b, nullptr, nullptr, nullptr, out, STREAM(stream));
  if (int e = DISPATCH_T(P, conv_misc)(P, CM_DOT, nullptr, nullptr, a, b, nullptr, nullptr, nullptr, STREAM(stream)))
    return e;
  if (int e = fetch_scal(P, 1, STREAM(stream))) return e;
  *out = P.h_scal[0];
  return ADP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Host-only introspection of the deterministic-sum layout (no device needed):
// lets CPU tests evaluate the exact tree the kernels evaluate.
extern "C" int adp_sum_layout(int64_t n, int32_t np_rule, int64_t* n_leaves, int32_t* n_sub, int32_t* top_prog,
                              int64_t* leaf_start, int64_t leaf_cap, int32_t* sub_leaf, int32_t* sub_prog,
                              int64_t sub_cap, int32_t* words, int64_t words_cap, int64_t* n_words) {
  adp::ProgPool pool;
  adp::SumHost s;
  adp::build_sum(s, n, np_rule != 0, pool);
  *n_leaves = s.nLeaves;
  *n_sub = s.nSub;
  *top_prog = s.regular ? -1 : s.top_prog;   // -1: perfect tree (zero-padded), subtrees of 2048 leaves
  *n_words = (int64_t)pool.words.size();
  if ((int64_t)s.leaf_start.size() > leaf_cap || (int64_t)s.sub_leaf.size() > sub_cap + 1 ||
      (int64_t)pool.words.size() > words_cap)
    return fail(ADP_ERR_ARG, "buffer too small");
  for (size_t i = 0; i < s.leaf_start.size(); ++i) leaf_start[i] = s.leaf_start[i];
  for (size_t i = 0; i < s.sub_leaf.size(); ++i) sub_leaf[i] = s.sub_leaf[i];
  for (size_t i = 0; i < s.sub_prog.size(); ++i) sub_prog[i] = s.sub_prog[i];
  for (size_t i = 0; i < pool.words.size(); ++i) words[i] = pool.words[i];
  return ADP_OK;
}

extern "C" int adp_prox_grad(adp_plan* p, const adp_lower* lp, const void* x0, void* x_out, int32_t n_iters,
                             double step, void* stream) {
  if (!p || !lp || !x0 || !x_out || !lp->kernel || !lp->y) return fail(ADP_ERR_ARG, "null argument");
  if (n_iters < 0) return fail(ADP_ERR_ARG, "n_iters must be >= 0");
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DENSE1D)
    return fail(ADP_ERR_UNSUPPORTED, "fused prox-gradient: dense1d plans (compose apply/adjoint/adp_vec otherwise)");
  return dense_prox(P, lp, x0, x_out, n_iters, step, (cudaStream_t)stream);
}

// micro-benchmark of the solve's decision-point reduction (tools/bench_reduce.py)
extern "C" int adp_debug_bench_reduce(adp_plan* p, int32_t reps, double* ms, void* stream) {
  if (!p || !ms || reps < 1) return fail(ADP_ERR_ARG, "bad argument");
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D || P.d.dtype != ADP_DTYPE_F64) return fail(ADP_ERR_UNSUPPORTED, "f64 conv");
  cudaStream_t st = (cudaStream_t)stream;
  ConvArgs<double> a = conv_base<double>(P);
  a.mode = CM_BENCH_REDUCE;
  a.max_iters = reps;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  if (int e = launch_coop(P, P.k_misc, a, st)) return e;
  cudaEventRecord(e1, st);
  CK(cudaEventSynchronize(e1));
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  *ms = t;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ADP_OK;
}

extern "C" int adp_plan_geometry(const adp_plan* p, int32_t* out) {
  if (!p || !out) return fail(ADP_ERR_ARG, "null argument");
  const PlanImpl& P = p->impl;
  const ConvGeom& g = P.g;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "geometry: depthwise2d plans only");
  const int32_t v[10] = {g.TH, g.TW, g.tilesH, g.tilesW, g.fused, g.leafL, g.rwb, P.k_solve.grid, g.threads,
                         (int32_t)P.smem};
  for (int i = 0; i < 10; ++i) out[i] = v[i];
  return ADP_OK;
}

extern "C" int adp_plan_probe(const adp_plan_desc* desc, int32_t* out) {
  if (!desc || !out) return fail(ADP_ERR_ARG, "null argument");
  if (desc->layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "probe: depthwise2d plans only");
  if (desc->H < 1 || desc->W < 1 || desc->C < 1 || desc->kh < 1 || desc->kw < 1 || desc->kh % 2 == 0 ||
      desc->kw % 2 == 0)
    return fail(ADP_ERR_ARG, "bad shape");
  adp_plan tmp;
  tmp.impl.d = *desc;
  tmp.impl.esize = desc->dtype == ADP_DTYPE_F32 ? 4 : 8;
  tmp.impl.probe_only = true;
  if (int e = conv_plan_init(tmp.impl)) return e;
  const ConvGeom& g = tmp.impl.g;
  const int32_t v[10] = {g.TH, g.TW, g.tilesH, g.tilesW, g.fused, g.leafL, g.rwb, 0, g.threads, (int32_t)tmp.impl.smem};
  for (int i = 0; i < 10; ++i) out[i] = v[i];
  return ADP_OK;
}

extern "C" int adp_slab_step(adp_plan* p, const adp_lower* lp, int32_t op, const void* x, const void* xp, void* out,
                  double beta, double L, void* stream) {
  if (!p || !x) return fail(ADP_ERR_ARG, "null argument");
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "slab steps: depthwise2d plans only");
  if (op < 0 || op > 4) return fail(ADP_ERR_ARG, "slab step: unknown op");
  const bool needs_lower = op != 3;
  if (needs_lower && (!lp || !lp->kernel)) return fail(ADP_ERR_ARG, "slab step: lower problem / kernel missing");
  if ((op == 0 || op == 1 || op == 4) && (!lp->y || lp->reg != ADP_REG_TV))
    return fail(ADP_ERR_UNSUPPORTED, "slab steps: TV lower problems with data y");
  if ((op == 0 || op == 1) && !xp) return fail(ADP_ERR_ARG, "slab step: x_prev missing");
  if ((op <= 2) && !out) return fail(ADP_ERR_ARG, "slab step: output missing");
  if (op == 2 && !(L != 0.0)) return fail(ADP_ERR_ARG, "slab power step: zero scale");
  return DISPATCH_T(P, conv_slab_step)(P, needs_lower ? lp : nullptr, op, x, xp, out, beta, L,
                                      (cudaStream_t)stream);
}

extern "C" int adp_slab_units(adp_plan* p, int32_t which, int64_t* n_units, int64_t* own, double* dst,
                              void* stream) {
  if (!p || !n_units || !own) return fail(ADP_ERR_ARG, "null argument");
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "slab units: depthwise2d plans only");
  if (which < 0 || which > 6) return fail(ADP_ERR_ARG, "slab units: unknown sum");
  const SumDev* sds[7] = {&P.s_fit, &P.s_tv, &P.s_fitc, &P.s_tvc, &P.s_t0, &P.s_t1, &P.s_t2};
  const SumDev& sd = *sds[which];
  if (!sd.regular) return fail(ADP_ERR_UNSUPPORTED, "slab units: irregular (program) sum");
  *n_units = P.units_n[which];
  for (int j = 0; j < 4; ++j) own[j] = P.units_own[which][j];
  if (dst) {
    const double* src = sd.nSub > 1 ? sd.sub_vals : sd.leaf_vals;
    for (int j = 0; j < 4; j += 2) {
      const int64_t a = own[j], b = own[j + 1];
      if (b > a)
        CK(cudaMemcpyAsync(dst + a, src + a, (size_t)(b - a) * sizeof(double), cudaMemcpyDeviceToDevice,
                           (cudaStream_t)stream));
    }
  }
  return ADP_OK;
}

// ---- row-slab hypergradient (multigpu.SlabHypergradient) -----------------
// One step of the hypergradient's Jacobi-PCG (hypergradient.py:35-84 on
// lower_hess_vec / lower_hess_diag, lower_solvers.py:66-80) over a slab +
// ghosts, stopping after phase 1 of its sums (adp_slab_units + adp_fold_units
// assemble them across ranks).  op 0: TV weights + unfloored diagonal of
// H(x~ = in0), *scal = max over the owned pixels; op 1: floor s, invert,
// r = in0 (- H q if flag), q = out0 (zeroed unless flag), s = out1, sums
// <r, s>, <r, r>; op 2: flag 0/1: p = in0 (+ s * in1) -> out0, H p, <p, Hp>;
// flag 2: ||H in0 - in1||^2 (true residual), Vbuf out0; flag 3: H in0 (warm
// start), Vbuf out0; op 3: q (out0) += s p (in0), r -= s H p, s (out1) = M^-1 r,
// sums <r, s>, <r, r>.
extern "C" int adp_slab_cg(adp_plan* p, const adp_lower* lp, int32_t op, const void* in0, const void* in1,
                           void* out0, void* out1, double s, int32_t flag, double* scal, void* stream) {
  if (int e = check_lower(p, lp)) return e;
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "slab CG: depthwise2d plans only");
  if (op < 0 || op > 3) return fail(ADP_ERR_ARG, "slab CG: unknown op");
  if (!in0 || (op != 0 && !out0) || ((op == 1 || op == 3) && !out1)) return fail(ADP_ERR_ARG, "slab CG: null argument");
  if (op == 2 && (flag < 0 || flag > 3 || (flag != 0 && flag != 3 && !in1))) return fail(ADP_ERR_ARG, "slab CG: bad flag");
  if (int e = DISPATCH_T(P, conv_slab_cg)(P, lp, op, in0, in1, out0, out1, s, flag, STREAM(stream))) return e;
  if (op == 0) {
    if (int e = fetch_scal(P, 1, STREAM(stream))) return e;
    if (scal) *scal = P.h_scal[0];
  }
  return ADP_OK;
}

// UpperProblem.fit_value / upper_fit_grad (problems.py:48-50,
// hypergradient.py:87-89) over a slab: R = A x - y, grad_out = 2 A^T R (owned
// rows valid), phase 1 of sum(R^2) (units 0) and ||grad||^2 (units 4).
extern "C" int adp_slab_upper(adp_plan* p, const void* A_kernel, const void* x, const void* y_delta, void* grad_out,
                              void* stream) {
  if (!p || !A_kernel || !x || !y_delta) return fail(ADP_ERR_ARG, "null argument");
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "slab upper: depthwise2d plans only");
  if (!P.g.fused) return fail(ADP_ERR_UNSUPPORTED, "slab upper: needs the row-aligned (fused) sum layout");
  return DISPATCH_T(P, conv_misc)(P, CM_SLAB_UPPER, nullptr, A_kernel, x, nullptr, grad_out, nullptr, y_delta,
                                  STREAM(stream));
}

// mixed_second_transpose (hypergradient.py:92-104) over a slab: R = B x~ - y,
// BP = B q, then the kernel_gram_correlation partials of the slab's owned
// groups into part (adp_kgc_groups doubles x groups, zero elsewhere; the
// ranks sum the vectors and adp_kgc_final folds them in group order).
extern "C" int adp_slab_mixed(adp_plan* p, const adp_lower* lp, const void* x_tilde, const void* q, double* part,
                              void* stream) {
  if (int e = check_lower(p, lp)) return e;
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "slab mixed: depthwise2d plans only");
  if (!x_tilde || !q || !part) return fail(ADP_ERR_ARG, "null argument");
  if ((P.g.row0 + P.g.own0) % 16 || ((P.g.row0 + P.g.own1) % 16 && P.g.row0 + P.g.own1 != P.g.Hg))
    return fail(ADP_ERR_ARG, "slab mixed: owned rows must be 16-row aligned");
  void* resid = P.ws[3];  // R
  void* bq = P.ws[12];    // BP
  if (int e = DISPATCH_T(P, conv_misc)(P, CM_SLAB_MIXED_PREP, lp, nullptr, x_tilde, q, nullptr, nullptr, nullptr,
                                       STREAM(stream)))
    return e;
  return DISPATCH_T(P, conv_kgc)(P, x_tilde, bq, q, resid, nullptr, 2.0, STREAM(stream), part);
}

// plan execution flags: bit 0 = TMA tile boxes (c2 kernel), bit 1 = host-stepped
// high-occupancy solve (conv2d_step.cu)
extern "C" int adp_plan_flags(adp_plan* p, int32_t* flags) {
  if (!p || !flags) return fail(ADP_ERR_ARG, "null argument");
  *flags = (p->impl.tma ? 1 : 0) | (p->impl.step ? 2 : 0) | (p->impl.step && p->impl.tail.on ? 4 : 0) |
           (p->impl.step && p->impl.d_tflag ? 8 : 0) | (p->impl.step && p->impl.d_tflag && p->impl.ovl_b ? 16 : 0);
  return ADP_OK;
}

extern "C" int adp_plan_profile(adp_plan* p, int32_t enable) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  p->impl.profile = enable > 0 ? enable : 0;   // sampling period in iterations (1: every launch)
  return ADP_OK;
}

extern "C" int adp_kgc_groups(adp_plan* p, int32_t* ngroups, int32_t* ntaps) {
  if (!p || !ngroups || !ntaps) return fail(ADP_ERR_ARG, "null argument");
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "kgc groups: depthwise2d plans only");
  *ngroups = P.kgc_groups;
  *ntaps = P.g.kh * P.g.kw * P.g.C;
  return ADP_OK;
}

extern "C" int adp_kgc_final(adp_plan* p, const double* part, void* out, double scale, void* stream) {
  if (!p || !part || !out) return fail(ADP_ERR_ARG, "null argument");
  PlanImpl& P = p->impl;
  if (P.d.layout != ADP_LAYOUT_DEPTHWISE2D) return fail(ADP_ERR_UNSUPPORTED, "kgc final: depthwise2d plans only");
  return DISPATCH_T(P, conv_kgc_final)(P, part, out, scale, STREAM(stream));
}

// Debug: enable (enable = 1) per-phase %globaltimer stamps of the next solves
// (first 64 iterations, 16 slots each); enable = 0 copies them to host_out
// (64 * 16 + 256 uint64: phases, reduce and per-warp stage-B sub-phase cycles) and disables.
extern "C" int adp_debug_trace(adp_plan* p, int32_t enable, uint64_t* host_out) {
  if (!p) return fail(ADP_ERR_ARG, "null plan");
  PlanImpl& P = p->impl;
  const size_t bytes = (64 * 16 + 256) * sizeof(unsigned long long);   // + sub-phase stamps
  if (enable) {
    if (!P.d_trace) CK(cudaMalloc(&P.d_trace, bytes));
    CK(cudaMemset(P.d_trace, 0, bytes));
    return ADP_OK;
  }
  if (P.d_trace) {
    CK(cudaDeviceSynchronize());
    if (host_out) CK(cudaMemcpy(host_out, P.d_trace, bytes, cudaMemcpyDeviceToHost));
    cudaFree(P.d_trace);
    P.d_trace = nullptr;
  }
  return ADP_OK;
}
