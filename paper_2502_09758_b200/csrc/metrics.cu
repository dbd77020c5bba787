// Quality metrics of the reference's metrics_io.py (PSNR, SSIM, relative L2)
// on the device, with the reference's rounding:
//
//   * np.sum / np.mean over a contiguous array = NumPy pairwise summation
//     (leaves of <= 128 with 8 accumulator chains, split at n/2 rounded down
//     to a multiple of 8).  The recursion tree is laid out on the host once
//     per length (leaf starts + internal nodes grouped by height) and
//     evaluated on the device: one 8-lane group per leaf, then one small
//     launch per tree level.  k equal-length segments are summed together.
//   * ssim's five ndimage.correlate passes (11x11 window, mode="constant")
//     restricted to the interior windows the reference keeps
//     (out[half:-half, half:-half]), taps in row-major order as
//     acc = acc + v * w, the products x*x, y*y, x*y rounded first as the
//     reference's temporaries are; then num / den per pixel in the
//     reference's expression order (metrics_io.py:66-75).
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <vector>
#include "adp_device.cuh"
#include "../../include/adp_b200.h"

namespace adp {
int dense_fail(int code, const char* m);

// ---------------------------------------------------------------------------
// Host layout of NumPy's pairwise recursion for n elements.
struct PwLayout {
  int64_t n = 0;
  int nLeaves = 0, nNodes = 0;           // values: [0, nLeaves) leaves, then internal nodes
  int root = 0;
  std::vector<int> level_off;            // internal nodes of height h: [level_off[h-1], level_off[h])
  int64_t* d_starts = nullptr;           // nLeaves + 1
  int* d_nodes = nullptr;                // 3 ints per internal node: out, left, right (by height)
  ~PwLayout() {
    if (d_starts) cudaFree(d_starts);
    if (d_nodes) cudaFree(d_nodes);
  }
};

namespace {
struct PwBuild {
  std::vector<int64_t> starts;
  struct Node { int l, r, h; };
  std::vector<Node> nodes;        // internal, in creation order (ids nLeaves + index)
  std::vector<int> height;        // per value id (leaves 0), filled at the end
  // returns a value id: leaves >= 0 as leaf index, internal as -(1 + node index)
  int rec(int64_t s, int64_t n, int& h_out) {
    if (n <= 128) {
      starts.push_back(s);
      h_out = 0;
      return (int)starts.size() - 1;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    int hl = 0, hr = 0;
    const int a = rec(s, n2, hl);
    const int b = rec(s + n2, n - n2, hr);
    nodes.push_back({a, b, std::max(hl, hr) + 1});
    h_out = std::max(hl, hr) + 1;
    return -(int)nodes.size();
  }
};
}  // namespace

static std::mutex g_pw_mu;
static std::map<int64_t, std::unique_ptr<PwLayout>> g_pw;

static PwLayout* pw_layout(int64_t n) {
  std::lock_guard<std::mutex> lk(g_pw_mu);
  auto it = g_pw.find(n);
  if (it != g_pw.end()) return it->second.get();
  PwBuild b;
  int hroot = 0;
  const int root = b.rec(0, n, hroot);
  auto L = std::make_unique<PwLayout>();
  L->n = n;
  L->nLeaves = (int)b.starts.size();
  L->nNodes = (int)b.nodes.size();
  b.starts.push_back(n);
  auto vid = [&](int id) { return id >= 0 ? id : L->nLeaves + (-id - 1); };
  L->root = vid(root);
  // group internal nodes by height (children always have smaller heights)
  std::vector<int> host;
  L->level_off.assign(1, 0);
  for (int h = 1; h <= hroot; ++h) {
    for (int i = 0; i < L->nNodes; ++i)
      if (b.nodes[i].h == h) {
        host.push_back(L->nLeaves + i);
        host.push_back(vid(b.nodes[i].l));
        host.push_back(vid(b.nodes[i].r));
      }
    L->level_off.push_back((int)host.size() / 3);
  }
  if (cudaMalloc(&L->d_starts, b.starts.size() * sizeof(int64_t)) != cudaSuccess) return nullptr;
  cudaMemcpy(L->d_starts, b.starts.data(), b.starts.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (!host.empty()) {
    if (cudaMalloc(&L->d_nodes, host.size() * sizeof(int)) != cudaSuccess) return nullptr;
    cudaMemcpy(L->d_nodes, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice);
  }
  PwLayout* r = L.get();
  g_pw[n] = std::move(L);
  return r;
}

// Element sources: segment `seg` of k, element i of n.
struct SrcPlain {
  const double* x;
  int64_t n;
  __device__ double operator()(int seg, int64_t i) const { return x[seg * n + i]; }
};
struct SrcSqDiff {   // (x - ref) ** 2  (metrics_io.py:34)
  const double* x;
  const double* y;
  int64_t n;
  __device__ double operator()(int seg, int64_t i) const {
    const double d = x[seg * n + i] - y[seg * n + i];
    return d * d;
  }
};

// One 8-lane group per leaf (k * nLeaves groups).  Lane j of the group runs
// accumulator chain r[j]; xor-shuffles give ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// in lane 0, which then adds the tail sequentially (pairwise_sum's block branch).
template <class Src>
__global__ void __launch_bounds__(256) pw_leaves_kernel(Src src, const int64_t* __restrict__ starts, int nLeaves,
                                                        int k, int stride, double* __restrict__ vals) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int j = threadIdx.x & 7;
  const bool act = g < (int64_t)k * nLeaves;
  const int seg = act ? (int)(g / nLeaves) : 0;
  const int leaf = act ? (int)(g - (int64_t)seg * nLeaves) : 0;
  const int64_t s = act ? starts[leaf] : 0;
  const int n = act ? (int)(starts[leaf + 1] - s) : 0;
  double acc = 0.0;
  if (n >= 8 && j < 8) {
    const int nfull = n - (n % 8);
    acc = src(seg, s + j);
    for (int i = 8; i < nfull; i += 8) acc = acc + src(seg, s + i + j);
  }
  acc = acc + __shfl_xor_sync(kFull, acc, 1);
  acc = acc + __shfl_xor_sync(kFull, acc, 2);
  acc = acc + __shfl_xor_sync(kFull, acc, 4);
  if (act && j == 0) {
    double res;
    if (n < 8) {
      res = 0.0;
      for (int i = 0; i < n; ++i) res = res + src(seg, s + i);
    } else {
      res = acc;
      for (int i = n - (n % 8); i < n; ++i) res = res + src(seg, s + i);
    }
    vals[(int64_t)seg * stride + leaf] = res;
  }
}

__global__ void pw_level_kernel(const int* __restrict__ nodes, int cnt, int k, int stride, double* vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)k * cnt) return;
  const int seg = (int)(t / cnt), i = (int)(t - (int64_t)seg * cnt);
  double* v = vals + (int64_t)seg * stride;
  v[nodes[3 * i]] = v[nodes[3 * i + 1]] + v[nodes[3 * i + 2]];
}

template <class Src>
static int pw_sum(const Src& src, int k, int64_t n, double* out, cudaStream_t st) {
  if (n == 0) {
    for (int i = 0; i < k; ++i) out[i] = 0.0;
    return ADP_OK;
  }
  PwLayout* L = pw_layout(n);
  if (!L) return dense_fail(ADP_ERR_CUDA, "pairwise layout allocation failed");
  const int stride = L->nLeaves + L->nNodes;
  double* vals = nullptr;
  if (cudaMallocAsync((void**)&vals, (size_t)k * stride * sizeof(double), st) != cudaSuccess)
    return dense_fail(ADP_ERR_CUDA, "pairwise scratch allocation failed");
  const int64_t threads = (int64_t)k * L->nLeaves * 8;
  pw_leaves_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(src, L->d_starts, L->nLeaves, k, stride, vals);
  for (size_t h = 1; h < L->level_off.size(); ++h) {
    const int cnt = L->level_off[h] - L->level_off[h - 1];
    const int64_t t = (int64_t)k * cnt;
    pw_level_kernel<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(L->d_nodes + 3 * L->level_off[h - 1], cnt, k,
                                                                 stride, vals);
  }
  cudaMemcpy2DAsync(out, sizeof(double), vals + L->root, (size_t)stride * sizeof(double), sizeof(double), k,
                    cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(vals, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return dense_fail(ADP_ERR_CUDA, cudaGetErrorString(e));
  return ADP_OK;
}

// ---------------------------------------------------------------------------
// SSIM map: one CTA per (TH x TW) block of interior outputs of one channel.
constexpr int kSsimK = 11, kSsimR = 5, kSsimTH = 16, kSsimTW = 32;
constexpr int kSsimSH = kSsimTH + 2 * kSsimR, kSsimSW = kSsimTW + 2 * kSsimR;

struct SsimArgs {
  const double* x;
  const double* y;
  double* map;          // (C, Ho, Wo)
  int H, W, C, Ho, Wo;
  double c1, c2;
  double w[kSsimK * kSsimK];
};

__global__ void __launch_bounds__(256) ssim_map_kernel(const __grid_constant__ SsimArgs a) {
  __shared__ double sx[kSsimSH][kSsimSW], sy[kSsimSH][kSsimSW], sxx[kSsimSH][kSsimSW], syy[kSsimSH][kSsimSW],
      sxy[kSsimSH][kSsimSW];
  const int c = blockIdx.z;
  const int oh0 = blockIdx.y * kSsimTH, ow0 = blockIdx.x * kSsimTW;   // interior output origin
  // input rows/cols [oh0, oh0 + SH) x [ow0, ow0 + SW) (interior output (i, j) = image (i + R, j + R))
  for (int t = threadIdx.x; t < kSsimSH * kSsimSW; t += blockDim.x) {
    const int r = t / kSsimSW, q = t - r * kSsimSW;
    const int h = oh0 + r, w = ow0 + q;
    double xv = 0.0, yv = 0.0;
    if (h < a.H && w < a.W) {
      const int64_t o = ((int64_t)h * a.W + w) * a.C + c;
      xv = a.x[o];
      yv = a.y[o];
    }
    sx[r][q] = xv;
    sy[r][q] = yv;
    sxx[r][q] = xv * xv;
    syy[r][q] = yv * yv;
    sxy[r][q] = xv * yv;
  }
  __syncthreads();
  const int q = threadIdx.x & 31, r0 = threadIdx.x >> 5;   // 8 row groups x 32 columns, 2 rows each
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = r0 + 8 * rr;
    const int oh = oh0 + r, ow = ow0 + q;
    double mx = 0.0, my = 0.0, fxx = 0.0, fyy = 0.0, fxy = 0.0;
#pragma unroll
    for (int i = 0; i < kSsimK; ++i)
#pragma unroll
      for (int j = 0; j < kSsimK; ++j) {
        const double wt = a.w[i * kSsimK + j];
        if (!(fabs(wt) > kDblEps)) continue;   // ndimage skips |w| <= DBL_EPSILON
        mx = mx + sx[r + i][q + j] * wt;
        my = my + sy[r + i][q + j] * wt;
        fxx = fxx + sxx[r + i][q + j] * wt;
        fyy = fyy + syy[r + i][q + j] * wt;
        fxy = fxy + sxy[r + i][q + j] * wt;
      }
    if (oh < a.Ho && ow < a.Wo) {
      const double vxx = fxx - mx * mx;
      const double vyy = fyy - my * my;
      const double vxy = fxy - mx * my;
      const double num = (2.0 * mx * my + a.c1) * (2.0 * vxy + a.c2);
      const double den = (mx * mx + my * my + a.c1) * (vxx + vyy + a.c2);
      a.map[((int64_t)c * a.Ho + oh) * a.Wo + ow] = num / den;
    }
  }
}

}  // namespace adp

using namespace adp;

extern "C" int adp_np_sum(int32_t op, int32_t k, int64_t n, const void* x, const void* y, double* out,
                          void* stream) {
  if (k < 1 || n < 0 || !out || (n > 0 && !x) || (op == 1 && n > 0 && !y))
    return dense_fail(ADP_ERR_ARG, "np_sum: bad arguments");
  if (n > ((int64_t)1 << 40)) return dense_fail(ADP_ERR_UNSUPPORTED, "np_sum: segment too long");
  cudaStream_t st = (cudaStream_t)stream;
  if (op == 0) return pw_sum(SrcPlain{(const double*)x, n}, k, n, out, st);
  if (op == 1) return pw_sum(SrcSqDiff{(const double*)x, (const double*)y, n}, k, n, out, st);
  return dense_fail(ADP_ERR_ARG, "np_sum: unknown op");
}

extern "C" int adp_ssim(int32_t H, int32_t W, int32_t C, const double* win, int32_t ksize, double c1, double c2,
                        const void* x, const void* ref, void* map_out, double* chan_sum, void* stream) {
  if (ksize != kSsimK) return dense_fail(ADP_ERR_UNSUPPORTED, "ssim: only the reference's 11x11 window");
  if (H < 0 || W < 0 || C < 1 || !win || !x || !ref || !chan_sum) return dense_fail(ADP_ERR_ARG, "ssim: bad arguments");
  const int Ho = H - 2 * kSsimR, Wo = W - 2 * kSsimR;
  if (Ho <= 0 || Wo <= 0) return dense_fail(ADP_ERR_ARG, "ssim: image smaller than the window");
  cudaStream_t st = (cudaStream_t)stream;
  SsimArgs a;
  a.x = (const double*)x;
  a.y = (const double*)ref;
  a.H = H;
  a.W = W;
  a.C = C;
  a.Ho = Ho;
  a.Wo = Wo;
  a.c1 = c1;
  a.c2 = c2;
  for (int i = 0; i < kSsimK * kSsimK; ++i) a.w[i] = win[i];
  const size_t mbytes = (size_t)C * Ho * Wo * sizeof(double);
  double* map = (double*)map_out;
  if (!map && cudaMallocAsync((void**)&map, mbytes, st) != cudaSuccess)
    return dense_fail(ADP_ERR_CUDA, "ssim: map allocation failed");
  a.map = map;
  dim3 grid((Wo + kSsimTW - 1) / kSsimTW, (Ho + kSsimTH - 1) / kSsimTH, C);
  ssim_map_kernel<<<grid, 256, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dense_fail(ADP_ERR_CUDA, cudaGetErrorString(e));
  const int rc = pw_sum(SrcPlain{map, (int64_t)Ho * Wo}, C, (int64_t)Ho * Wo, chan_sum, st);
  if (!map_out) cudaFreeAsync(map, st);
  return rc;
}
