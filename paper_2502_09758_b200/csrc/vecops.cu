// Plan-free vector primitives for the generic cg_solve(callable) API path
// (hypergradient.py:35-84 with an arbitrary hess_vec): elementwise updates in
// the reference's expression order and deterministic inner products
// (fixed 256-block grid, fixed tree).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include "adp_device.cuh"
#include "../../include/adp_b200.h"

namespace adp {
int dense_fail(int code, const char* m);

constexpr int kVecBlocks = 256;

template <typename T>
__global__ void vec_elementwise(int op, int64_t n, double a, const T* x, const T* y, T* out) {
  const T ta = T(a);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    switch (op) {
      case 0: out[i] = x[i] + ta * y[i]; break;   // q + a * p
      case 1: out[i] = x[i] - ta * y[i]; break;   // r - a * hp
      case 2: out[i] = x[i] * y[i]; break;        // inv_diag * r
      case 3: out[i] = T(1) / x[i]; break;        // 1.0 / precond_diag
      case 4: out[i] = x[i] - y[i]; break;        // rhs - H q
      case 5: out[i] = x[i]; break;               // copy
      case 6: {                                   // prox_l1(x, a) = sign(x) * max(|x| - a, 0) (np semantics)
        const T u = x[i], m = fabs(u) - ta;
        const T mx = (m > T(0) || m != m) ? m : T(0);
        const T sg = u > T(0) ? T(1) : (u < T(0) ? T(-1) : (u == T(0) ? T(0) : u));
        out[i] = sg * mx;
        break;
      }
      case 7: out[i] = fabs(y[i]) > ta ? x[i] : T(0); break;   // np.where(|u| > thr, w, 0.0)
      default: break;
    }
  }
}

template <typename T>
__global__ void vec_reduce_partial(int op, int64_t n, const T* x, const T* y, double* part) {
  __shared__ double red[64];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (op == 0) acc += (double)x[i] * (double)y[i];
    else acc += (x[i] <= T(0)) ? 1.0 : 0.0;
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void vec_reduce_final(const double* part, double* out) {
  __shared__ double red[64];
  double v = threadIdx.x < kVecBlocks ? part[threadIdx.x] : 0.0;
  const double t = block_sum(v, red);
  if (threadIdx.x == 0) *out = t;
}

}  // namespace adp

using namespace adp;

extern "C" int adp_vec(int32_t op, int64_t n, int32_t dtype, double a, const void* x, const void* y, void* out,
                       double* red_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  static thread_local double* d_part = nullptr;
  static thread_local double* h_out = nullptr;
  if (n < 0) return dense_fail(ADP_ERR_ARG, "negative length");
  if (op < 10) {
    if (n == 0) return ADP_OK;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 4096);
    if (dtype == ADP_DTYPE_F32)
      vec_elementwise<float><<<grid, 256, 0, st>>>(op, n, a, (const float*)x, (const float*)y, (float*)out);
    else
      vec_elementwise<double><<<grid, 256, 0, st>>>(op, n, a, (const double*)x, (const double*)y, (double*)out);
  } else {
    if (!d_part) {
      if (cudaMalloc(&d_part, (kVecBlocks + 1) * sizeof(double)) != cudaSuccess ||
          cudaMallocHost(&h_out, sizeof(double)) != cudaSuccess)
        return dense_fail(ADP_ERR_CUDA, "allocation failed");
    }
    const int rop = op - 10;  // 0: dot, 1: count(x <= 0)
    if (dtype == ADP_DTYPE_F32)
      vec_reduce_partial<float><<<kVecBlocks, 256, 0, st>>>(rop, n, (const float*)x, (const float*)y, d_part);
    else
      vec_reduce_partial<double><<<kVecBlocks, 256, 0, st>>>(rop, n, (const double*)x, (const double*)y, d_part);
    vec_reduce_final<<<1, 256, 0, st>>>(d_part, d_part + kVecBlocks);
    cudaMemcpyAsync(h_out, d_part + kVecBlocks, sizeof(double), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return dense_fail(ADP_ERR_CUDA, "vec reduce failed");
    *red_out = *h_out;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dense_fail(ADP_ERR_CUDA, cudaGetErrorString(e));
  return ADP_OK;
}

// ---------------------------------------------------------------------------
// FP64 roof microbenchmark: 8 independent DFMA chains per thread, 148 SMs x
// full occupancy; reports sustained DFMA TFLOP/s (2 flop per DFMA) for the
// roofline denominator (MEASURED_PEAKS.json carries no FP64 figure).
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
  double r0 = threadIdx.x * 1e-9, r1 = r0 + 1e-9, r2 = r0 + 2e-9, r3 = r0 + 3e-9;
  double r4 = r0 + 4e-9, r5 = r0 + 5e-9, r6 = r0 + 6e-9, r7 = r0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
      r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b);
    }
  }
  const double s = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  if (s == 1234.5) out[0] = s;  // keep the chains alive
}

extern "C" int adp_fp64_peak(double* tflops, double* ms, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dfma_peak_kernel, 256, 0);
  const int grid = sms * nb, iters = 4096;
  double* d_out = nullptr;
  if (cudaMalloc(&d_out, sizeof(double)) != cudaSuccess) return dense_fail(ADP_ERR_CUDA, "alloc");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_peak_kernel<<<grid, 256, 0, st>>>(d_out, 64, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, st);
    dfma_peak_kernel<<<grid, 256, 0, st>>>(d_out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    best = t < best ? t : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d_out);
  const double flops = 2.0 * 8.0 * 16.0 * (double)iters * 256.0 * (double)grid;
  *ms = best;
  *tflops = flops / (best * 1e-3) / 1e12;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dense_fail(ADP_ERR_CUDA, cudaGetErrorString(e));
  return ADP_OK;
}

// ---------------------------------------------------------------------------
// Perfect-tree folds of assembled sum units (row-slab reductions): one CTA
// per sum, the same zero-padded perfect tree the persistent kernels use.
namespace adp {
struct FoldArgs {
  const double* u[8];
  int n[8];
  double* out;
};
constexpr int kFoldMax = 16384;

__global__ void __launch_bounds__(1024) fold_units_kernel(FoldArgs f) {
  extern __shared__ __align__(16) double fsm[];
  const double r = tree_reduce_cta(f.u[blockIdx.x], f.n[blockIdx.x], fsm, fsm + kFoldMax);
  if (threadIdx.x == 0) f.out[blockIdx.x] = r;
}
}  // namespace adp

extern "C" int adp_fold_units(int32_t k, const double* const* units, const int64_t* n, double* out, void* stream) {
  using namespace adp;
  if (k < 1 || k > 8 || !units || !n || !out) return dense_fail(ADP_ERR_ARG, "fold: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  FoldArgs f{};
  for (int i = 0; i < k; ++i) {
    if (n[i] < 0 || n[i] > kFoldMax) return dense_fail(ADP_ERR_UNSUPPORTED, "fold: more than 16384 units");
    if (n[i] > 0 && !units[i]) return dense_fail(ADP_ERR_ARG, "fold: null unit vector");
    f.u[i] = units[i];
    f.n[i] = (int)n[i];
  }
  const size_t smem = (size_t)(kFoldMax + 64) * sizeof(double);
  if (cudaFuncSetAttribute(fold_units_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return dense_fail(ADP_ERR_CUDA, "fold: smem attribute");
  double* d_out = nullptr;
  if (cudaMallocAsync((void**)&d_out, 8 * sizeof(double), st) != cudaSuccess) return dense_fail(ADP_ERR_CUDA, "fold: alloc");
  f.out = d_out;
  fold_units_kernel<<<k, 1024, smem, st>>>(f);
  cudaMemcpyAsync(out, d_out, k * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_out, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return dense_fail(ADP_ERR_CUDA, cudaGetErrorString(e));
  return ADP_OK;
}
