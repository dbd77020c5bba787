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
