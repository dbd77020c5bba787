// Microbenchmark: per-CTA tile-box load (global -> shared) cost in SM cycles,
// LDG+STS vs cp.async, fresh kernel vs after a grid-wide fence pattern.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ldg(const double* __restrict__ x, long long* out, int n_per_cta, int reps, int fence) {
  extern __shared__ double s[];
  long long acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (fence && threadIdx.x == 0) __threadfence();
    __syncthreads();
    long long t0 = clock64();
    const double* src = x + (size_t)blockIdx.x * n_per_cta + (size_t)(r % 4) * 1000;
    double v[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      int k = threadIdx.x + b * blockDim.x;
      v[b] = k < n_per_cta ? src[k] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      int k = threadIdx.x + b * blockDim.x;
      if (k < n_per_cta) s[k + (k >> 2)] = v[b];
    }
    __syncthreads();
    acc += clock64() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / reps;
}
__global__ void k_cpa(const double* __restrict__ x, long long* out, int n_per_cta, int reps, int fence) {
  extern __shared__ double s[];
  long long acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (fence && threadIdx.x == 0) __threadfence();
    __syncthreads();
    long long t0 = clock64();
    const double* src = x + (size_t)blockIdx.x * n_per_cta + (size_t)(r % 4) * 1000;
    for (int k = threadIdx.x; k < n_per_cta; k += blockDim.x) {
      unsigned d = (unsigned)__cvta_generic_to_shared(s + k + (k >> 2));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src + k) : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    acc += clock64() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / reps;
}
int main() {
  const int ctas = 128, threads = 128, n = 1932, reps = 50;
  double* x; long long* o; long long h[ctas];
  cudaMalloc(&x, (size_t)ctas * n * 8 + 8 * 8000); cudaMemset(x, 0, (size_t)ctas * n * 8 + 8 * 8000);
  cudaMalloc(&o, ctas * 8);
  for (int f = 0; f < 2; ++f) {
    k_ldg<<<ctas, threads, 20000>>>(x, o, n, reps, f); cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
    printf("LDG+STS  fence=%d: %lld cycles per 15 KB tile (CTA 0), %lld (CTA 77)\n", f, h[0], h[77]);
    k_cpa<<<ctas, threads, 20000>>>(x, o, n, reps, f); cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
    printf("cp.async fence=%d: %lld cycles per 15 KB tile (CTA 0), %lld (CTA 77)\n", f, h[0], h[77]);
  }
  return 0;
}
