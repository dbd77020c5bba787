// Microbenchmark: formulations of the strict (DMUL+DADD, row-major tap order)
// K = 15 register-blocked stencil at c3 geometry (one channel per CTA).
// RW outputs per row per thread, RH output rows per thread; input rows are
// walked once each and applied to every output row that uses them (per
// output the taps stay in row-major order).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int K = 15, R = K / 2, TW = 64;
constexpr int H = 512, W = 512, C = 3;

__device__ __forceinline__ double madd(double a, double x, double w) { return __dadd_rn(a, __dmul_rn(x, w)); }

template <int RW>
__device__ __forceinline__ int sk(int c) { return RW == 1 ? c : c + c / RW; }

__constant__ double cw[C * K * K];

template <int TH, int RW, int RH, int CW>
__global__ void __launch_bounds__((TH / RH) * (TW / RW)) stage(const double* __restrict__ x, const double* __restrict__ y,
                                                              const double* __restrict__ kern, double* __restrict__ out) {
  constexpr int SH = TH + 2 * R + 2, SWL = TW + 2 * R + 2, SWP = SWL + SWL / RW + 1;
  __shared__ __align__(16) double ws[K * K + 1];
  extern __shared__ double pl[];
  const int tilesW = W / TW;
  const int tile = blockIdx.x / C, ch = blockIdx.x % C;
  const int h0 = (tile / tilesW) * TH, w0 = (tile % tilesW) * TW;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) ws[e] = kern[e * C + ch];
  const int gh0 = h0 - R - 1, gw0 = w0 - R - 1;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int sr = threadIdx.x >> 5; sr < SH; sr += nw) {
    const int gh = gh0 + sr;
    const bool rok = gh >= 0 && gh < H;
    for (int e = lane; e < SWL; e += 32) {
      const int gw = gw0 + e;
      const bool ok = rok && gw >= 0 && gw < W;
      const unsigned d = (unsigned)__cvta_generic_to_shared(pl + sr * SWP + sk<RW>(e));
      const double* s = ok ? x + ((size_t)gh * W + gw) * C + ch : x;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(s), "r"(ok ? 8 : 0) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  constexpr int TPR = TW / RW;
  const int ty = threadIdx.x / TPR, tx = threadIdx.x % TPR;
  const int hb = h0 + ty * RH;
  __syncthreads();
  double acc[RH][RW];
#pragma unroll
  for (int q = 0; q < RH; ++q)
#pragma unroll
    for (int o = 0; o < RW; ++o) acc[q][o] = 0.0;
  const double* base = pl + (ty * RH + 1) * SWP + sk<RW>(tx * RW);
  // input row m (0 .. K + RH - 2) feeds output row q with kernel row i = m - q
#pragma unroll
  for (int m = 0; m < K + RH - 1; ++m) {
    const double* row = base + m * SWP;
    double win[K + RW - 1];
#pragma unroll
    for (int e = 0; e < K + RW - 1; ++e) win[e] = row[sk<RW>(1 + e)];
#pragma unroll
    for (int q = 0; q < RH; ++q) {
      const int i = m - q;
      if (i < 0 || i >= K) continue;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const double wt = CW ? cw[ch * K * K + i * K + j] : ws[i * K + j];
#pragma unroll
        for (int o = 0; o < RW; ++o) acc[q][o] = madd(acc[q][o], win[o + j], wt);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < RH; ++q)
#pragma unroll
    for (int o = 0; o < RW; ++o) {
      const size_t gi = ((size_t)(hb + q) * W + w0 + tx * RW + o) * C + ch;
      out[gi] = acc[q][o] - y[gi];
    }
}

template <int TH, int RW, int RH, int CW = 0>
void run(const double* x, const double* y, const double* k, double* out) {
  constexpr int SH = TH + 2 * R + 2, SWL = TW + 2 * R + 2, SWP = SWL + SWL / RW + 1;
  const size_t smem = (size_t)SH * SWP * sizeof(double);
  const int threads = (TH / RH) * (TW / RW);
  cudaFuncSetAttribute(stage<TH, RW, RH, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, stage<TH, RW, RH, CW>);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, stage<TH, RW, RH, CW>, threads, smem);
  const int grid = (H / TH) * (W / TW) * C;
  for (int w = 0; w < 3; ++w) stage<TH, RW, RH, CW><<<grid, threads, smem>>>(x, y, k, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 400;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) stage<TH, RW, RH, CW><<<grid, threads, smem>>>(x, y, k, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = 1e3 * ms / reps;
  const double taps = (double)H * W * C * K * K;
  printf("%s TH=%2d RW=%d RH=%d threads=%3d regs=%3d CTAs/SM=%2d: %6.2f us/pass %.2f Ttap/s (%s)\n", CW ? "const" : "smem ", TH, RW, RH, threads,
         fa.numRegs, nb, us, taps / us / 1e6, cudaGetErrorString(cudaGetLastError()));
}

__global__ void spin(double* o, int n) {
  double a = threadIdx.x, c0 = 0.5;
  for (int i = 0; i < n; ++i) c0 = fma(a, 1.0000001, c0);
  if (c0 == 1.2345) o[0] = 1;
}

int main() {
  const size_t n = (size_t)H * W * C;
  double *x, *y, *k, *out;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&y, n * 8);
  cudaMalloc(&out, n * 8);
  cudaMalloc(&k, K * K * C * 8);
  cudaMemset(x, 0, n * 8);
  cudaMemset(y, 0, n * 8);
  cudaMemset(k, 0, K * K * C * 8);
  for (int w = 0; w < 20; ++w) spin<<<148 * 4, 512>>>(out, 200000);   // clocks up before timing
  cudaDeviceSynchronize();
  run<16, 4, 1>(x, y, k, out);
  run<16, 4, 1, 1>(x, y, k, out);
  run<16, 4, 2, 1>(x, y, k, out);
  run<16, 8, 1, 1>(x, y, k, out);
  run<16, 2, 4, 1>(x, y, k, out);
  run<16, 4, 4, 1>(x, y, k, out);
  run<16, 4, 2>(x, y, k, out);
  run<16, 4, 4>(x, y, k, out);
  run<16, 8, 1>(x, y, k, out);
  run<16, 8, 2>(x, y, k, out);
  run<16, 2, 4>(x, y, k, out);
  run<32, 4, 4>(x, y, k, out);
  run<32, 4, 8>(x, y, k, out);
  run<16, 2, 8>(x, y, k, out);
  run<16, 4, 1>(x, y, k, out);
  return 0;
}
