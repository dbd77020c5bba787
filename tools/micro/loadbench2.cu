// The engine's row-per-warp loader (c2 geometry) in isolation, with and
// without other CTAs having just written the source (grid sync between).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
constexpr int kJ = 8;
__device__ __forceinline__ int sk(int c) { return c + (c >> 2); }
__global__ void k(double* x, long long* out, int reps, int write_first) {
  extern __shared__ double s[];
  cg::grid_group grid = cg::this_grid();
  const int H = 256, W = 256, C = 1, SH = 14, SWP = 138 + 34 + 1, rowE = 138;
  const unsigned mC = (1u << 20);
  const int tilesW = 2;
  const int tile = blockIdx.x, h0 = (tile / tilesW) * 4, w0 = (tile % tilesW) * 128;
  const int gh0 = h0 - 5, gw0 = w0 - 5;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  long long acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (write_first) {  // every CTA rewrites its own tile pixels, then grid sync
      for (int i = threadIdx.x; i < 512; i += blockDim.x) x[(h0 + i / 128) * W + w0 + (i % 128)] = r + i;
      grid.sync();
    }
    __syncthreads();
    long long t0 = clock64();
    for (int sr0 = threadIdx.x >> 5; sr0 < SH; sr0 += 2 * nw) {
      double v[2][kJ];
      int off[2][kJ];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int sr = sr0 + rr * nw;
        const int gh = gh0 + sr;
        const bool rowok = sr < SH && gh >= 0 && gh < H;
        const long long rowbase = ((long long)gh * W + gw0) * C;
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
          const int e = lane + 32 * j;
          const int px = (int)(((unsigned long long)(unsigned)e * mC) >> 20);
          const int c = e - px * C;
          const int gw = gw0 + px;
          const bool ok = rowok && e < rowE && (unsigned)gw < (unsigned)W;
          off[rr][j] = (sr < SH && e < rowE) ? c * SH * SWP + sr * SWP + sk(px) : -1;
          v[rr][j] = ok ? x[rowbase + e] : 0.0;
        }
      }
#pragma unroll
      for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int j = 0; j < kJ; ++j)
          if (off[rr][j] >= 0) s[off[rr][j]] = v[rr][j];
    }
    __syncthreads();
    acc += clock64() - t0;
    if (write_first) grid.sync();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc / reps;
}
int main() {
  double* x; long long* o; long long h[128];
  cudaMalloc(&x, 256 * 256 * 8); cudaMemset(x, 0, 256 * 256 * 8);
  cudaMalloc(&o, 128 * 8);
  for (int wf = 0; wf < 2; ++wf) {
    int reps = 50;
    void* args[] = {&x, &o, &reps, &wf};
    cudaLaunchCooperativeKernel((void*)k, 128, 128, args, 20000, 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
    printf("engine loader, write_first=%d: %lld cycles (CTA 0), %lld (CTA 77) [%s]\n", wf, h[0], h[77], cudaGetErrorString(e));
  }
  return 0;
}
