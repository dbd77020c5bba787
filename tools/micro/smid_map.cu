// Which SM does each CTA of a 2-CTAs-per-SM grid land on, and when does it start?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(384, 2) k(int* smid, unsigned long long* t0, int spin) {
  extern __shared__ double sm[];
  unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) { smid[blockIdx.x] = s; t0[blockIdx.x] = t; }
  double a = threadIdx.x;
  for (int i = 0; i < spin; ++i) a = a * 1.0000001 + 0.5;
  sm[threadIdx.x] = a;
}
int main() {
  const int G = 1032;
  int* d; unsigned long long* t; cudaMalloc(&d, G * 4); cudaMalloc(&t, G * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 109056);
  k<<<G, 384, 109056>>>(d, t, 20000); cudaDeviceSynchronize();
  k<<<G, 384, 109056>>>(d, t, 20000); cudaDeviceSynchronize();
  int h[G]; unsigned long long ht[G];
  cudaMemcpy(h, d, G * 4, cudaMemcpyDeviceToHost); cudaMemcpy(ht, t, G * 8, cudaMemcpyDeviceToHost);
  unsigned long long m = ht[0]; for (int i = 0; i < G; ++i) if (ht[i] < m) m = ht[i];
  for (int i = 0; i < 310; ++i) printf("%d:%d@%llu ", i, h[i], (ht[i] - m) / 100);
  printf("\n");
  // pairs sharing an SM among the first 296
  int first[256]; for (int i = 0; i < 256; ++i) first[i] = -1;
  int same_half = 0;
  for (int i = 0; i < 296; ++i) { if (first[h[i]] < 0) first[h[i]] = i; else if ((first[h[i]] < 148) == (i < 148)) ++same_half; }
  printf("pairs within the same half of the first wave: %d\n", same_half);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
