// Grid-barrier latency micro-benchmark (cooperative launch, one CTA per SM).
//   V0: __syncthreads; t0: fence + atomicAdd + acquire-spin + fence (the engine's GridBarrier)
//   V1: __syncthreads; t0: red.release.gpu + ld.acquire spin
//   V2: flag array: CTA b stores epoch to flag[b] (st.release); threads t < G spin on flag[t]
//   V3: two-level counters (16 groups), last arriver of a group bumps the top counter
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barbench barbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__global__ void bar_kernel(int variant, int iters, unsigned* cnt, unsigned* flags, unsigned* grp, double* sink) {
  const unsigned G = gridDim.x;
  unsigned target = 0;
  double acc = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    acc = acc * 1.0000001 + 1.0;   // a little "work"
    if (variant == 0) {
      __syncthreads();
      if (threadIdx.x == 0) {
        target += G;
        __threadfence();
        atomicAdd(cnt, 1u);
        while ((int)(ld_acq(cnt) - target) < 0) {
        }
        __threadfence();
      }
      __syncthreads();
    } else if (variant == 1) {
      __syncthreads();
      if (threadIdx.x == 0) {
        target += G;
        red_rel(cnt, 1u);
        while ((int)(ld_acq(cnt) - target) < 0) {
        }
      }
      __syncthreads();
    } else if (variant == 2) {
      const unsigned epoch = it + 1;
      __syncthreads();
      if (threadIdx.x == 0) st_rel(flags + blockIdx.x * 32, epoch);   // one flag per 128-byte line
      if (threadIdx.x < G) {
        while ((int)(ld_acq(flags + threadIdx.x * 32) - epoch) < 0) {
        }
      }
      __syncthreads();
    } else {
      // two-level: groups of 16 CTAs
      const unsigned ng = (G + 15) / 16, gi = blockIdx.x / 16;
      const unsigned gsz = min(16u, G - gi * 16);
      const unsigned epoch = it + 1;
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned old = atom_add_acqrel(grp + gi * 32, 1u);
        if (old + 1 == epoch * gsz) red_rel(cnt, 1u);
        while ((int)(ld_acq(cnt) - epoch * ng) < 0) {
        }
      }
      __syncthreads();
    }
  }
  if (acc == -1.0) *sink = acc;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned *cnt, *flags, *grp;
  double* sink;
  cudaMalloc(&cnt, 256);
  cudaMalloc(&flags, 148 * 128 * 2);
  cudaMalloc(&grp, 64 * 128);
  cudaMalloc(&sink, 8);
  const int iters = 2000;
  for (int threads : {256, 512}) {
    for (int v = 0; v < 4; ++v) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(cnt, 0, 256);
        cudaMemset(flags, 0, 148 * 128 * 2);
        cudaMemset(grp, 0, 64 * 128);
        int variant = v, it = iters;
        void* args[] = {&variant, &it, &cnt, &flags, &grp, &sink};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_kernel, dim3(sms), dim3(threads), args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (e != cudaSuccess) {
          printf("launch failed: %s\n", cudaGetErrorString(e));
          return 1;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("threads %d variant %d: %.3f us per barrier\n", threads, v, best * 1e3f / iters);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
