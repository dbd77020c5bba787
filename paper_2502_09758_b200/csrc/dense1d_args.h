// Kernel-argument block of the dense 1-D engine (host + device).
#pragma once
#include "adp_types.h"

namespace adp {

template <typename T>
struct DenseArgs {
  int n, G, rows_per, b_smem;   // size, grid, rows of B per CTA, B slice cached in smem
  const T* B;                    // (n, n) row-major operator
  const T* ydat;
  double alpha, l1, l2, nu, regcurv;
  int reg;
  int method, adaptive, max_iters;
  double tol, mu, step_given, lip_cached;
  int power_max_iters;
  double power_tol;
  const T* v0; const T* x0; T* out;
  const T* xt; const T* rhs; T* Q; const T* diag_in; int warm;
  T* rowbuf;                     // n: GEMV row results (exchanged)
  double* part;                  // G x n: B^T partials (exchanged)
  SumDev s_n;                    // numpy-pairwise program over n elements
  unsigned int* bar;
  SolveOut* sres;
  CGOut* cres;
  double* scal;
  int mode;
  int reg_only;                  // regularizer alone (operator term dropped)
  int nofloor;
  const T* in0; const T* in1; T* out0; T* out1;
  double pstep, pthr; int piters;   // prox_grad_iterations (DM_PROX)
  T* gvec;                       // non-null: the replicated vectors live in global memory (large n),
                                 //   CTA b's kDenseVecs vectors at gvec + (b * kDenseVecs + k) * vpitch
  int64_t vpitch;
  int plen;                      // words of the sum program s_n (cached in shared memory with the leaf starts)
  int cluster;                   // 1: the grid is ONE thread-block cluster (n <= 256: c1): GEMV row results and
                                 //    B^T partials are exchanged through distributed shared memory and
                                 //    cluster barriers instead of global memory and the grid barrier
};

struct DenseKernelSet {
  const void* solve;
  const void* cg;
  const void* misc;
};
DenseKernelSet dense_kernels_f64();
DenseKernelSet dense_kernels_f32();

}  // namespace adp
