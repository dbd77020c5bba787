// Host-stepped solve: in-kernel ("tail") evaluation of the decision sums.
//
// The stage kernels that produce sum leaves (candidate value + speculative
// stage A, non-speculative stage A) finish with a ticketed fold instead of a
// separate reduction launch: the last CTA of a tile row folds that row's
// leaves (a power-of-two run of the perfect pairwise tree) into sub-values,
// and the last tile row of the candidate half folds the sub-values of all six
// sums and writes them, then a sequence number, to mapped pinned host memory.
// The tree is the one reduce_k evaluates (perfect binary tree in leaf order,
// zero padded), so the sums are bitwise those of step_reduce_kernel; only the
// distribution of the work differs.  The candidate CTAs come first in the
// grid, so the host has the decision while the speculative half still runs
// and the next launch is queued before the kernel ends.
#pragma once

namespace adp {

struct StepTail {
  double* sub;          // sub-values, see the offsets below (11 * nG doubles)
  unsigned int* cnt;    // [nG] candidate-half tickets, [nG] stage-A tickets, [1] top ticket (zero between launches)
  int on;               // 0: no tail (the host launches step_reduce_kernel)
  int nG;               // groups = tile rows (power of two)
  int GL;               // leaves of an N-element sum per group (power of two, <= 1024)
  int tW;               // tiles per group (power of two)
  int setA;             // (fit, tv) set the stage-A pass of this launch writes: 0 / 1
  int setR;             // (fit, tv) set the decision of this launch reads
  // sub-value offsets (doubles)
  __host__ __device__ int o_fit(int set) const { return set * nG; }
  __host__ __device__ int o_tv(int set) const { return 2 * nG + set * 2 * nG; }
  __host__ __device__ int o_fitc() const { return 6 * nG; }
  __host__ __device__ int o_tvc() const { return 7 * nG; }
  __host__ __device__ int o_t0() const { return 9 * nG; }
  __host__ __device__ int o_t1() const { return 10 * nG; }
};

}  // namespace adp
