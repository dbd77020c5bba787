// Instantiation: RW = 4 solve kernels (c3, c4, c5 and the fp32 mode) bounded
// at kSolveT384 threads per CTA, so they get 168 registers per thread
// instead of spilling at the 512-thread cap of 128.
#include "conv2d_kernels.cuh"

namespace adp {
const void* conv_solve_t384(int dtype, int fast) {
  if (dtype == 1) return (const void*)conv_solve_kernel<float, true, 4, 0, kSolveT384>;
  return fast ? (const void*)conv_solve_kernel<double, true, 4, 0, kSolveT384>
              : (const void*)conv_solve_kernel<double, false, 4, 0, kSolveT384>;
}
}  // namespace adp
