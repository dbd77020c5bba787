// Instantiation: the c2 solve kernels (float64, RW = 2) with the 9x9 stencil
// as a compile-time size, so the persistent kernel carries no other stencil
// variant (compact hot loop; SURVEY.md §8 c2 is latency-bound).
#include "conv2d_kernels.cuh"

namespace adp {
const void* conv_solve_k9(int fast) {
  return fast ? (const void*)conv_solve_kernel<double, true, 2, 9> : (const void*)conv_solve_kernel<double, false, 2, 9>;
}
const void* conv_solve_k9_tma(int fast) {
  return fast ? (const void*)conv_solve_kernel<double, true, 2, 9, 512, true>
              : (const void*)conv_solve_kernel<double, false, 2, 9, 512, true>;
}
}  // namespace adp
