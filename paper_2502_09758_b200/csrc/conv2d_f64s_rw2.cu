// Instantiation: double, strict (reference order, no FMA) stencils, RW = 2
// (small single-channel problems: more warps per SM).
#include "conv2d_kernels.cuh"

namespace adp {
ConvKernelSet conv_kernels_f64s_rw2() {
  ConvKernelSet k;
  k.solve = (const void*)conv_solve_kernel<double, false, 2>;
  k.cg = (const void*)conv_cg_kernel<double, false, 2>;
  k.misc = (const void*)conv_misc_kernel<double, false, 2>;
  k.kgc_part = (const void*)kgc_partial_kernel<double>;
  k.kgc_final = (const void*)kgc_final_kernel<double>;
  return k;
}
}  // namespace adp
