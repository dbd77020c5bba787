// Instantiation: float, FMA stencils.
#include "conv2d_kernels.cuh"

namespace adp {
ConvKernelSet conv_kernels_f32() {
  ConvKernelSet k;
  k.solve = (const void*)conv_solve_kernel<float, true, 4>;
  k.cg = (const void*)conv_cg_kernel<float, true, 4>;
  k.misc = (const void*)conv_misc_kernel<float, true, 4>;
  k.kgc_part = (const void*)kgc_partial_kernel<float>;
  k.kgc_final = (const void*)kgc_final_kernel<float>;
  return k;
}
}  // namespace adp
