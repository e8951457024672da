// multi_r.cu — instantiation of the fused multi-r sweep kernel for BASELINE C5's r set (own
// translation unit: it is the largest kernel and builds in parallel with the others).
#include "adct_kernels.cuh"

namespace adct {
CompressKernel multi_kernel_c5() { return &k_compress_multi<RSetC5>; }
CompressKernel sweep_inc_kernel_c5() { return &k_compress_sweep_inc<0>; }
}  // namespace adct
