// exact_parts.cu — compile-time-r instantiations of the exact u64 SSE kernel (adct_compress_sse576)
// for BASELINE C5's r set; any other r uses the runtime-mask instantiation k_compress_exact<2>.
#include "adct_kernels.cuh"

namespace adct {
CompressKernel exact_kernel(int r) {
  switch (r) {
    case 1: return &k_compress_exact<2, 1>;
    case 3: return &k_compress_exact<2, 3>;
    case 6: return &k_compress_exact<2, 6>;
    case 10: return &k_compress_exact<2, 10>;
    case 15: return &k_compress_exact<2, 15>;
    case 21: return &k_compress_exact<2, 21>;
    case 28: return &k_compress_exact<2, 28>;
    case 36: return &k_compress_exact<2, 36>;
    default: return nullptr;
  }
}
}  // namespace adct
