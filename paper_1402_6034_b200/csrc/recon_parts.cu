// recon_parts.cu — compile-time-r instantiations of the compress + reconstruction-store kernel for
// BASELINE C5's r set (own translation unit: builds in parallel with the others).  Any other r, and
// the quantiser, use the runtime-mask instantiation k_compress_recon<MODE, RECON> (adct_api.cu).
#include "adct_kernels.cuh"

namespace adct {
template <int RECON> static ReconKernel zonal_recon(int r) {
  switch (r) {
    case 1: return &k_compress_recon<MODE_ZONAL, RECON, 1>;
    case 3: return &k_compress_recon<MODE_ZONAL, RECON, 3>;
    case 6: return &k_compress_recon<MODE_ZONAL, RECON, 6>;
    case 10: return &k_compress_recon<MODE_ZONAL, RECON, 10>;
    case 15: return &k_compress_recon<MODE_ZONAL, RECON, 15>;
    case 21: return &k_compress_recon<MODE_ZONAL, RECON, 21>;
    case 28: return &k_compress_recon<MODE_ZONAL, RECON, 28>;
    case 36: return &k_compress_recon<MODE_ZONAL, RECON, 36>;
    default: return nullptr;
  }
}
ReconKernel zonal_recon_kernel(int r, int recon) {
  return recon == REC_F32 ? zonal_recon<REC_F32>(r) : recon == REC_U8 ? zonal_recon<REC_U8>(r) : nullptr;
}
}  // namespace adct
