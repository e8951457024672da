// zonal_part3.cu — instantiations of the compile-time-r zonal compress kernel for
// r = 49..64 (split over four translation units so nvcc builds them in parallel).
#include "adct_kernels.cuh"

namespace adct {
CompressKernel zonal_kernel_part3(int r) {
  switch (r) {
    case 49: return &k_compress<49, MODE_ZONAL, REC_NONE>;
    case 50: return &k_compress<50, MODE_ZONAL, REC_NONE>;
    case 51: return &k_compress<51, MODE_ZONAL, REC_NONE>;
    case 52: return &k_compress<52, MODE_ZONAL, REC_NONE>;
    case 53: return &k_compress<53, MODE_ZONAL, REC_NONE>;
    case 54: return &k_compress<54, MODE_ZONAL, REC_NONE>;
    case 55: return &k_compress<55, MODE_ZONAL, REC_NONE>;
    case 56: return &k_compress<56, MODE_ZONAL, REC_NONE>;
    case 57: return &k_compress<57, MODE_ZONAL, REC_NONE>;
    case 58: return &k_compress<58, MODE_ZONAL, REC_NONE>;
    case 59: return &k_compress<59, MODE_ZONAL, REC_NONE>;
    case 60: return &k_compress<60, MODE_ZONAL, REC_NONE>;
    case 61: return &k_compress<61, MODE_ZONAL, REC_NONE>;
    case 62: return &k_compress<62, MODE_ZONAL, REC_NONE>;
    case 63: return &k_compress<63, MODE_ZONAL, REC_NONE>;
    case 64: return &k_compress<64, MODE_ZONAL, REC_NONE>;
    default: return nullptr;
  }
}
}  // namespace adct
