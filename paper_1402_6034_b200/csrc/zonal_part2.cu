// zonal_part2.cu — instantiations of the compile-time-r zonal compress kernel for
// r = 33..48 (split over four translation units so nvcc builds them in parallel).
#include "adct_kernels.cuh"

namespace adct {
CompressKernel zonal_kernel_part2(int r) {
  switch (r) {
    case 33: return &k_compress<33, MODE_ZONAL, REC_NONE>;
    case 34: return &k_compress<34, MODE_ZONAL, REC_NONE>;
    case 35: return &k_compress<35, MODE_ZONAL, REC_NONE>;
    case 36: return &k_compress<36, MODE_ZONAL, REC_NONE>;
    case 37: return &k_compress<37, MODE_ZONAL, REC_NONE>;
    case 38: return &k_compress<38, MODE_ZONAL, REC_NONE>;
    case 39: return &k_compress<39, MODE_ZONAL, REC_NONE>;
    case 40: return &k_compress<40, MODE_ZONAL, REC_NONE>;
    case 41: return &k_compress<41, MODE_ZONAL, REC_NONE>;
    case 42: return &k_compress<42, MODE_ZONAL, REC_NONE>;
    case 43: return &k_compress<43, MODE_ZONAL, REC_NONE>;
    case 44: return &k_compress<44, MODE_ZONAL, REC_NONE>;
    case 45: return &k_compress<45, MODE_ZONAL, REC_NONE>;
    case 46: return &k_compress<46, MODE_ZONAL, REC_NONE>;
    case 47: return &k_compress<47, MODE_ZONAL, REC_NONE>;
    case 48: return &k_compress<48, MODE_ZONAL, REC_NONE>;
    default: return nullptr;
  }
}
}  // namespace adct
