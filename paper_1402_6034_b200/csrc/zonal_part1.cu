// zonal_part1.cu — instantiations of the compile-time-r zonal compress kernel for
// r = 17..32 (split over four translation units so nvcc builds them in parallel).
#include "adct_kernels.cuh"

namespace adct {
CompressKernel zonal_kernel_part1(int r) {
  switch (r) {
    case 17: return &k_compress<17, MODE_ZONAL, REC_NONE>;
    case 18: return &k_compress<18, MODE_ZONAL, REC_NONE>;
    case 19: return &k_compress<19, MODE_ZONAL, REC_NONE>;
    case 20: return &k_compress<20, MODE_ZONAL, REC_NONE>;
    case 21: return &k_compress<21, MODE_ZONAL, REC_NONE>;
    case 22: return &k_compress<22, MODE_ZONAL, REC_NONE>;
    case 23: return &k_compress<23, MODE_ZONAL, REC_NONE>;
    case 24: return &k_compress<24, MODE_ZONAL, REC_NONE>;
    case 25: return &k_compress<25, MODE_ZONAL, REC_NONE>;
    case 26: return &k_compress<26, MODE_ZONAL, REC_NONE>;
    case 27: return &k_compress<27, MODE_ZONAL, REC_NONE>;
    case 28: return &k_compress<28, MODE_ZONAL, REC_NONE>;
    case 29: return &k_compress<29, MODE_ZONAL, REC_NONE>;
    case 30: return &k_compress<30, MODE_ZONAL, REC_NONE>;
    case 31: return &k_compress<31, MODE_ZONAL, REC_NONE>;
    case 32: return &k_compress<32, MODE_ZONAL, REC_NONE>;
    default: return nullptr;
  }
}
}  // namespace adct
