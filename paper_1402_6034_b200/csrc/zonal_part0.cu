// zonal_part0.cu — instantiations of the compile-time-r zonal compress kernel for
// r = 1..16 (split over four translation units so nvcc builds them in parallel).
#include "adct_kernels.cuh"

namespace adct {
CompressKernel zonal_kernel_part0(int r) {
  switch (r) {
    case 1: return &k_compress<1, MODE_ZONAL, REC_NONE>;
    case 2: return &k_compress<2, MODE_ZONAL, REC_NONE>;
    case 3: return &k_compress<3, MODE_ZONAL, REC_NONE>;
    case 4: return &k_compress<4, MODE_ZONAL, REC_NONE>;
    case 5: return &k_compress<5, MODE_ZONAL, REC_NONE>;
    case 6: return &k_compress<6, MODE_ZONAL, REC_NONE>;
    case 7: return &k_compress<7, MODE_ZONAL, REC_NONE>;
    case 8: return &k_compress<8, MODE_ZONAL, REC_NONE>;
    case 9: return &k_compress<9, MODE_ZONAL, REC_NONE>;
    case 10: return &k_compress<10, MODE_ZONAL, REC_NONE>;
    case 11: return &k_compress<11, MODE_ZONAL, REC_NONE>;
    case 12: return &k_compress<12, MODE_ZONAL, REC_NONE>;
    case 13: return &k_compress<13, MODE_ZONAL, REC_NONE>;
    case 14: return &k_compress<14, MODE_ZONAL, REC_NONE>;
    case 15: return &k_compress<15, MODE_ZONAL, REC_NONE>;
    case 16: return &k_compress<16, MODE_ZONAL, REC_NONE>;
    default: return nullptr;
  }
}
}  // namespace adct
