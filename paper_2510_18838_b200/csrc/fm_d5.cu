// fm_d5.cu -- dimension-5 radius search kernels (count / fill).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DIM(5)
}  // namespace fm
