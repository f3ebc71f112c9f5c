// fm_d4.cu -- dimension-4 radius search kernels (count / fill).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DIM(4)
}  // namespace fm
