// fm_d2.cu -- dimension-2 radius search kernels (count / fill).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DIM(2)
}  // namespace fm
