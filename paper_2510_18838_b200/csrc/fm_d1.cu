// fm_d1.cu -- dimension-1 radius search kernels (count / fill).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DIM(1)
}  // namespace fm
