// fm_d3.cu -- dimension-3 radius search kernels (count / fill).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DIM(3)
}  // namespace fm
