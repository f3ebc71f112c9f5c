// fm_d3_p2.cu -- dimension-3, degree-2 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(3, 2)
}  // namespace fm
