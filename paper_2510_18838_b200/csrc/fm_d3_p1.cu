// fm_d3_p1.cu -- dimension-3, degree-1 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(3, 1)
}  // namespace fm
