// fm_d3_p0.cu -- dimension-3, degree-0 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(3, 0)
}  // namespace fm
