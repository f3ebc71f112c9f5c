// fm_d3_p3.cu -- dimension-3, degree-3 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(3, 3)
}  // namespace fm
