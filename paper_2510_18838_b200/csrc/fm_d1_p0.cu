// fm_d1_p0.cu -- dimension-1, degree-0 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(1, 0)
}  // namespace fm
