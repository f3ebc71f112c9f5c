// fm_d2_p0.cu -- dimension-2, degree-0 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(2, 0)
}  // namespace fm
