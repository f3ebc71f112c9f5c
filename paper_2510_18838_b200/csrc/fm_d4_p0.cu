// fm_d4_p0.cu -- dimension-4, degree-0 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(4, 0)
}  // namespace fm
