// fm_d5_p0.cu -- dimension-5, degree-0 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(5, 0)
}  // namespace fm
