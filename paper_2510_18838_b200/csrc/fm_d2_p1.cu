// fm_d2_p1.cu -- dimension-2, degree-1 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(2, 1)
}  // namespace fm
