// fm_d2_p3.cu -- dimension-2, degree-3 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(2, 3)
}  // namespace fm
