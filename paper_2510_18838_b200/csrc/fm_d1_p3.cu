// fm_d1_p3.cu -- dimension-1, degree-3 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(1, 3)
}  // namespace fm
