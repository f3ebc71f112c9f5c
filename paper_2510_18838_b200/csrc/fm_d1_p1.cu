// fm_d1_p1.cu -- dimension-1, degree-1 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(1, 1)
}  // namespace fm
