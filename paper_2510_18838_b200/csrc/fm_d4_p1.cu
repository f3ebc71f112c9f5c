// fm_d4_p1.cu -- dimension-4, degree-1 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(4, 1)
}  // namespace fm
