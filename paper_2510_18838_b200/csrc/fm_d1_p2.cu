// fm_d1_p2.cu -- dimension-1, degree-2 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(1, 2)
}  // namespace fm
