// fm_d2_p2.cu -- dimension-2, degree-2 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(2, 2)
}  // namespace fm
