// fm_d4_p2.cu -- dimension-4, degree-2 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(4, 2)
}  // namespace fm
