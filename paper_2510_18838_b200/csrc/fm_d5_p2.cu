// fm_d5_p2.cu -- dimension-5, degree-2 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(5, 2)
}  // namespace fm
