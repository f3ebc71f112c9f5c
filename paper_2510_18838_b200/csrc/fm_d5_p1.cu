// fm_d5_p1.cu -- dimension-5, degree-1 fit kernels (fused search+fit, fit_many).
#include "fm_kernels.cuh"

namespace fm {
FM_DEFINE_DEG(5, 1)
}  // namespace fm
