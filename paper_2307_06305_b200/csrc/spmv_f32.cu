// float instantiations of the SpMV kernel family (spmv_kernels.cuh).
#include "spmv_kernels.cuh"

namespace dacsr {
int launch_values_f32(const dacsr_matrix_t* a, const Req& q) { return by_kind<float>(a, q); }
}  // namespace dacsr
