// double instantiations of the SpMV kernel family (spmv_kernels.cuh).
#include "spmv_kernels.cuh"

namespace dacsr {
int launch_values_f64(const dacsr_matrix_t* a, const Req& q) { return by_kind<double>(a, q); }
}  // namespace dacsr
