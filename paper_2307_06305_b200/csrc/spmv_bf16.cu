// bfloat16 instantiations of the SpMV kernel family (spmv_kernels.cuh); the
// 16-bit numerics are described in spmv_f16.cu.
#include "spmv_kernels.cuh"

namespace dacsr {
int launch_values_bf16(const dacsr_matrix_t* a, const Req& q) {
  return by_kind<__nv_bfloat16>(a, q);
}
}  // namespace dacsr
