// binary16 instantiations of the SpMV kernel
// family (spmv_kernels.cuh): values, x and y stored in 16 bits, products
// exact in float32 (11x11 / 8x8 significand bits), accumulated in float64 in
// the selected order, one rounding on the store.  An extension along the
// width lattice of model.py:21-74 (the reference kernels stop at f32).
#include "spmv_kernels.cuh"

namespace dacsr {
int launch_values_f16(const dacsr_matrix_t* a, const Req& q) { return by_kind<__half>(a, q); }
}  // namespace dacsr
