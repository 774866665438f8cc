// Builder of the sliced device layout (dacsr_slices_t, include/dacsr_b200.h).
//
// The reference stores a matrix as three flat row-major arrays
// (core.py:148-267) and its kernels walk each row's entries in order
// (_numba_kernels.py:82-91).  On the GPU one lane owns one row; reading
// row-major arrays lane-per-row is a strided access, which is why WSTREAM
// stages every 32-row chunk through shared memory.  The sliced layout is the
// same entries re-laid once per matrix so that entry j of the 32 rows of a
// slice is one contiguous run: the SpMV then streams it from HBM with plain
// coalesced loads.  The entries are copied bit-for-bit (raw element
// copies), the order inside a row is unchanged, so every row's exact naive
// fold — and hence y — is identical to the CSR-layout kernels.
//
// Passes (warp per slice), scans by the caller in between:
//   count        : row_len (uint8, 255 = longer than 254), per main slice
//                  32*W_s and its medium / long row counts
//   fill         : main entries to slot slice_ptr[s] + 32*j + lane (padding
//                  zeroed), medium / long rows (ascending) to their lists
//   medium_count : 32 * width of each medium slice (32 listed rows)
//   medium_fill  : medium entries to m_slice_ptr[m] + 32*j + lane

#include <algorithm>

#include "device_common.cuh"

namespace dacsr {
namespace {

template <class RP>
__global__ void slices_count_kernel(const RP* __restrict__ rp, int64_t rs, int64_t re,
                                    int max_len, int medium_len, uint8_t* __restrict__ row_len,
                                    int32_t* __restrict__ slot_counts,
                                    int32_t* __restrict__ medium_counts,
                                    int32_t* __restrict__ long_counts) {
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (re - rs + 31) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < nsl;
       c += nw) {
    const int64_t r = rs + 32 * c + lane;
    const bool in = r < re;
    int64_t l = 0;
    if (in) l = static_cast<int64_t>(rp[r + 1]) - static_cast<int64_t>(rp[r]);
    if (in) row_len[r - rs] = l > 254 ? uint8_t(255) : static_cast<uint8_t>(l);
    const bool main = in && l <= max_len;
    const bool medium = in && l > max_len && l <= medium_len;
    const bool lng = in && l > medium_len;
    const unsigned w = __reduce_max_sync(0xffffffffu, main ? static_cast<unsigned>(l) : 0u);
    const unsigned bm = __ballot_sync(0xffffffffu, medium);
    const unsigned bl = __ballot_sync(0xffffffffu, lng);
    if (lane == 0) {
      slot_counts[c] = static_cast<int32_t>(32 * w);
      medium_counts[c] = __popc(bm);
      long_counts[c] = __popc(bl);
    }
  }
}

// IT / VB: raw element types of the same width as the inner / value arrays
template <class RP, class IT, class VB>
__global__ void slices_fill_kernel(const RP* __restrict__ rp, const IT* __restrict__ ci,
                                   const VB* __restrict__ v, int64_t rs, int64_t re, int max_len,
                                   int medium_len, const int64_t* __restrict__ slice_ptr,
                                   const uint8_t* __restrict__ row_len,
                                   const int64_t* __restrict__ medium_ptr,
                                   const int64_t* __restrict__ long_ptr, IT* __restrict__ s_ci,
                                   VB* __restrict__ s_v, int64_t* __restrict__ medium_rows,
                                   int64_t* __restrict__ long_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (re - rs + 31) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const unsigned below = (1u << lane) - 1u;
  for (int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < nsl;
       c += nw) {
    const int64_t r = rs + 32 * c + lane;
    const bool in = r < re;
    int64_t l = 0, b = 0;
    if (in) {
      b = static_cast<int64_t>(rp[r]);
      l = static_cast<int64_t>(rp[r + 1]) - b;
    }
    const bool main = in && l <= max_len;
    const bool medium = in && l > max_len && l <= medium_len;
    const bool lng = in && l > medium_len;
    const int n = main ? static_cast<int>(l) : 0;
    const int64_t p0 = slice_ptr[c];
    const int width = static_cast<int>((slice_ptr[c + 1] - p0) >> 5);
    for (int j = 0; j < width; ++j) {
      const int64_t slot = p0 + 32 * j + lane;
      if (j < n) {
        s_ci[slot] = ci[b + j];
        s_v[slot] = v[b + j];
      } else {
        s_ci[slot] = IT(0);
        s_v[slot] = VB(0);
      }
    }
    const unsigned bm = __ballot_sync(0xffffffffu, medium);
    const unsigned bl = __ballot_sync(0xffffffffu, lng);
    if (medium) medium_rows[medium_ptr[c] + __popc(bm & below)] = r;
    if (lng) long_rows[long_ptr[c] + __popc(bl & below)] = r;
  }
}

// medium slice m = rows medium_rows[32m .. 32m + 31]
__global__ void medium_count_kernel(const int64_t* __restrict__ rows, int64_t n_rows,
                                    int64_t row0, const uint8_t* __restrict__ row_len,
                                    int32_t* __restrict__ slot_counts) {
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (n_rows + 31) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < nsl;
       c += nw) {
    const int64_t k = 32 * c + lane;
    const unsigned l = k < n_rows ? row_len[rows[k] - row0] : 0u;
    const unsigned w = __reduce_max_sync(0xffffffffu, l);
    if (lane == 0) slot_counts[c] = static_cast<int32_t>(32 * w);
  }
}

template <class RP, class IT, class VB>
__global__ void medium_fill_kernel(const RP* __restrict__ rp, const IT* __restrict__ ci,
                                   const VB* __restrict__ v, const int64_t* __restrict__ rows,
                                   int64_t n_rows, const int64_t* __restrict__ m_ptr,
                                   IT* __restrict__ s_ci, VB* __restrict__ s_v) {
  const int lane = threadIdx.x & 31;
  const int64_t nsl = (n_rows + 31) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < nsl;
       c += nw) {
    const int64_t k = 32 * c + lane;
    int64_t b = 0;
    int n = 0;
    if (k < n_rows) {
      const int64_t r = rows[k];
      b = static_cast<int64_t>(rp[r]);
      n = static_cast<int>(static_cast<int64_t>(rp[r + 1]) - b);
    }
    const int64_t p0 = m_ptr[c];
    const int width = static_cast<int>((m_ptr[c + 1] - p0) >> 5);
    for (int j = 0; j < width; ++j) {
      const int64_t slot = p0 + 32 * j + lane;
      s_ci[slot] = j < n ? ci[b + j] : IT(0);
      s_v[slot] = j < n ? v[b + j] : VB(0);
    }
  }
}

int grid_for(int64_t nslices) {
  const int64_t blocks = (nslices + 7) / 8;  // 8 warps per block
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 64)));
}

const int kBytes[8] = {1, 2, 4, 8, 4, 8, 2, 2};

// launch kernel template K<RP, IT, VB> with the value width of `a`
template <class RP, class IT, class F>
int by_value_bytes(const dacsr_matrix_t* a, F&& f) {
  switch (kBytes[a->values_dtype]) {
    case 8: return f(RP(), IT(), uint64_t());
    case 4: return f(RP(), IT(), uint32_t());
    case 2: return f(RP(), IT(), uint16_t());
    default: return DACSR_ERR_DTYPE;
  }
}
template <class RP, class F>
int by_inner_bytes(const dacsr_matrix_t* a, F&& f) {
  switch (kBytes[a->colids_dtype]) {
    case 1: return by_value_bytes<RP, uint8_t>(a, f);
    case 2: return by_value_bytes<RP, uint16_t>(a, f);
    case 4: return by_value_bytes<RP, uint32_t>(a, f);
    case 8: return by_value_bytes<RP, uint64_t>(a, f);
    default: return DACSR_ERR_DTYPE;
  }
}
template <class F>
int by_types(const dacsr_matrix_t* a, F&& f) {
  if (a->rowptr_dtype == DACSR_I64) return by_inner_bytes<int64_t>(a, f);
  return by_inner_bytes<int32_t>(a, f);
}

bool dtypes_ok(const dacsr_matrix_t* a) {
  return a->values_dtype >= DACSR_F32 && a->values_dtype <= DACSR_BF16 && a->colids_dtype >= 0 &&
         a->colids_dtype <= DACSR_I64 && (a->rowptr_dtype == DACSR_I32 || a->rowptr_dtype == DACSR_I64);
}

}  // namespace
}  // namespace dacsr

using namespace dacsr;

extern "C" {

int dacsr_slices_count(const dacsr_matrix_t* a, int64_t rs, int64_t re, int32_t max_len,
                       int32_t medium_len, uint8_t* row_len, int32_t* slot_counts,
                       int32_t* medium_counts, int32_t* long_counts, void* stream) {
  if (!a || !a->rowptr || rs < 0 || re < rs || re > a->nrows || max_len < 1 ||
      medium_len < max_len || medium_len > 254 ||
      (re > rs && (!row_len || !slot_counts || !medium_counts || !long_counts)))
    return DACSR_ERR_ARG;
  if (!dtypes_ok(a)) return DACSR_ERR_DTYPE;
  const int64_t nsl = (re - rs + 31) >> 5;
  if (nsl == 0) return DACSR_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const int g = grid_for(nsl);
  if (a->rowptr_dtype == DACSR_I64)
    slices_count_kernel<int64_t><<<g, 256, 0, st>>>(static_cast<const int64_t*>(a->rowptr), rs,
                                                    re, max_len, medium_len, row_len, slot_counts,
                                                    medium_counts, long_counts);
  else
    slices_count_kernel<int32_t><<<g, 256, 0, st>>>(static_cast<const int32_t*>(a->rowptr), rs,
                                                    re, max_len, medium_len, row_len, slot_counts,
                                                    medium_counts, long_counts);
  return check_launch("slices_count_kernel");
}

static bool slices_ok(const dacsr_matrix_t* a, const dacsr_slices_t* s) {
  return a && s && a->rowptr && s->row_start >= 0 && s->row_end >= s->row_start &&
         s->row_end <= a->nrows && s->nslices == ((s->row_end - s->row_start + 31) >> 5) &&
         s->slice_ptr && s->row_len && s->max_len >= 1 && s->medium_len >= s->max_len &&
         s->medium_len <= 254 && (s->total == 0 || (s->inner && s->values)) &&
         (a->nnz == 0 || (a->colids && a->values)) &&
         (s->n_medium == 0 || s->medium_rows) && (s->n_long == 0 || s->long_rows) &&
         s->m_nslices == ((s->n_medium + 31) >> 5);
}

int dacsr_slices_fill(const dacsr_matrix_t* a, const dacsr_slices_t* s, const int64_t* medium_ptr,
                      const int64_t* long_ptr, void* stream) {
  if (!slices_ok(a, s) || !medium_ptr || !long_ptr) return DACSR_ERR_ARG;
  if (!dtypes_ok(a)) return DACSR_ERR_DTYPE;
  if (s->nslices == 0) return DACSR_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const int g = grid_for(s->nslices);
  return by_types(a, [&](auto rp0, auto it0, auto vb0) {
    using RP = decltype(rp0);
    using IT = decltype(it0);
    using VB = decltype(vb0);
    slices_fill_kernel<RP, IT, VB><<<g, 256, 0, st>>>(
        static_cast<const RP*>(a->rowptr), static_cast<const IT*>(a->colids),
        static_cast<const VB*>(a->values), s->row_start, s->row_end, s->max_len, s->medium_len,
        s->slice_ptr, s->row_len, medium_ptr, long_ptr, static_cast<IT*>(const_cast<void*>(s->inner)),
        static_cast<VB*>(const_cast<void*>(s->values)), const_cast<int64_t*>(s->medium_rows),
        const_cast<int64_t*>(s->long_rows));
    return check_launch("slices_fill_kernel");
  });
}

int dacsr_slices_medium_count(const dacsr_slices_t* s, int32_t* m_slot_counts, void* stream) {
  if (!s || !s->row_len || s->n_medium < 0 || (s->n_medium > 0 && (!s->medium_rows || !m_slot_counts)))
    return DACSR_ERR_ARG;
  if (s->n_medium == 0) return DACSR_OK;
  const int64_t msl = (s->n_medium + 31) >> 5;
  medium_count_kernel<<<grid_for(msl), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      s->medium_rows, s->n_medium, s->row_start, s->row_len, m_slot_counts);
  return check_launch("medium_count_kernel");
}

int dacsr_slices_medium_fill(const dacsr_matrix_t* a, const dacsr_slices_t* s, void* stream) {
  if (!slices_ok(a, s) || (s->n_medium > 0 && (!s->m_slice_ptr || (s->m_total > 0 && (!s->m_inner || !s->m_values)))))
    return DACSR_ERR_ARG;
  if (!dtypes_ok(a)) return DACSR_ERR_DTYPE;
  if (s->n_medium == 0) return DACSR_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const int g = grid_for(s->m_nslices);
  return by_types(a, [&](auto rp0, auto it0, auto vb0) {
    using RP = decltype(rp0);
    using IT = decltype(it0);
    using VB = decltype(vb0);
    medium_fill_kernel<RP, IT, VB><<<g, 256, 0, st>>>(
        static_cast<const RP*>(a->rowptr), static_cast<const IT*>(a->colids),
        static_cast<const VB*>(a->values), s->medium_rows, s->n_medium, s->m_slice_ptr,
        static_cast<IT*>(const_cast<void*>(s->m_inner)), static_cast<VB*>(const_cast<void*>(s->m_values)));
    return check_launch("medium_fill_kernel");
  });
}

}  // extern "C"
