// Seeded, counter-based generator for the random banded configurations
// C3 (n = 2^24, Poisson(16), k <= 64) and C5 (n = 2^28, Poisson(8), k <= 32)
// of BASELINE.json.  Each row is a pure function of (seed, row), so any row
// range can be generated on any rank without communication, and the CPU
// checker (oracle/gen_oracle.c) can verify individual rows of a matrix that
// never exists on the host.
//
// Row r: k = clip(Poisson(lambda), 1, kmax) by inversion of a cdf table;
// k-1 distinct offsets uniform on [-b, b] \ {0} (rejection of repeats);
// offsets with r+off outside [0, n) dropped; diagonal added; ascending.
// value(r, off): piecewise-linear normal quantile of a 53-bit hash, exact
// IEEE operations only (bit-identical on host and device).

#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "device_common.cuh"

namespace dacsr {
namespace {

constexpr uint64_t kValueSalt = 0x5851F42D4C957F2DULL;
constexpr int kMaxRow = 128;

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t key(uint64_t seed, uint64_t r, uint64_t j) {
  return splitmix(splitmix(seed ^ (r * 0xD1B54A32D192ED03ULL)) + j);
}

__device__ __forceinline__ double normal_of(uint64_t h, const double* __restrict__ table) {
  const uint64_t i = h >> 52;
  const double f = __dmul_rn(static_cast<double>((h >> 11) & ((1ULL << 41) - 1)),
                             1.0 / 2199023255552.0);
  const double lo = ldg(table + i), hi = ldg(table + i + 1);
  return __dadd_rn(lo, __dmul_rn(f, __dsub_rn(hi, lo)));
}

// sorted in-range offsets of row r into off[]; returns the count
__device__ int row_offsets(int64_t n, int64_t b, int kmax, uint64_t seed,
                           const double* __restrict__ cdf, int64_t r, int32_t* off) {
  const double u = __dmul_rn(static_cast<double>(key(seed, r, 0) >> 11), 1.0 / 9007199254740992.0);
  int k = 0;
  while (k < kmax && u >= ldg(cdf + k)) ++k;
  k = max(k, 1);
  const uint64_t span = 2ull * static_cast<uint64_t>(b);
  int32_t drawn[kMaxRow];
  int nd = 0;
  for (uint64_t j = 1; nd < k - 1; ++j) {
    const uint64_t t = ((key(seed, r, j) >> 32) * span) >> 32;
    const int32_t o = static_cast<int32_t>(static_cast<int64_t>(t) < b ? static_cast<int64_t>(t) - b
                                                                       : static_cast<int64_t>(t) - b + 1);
    bool seen = false;
    for (int q = 0; q < nd; ++q) seen |= drawn[q] == o;
    if (!seen) drawn[nd++] = o;
  }
  int m = 0;
  off[m++] = 0;
  for (int q = 0; q < nd; ++q) {
    const int64_t c = r + drawn[q];
    if (c >= 0 && c < n) off[m++] = drawn[q];
  }
  for (int a = 1; a < m; ++a) {  // insertion sort, m <= kmax
    const int32_t v = off[a];
    int c = a - 1;
    while (c >= 0 && off[c] > v) {
      off[c + 1] = off[c];
      --c;
    }
    off[c + 1] = v;
  }
  return m;
}

__global__ void counts_kernel(int64_t n, int64_t b, int kmax, uint64_t seed, const double* cdf,
                              int64_t r0, int64_t r1, int32_t* counts) {
  int32_t off[kMaxRow];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < r1;
       r += stride)
    counts[r - r0] = row_offsets(n, b, kmax, seed, cdf, r, off);
}

template <class RP, class VT>
__global__ void fill_kernel(int64_t n, int64_t b, int kmax, uint64_t seed, const double* cdf,
                            const double* table, int64_t r0, int64_t r1, const RP* rowptr,
                            int16_t* offsets, int32_t* colids, VT* values) {
  int32_t off[kMaxRow];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = r0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < r1;
       r += stride) {
    const int m = row_offsets(n, b, kmax, seed, cdf, r, off);
    const int64_t at = static_cast<int64_t>(rowptr[r - r0]);
    for (int q = 0; q < m; ++q) {
      if (offsets) offsets[at + q] = static_cast<int16_t>(off[q]);
      if (colids) colids[at + q] = static_cast<int32_t>(r + off[q]);
      const double v = normal_of(key(seed ^ kValueSalt, r, static_cast<uint64_t>(off[q] + b)), table);
      store_rounded(values + at + q, v);
    }
  }
}

template <class VT>
__global__ void normal_kernel(uint64_t seed, int64_t i0, int64_t i1, const double* table, VT* out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = i0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < i1;
       i += stride)
    store_rounded(out + (i - i0), normal_of(key(seed, i, 0), table));
}

struct Widen {
  __host__ __device__ int64_t operator()(int32_t v) const { return v; }
};

int grid_rows(int64_t rows) {
  const int64_t g = (rows + 127) / 128;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 64)));
}

}  // namespace
}  // namespace dacsr

using namespace dacsr;

extern "C" {

int dacsr_gen_banded_counts(int64_t n, int64_t b, int32_t kmax, uint64_t seed, const double* cdf,
                            int64_t r0, int64_t r1, int32_t* counts, void* stream) {
  // kmax - 1 distinct non-zero offsets must exist in [-b, b]
  if (b <= 0 || kmax < 1 || kmax > 64 || kmax - 1 > 2 * b || !cdf || r0 < 0 || r1 < r0 || r1 > n ||
      (r1 > r0 && !counts))
    return DACSR_ERR_ARG;
  if (r1 == r0) return DACSR_OK;
  counts_kernel<<<grid_rows(r1 - r0), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      n, b, kmax, seed, cdf, r0, r1, counts);
  return check_launch("counts_kernel");
}

int dacsr_gen_banded_fill(int64_t n, int64_t b, int32_t kmax, uint64_t seed, const double* cdf,
                          const double* table, int64_t r0, int64_t r1, const void* rowptr,
                          int32_t rdt, int16_t* offsets, int32_t* colids, void* values,
                          int32_t vdt, void* stream) {
  if (b <= 0 || kmax < 1 || kmax > 64 || kmax - 1 > 2 * b || !cdf || !table || r0 < 0 || r1 < r0 ||
      r1 > n || !rowptr ||
      !values)
    return DACSR_ERR_ARG;
  if (r1 == r0) return DACSR_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const int g = grid_rows(r1 - r0);
  const bool r64 = rdt == DACSR_I64;
  if (rdt != DACSR_I64 && rdt != DACSR_I32) return DACSR_ERR_DTYPE;
  if (vdt == DACSR_F64) {
    if (r64) fill_kernel<int64_t, double><<<g, 128, 0, st>>>(n, b, kmax, seed, cdf, table, r0, r1, static_cast<const int64_t*>(rowptr), offsets, colids, static_cast<double*>(values));
    else fill_kernel<int32_t, double><<<g, 128, 0, st>>>(n, b, kmax, seed, cdf, table, r0, r1, static_cast<const int32_t*>(rowptr), offsets, colids, static_cast<double*>(values));
  } else if (vdt == DACSR_F32) {
    if (r64) fill_kernel<int64_t, float><<<g, 128, 0, st>>>(n, b, kmax, seed, cdf, table, r0, r1, static_cast<const int64_t*>(rowptr), offsets, colids, static_cast<float*>(values));
    else fill_kernel<int32_t, float><<<g, 128, 0, st>>>(n, b, kmax, seed, cdf, table, r0, r1, static_cast<const int32_t*>(rowptr), offsets, colids, static_cast<float*>(values));
  } else {
    return DACSR_ERR_DTYPE;
  }
  return check_launch("fill_kernel");
}

int dacsr_gen_normal(uint64_t seed, int64_t i0, int64_t i1, const double* table, void* out,
                     int32_t vdt, void* stream) {
  if (!table || i1 < i0 || (i1 > i0 && !out)) return DACSR_ERR_ARG;
  if (i1 == i0) return DACSR_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const int g = grid_rows(i1 - i0);
  if (vdt == DACSR_F64) normal_kernel<double><<<g, 128, 0, st>>>(seed, i0, i1, table, static_cast<double*>(out));
  else if (vdt == DACSR_F32) normal_kernel<float><<<g, 128, 0, st>>>(seed, i0, i1, table, static_cast<float*>(out));
  else return DACSR_ERR_DTYPE;
  return check_launch("normal_kernel");
}

int dacsr_counts_to_rowptr(const int32_t* counts, int64_t m, void* rowptr, int32_t rdt, void* temp,
                           size_t* temp_bytes, void* stream) {
  if (!temp_bytes || m < 0 || (rdt != DACSR_I32 && rdt != DACSR_I64)) return DACSR_ERR_ARG;
  auto st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (rdt == DACSR_I64) {
    auto it = cub::TransformInputIterator<int64_t, Widen, const int32_t*>(counts, Widen());
    int64_t* out = static_cast<int64_t*>(rowptr);
    e = cub::DeviceScan::InclusiveSum(temp, *temp_bytes, it, temp ? out + 1 : out, m, st);
    if (e == cudaSuccess && temp) e = cudaMemsetAsync(out, 0, sizeof(int64_t), st);
  } else {
    int32_t* out = static_cast<int32_t*>(rowptr);
    e = cub::DeviceScan::InclusiveSum(temp, *temp_bytes, counts, temp ? out + 1 : out, m, st);
    if (e == cudaSuccess && temp) e = cudaMemsetAsync(out, 0, sizeof(int32_t), st);
  }
  if (e != cudaSuccess) {
    set_last_error("counts_to_rowptr", e);
    return DACSR_ERR_CUDA;
  }
  return DACSR_OK;
}

}  // extern "C"
