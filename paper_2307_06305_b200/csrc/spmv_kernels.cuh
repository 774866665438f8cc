// Kernel templates and launchers shared by the per-value-type translation
// units (spmv_f64.cu, spmv_f32.cu, spmv_f16.cu, spmv_bf16.cu); spmv.cu holds the C ABI.
// See spmv.cu for the kernel family.
#pragma once

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "device_common.cuh"

namespace dacsr {

constexpr int kMaxThreads = 512;
constexpr int kMaxStages = 4;
constexpr int kMaxLong = 64;      // rows > long_len starting in one chunk (<= cap/long_len+1)
constexpr int kLongChunk = 512;   // products per cooperative round (x2 buffers)
constexpr int kScratchBytes = 2 * kLongChunk * 8;

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------- kernel args
template <int KIND, class RP, class CI, class VT>
struct Mat {
  const RP* __restrict__ rp;
  const CI* __restrict__ ci;
  const VT* __restrict__ v;
  const VT* __restrict__ x;
  VT* __restrict__ y;
  int64_t xoff;
  int64_t nrows, ncols, nnz;  // bounds for the checked build
  __device__ __forceinline__ int64_t col(int64_t r, CI c) const {
    return (KIND == DACSR_KIND_DA ? r + static_cast<int64_t>(c) : static_cast<int64_t>(c)) +
           xoff;
  }
  // entry i of row r: checked build verifies i, the row and the column
  __device__ __forceinline__ void check(int64_t r, int64_t i, CI c) const {
    DACSR_CHECK(r >= 0 && r < nrows);
    DACSR_CHECK(i >= 0 && i < nnz);
    DACSR_CHECK(col(r, c) - xoff >= 0 && col(r, c) - xoff < ncols);
    (void)r; (void)i; (void)c;
  }
  __device__ __forceinline__ double prod_global(int64_t r, int64_t i) const {
    const CI c = ldg(ci + i);
    check(r, i, c);
    return product(ldg(v + i), ldg(x + col(r, c)));
  }
};

struct Scal {
  double alpha, beta;
  int order;
  int64_t long_len;
  // alpha read from device memory at the epilogue (power iteration: the
  // previous norm's 1/s, computed on the device); nullptr: `alpha`
  const double* alpha_dev = nullptr;
  // TILED only: sum of y^2 of every 512-row group in the fixed group tree
  // (aux.cu group_sumsq), stored at group_sumsq[row / 512]; nullptr: off
  double* group_sumsq = nullptr;
  __device__ __forceinline__ double a() const { return alpha_dev ? __ldg(alpha_dev) : alpha; }
};

struct Chunks {
  const int64_t* block_rows;
  int64_t base, end, nblocks;
  int cap, stages;
};

// --------------------------------------------------- block reduce (TREE)
__device__ __forceinline__ double block_sum_tree(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < nw ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
  }
  __syncthreads();
  return t;  // valid in thread 0
}

// Entry i of row r as seen by a CTA whose chunk [lo, hi) sits in smem.
template <int KIND, class RP, class CI, class VT>
struct StagedGet {
  const Mat<KIND, RP, CI, VT>& m;
  const VT* sv;
  const CI* si;
  int64_t lo, hi, r;
  __device__ __forceinline__ double operator()(int64_t i) const {
    if (i < hi) {
      const int k = static_cast<int>(i - lo);
      DACSR_CHECK(i >= lo);
      m.check(r, i, si[k]);
      return product(sv[k], ldg(m.x + m.col(r, si[k])));
    }
    return m.prod_global(r, i);
  }
};

// One long row, reduced by the whole CTA.
template <int KIND, class RP, class CI, class VT>
__device__ void long_row(const Mat<KIND, RP, CI, VT>& m, const Scal& s, int64_t r, int64_t lo,
                         int64_t hi, const VT* sv, const CI* si, double* scratch) {
  const int64_t b = ldg(m.rp + r), e = ldg(m.rp + r + 1), len = e - b;
  StagedGet<KIND, RP, CI, VT> get{m, sv, si, lo, hi, r};
  if (s.order == DACSR_ORDER_TREE) {
    double part = 0.0;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) part = __dadd_rn(part, get(i));
    const double t = block_sum_tree(part, scratch);
    if (threadIdx.x == 0) epilogue(m.y, r, t, s.a(), s.beta);
    __syncthreads();
    return;
  }
  // exact: warps 1.. produce products of round c+1 while thread 0 folds
  // round c in the reference order.
  const int64_t rounds = (len + kLongChunk - 1) / kLongChunk;
  const int producers = blockDim.x - 32;
  const int pid = threadIdx.x - 32;
  auto produce = [&](int64_t c) {
    double* buf = scratch + (c & 1) * kLongChunk;
    const int64_t start = b + c * kLongChunk;
    const int n = static_cast<int>(min64(kLongChunk, e - start));
    for (int k = pid; k < n; k += producers) buf[k] = get(start + k);
  };
  OrderedAcc acc;
  if (threadIdx.x == 0) acc.init(s.order, len);
  if (pid >= 0 && rounds > 0) produce(0);
  __syncthreads();
  for (int64_t c = 0; c < rounds; ++c) {
    if (pid >= 0 && c + 1 < rounds) produce(c + 1);
    if (threadIdx.x == 0) {
      const double* buf = scratch + (c & 1) * kLongChunk;
      const int64_t start = c * kLongChunk;
      const int n = static_cast<int>(min64(kLongChunk, len - start));
      acc.add_many(buf, n);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) epilogue(m.y, r, acc.result(), s.a(), s.beta);
  __syncthreads();
}

// Rows [r0, r1) whose entries are (mostly) staged in smem at [lo, hi).
// Ends after a __syncthreads: the stage may be overwritten afterwards.
template <int KIND, class RP, class CI, class VT>
__device__ void process_rows(const Mat<KIND, RP, CI, VT>& m, const Scal& s, int64_t r0,
                             int64_t r1, int64_t lo, int64_t hi, const VT* sv, const CI* si,
                             int64_t* long_rows, int* n_long, double* scratch) {
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const int64_t b = ldg(m.rp + r), e = ldg(m.rp + r + 1);
    if (e - b > s.long_len) {
      long_rows[atomicAdd(n_long, 1)] = r;
      continue;
    }
    StagedGet<KIND, RP, CI, VT> get{m, sv, si, lo, hi, r};
    epilogue(m.y, r, row_sum(s.order, b, e, get), s.a(), s.beta);
  }
  __syncthreads();
  const int nl = *n_long;
  for (int k = 0; k < nl; ++k) long_row(m, s, long_rows[k], lo, hi, sv, si, scratch);
}

// ------------------------------------------------- ROWBLOCK (persistent)
template <int KIND, class RP, class CI, class VT>
__global__ void __launch_bounds__(kMaxThreads, 2)
    rowblock_kernel(Mat<KIND, RP, CI, VT> m, Scal s, Chunks p) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ int64_t long_rows[kMaxLong];
  __shared__ int n_long;

  const int64_t nb = p.nblocks;
  if (blockIdx.x >= nb) return;
  const int64_t mine = (nb - 1 - blockIdx.x) / gridDim.x + 1;
  const int cap = p.cap, stages = p.stages;
  const size_t vbytes = static_cast<size_t>(cap) * sizeof(VT);
  const size_t stage_bytes = static_cast<size_t>(cap) * (sizeof(VT) + sizeof(CI));
  double* scratch = reinterpret_cast<double*>(dsm + stages * stage_bytes);
  const int64_t copy_end = p.end & ~int64_t(15);

  auto lo_of = [&](int64_t b) { return p.base + b * cap; };
  auto hi_of = [&](int64_t b) {
    const int64_t lo = lo_of(b), hi = min(lo + cap, copy_end);
    return hi > lo ? hi : lo;
  };
  auto issue = [&](int64_t k) {
    const int64_t b = blockIdx.x + k * gridDim.x;
    const int st = static_cast<int>(k % stages);
    const int64_t lo = lo_of(b), hi = hi_of(b);
    if (hi > lo) {
      const uint32_t n = static_cast<uint32_t>(hi - lo);
      unsigned char* dst = dsm + st * stage_bytes;
      mbar_arrive_expect_tx(&full[st], n * static_cast<uint32_t>(sizeof(VT) + sizeof(CI)));
      bulk_copy_g2s(dst, m.v + lo, n * sizeof(VT), &full[st]);
      bulk_copy_g2s(dst + vbytes, m.ci + lo, n * sizeof(CI), &full[st]);
    }
  };

  if (threadIdx.x == 0) {
    for (int st = 0; st < stages; ++st) mbar_init(&full[st], 1);
    mbar_fence_init();
    n_long = 0;
    for (int64_t k = 0; k < min64(stages, mine); ++k) issue(k);
  }
  __syncthreads();

  for (int64_t k = 0; k < mine; ++k) {
    const int64_t b = blockIdx.x + k * gridDim.x;
    const int st = static_cast<int>(k % stages);
    const int64_t r0 = ldg(p.block_rows + b), r1 = ldg(p.block_rows + b + 1);
    const int64_t lo = lo_of(b), hi = hi_of(b);
    if (hi > lo) mbar_wait(&full[st], static_cast<uint32_t>((k / stages) & 1));
    const unsigned char* stage = dsm + st * stage_bytes;
    process_rows(m, s, r0, r1, lo, hi, reinterpret_cast<const VT*>(stage),
                 reinterpret_cast<const CI*>(stage + vbytes), long_rows, &n_long, scratch);
    if (threadIdx.x == 0) {
      n_long = 0;
      if (k + stages < mine) {
        fence_proxy_async_smem();
        issue(k + stages);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------- STAGED (fixed rows per CTA)
template <int KIND, class RP, class CI, class VT>
__global__ void __launch_bounds__(256, 4)
    staged_kernel(Mat<KIND, RP, CI, VT> m, Scal s, int64_t row_start, int64_t row_end, int scap) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int64_t long_rows[256];
  __shared__ int n_long;
  __shared__ int64_t s_lo, s_hi;

  const int64_t r0 = row_start + static_cast<int64_t>(blockIdx.x) * blockDim.x;
  const int64_t r1 = min64(r0 + blockDim.x, row_end);
  const size_t vbytes = static_cast<size_t>(scap) * sizeof(VT);
  double* scratch = reinterpret_cast<double*>(dsm + static_cast<size_t>(scap) * (sizeof(VT) + sizeof(CI)));
  if (threadIdx.x == 0) {
    const int64_t e0 = ldg(m.rp + r0), e1 = ldg(m.rp + r1);
    const int64_t lo = e0 & ~int64_t(15);
    int64_t hi = min64(e1 & ~int64_t(15), lo + scap);
    if (hi < lo) hi = lo;
    s_lo = lo;
    s_hi = hi;
    n_long = 0;
    mbar_init(&bar, 1);
    mbar_fence_init();
    if (hi > lo) {
      const uint32_t n = static_cast<uint32_t>(hi - lo);
      mbar_arrive_expect_tx(&bar, n * static_cast<uint32_t>(sizeof(VT) + sizeof(CI)));
      bulk_copy_g2s(dsm, m.v + lo, n * sizeof(VT), &bar);
      bulk_copy_g2s(dsm + vbytes, m.ci + lo, n * sizeof(CI), &bar);
    }
  }
  __syncthreads();
  const int64_t lo = s_lo, hi = s_hi;
  if (hi > lo) mbar_wait(&bar, 0);
  process_rows(m, s, r0, r1, lo, hi, reinterpret_cast<const VT*>(dsm),
               reinterpret_cast<const CI*>(dsm + vbytes), long_rows, &n_long, scratch);
}

// ----------------------------------------------------------- SCALAR
template <int KIND, class RP, class CI, class VT>
__global__ void __launch_bounds__(256)
    scalar_kernel(Mat<KIND, RP, CI, VT> m, Scal s, int64_t row_start, int64_t row_end) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = row_start + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       r < row_end; r += stride) {
    const int64_t b = ldg(m.rp + r), e = ldg(m.rp + r + 1);
    auto get = [&](int64_t i) { return m.prod_global(r, i); };
    epilogue(m.y, r, row_sum(s.order, b, e, get), s.a(), s.beta);
  }
}

// ----------------------------------------------------------- VECTOR<G>
template <int G, int KIND, class RP, class CI, class VT>
__global__ void __launch_bounds__(256)
    vector_kernel(Mat<KIND, RP, CI, VT> m, Scal s, int64_t row_start, int64_t row_end) {
  constexpr int kGroups = 32 / G;
  const int lane = threadIdx.x & 31, sub = lane % G, grp = lane / G;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t base = row_start + warp * kGroups; base < row_end; base += nwarps * kGroups) {
    const int64_t r = base + grp;
    double acc = 0.0;
    int64_t b = 0, e = 0;
    if (r < row_end) {
      b = ldg(m.rp + r);
      e = ldg(m.rp + r + 1);
    }
    for (int64_t i = b + sub; i < e; i += G) acc = __dadd_rn(acc, m.prod_global(r, i));
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (sub == 0 && r < row_end) epilogue(m.y, r, acc, s.a(), s.beta);
  }
}

// ------------------------------------------------- WSTREAM (warp streams)
// Each warp owns chunks of 32 consecutive rows (one per lane), chunk c =
// gw, gw + W, ... (persistent grid).  The chunk's entries [A, A + VCAP)
// (A = first entry rounded down to 16 bytes of both arrays) are moved into a
// warp-private shared-memory slot by the TMA bulk-copy engine: lane 0 issues
// one cp.async.bulk per array, completion is tracked by a per-slot mbarrier
// (expect_tx).  Two slots per warp: the copy of the warp's next chunk is in
// flight while the lanes reduce the current one — no registers spent on
// staging, no CTA-wide barrier, warps pipeline independently.  Rows are
// reduced one lane per row in the exact reference order; entries past the
// staged window come from global; rows longer than long_len are reduced by
// the whole warp after the others.
// Shared-memory layout of one warp: two slots of `vcap` entries (values,
// then inner indices, each 16-byte aligned).  vcap is chosen per matrix by
// the planner (a multiple of 16 covering ~99% of the 32-row chunks).
template <class RP, class CI, class VT>
struct WarpChunk {
  static constexpr int kSlots = 2;
  // entries per 16-byte vector of the narrower array: window alignment
  static constexpr int kAlign = 16 / (sizeof(VT) < sizeof(CI) ? sizeof(VT) : sizeof(CI));
  __host__ __device__ static constexpr int value_bytes(int vcap) {
    return vcap * static_cast<int>(sizeof(VT));
  }
  __host__ __device__ static constexpr int slot_bytes(int vcap) {
    return value_bytes(vcap) + ((vcap * static_cast<int>(sizeof(CI)) + 15) & ~15);
  }
  __host__ __device__ static constexpr int warp_bytes(int vcap) { return kSlots * slot_bytes(vcap); }
};

// One row reduced by a whole warp.  TREE: lane partial sums + shfl tree.
// Exact: 128 products per batch go to a warp scratch in shared memory and
// lane 0 folds them in the reference order, while the next batch's gathers
// are already in flight.
template <int KIND, class RP, class CI, class VT>
__device__ __noinline__ void warp_long_row(const Mat<KIND, RP, CI, VT> m, Scal s, int64_t r,
                                           int64_t b, int64_t e, const VT* sv, const CI* si,
                                           int64_t A, int64_t H, int lane, double* scratch) {
  auto get = [&](int64_t i) -> double {
    if (i < H) {
      const int k = static_cast<int>(i - A);
      DACSR_CHECK(i >= A);
      m.check(r, i, si[k]);
      return product(sv[k], ldg(m.x + m.col(r, si[k])));
    }
    return m.prod_global(r, i);
  };
  if (s.order == DACSR_ORDER_TREE) {
    double part = 0.0;
    for (int64_t i = b + lane; i < e; i += 32) part = __dadd_rn(part, get(i));
    for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
    if (lane == 0) epilogue(m.y, r, part, s.a(), s.beta);
    return;
  }
  constexpr int kPer = 4;  // products per lane per batch
  OrderedAcc acc;
  acc.init(s.order, e - b);
  double p[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int64_t i = b + u * 32 + lane;
    p[u] = i < e ? get(i) : 0.0;
  }
  for (int64_t base = b; base < e; base += 32 * kPer) {
    __syncwarp();
#pragma unroll
    for (int u = 0; u < kPer; ++u) scratch[u * 32 + lane] = p[u];
    __syncwarp();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {  // next batch in flight during the fold
      const int64_t i = base + 32 * kPer + u * 32 + lane;
      p[u] = i < e ? get(i) : 0.0;
    }
    if (lane == 0) {
      const int n = static_cast<int>(min64(32 * kPer, e - base));
      // (through OrderedAcc::add the fold ran at ~100 cycles per entry:
      // C4's longest row, 1055 entries, took as long as the rest of the
      // kernel; add_many folds aligned blocks as bare addition chains)
      acc.add_many(scratch, n);
    }
  }
  __syncwarp();
  if (lane == 0) epilogue(m.y, r, acc.result(), s.a(), s.beta);
}

// Chunks the planner listed as not fitting the staging window: one warp per
// chunk, rows reduced from global in the exact order, long rows by the warp.
template <int KIND, class RP, class CI, class VT>
__device__ __noinline__ void complex_chunks(const Mat<KIND, RP, CI, VT> m, Scal s, int64_t rs,
                                            int64_t re, const int64_t* __restrict__ chunks,
                                            int64_t n_chunks, int rows_per_chunk, int cta,
                                            int n_ctas, double* scratch) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(n_ctas) * (blockDim.x >> 5);
  double* wscratch = scratch + (threadIdx.x >> 5) * 128;
  const int sub = rows_per_chunk / 32;  // 32-row pieces per listed chunk
  for (int64_t w = static_cast<int64_t>(cta) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       w < n_chunks * sub; w += nw) {
    const int64_t r = rs + rows_per_chunk * ldg(chunks + w / sub) + 32 * (w % sub) + lane;
    int64_t b = 0, e = 0;
    if (r < re) {
      b = ldg(m.rp + r);
      e = ldg(m.rp + r + 1);
    }
    const bool is_long = (e - b) > s.long_len;
    if (r < re && !is_long) {
      auto get = [&](int64_t i) { return m.prod_global(r, i); };
      epilogue(m.y, r, row_sum(s.order, b, e, get), s.a(), s.beta);
    }
    unsigned longs = __ballot_sync(0xffffffffu, r < re && is_long);
    while (longs) {
      const int src = __ffs(longs) - 1;
      longs &= longs - 1;
      const int64_t lb = __shfl_sync(0xffffffffu, b, src), le = __shfl_sync(0xffffffffu, e, src);
      warp_long_row(m, s, r - lane + src, lb, le, static_cast<const VT*>(nullptr),
                    static_cast<const CI*>(nullptr), 0, 0, lane, wscratch);
    }
  }
}

// Fully staged row, exact order, from the warp's smem slot.
// xr = &x[column base of this row]; all gathers of a batch are issued before
// the first product is folded.
// Eight gathers x[xr + off[u]] for u < cnt, issued by ONE asm statement so
// the compiler cannot interleave the fold between them: all eight are in
// flight before the first product is formed (ILP 8 per lane).
__device__ __forceinline__ void gather8(const double* xr, const int* off, int cnt, double* v) {
  const double* p[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) p[u] = xr + off[u];
  asm volatile(
      "{\n\t.reg .pred q<8>;\n\t"
      "setp.gt.s32 q0, %16, 0;\n\tsetp.gt.s32 q1, %16, 1;\n\t"
      "setp.gt.s32 q2, %16, 2;\n\tsetp.gt.s32 q3, %16, 3;\n\t"
      "setp.gt.s32 q4, %16, 4;\n\tsetp.gt.s32 q5, %16, 5;\n\t"
      "setp.gt.s32 q6, %16, 6;\n\tsetp.gt.s32 q7, %16, 7;\n\t"
      "@q0 ld.global.nc.f64 %0, [%8];\n\t@q1 ld.global.nc.f64 %1, [%9];\n\t"
      "@q2 ld.global.nc.f64 %2, [%10];\n\t@q3 ld.global.nc.f64 %3, [%11];\n\t"
      "@q4 ld.global.nc.f64 %4, [%12];\n\t@q5 ld.global.nc.f64 %5, [%13];\n\t"
      "@q6 ld.global.nc.f64 %6, [%14];\n\t@q7 ld.global.nc.f64 %7, [%15];\n\t}"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]),
        "=d"(v[7])
      : "l"(p[0]), "l"(p[1]), "l"(p[2]), "l"(p[3]), "l"(p[4]), "l"(p[5]), "l"(p[6]), "l"(p[7]),
        "r"(cnt));
}
__device__ __forceinline__ void gather8(const float* xr, const int* off, int cnt, float* v) {
  const float* p[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) p[u] = xr + off[u];
  asm volatile(
      "{\n\t.reg .pred q<8>;\n\t"
      "setp.gt.s32 q0, %16, 0;\n\tsetp.gt.s32 q1, %16, 1;\n\t"
      "setp.gt.s32 q2, %16, 2;\n\tsetp.gt.s32 q3, %16, 3;\n\t"
      "setp.gt.s32 q4, %16, 4;\n\tsetp.gt.s32 q5, %16, 5;\n\t"
      "setp.gt.s32 q6, %16, 6;\n\tsetp.gt.s32 q7, %16, 7;\n\t"
      "@q0 ld.global.nc.f32 %0, [%8];\n\t@q1 ld.global.nc.f32 %1, [%9];\n\t"
      "@q2 ld.global.nc.f32 %2, [%10];\n\t@q3 ld.global.nc.f32 %3, [%11];\n\t"
      "@q4 ld.global.nc.f32 %4, [%12];\n\t@q5 ld.global.nc.f32 %5, [%13];\n\t"
      "@q6 ld.global.nc.f32 %6, [%14];\n\t@q7 ld.global.nc.f32 %7, [%15];\n\t}"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7])
      : "l"(p[0]), "l"(p[1]), "l"(p[2]), "l"(p[3]), "l"(p[4]), "l"(p[5]), "l"(p[6]), "l"(p[7]),
        "r"(cnt));
}

template <int ORDER, class CI, class VT>
__device__ __forceinline__ double staged_dot(const VT* pv, const CI* pi, int n,
                                             const VT* __restrict__ xr) {
  if constexpr (ORDER == DACSR_ORDER_NAIVE) {
    double acc = 0.0;
    for (int j = 0; j < n; j += 8) {
      const int cnt = n - j;
      VT xv[8];
      if constexpr (sizeof(VT) == 8) {
        // f64: one asm statement for the 8 gathers (measured: 7 of 8 issued
        // before the first fold vs 4+4 from the plain loop; C2 33.2 -> 32.4 us)
        int off[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) off[u] = u < cnt ? static_cast<int>(pi[j + u]) : 0;
        gather8(xr, off, cnt, xv);
      } else {
        // f32: the plain loop measured faster (26.9 vs 29.1 us on C2 f32)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (u < cnt) xv[u] = ldg(xr + pi[j + u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < cnt) acc = __dadd_rn(acc, product(pv[j + u], xv[u]));
    }
    return acc;
  } else {
    auto get = [&](int64_t i) -> double { return product(pv[i], ldg(xr + pi[i])); };
    return ORDER == DACSR_ORDER_MACC3 ? sum_macc3(0, n, get) : sum_strip4(0, n, get);
  }
}

__device__ __forceinline__ void cp_async_4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Chunks of 32 rows whose entries [first, last) fit the staging window
// [A, A + VCAP) with A = first rounded down to 16 bytes ("simple").  The
// planner lists the others; the hot kernel skips them.
template <class IT>
__device__ __forceinline__ bool chunk_fits(IT first, IT last, int vcap, int align, IT last_aligned) {
  const IT A = first & ~static_cast<IT>(align - 1);
  IT H = A + vcap;
  if (H > last_aligned) H = last_aligned;
  return last <= H;
}

// 64 registers (4 CTAs/SM): measured faster than 48 registers at 5 CTAs/SM
// (C2: 33.5 vs 39.0 us) — the gather batch needs the registers for ILP.
#ifndef DACSR_WSTREAM_MINB
#define DACSR_WSTREAM_MINB 4
#endif
template <int KIND, class RP, class CI, class VT, int ORDER, int RPL>
__global__ void __launch_bounds__(256, DACSR_WSTREAM_MINB)
    wstream_kernel(Mat<KIND, RP, CI, VT> m, Scal s, int64_t rs, int64_t re, int64_t nnz,
                   const int64_t* complex_list, int64_t n_complex, int side_ctas, int vcap) {
  using WC = WarpChunk<RP, CI, VT>;
  constexpr int kRows = 32 * RPL;         // rows per chunk (RPL per lane)
  constexpr int kRpSlot = kRows + 8;      // rowptr values per slot (kRows + 1 used)
  const int kSlot = WC::slot_bytes(vcap), kVB = WC::value_bytes(vcap);
  extern __shared__ __align__(128) unsigned char dsm[];
  // Programmatic dependent launch: the next launch in the stream may start
  // its prologue (matrix-only reads) while this grid drains; x and y are
  // touched only after griddepcontrol.wait (the previous grid complete).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // the first side_ctas CTAs take the planner's complex chunks, so they are
  // resident from the start and overlap the streaming CTAs
  if (static_cast<int>(blockIdx.x) < side_ctas) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    complex_chunks(m, s, rs, re, complex_list, n_complex, kRows, blockIdx.x, side_ctas,
                   reinterpret_cast<double*>(dsm));
    return;
  }
  const int cta = blockIdx.x - side_ctas, n_cta = gridDim.x - side_ctas;
  using IT = RP;  // entry positions fit the rowptr type
  __shared__ __align__(8) uint64_t bars[8][WC::kSlots];
  __shared__ RP rps[8][3][kRpSlot];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* wbase = dsm + wib * WC::warp_bytes(vcap);
  uint64_t* bar = bars[wib];
  RP (*rp_slot)[kRpSlot] = rps[wib];
  const int W = n_cta * (blockDim.x >> 5);
  const int gw = cta * (blockDim.x >> 5) + wib;
  const int nchunks = static_cast<int>((re - rs + kRows - 1) / kRows);
  if (gw >= nchunks) return;
  const IT last_aligned = static_cast<IT>(nnz & ~int64_t(WC::kAlign - 1));

  if (lane == 0) {
    for (int k = 0; k < WC::kSlots; ++k) mbar_init(&bar[k], 1);
    mbar_fence_init();
  }
  // rowptr slice of chunk c: lane l copies rowptr[rs + kRows*c + 32q + l + 1]
  // (clamped) for q < RPL, lane 0 also rowptr[rs + kRows*c]
  auto fetch_rp = [&](int c, int slot) {
    if (c < nchunks) {
      const int64_t row0 = rs + kRows * static_cast<int64_t>(c);
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const RP* src = m.rp + min64(row0 + 32 * q + lane + 1, re);
        if constexpr (sizeof(RP) == 8) cp_async_8(&rp_slot[slot][32 * q + lane + 1], src);
        else cp_async_4(&rp_slot[slot][32 * q + lane + 1], src);
      }
      if (lane == 0) {
        if constexpr (sizeof(RP) == 8) cp_async_8(&rp_slot[slot][0], m.rp + row0);
        else cp_async_4(&rp_slot[slot][0], m.rp + row0);
      }
    }
    cp_async_commit();
  };
  // lane 0: the chunk's entries via the TMA bulk-copy engine
  auto issue = [&](int slot, IT first) {
    const IT A = first & ~static_cast<IT>(WC::kAlign - 1);
    IT H = A + vcap;
    if (H > last_aligned) H = last_aligned;
    if (H > A) {
      const uint32_t n = static_cast<uint32_t>(H - A);
      unsigned char* dst = wbase + slot * kSlot;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bar[slot], n * static_cast<uint32_t>(sizeof(VT) + sizeof(CI)));
      bulk_copy_g2s(dst, m.v + A, n * sizeof(VT), &bar[slot]);
      bulk_copy_g2s(dst + kVB, m.ci + A, ((n * sizeof(CI)) + 15) & ~15u, &bar[slot]);
    }
  };
  auto fits = [&](int slot) {
    return chunk_fits<IT>(rp_slot[slot][0], rp_slot[slot][kRows], vcap, WC::kAlign, last_aligned);
  };
  // a chunk's entries are copied (and waited for) iff it fits and is not
  // empty; both sides evaluate this same predicate
  auto staged = [&](int slot) {
    const IT A = rp_slot[slot][0] & ~static_cast<IT>(WC::kAlign - 1);
    return fits(slot) && rp_slot[slot][kRows] > A;
  };

  fetch_rp(gw, 0);
  fetch_rp(gw + W, 1);
  cp_async_wait<1>();
  __syncwarp();
  // per chunk, `fits` and `staged` are evaluated once (when its rowptr
  // slice lands) and carried to the iteration that consumes the chunk
  bool fits_cur = fits(0), staged_cur = staged(0);
  if (lane == 0 && staged_cur) issue(0, rp_slot[0][0]);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // x / y from here on
  uint32_t phase = 0;
  int rslot = 0;
  int k = 0;
  const VT* __restrict__ xbase = m.x + m.xoff;
  for (int c = gw; c < nchunks; c += W, ++k) {
    const int dslot = k & 1;
    const int rnext = rslot == 2 ? 0 : rslot + 1;
    const int rnn = rnext == 2 ? 0 : rnext + 1;
    cp_async_wait<0>();  // rowptr of chunk c + W (issued last iteration)
    __syncwarp();
    const bool has_next = c + W < nchunks;
    const bool fits_next = has_next && fits(rnext);
    const bool staged_next = fits_next && staged(rnext);
    if (lane == 0 && staged_next) issue(dslot ^ 1, rp_slot[rnext][0]);
    fetch_rp(c + 2 * W, rnn);
    if (fits_cur) {  // warp-uniform: complex chunks belong to the side CTAs
      if (staged_cur) {
        mbar_wait(&bar[dslot], (phase >> dslot) & 1u);
        phase ^= 1u << dslot;
      }
      const IT A = rp_slot[rslot][0] & ~static_cast<IT>(WC::kAlign - 1);
      const VT* sv = reinterpret_cast<const VT*>(wbase + dslot * kSlot);
      const CI* si = reinterpret_cast<const CI*>(wbase + dslot * kSlot + kVB);
      const int64_t row0 = rs + kRows * static_cast<int64_t>(c);
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const int rl = 32 * q + lane;
        if (row0 + rl < re) {
          const int64_t r = row0 + rl;
          const IT b = rp_slot[rslot][rl], e = rp_slot[rslot][rl + 1];
          const int kk = static_cast<int>(b - A);
          DACSR_CHECK(kk >= 0 && kk + (e - b) <= vcap && e >= b);
#ifdef DACSR_CHECKED
          for (int j = 0; j < static_cast<int>(e - b); ++j)
            m.check(r, b + j, reinterpret_cast<const CI*>(wbase + dslot * kSlot + kVB)[kk + j]);
#endif
          const VT* xr = KIND == DACSR_KIND_DA ? xbase + r : xbase;
          epilogue(m.y, r, staged_dot<ORDER>(sv + kk, si + kk, static_cast<int>(e - b), xr),
                   s.a(), s.beta);
        }
      }
    }
    __syncwarp();
    fits_cur = fits_next;
    staged_cur = staged_next;
    rslot = rnext;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------- SLICED (lane per row)
// The sliced layout (dacsr_slices_t): slice s = 32 rows, entry j of the
// row in lane l at slot slice_ptr[s] + 32*j + l.  A warp takes one slice;
// for each j the 32 lanes load one contiguous run of offsets and one of
// values straight from HBM (fully coalesced, no shared-memory staging, no
// per-chunk barrier), gather x at row + offset and fold in the exact naive
// order.  Rows longer than the layout's max_len ("spill rows") are reduced
// from the CSR arrays by the first side_ctas CTAs.
template <class CI, class VT>
struct SliceArgs {
  const int64_t* __restrict__ ptr;
  const uint8_t* __restrict__ len;
  const CI* __restrict__ ci;
  const VT* __restrict__ v;
  int64_t row0, total;
  int max_len;
  // medium rows, 32 per medium slice
  const int64_t* __restrict__ mrows;
  const int64_t* __restrict__ mptr;
  const CI* __restrict__ mci;
  const VT* __restrict__ mv;
  int64_t n_medium, m_nslices, m_total;
  // long rows (warp per row)
  const int64_t* __restrict__ lrows;
  int64_t n_long;
};

// evict-first loads for the operator (read once per SpMV) so x stays in L2
template <class T>
__device__ __forceinline__ T ldcs(const T* p) {
  return __ldcs(p);
}
template <>
__device__ __forceinline__ int64_t ldcs<int64_t>(const int64_t* p) {
  return static_cast<int64_t>(__ldcs(reinterpret_cast<const long long*>(p)));
}
template <>
__device__ __forceinline__ __nv_bfloat16 ldcs<__nv_bfloat16>(const __nv_bfloat16* p) {
  const unsigned short b = __ldcs(reinterpret_cast<const unsigned short*>(p));
  return __ushort_as_bfloat16(b);
}
template <>
__device__ __forceinline__ __half ldcs<__half>(const __half* p) {
  const unsigned short b = __ldcs(reinterpret_cast<const unsigned short*>(p));
  return __ushort_as_half(b);
}

// Long rows (listed ascending) inside [rs, re): one warp per row, exact
// order (products staged per batch, lane 0 folds), from the CSR arrays.
template <int KIND, class RP, class CI, class VT>
__device__ __noinline__ void long_rows(const Mat<KIND, RP, CI, VT> m, Scal s, int64_t rs,
                                       int64_t re, const int64_t* __restrict__ list,
                                       int64_t n_list, int cta, int n_ctas, double* scratch) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = static_cast<int64_t>(n_ctas) * (blockDim.x >> 5);
  double* wscratch = scratch + (threadIdx.x >> 5) * 128;
  for (int64_t w = static_cast<int64_t>(cta) * (blockDim.x >> 5) + (threadIdx.x >> 5); w < n_list;
       w += nw) {
    const int64_t r = ldg(list + w);
    if (r < rs || r >= re) continue;  // warp-uniform
    const int64_t b = ldg(m.rp + r), e = ldg(m.rp + r + 1);
    warp_long_row(m, s, r, b, e, static_cast<const VT*>(nullptr), static_cast<const CI*>(nullptr),
                  0, 0, lane, wscratch);
  }
}

// TMA bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, multiple of 16)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// &base[off] as one IMAD.WIDE (32-bit signed offset scaled by the element
// size into a 64-bit address) — the compiler otherwise sign-extends the
// offset and forms the address with a 64-bit shift-add pair
template <class VT>
__device__ __forceinline__ const VT* elem_addr(const VT* base, int off) {
  const VT* p;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(p) : "r"(off), "n"(static_cast<int>(sizeof(VT))), "l"(base));
  return p;
}
template <class VT>
__device__ __forceinline__ const VT* elem_addr(const VT* base, int64_t off) {
  return base + off;
}

#ifndef DACSR_SLICED_MINB
#define DACSR_SLICED_MINB 4
#endif
#ifndef DACSR_SLICED_BATCH
#define DACSR_SLICED_BATCH 8
#endif
// 16-bit values (and f32 with _F32) may trade batch size for occupancy
#ifndef DACSR_SLICED_MINB_16
#define DACSR_SLICED_MINB_16 DACSR_SLICED_MINB
#endif
#ifndef DACSR_SLICED_BATCH_16
#define DACSR_SLICED_BATCH_16 DACSR_SLICED_BATCH
#endif
#ifndef DACSR_SLICED_MINB_32
#define DACSR_SLICED_MINB_32 DACSR_SLICED_MINB
#endif
#ifndef DACSR_SLICED_BATCH_32
#define DACSR_SLICED_BATCH_32 DACSR_SLICED_BATCH
#endif
template <class VT>
struct SlicedTune {
  static constexpr int minb = sizeof(VT) == 2 ? DACSR_SLICED_MINB_16
                              : sizeof(VT) == 4 ? DACSR_SLICED_MINB_32 : DACSR_SLICED_MINB;
  static constexpr int batch = sizeof(VT) == 2 ? DACSR_SLICED_BATCH_16
                               : sizeof(VT) == 4 ? DACSR_SLICED_BATCH_32 : DACSR_SLICED_BATCH;
};
#ifndef DACSR_SLICED_PREFETCH
#define DACSR_SLICED_PREFETCH 1
#endif
#ifndef DACSR_SLICED_LDCS
#define DACSR_SLICED_LDCS 1
#endif
#ifndef DACSR_SLICED_LATE_VALUES
#define DACSR_SLICED_LATE_VALUES 0
#endif


// One lane's row of a slice in the exact naive order.  li(j) / lv(j) load
// entry j of the lane's row (offset / value) from wherever the slice sits
// (HBM or the warp's shared-memory stage).  Slots past the lane's n load
// nothing and contribute +0 * +0 = +0; acc + (+0) == acc bit-for-bit since
// the naive sum from +0.0 never holds -0.0, so the fold needs no select.
template <int B, class OT, int KIND, class RP, class CI, class VT, class LI, class LV>
__device__ __forceinline__ double slice_row_dot(const Mat<KIND, RP, CI, VT>& m, int64_t r,
                                                int width, int n, const VT* xr, const LI& li,
                                                const LV& lv, int j0 = 0, double acc = 0.0) {
  for (int j = j0; j < width; j += B) {
    OT o[B];
    VT vv[B], xv[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const bool on = j + u < n;
      o[u] = on ? static_cast<OT>(li(j + u)) : OT(0);
      if (!DACSR_SLICED_LATE_VALUES) vv[u] = on ? lv(j + u) : VT(0);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const bool on = j + u < n;
      if (on) m.check(r, 0, static_cast<CI>(o[u]));
      xv[u] = on ? ldg(elem_addr(xr, o[u])) : VT(0);
    }
    if (DACSR_SLICED_LATE_VALUES) {
      // values after the gathers: the offsets are dead by then, so the
      // batch peaks at 2 x B values instead of 2.5 x B (same latency: the
      // values, prefetched into L2, arrive alongside the gathers)
#pragma unroll
      for (int u = 0; u < B; ++u) vv[u] = j + u < n ? lv(j + u) : VT(0);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) acc = __dadd_rn(acc, product(vv[u], xv[u]));
  }
  return acc;
}

// slice_row_dot with the next batch's offsets loaded while this batch's
// gathers and values are in flight: one memory round per batch instead of
// two (the medium slices' chains; the main slices of SLICED_PIPE pipeline
// across slices instead)
template <int B, class OT, int KIND, class RP, class CI, class VT, class LI, class LV>
__device__ __forceinline__ double slice_row_dot_pipe(const Mat<KIND, RP, CI, VT>& m, int64_t r,
                                                     int width, int n, const VT* xr,
                                                     const LI& li, const LV& lv) {
  OT o[B];
#pragma unroll
  for (int u = 0; u < B; ++u) o[u] = u < n ? static_cast<OT>(li(u)) : OT(0);
  double acc = 0.0;
  for (int j = 0; j < width; j += B) {
    VT vv[B], xv[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const bool on = j + u < n;
      if (on) m.check(r, 0, static_cast<CI>(o[u]));
      xv[u] = on ? ldg(elem_addr(xr, o[u])) : VT(0);
      vv[u] = on ? lv(j + u) : VT(0);
    }
    if (j + B < width) {
#pragma unroll
      for (int u = 0; u < B; ++u) o[u] = j + B + u < n ? static_cast<OT>(li(j + B + u)) : OT(0);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) acc = __dadd_rn(acc, product(vv[u], xv[u]));
  }
  return acc;
}

#ifndef DACSR_SLICED_MEDIUM_PIPE
#define DACSR_SLICED_MEDIUM_PIPE 1
#endif
// Medium slices t = first, first + stride, ... (32 listed rows each; lanes
// whose row is outside [rs, re) skip), straight from HBM.  Call after
// griddepcontrol.wait.
template <int B, class OT, int KIND, class RP, class CI, class VT>
__device__ __forceinline__ void medium_slices(const Mat<KIND, RP, CI, VT>& m, const Scal& s,
                                              const SliceArgs<CI, VT>& sl, int64_t rs,
                                              int64_t re, int64_t first, int64_t stride,
                                              int lane) {
  const VT* __restrict__ xb = m.x + m.xoff;
  for (int64_t t = first; t < sl.m_nslices; t += stride) {
    const int64_t p0 = ldg(sl.mptr + t);
    const int width = static_cast<int>((ldg(sl.mptr + t + 1) - p0) >> 5);
    const int64_t k = 32 * t + lane;
    int64_t r = -1;
    int n = -1;
    if (k < sl.n_medium) {
      r = ldg(sl.mrows + k);
      if (r >= rs && r < re) n = ldg(sl.len + (r - sl.row0));
    }
    const VT* xr = KIND == DACSR_KIND_DA ? xb + r : xb;
    asm("" : "+l"(xr));
    DACSR_CHECK(n <= width && width <= 254);
    DACSR_CHECK(n <= 0 || p0 + lane + 32 * (n - 1) < sl.m_total);
    const CI* pi = sl.mci + p0 + lane;
    const VT* pv = sl.mv + p0 + lane;
    double acc;
    if (DACSR_SLICED_MEDIUM_PIPE) {
      // the slice's two arrays into L2 (its later batches then wait for L2,
      // not HBM), and one memory round per batch: a medium slice is a chain
      // of dependent rounds on a warp whose main slices wait behind it
      if (lane == 0 && width > 0) {
        prefetch_l2_bulk(sl.mv + p0, static_cast<uint32_t>(32 * width * sizeof(VT)));
        prefetch_l2_bulk(sl.mci + p0, static_cast<uint32_t>(32 * width * sizeof(CI)) & ~15u);
      }
      acc = slice_row_dot_pipe<B, OT>(m, r, width, n, xr,
                                      [&](int j) { return ldcs(pi + 32 * j); },
                                      [&](int j) { return ldcs(pv + 32 * j); });
    } else {
      acc = slice_row_dot<B, OT>(m, r, width, n, xr, [&](int j) { return ldcs(pi + 32 * j); },
                                 [&](int j) { return ldcs(pv + 32 * j); });
    }
    if (n >= 0) epilogue(m.y, r, acc, s.a(), s.beta);
  }
}

// SLICED kernel.  Each warp first takes its share of the medium slices
// (rows outside [rs, re) skipped lane by lane), then its main slices of
// [rs, re); long rows go to the first side_ctas CTAs.  PIPE selects:
//  0  SLICED: every slice straight from HBM with coalesced loads; the
//     entries of the slice two steps ahead are pulled into L2 by a bulk
//     prefetch (slice metadata is loaded one step earlier still).
//  1  SLICED_PIPE: mode 0 with the next slice's first-batch offsets loaded
//     while this slice's gathers and values are in flight (one memory round
//     per slice instead of two), 80 registers.
// (Round 1 also had TMA-staged, warp-specialised-ring and offset-predicted
// modes; each was exact and slower on every BASELINE config — DESIGN.md
// keeps the measurements — and they were removed.)
// Programmatic dependent launch: slice metadata and operator loads may run
// before griddepcontrol.wait; the layout builders synchronize the stream
// before a layout is used, so the grid before a sliced launch never writes
// the operator arrays.
// SLICED_PIPE holds the next slice's offsets across the iteration: 80
// registers, 3 CTAs/SM (measured: 64 registers spill and run 27 % slower)
#ifndef DACSR_SLICED_PIPE_MINB
#define DACSR_SLICED_PIPE_MINB 3
#endif
#ifndef DACSR_SLICED_PIPE_VALUES
#define DACSR_SLICED_PIPE_VALUES 1
#endif
// SMALL: rows and layout positions fit 32 bits (the launcher checks): slice
// and row indices are then ints — half the registers and instructions of the
// 64-bit index arithmetic around each slice (the 64-register SLICED kernel
// spilled its row length in the loop)
#ifndef DACSR_SLICED_SMALL
#define DACSR_SLICED_SMALL 1
#endif
// compiler barrier that names v: code using v stays behind earlier volatile
// asm and memory operations (no instruction is emitted)
template <class T>
__device__ __forceinline__ void pin_after(T& v) {
  if constexpr (sizeof(T) == 8)
    asm volatile("" : "+d"(reinterpret_cast<double&>(v))::"memory");
  else if constexpr (sizeof(T) == 4)
    asm volatile("" : "+f"(reinterpret_cast<float&>(v))::"memory");
  else
    asm volatile("" : "+h"(reinterpret_cast<unsigned short&>(v))::"memory");
}
#ifndef DACSR_SLICED_RAW_LATE
#define DACSR_SLICED_RAW_LATE 1
#endif
template <int KIND, class RP, class CI, class VT, int PIPE, bool SMALL>
__global__ void __launch_bounds__(256, PIPE ? DACSR_SLICED_PIPE_MINB : SlicedTune<VT>::minb)
    sliced_kernel(Mat<KIND, RP, CI, VT> m, Scal s, SliceArgs<CI, VT> sl, int64_t rs64, int64_t re64,
                  int side_ctas, int flags) {
  using IX = typename std::conditional<SMALL, int, int64_t>::type;
  const IX rs = static_cast<IX>(rs64), re = static_cast<IX>(re64);
  const IX row0 = static_cast<IX>(sl.row0);
  constexpr int B = SlicedTune<VT>::batch;
  using OT = typename std::conditional<sizeof(CI) == 8, int64_t, int>::type;
  extern __shared__ __align__(128) unsigned char dsm[];
  // programmatic dependent launch: metadata and operator loads may start
  // while the previous grid drains; x / y only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (static_cast<int>(blockIdx.x) < side_ctas) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    long_rows(m, s, rs64, re64, sl.lrows, sl.n_long, blockIdx.x, side_ctas,
              reinterpret_cast<double*>(dsm));
    return;
  }
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const IX W = static_cast<IX>(gridDim.x - side_ctas) * static_cast<IX>(blockDim.x >> 5);
  const IX gw = static_cast<IX>(blockIdx.x - side_ctas) * static_cast<IX>(blockDim.x >> 5) + wib;
  const IX s0 = (rs - row0) >> 5, s1 = (re - row0 + 31) >> 5;
  const VT* __restrict__ xb = m.x + m.xoff;
  bool waited = false;

  // medium slices (few, up to medium_len wide): straight from HBM
  if (gw < sl.m_nslices) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    waited = true;
    medium_slices<B, OT>(m, s, sl, rs64, re64, gw, W, lane);
  }

  // main slices of [rs, re)
  IX c = s0 + gw;
  if (c >= s1) return;
  // slice metadata: raw loads now, arithmetic one iteration later (so the
  // loads are never waited on where they are issued).  l: the lane's row
  // length byte; 256 = not a row of this launch.
  struct Raw {
    IX a, b;
    int l;
  };
  struct Meta {
    IX p0;
    int width, n;
  };
  // kLate (8-byte values): the metadata loads are branch-free (the index
  // clamped, the length load predicated) so that they can sit in the block
  // of the operator loads, behind the next slice's offset loads; derive()
  // discards the values of a slice past the end.  4-byte values keep the
  // branch and the early position (measured: C2-f32 CSR 17.5 against 18.9 us)
  constexpr bool kLate = DACSR_SLICED_RAW_LATE && PIPE && sizeof(VT) == 8;
  auto load_raw = [&](IX cc) {
    Raw w{0, 0, 256};
    if constexpr (kLate) {
      const IX cq = cc < s1 ? cc : s1 - 1;
      w.a = static_cast<IX>(ldg(sl.ptr + cq));
      w.b = static_cast<IX>(ldg(sl.ptr + cq + 1));
      const IX r = row0 + 32 * cc + lane;
      if (cc < s1 && r >= rs && r < re) w.l = ldg(sl.len + (r - row0));
    } else if (cc < s1) {
      w.a = static_cast<IX>(ldg(sl.ptr + cc));
      w.b = static_cast<IX>(ldg(sl.ptr + cc + 1));
      const IX r = row0 + 32 * cc + lane;
      if (r >= rs && r < re) w.l = ldg(sl.len + (r - row0));
    }
    return w;
  };
  auto derive = [&](const Raw& w, IX cc) {
    Meta q;
    q.p0 = w.a;
    q.width = static_cast<int>((w.b - w.a) >> 5);
    if constexpr (kLate) q.width = cc < s1 ? q.width : 0;  // clamped loads past the end
    q.n = w.l > sl.max_len ? -1 : w.l;  // 256 (none) or a medium / long row
    return q;
  };
  // the slice's two arrays into L2 (bulk prefetch).  The whole warp issues
  // it with operands the compiler knows warp-uniform (REDUX of values every
  // lane holds alike): one UBLKPF each.  Issued by lane 0 alone the two
  // instructions cost a ~20-instruction leader-election loop each — a tenth
  // of a 7-entry slice's instructions.
#ifndef DACSR_SLICED_UNIFORM_PF
#define DACSR_SLICED_UNIFORM_PF 1
#endif
  auto stage = [&](const Meta& q) {
    if (!(DACSR_SLICED_PREFETCH && !(flags & DACSR_PLAN_NO_L2_PREFETCH))) return;
    if (DACSR_SLICED_UNIFORM_PF) {
      const int width = static_cast<int>(__reduce_max_sync(0xffffffffu, q.width));
      if (width <= 0) return;
      const uint32_t plo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(q.p0));
      uint32_t phi = 0;
      if constexpr (!SMALL)
        phi = __reduce_or_sync(0xffffffffu,
                               static_cast<uint32_t>(static_cast<int64_t>(q.p0) >> 32));
      const int64_t p0 = static_cast<int64_t>((static_cast<uint64_t>(phi) << 32) | plo);
      prefetch_l2_bulk(sl.v + p0, static_cast<uint32_t>(32 * width * sizeof(VT)));
      prefetch_l2_bulk(sl.ci + p0, static_cast<uint32_t>(32 * width * sizeof(CI)) & ~15u);
      return;
    }
    if (lane != 0 || q.width <= 0) return;
    prefetch_l2_bulk(sl.v + q.p0, static_cast<uint32_t>(32 * q.width * sizeof(VT)));
    prefetch_l2_bulk(sl.ci + q.p0, static_cast<uint32_t>(32 * q.width * sizeof(CI)) & ~15u);
  };
  if constexpr (PIPE) {
    // offsets one slice ahead: the first batch's offsets of the next slice
    // are loaded while this slice's gathers and values are in flight, so
    // each slice costs one memory round (gathers + values) instead of two
    // (offsets, then gathers).
    Meta cur = derive(load_raw(c), c);
    Meta nxt = derive(load_raw(c + W), c + W);
    stage(nxt);
    OT oc[B];
    // f32 values are cheap to hold too: the next slice's first-batch values
    // travel with its offsets (measured: f32 -5 % time; f64 would spill,
    // 16-bit values measured 7 % slower)
    constexpr bool kVals = sizeof(VT) == 4 && DACSR_SLICED_PIPE_VALUES;
    VT vc[kVals ? B : 1];
    auto load_offsets = [&](const Meta& q, OT* o) {
      const CI* pi = sl.ci + q.p0 + lane;
#pragma unroll
      for (int u = 0; u < B; ++u) o[u] = u < q.n ? static_cast<OT>(ldcs(pi + 32 * u)) : OT(0);
      if constexpr (kVals) {
        const VT* pv = sl.v + q.p0 + lane;
#pragma unroll
        for (int u = 0; u < B; ++u) vc[u] = u < q.n ? ldcs(pv + 32 * u) : VT(0);
      }
    };
    load_offsets(cur, oc);
    if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (; c < s1; c += W) {
      Raw raw2;
      if (!kLate) raw2 = load_raw(c + 2 * W);
      const IX r = row0 + 32 * c + lane;
      const VT* xr = KIND == DACSR_KIND_DA ? xb + r : xb;
      asm("" : "+l"(xr));
      DACSR_CHECK(cur.n <= cur.width && cur.width <= 254);
      DACSR_CHECK(cur.n <= 0 || cur.p0 + lane + 32 * (cur.n - 1) < sl.total);
      const VT* pv = sl.v + cur.p0 + lane;
      VT xv[B], vv[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const bool on = u < cur.n;
        if (on) m.check(r, 0, static_cast<CI>(oc[u]));
        xv[u] = on ? ldg(elem_addr(xr, oc[u])) : VT(0);
        if constexpr (kVals)
          vv[u] = vc[u];
        else
          vv[u] = on ? ldcs(pv + 32 * u) : VT(0);
      }
      load_offsets(nxt, oc);
      if (kLate) {
        // the metadata loads share a scoreboard with the offset loads (ptxas
        // has six): issued ahead of the gathers, the first gather address
        // waited for them — a memory latency per slice.  Behind the offset
        // loads they are covered by the wait for the values.
        asm volatile("" ::: "memory");
        raw2 = load_raw(c + 2 * W);
#pragma unroll
        for (int u = 0; u < B; ++u) pin_after(xv[u]);  // the sums stay behind these loads
      }
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u) acc = __dadd_rn(acc, product(vv[u], xv[u]));
      if (cur.width > B) {  // the rest of a wider slice: the plain loop
        const CI* pi = sl.ci + cur.p0 + lane;
        acc = slice_row_dot<B, OT>(m, r, cur.width, cur.n, xr,
                                   [&](int j) { return ldcs(pi + 32 * j); },
                                   [&](int j) { return ldcs(pv + 32 * j); }, B, acc);
      }
      if (cur.n >= 0) epilogue(m.y, r, acc, s.a(), s.beta);
      const Meta nxt2 = derive(raw2, c + 2 * W);
      stage(nxt2);
      cur = nxt;
      nxt = nxt2;
    }
    return;
  }
  Meta cur = derive(load_raw(c), c);
  Meta nxt = derive(load_raw(c + W), c + W);
  stage(nxt);
  if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (; c < s1; c += W) {
    const Raw raw2 = load_raw(c + 2 * W);
    const IX r = row0 + 32 * c + lane;
    const VT* xr = KIND == DACSR_KIND_DA ? xb + r : xb;
    // opaque base pointer: each gather is then one IMAD.WIDE off, xr
    // instead of re-deriving x + (xoff + r + off) in 64-bit index space
    asm("" : "+l"(xr));
    DACSR_CHECK(cur.n <= cur.width && cur.width <= 254);
    DACSR_CHECK(cur.n <= 0 || cur.p0 + lane + 32 * (cur.n - 1) < sl.total);
    const CI* pi = sl.ci + cur.p0 + lane;
    const VT* pv = sl.v + cur.p0 + lane;
    double acc;
    if (DACSR_SLICED_LDCS)
      acc = slice_row_dot<B, OT>(m, r, cur.width, cur.n, xr,
                                 [&](int j) { return ldcs(pi + 32 * j); },
                                 [&](int j) { return ldcs(pv + 32 * j); });
    else
      acc = slice_row_dot<B, OT>(m, r, cur.width, cur.n, xr,
                                 [&](int j) { return ldg(pi + 32 * j); },
                                 [&](int j) { return ldg(pv + 32 * j); });
    if (cur.n >= 0) epilogue(m.y, r, acc, s.a(), s.beta);
    const Meta nxt2 = derive(raw2, c + 2 * W);
    stage(nxt2);
    cur = nxt;
    nxt = nxt2;
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

template <class RP>
__global__ void classify_chunks_kernel(const RP* __restrict__ rp, int64_t rs, int64_t re,
                                       int rows, int vcap, int align, int64_t last_aligned,
                                       int64_t* out, unsigned long long* count) {
  const int64_t nchunks = (re - rs + rows - 1) / rows;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < nchunks;
       c += stride) {
    const int64_t first = static_cast<int64_t>(rp[rs + rows * c]);
    const int64_t last = static_cast<int64_t>(rp[min64(rs + rows * c + rows, re)]);
    if (!chunk_fits<int64_t>(first, last, vcap, align, last_aligned)) {
      const unsigned long long slot = atomicAdd(count, 1ull);
      out[slot] = c;
    }
  }
}

#include "tiled.cuh"

// one launch request (dacsr_spmv arguments after validation)
struct Req {
  const dacsr_plan_t* plan;
  int variant, order;
  const void* x;
  int64_t xoff;
  void* y;
  double alpha, beta;
  int64_t rs, re;
  cudaStream_t stream;
  const double* alpha_dev = nullptr;
  double* group_sumsq = nullptr;
};

// per-value-type launchers (one translation unit each)
int launch_values_f64(const dacsr_matrix_t* a, const Req& q);
int launch_values_f32(const dacsr_matrix_t* a, const Req& q);
int launch_values_f16(const dacsr_matrix_t* a, const Req& q);
int launch_values_bf16(const dacsr_matrix_t* a, const Req& q);

// ============================================================ host side
namespace {

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  return dev;
}

// SM count of the current device (cached per device)
int sm_count() {
  static int cached[64];
  static bool have[64];
  static std::mutex mu;
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) return 148;
  if (!have[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev] = v;
    have[dev] = true;
  }
  return cached[dev];
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Per-kernel launch configuration, computed once per (device, kernel, smem
// bytes): the max-dynamic-smem attribute and the occupancy query cost
// microseconds of host time, which would otherwise sit between back-to-back
// launches.  Function attributes are per device, so the attribute is raised
// once per (device, kernel) to that device's opt-in maximum (a cap, not a
// reservation), which keeps cached entries launchable.
struct LaunchCache {
  std::mutex mu;
  static constexpr int kMax = 256;
  const void* fn[kMax] = {};
  int dev[kMax] = {};
  size_t smem[kMax] = {};
  int per_sm[kMax] = {};
  int n = 0;
  const void* raised[kMax] = {};
  int raised_dev[kMax] = {};
  int n_raised = 0;
};

template <class K>
int cached_per_sm(K kern, int threads, size_t smem) {
  static LaunchCache cache;
  const void* key = reinterpret_cast<const void*>(kern);
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(cache.mu);
  for (int i = 0; i < cache.n; ++i)
    if (cache.fn[i] == key && cache.dev[i] == dev && cache.smem[i] == smem) return cache.per_sm[i];
  bool raised = false;
  for (int i = 0; i < cache.n_raised; ++i)
    raised |= cache.raised[i] == key && cache.raised_dev[i] == dev;
  if (!raised) {
    int optin = 227 * 1024;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return -1;
    const int dyn_max = optin - static_cast<int>(fa.sharedSizeBytes);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) !=
        cudaSuccess)
      return -1;
    if (cache.n_raised < LaunchCache::kMax) {
      cache.raised[cache.n_raised] = key;
      cache.raised_dev[cache.n_raised++] = dev;
    }
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess)
    return -1;
  per_sm = std::max(1, per_sm);
  if (cache.n < LaunchCache::kMax) {
    cache.fn[cache.n] = key;
    cache.dev[cache.n] = dev;
    cache.smem[cache.n] = smem;
    cache.per_sm[cache.n] = per_sm;
    ++cache.n;
  }
  return per_sm;
}


template <class VT, class CI>
int rowblock_stages(int cap) {
  const size_t stage = static_cast<size_t>(cap) * (sizeof(VT) + sizeof(CI));
  const size_t budget = 100 * 1024;
  int st = static_cast<int>(budget / stage);
  return std::max(2, std::min(kMaxStages, st));
}

template <int KIND, class RP, class CI, class VT>
int launch(const dacsr_matrix_t* a, const Req& q) {
  Mat<KIND, RP, CI, VT> m{static_cast<const RP*>(a->rowptr), static_cast<const CI*>(a->colids),
                          static_cast<const VT*>(a->values), static_cast<const VT*>(q.x),
                          static_cast<VT*>(q.y), q.xoff, a->nrows,
                          a->ncols > 0 ? a->ncols : INT64_MAX,
                          a->nnz > 0 ? a->nnz : INT64_MAX};
  const int64_t rows = q.re - q.rs;
  if (rows <= 0) return DACSR_OK;
  const int order = q.order;
  const bool exact = order != DACSR_ORDER_TREE;
  Scal s{q.alpha, q.beta, order, 0, q.alpha_dev, q.group_sumsq};
  // the fused group sums exist in the TILED epilogue only
  if (q.group_sumsq && q.variant != DACSR_VARIANT_TILED) return DACSR_ERR_VARIANT;
  const int sms = sm_count();
  const bool can_bulk = aligned16(a->values) && aligned16(a->colids);

  switch (q.variant) {
    case DACSR_VARIANT_ROWBLOCK: {
      const dacsr_plan_t* p = q.plan;
      if (!p || p->row_start != q.rs || p->row_end != q.re || !p->block_rows) return DACSR_ERR_PLAN;
      if (p->cap <= 0 || (p->cap & 15) || !can_bulk) return DACSR_ERR_PLAN;
      // at most cap/long_len + 1 long rows can start inside one chunk
      s.long_len = std::max<int64_t>(p->long_len, p->cap / (kMaxLong - 2));
      const int stages = rowblock_stages<VT, CI>(p->cap);
      const size_t smem = static_cast<size_t>(stages) * p->cap * (sizeof(VT) + sizeof(CI)) + kScratchBytes;
      auto kern = rowblock_kernel<KIND, RP, CI, VT>;
      const int threads = kMaxThreads;
      const int per_sm = cached_per_sm(kern, threads, smem);
      if (per_sm < 0) return check_launch("rowblock launch config");
      const int64_t grid = std::min<int64_t>(p->nblocks, static_cast<int64_t>(sms) * per_sm);
      Chunks c{p->block_rows, p->entry_base, p->entry_end, p->nblocks, p->cap, stages};
      kern<<<static_cast<unsigned>(grid), threads, smem, q.stream>>>(m, s, c);
      return check_launch("rowblock_kernel");
    }
    case DACSR_VARIANT_STAGED: {
      const int threads = 256;
      // capacity: 2x the mean entries of a 256-row block, at most 64 KiB
      // (the reference-named entry points pass nnz = 0: assume 16 per row)
      const double mean = a->nnz > 0 && a->nrows ? static_cast<double>(a->nnz) / a->nrows : 16.0;
      int scap = static_cast<int>(std::min(65536.0 / (sizeof(VT) + sizeof(CI)),
                                           std::max(512.0, 2.0 * mean * threads)));
      scap &= ~15;
      if (!can_bulk) scap = 0;
      s.long_len = std::max<int64_t>(256, static_cast<int64_t>(8 * mean));
      const size_t smem = static_cast<size_t>(scap) * (sizeof(VT) + sizeof(CI)) + kScratchBytes;
      auto kern = staged_kernel<KIND, RP, CI, VT>;
      if (cached_per_sm(kern, threads, smem) < 0) return check_launch("staged launch config");
      const int64_t grid = (rows + threads - 1) / threads;
      kern<<<static_cast<unsigned>(grid), threads, smem, q.stream>>>(m, s, q.rs, q.re, scap);
      return check_launch("staged_kernel");
    }
    case DACSR_VARIANT_SCALAR: {
      const int threads = 256;
      const int64_t grid = std::min<int64_t>((rows + threads - 1) / threads, sms * 16);
      scalar_kernel<KIND, RP, CI, VT><<<static_cast<unsigned>(grid), threads, 0, q.stream>>>(
          m, s, q.rs, q.re);
      return check_launch("scalar_kernel");
    }
    case DACSR_VARIANT_VECTOR2:
    case DACSR_VARIANT_VECTOR4:
    case DACSR_VARIANT_VECTOR8:
    case DACSR_VARIANT_VECTOR16:
    case DACSR_VARIANT_WARP: {
      (void)exact;  // vector variants always combine lanes with a tree
      const int threads = 256;
      const int g = 2 << (q.variant - DACSR_VARIANT_VECTOR2);
      const int64_t rows_per_cta = threads / g;
      const int64_t grid = std::min<int64_t>((rows + rows_per_cta - 1) / rows_per_cta, sms * 16);
      const unsigned gr = static_cast<unsigned>(std::max<int64_t>(grid, 1));
      switch (g) {
        case 2: vector_kernel<2, KIND, RP, CI, VT><<<gr, threads, 0, q.stream>>>(m, s, q.rs, q.re); break;
        case 4: vector_kernel<4, KIND, RP, CI, VT><<<gr, threads, 0, q.stream>>>(m, s, q.rs, q.re); break;
        case 8: vector_kernel<8, KIND, RP, CI, VT><<<gr, threads, 0, q.stream>>>(m, s, q.rs, q.re); break;
        case 16: vector_kernel<16, KIND, RP, CI, VT><<<gr, threads, 0, q.stream>>>(m, s, q.rs, q.re); break;
        default: vector_kernel<32, KIND, RP, CI, VT><<<gr, threads, 0, q.stream>>>(m, s, q.rs, q.re); break;
      }
      return check_launch("vector_kernel");
    }
    case DACSR_VARIANT_WSTREAM: {
      const dacsr_plan_t* p = q.plan;
      if (!p || p->chunk_vcap <= 0 || (p->chunk_rows != 32 && p->chunk_rows != 64) ||
          p->row_start != q.rs || p->row_end != q.re ||
          (p->n_complex > 0 && !p->complex_chunks) || !can_bulk)
        return DACSR_ERR_PLAN;
      if (order == DACSR_ORDER_MACC3 || order == DACSR_ORDER_STRIP4) {
        // warp streams specialise the naive order; the others run row blocks
        Req r2 = q;
        r2.variant = p->block_rows ? DACSR_VARIANT_ROWBLOCK : DACSR_VARIANT_STAGED;
        return launch<KIND, RP, CI, VT>(a, r2);
      }
      const int vcap = p->chunk_vcap;
      // side CTAs need 128 doubles of scratch per warp
      const size_t per_warp = std::max<size_t>(WarpChunk<RP, CI, VT>::warp_bytes(vcap), 128 * 8);
      // up to 8 warps per CTA within ~200 KiB of shared memory
      const int warps = static_cast<int>(std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per_warp)));
      const int threads = 32 * warps;
      s.long_len = std::max<int64_t>(p->long_len, 32);
      auto kern = p->chunk_rows == 64 ? wstream_kernel<KIND, RP, CI, VT, DACSR_ORDER_NAIVE, 2>
                                      : wstream_kernel<KIND, RP, CI, VT, DACSR_ORDER_NAIVE, 1>;
      const size_t smem = per_warp * warps;
      int per_sm = cached_per_sm(kern, threads, smem);
      if (per_sm < 0) return check_launch("wstream launch config");
      if (p->ctas_per_sm > 0) per_sm = std::min(per_sm, static_cast<int>(p->ctas_per_sm));
      const int64_t chunks = (rows + p->chunk_rows - 1) / p->chunk_rows;
      // all CTAs co-resident; the complex chunks get at most 1/8 of the
      // slots (they loop), the streaming grid the rest
      const int64_t slots = static_cast<int64_t>(sms) * per_sm;
      const int side = p->n_complex > 0
                           ? static_cast<int>(std::min<int64_t>((p->n_complex + warps - 1) / warps,
                                                                std::max<int64_t>(1, slots / 8)))
                           : 0;
      const int64_t grid = std::min<int64_t>((chunks + warps - 1) / warps, std::max<int64_t>(slots - side, slots / 2));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(std::max<int64_t>(grid, 1) + side));
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = q.stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const int64_t nnz = a->nnz;
      const int64_t* cl = p->complex_chunks;
      const int64_t ncx = p->n_complex;
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, m, s, q.rs, q.re, nnz, cl, ncx, side, vcap);
      if (e != cudaSuccess) {
        set_last_error("wstream_kernel launch", e);
        return DACSR_ERR_CUDA;
      }
      return check_launch("wstream_kernel");
    }
    case DACSR_VARIANT_SLICED:
    case DACSR_VARIANT_SLICED_PIPE: {
      const dacsr_plan_t* p = q.plan;
      if (!p || !p->slices) return DACSR_ERR_PLAN;
      const dacsr_slices_t* sd = p->slices;
      if (q.rs < sd->row_start || q.re > sd->row_end || sd->max_len < 1 ||
          sd->medium_len < sd->max_len || sd->medium_len > 254 || !sd->slice_ptr ||
          !sd->row_len || (sd->total > 0 && (!sd->inner || !sd->values)) ||
          (sd->n_medium > 0 && (!sd->medium_rows || !sd->m_slice_ptr ||
                                (sd->m_total > 0 && (!sd->m_inner || !sd->m_values)))) ||
          sd->m_nslices != ((sd->n_medium + 31) >> 5) || (sd->n_long > 0 && !sd->long_rows) ||
          sd->row_end - sd->row_start >= (int64_t(1) << 31))  // rows kept as int32 offsets
        return DACSR_ERR_PLAN;
      if (order == DACSR_ORDER_MACC3 || order == DACSR_ORDER_STRIP4) {
        // the sliced loop specialises the naive order; the others run row blocks
        Req r2 = q;
        r2.variant = p->block_rows && p->row_start == q.rs && p->row_end == q.re
                         ? DACSR_VARIANT_ROWBLOCK
                         : DACSR_VARIANT_STAGED;
        return launch<KIND, RP, CI, VT>(a, r2);
      }
      SliceArgs<CI, VT> sa{sd->slice_ptr, sd->row_len, static_cast<const CI*>(sd->inner),
                           static_cast<const VT*>(sd->values), sd->row_start, sd->total,
                           sd->max_len, sd->medium_rows, sd->m_slice_ptr,
                           static_cast<const CI*>(sd->m_inner), static_cast<const VT*>(sd->m_values),
                           sd->n_medium, sd->m_nslices, sd->m_total, sd->long_rows, sd->n_long};
      constexpr int warps = 8, threads = 32 * warps;
      const size_t smem = sd->n_long > 0 ? static_cast<size_t>(warps) * 128 * 8 : 0;
      // 32-bit slice / row / position indices when they fit: 7-16 % faster
      // on the regular stencils, 3 % on C4 (measured 9 % slower there while
      // C4's longest row still set the kernel's time)
      const bool small = DACSR_SLICED_SMALL && a->nrows < (int64_t(1) << 31) - 64 &&
                         sd->total < (int64_t(1) << 31) - (int64_t(1) << 16);
      const bool pipe = q.variant == DACSR_VARIANT_SLICED_PIPE;
      auto kern = small ? (pipe ? sliced_kernel<KIND, RP, CI, VT, 1, true>
                                : sliced_kernel<KIND, RP, CI, VT, 0, true>)
                        : (pipe ? sliced_kernel<KIND, RP, CI, VT, 1, false>
                                : sliced_kernel<KIND, RP, CI, VT, 0, false>);
      int per_sm = cached_per_sm(kern, threads, smem);
      if (per_sm < 0) return check_launch("sliced launch config");
      if (p->ctas_per_sm > 0) per_sm = std::min(per_sm, static_cast<int>(p->ctas_per_sm));
      const int64_t slots = static_cast<int64_t>(sms) * per_sm;
      const int64_t nsl = ((q.re - sd->row_start + 31) >> 5) - ((q.rs - sd->row_start) >> 5) +
                          sd->m_nslices;
      // long rows: DACSR_SLICED_LONG_PER_WARP rows per warp of the side
      // CTAs, at most 1/8 of the resident CTAs (a side CTA's slot idles once
      // its rows are done: one row per warp left 34 of C4's 444 slots idle
      // for most of the kernel)
#ifndef DACSR_SLICED_LONG_PER_WARP
#define DACSR_SLICED_LONG_PER_WARP 4
#endif
      constexpr int64_t kLongPerCta = static_cast<int64_t>(warps) * DACSR_SLICED_LONG_PER_WARP;
      const int side = sd->n_long > 0
                           ? static_cast<int>(std::min<int64_t>((sd->n_long + kLongPerCta - 1) / kLongPerCta,
                                                                std::max<int64_t>(1, slots / 8)))
                           : 0;
      const int64_t grid = std::min<int64_t>((nsl + warps - 1) / warps,
                                             std::max<int64_t>(slots - side, slots / 2));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(std::max<int64_t>(grid, 1) + side));
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = q.stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, m, s, sa, q.rs, q.re, side,
                                         static_cast<int>(p->flags));
      if (e != cudaSuccess) {
        set_last_error("sliced_kernel launch", e);
        return DACSR_ERR_CUDA;
      }
      return check_launch("sliced_kernel");
    }
    case DACSR_VARIANT_TILED: {
      const dacsr_plan_t* p = q.plan;
      if (!p || !p->tiles) return DACSR_ERR_PLAN;
      const dacsr_tiles_t* td = p->tiles;
      if (q.rs < td->row_start || q.re > td->row_end || td->tile_cols < 64 ||
          td->step_group != DACSR_TILED_G ||
          td->tile_cols > 65536 || (td->tile_cols & 15) ||
          td->ngroups != (td->row_end - td->row_start + 511) / 512 ||
          (td->ngroups > 0 && (!td->ent_ptr || !td->cnt_ptr || !td->tile_lo || !td->skip)) ||
          (td->nblocks > 0 && (!td->counts || !td->order || !td->masks)) || (td->total > 0 && (!td->inner || !td->values)) ||
          (td->n_ovf > 0 && !td->ovf_rows) || (a->nnz > 0 && (!a->colids || !a->values)))
        return DACSR_ERR_PLAN;
      // fused group sums: whole 512-row groups of y (y index 0 on a group
      // boundary), no rows left to the warp-per-row pass
      if (q.group_sumsq &&
          ((td->row_start & 511) || ((q.rs - td->row_start) & 511) ||
           (q.re != td->row_end && ((q.re - td->row_start) & 511)) || td->n_ovf > 0 ||
           order == DACSR_ORDER_MACC3 || order == DACSR_ORDER_STRIP4))
        return DACSR_ERR_PLAN;
      if (order == DACSR_ORDER_MACC3 || order == DACSR_ORDER_STRIP4) {
        // the tiled fold specialises the naive order; the others run row blocks
        Req r2 = q;
        r2.variant = p->block_rows && p->row_start == q.rs && p->row_end == q.re
                         ? DACSR_VARIANT_ROWBLOCK
                         : DACSR_VARIANT_STAGED;
        return launch<KIND, RP, CI, VT>(a, r2);
      }
      const int xbuf = td->tile_cols + static_cast<int>(16 / sizeof(VT));
      const size_t smem = tiled_smem_bytes<VT>(xbuf);
      if (smem > 227 * 1024) return DACSR_ERR_PLAN;  // tile_cols too wide for the x ring
      const int threads = 32 * (kTileWarps + 1);
      auto kern = tiled_kernel<KIND, RP, CI, VT>;
      int per_sm = cached_per_sm(kern, threads, smem);
      if (per_sm < 0) return check_launch("tiled launch config");
      const int64_t g_first = (q.rs - td->row_start) / 512;
      const int64_t g_last = (q.re - td->row_start + 511) / 512;
      const int64_t nchunks = (g_last - g_first + kTileWarps - 1) / kTileWarps;
      const int64_t grid = std::max<int64_t>(
          1, std::min<int64_t>(std::max<int64_t>(nchunks, (td->n_ovf + kTileWarps - 1) / kTileWarps),
                               static_cast<int64_t>(sms) * per_sm));
      TileArgs<CI, VT> ta{td->ent_ptr, td->cnt_ptr, td->tile_lo, td->counts, td->order, td->masks, td->skip,
                          static_cast<const CI*>(td->inner), static_cast<const VT*>(td->values),
                          td->ovf_rows, td->row_start, td->col0, td->cmax, td->total, td->n_ovf,
                          td->tile_cols};
      kern<<<static_cast<unsigned>(grid), threads, smem, q.stream>>>(m, s, ta, g_first, g_last,
                                                                     q.rs, q.re, xbuf);
      return check_launch("tiled_kernel");
    }
    default:
      return DACSR_ERR_VARIANT;
  }
}

template <int KIND, class RP, class VT>
int by_colids(const dacsr_matrix_t* a, const Req& q) {
  if constexpr (KIND == DACSR_KIND_DA) {
    switch (a->colids_dtype) {
      case DACSR_I8: return launch<KIND, RP, int8_t, VT>(a, q);
      case DACSR_I16: return launch<KIND, RP, int16_t, VT>(a, q);
      case DACSR_I32: return launch<KIND, RP, int32_t, VT>(a, q);
      default: return DACSR_ERR_DTYPE;
    }
  } else {
    switch (a->colids_dtype) {
      case DACSR_I32: return launch<KIND, RP, int32_t, VT>(a, q);
      case DACSR_I64: return launch<KIND, RP, int64_t, VT>(a, q);
      default: return DACSR_ERR_DTYPE;
    }
  }
}

template <int KIND, class VT>
int by_rowptr(const dacsr_matrix_t* a, const Req& q) {
  if (a->rowptr_dtype == DACSR_I32) return by_colids<KIND, int32_t, VT>(a, q);
  if (a->rowptr_dtype == DACSR_I64) return by_colids<KIND, int64_t, VT>(a, q);
  return DACSR_ERR_DTYPE;
}

// every (kind, rowptr, colids) combination for one value type
template <class VT>
int by_kind(const dacsr_matrix_t* a, const Req& q) {
  if (a->kind == DACSR_KIND_DA) return by_rowptr<DACSR_KIND_DA, VT>(a, q);
  if (a->kind == DACSR_KIND_CSR) return by_rowptr<DACSR_KIND_CSR, VT>(a, q);
  return DACSR_ERR_DTYPE;
}

}  // namespace
}  // namespace dacsr
