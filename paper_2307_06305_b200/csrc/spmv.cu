// SpMV kernels for CSR and DA-CSR on sm_100a, and their C-ABI launchers.
//
// Replaces the reference's compiled inner loops
// (/root/reference/pkg/src/dacsr/spmv/_numba_kernels.py:12-160) behind the
// kernel-plugin boundary (spmv/__init__.py:88-101).  Kernel family:
//
//  ROWBLOCK  persistent, nnz-balanced.  Entry chunk b = [base + b*cap,
//            base + (b+1)*cap) is streamed into shared memory by the TMA
//            bulk-copy engine (cp.async.bulk + mbarrier, `stages`-deep ring
//            per CTA, no register staging) — values and offsets are the
//            ~93% of the bytes and move as a pure memcpy.  The rows whose
//            first entry lies in the chunk (plan.block_rows) are reduced one
//            thread per row in the reference's exact order; the few entries
//            of a row that spill past the chunk are read from global.  Rows
//            longer than long_len are reduced by the whole CTA (exact:
//            products staged in smem, one thread sums in order, pipelined;
//            TREE: block tree).
//  STAGED    the same row engine with fixed rows per CTA and a one-shot bulk
//            copy; needs no plan (the reference-named entry points).
//  SCALAR    thread per row straight from global (exact orders).
//  VECTOR<G> G lanes per row, lane-strided partial sums, __shfl_xor tree.
//
// Column of entry i in row r: CSR colids[i]; DA r + colids[i] (the shifted
// base of PAPER.md Snippet 2); plus x_offset for rank-local halo buffers.

#include "spmv_kernels.cuh"

namespace dacsr {

// ------------------------------------------------------------- error state
namespace {
thread_local char g_last_error[256] = "";
}

void set_last_error(const char* what, cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%d)", what, cudaGetErrorString(e),
           static_cast<int>(e));
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error(what, e);
    return DACSR_ERR_CUDA;
  }
  return DACSR_OK;
}

}  // namespace dacsr

using namespace dacsr;

extern "C" {

const char* dacsr_version(void) { return "dacsr_b200 0.1.0 (sm_100a)"; }

const char* dacsr_last_error(void) { return g_last_error; }

int32_t dacsr_tiles_step_group(void) { return DACSR_TILED_G; }

int32_t dacsr_tiles_max_cols(int32_t values_dtype) {
  static const int kB[8] = {1, 2, 4, 8, 4, 8, 2, 2};
  if (values_dtype < DACSR_F32 || values_dtype > DACSR_BF16) return 0;
  const size_t vb = kB[values_dtype];
  const size_t budget = 227 * 1024;
  const size_t fixed = size_t(kTileWarps) * (kTileRows + 1) * 32 * 8 + 16 * kTileXBufs;
  if (budget <= fixed) return 0;
  // kTileXBufs x ((T + 16 / vb) * vb rounded up to 128 bytes) must fit
  const size_t per_buf = ((budget - fixed) / kTileXBufs) & ~size_t(127);
  int64_t t = static_cast<int64_t>(per_buf / vb) - static_cast<int64_t>(16 / vb);
  t &= ~int64_t(15);
  return static_cast<int32_t>(std::min<int64_t>(t, 65536));
}

// Selection by row statistics (measured per config):
//  * scattered gathers (random wide bands, C3/C5): TILED, x staged in smem;
//  * everything else with enough rows (stencils, RCM orders, skew: C1, C2,
//    C4): SLICED_PIPE on the sliced layout (medium / long rows handled
//    inside the launch);
//  * tiny matrices, and regular ones up to 8 M entries: SCALAR (no derived
//    layout worth building);
//  * the MACC3 / STRIP4 orders: ROWBLOCK (the layout kernels specialise
//    the naive order); long-row TREE: vector / warp kernels.
int32_t dacsr_select_variant(const dacsr_stats_t* st, int32_t order) {
  if (!st) return DACSR_VARIANT_STAGED;
  if (order == DACSR_ORDER_TREE && st->mean_len >= 48.0)
    return st->mean_len >= 256.0 ? DACSR_VARIANT_WARP : DACSR_VARIANT_VECTOR16;
  if (order == DACSR_ORDER_MACC3 || order == DACSR_ORDER_STRIP4) return DACSR_VARIANT_ROWBLOCK;
  if (st->rows < 4096) return DACSR_VARIANT_SCALAR;
  if (st->scatter > 0.5 && st->mean_len >= 2.0) return DACSR_VARIANT_TILED;
  // small regular operators (C1: 5 M entries, L2-resident once warm): the
  // thread-per-row kernel straight from the CSR arrays wins (9.2 against
  // 12.7 us warm, 18.8 against 20.5 cold) and needs no derived layout; from
  // C2's size on (14.6 M entries) the sliced layout is faster
  if (st->nnz <= (int64_t(8) << 20) && st->max_len <= 64 && st->cv_len <= 0.5)
    return DACSR_VARIANT_SCALAR;
  return DACSR_VARIANT_SLICED_PIPE;
}

int dacsr_plan_chunks(const dacsr_matrix_t* a, int64_t rs, int64_t re, int32_t chunk_rows,
                      int32_t vcap, int64_t* chunks_dev, void* count_scratch_dev,
                      dacsr_plan_t* inout, void* stream) {
  if (!a || !inout || !chunks_dev || !count_scratch_dev || rs < 0 || re < rs || re > a->nrows ||
      vcap < 64 || vcap > 16384 || (vcap & 15) || (chunk_rows != 32 && chunk_rows != 64))
    return DACSR_ERR_ARG;
  static const int kBytes[8] = {1, 2, 4, 8, 4, 8, 2, 2};
  if (a->values_dtype < 0 || a->values_dtype > 7 || a->colids_dtype < 0 || a->colids_dtype > 5)
    return DACSR_ERR_DTYPE;
  const int narrow = std::min(kBytes[a->values_dtype], kBytes[a->colids_dtype]);
  const int align = 16 / narrow;
  const int64_t last_aligned = a->nnz & ~static_cast<int64_t>(align - 1);
  auto st = static_cast<cudaStream_t>(stream);
  auto* count = static_cast<unsigned long long*>(count_scratch_dev);
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) {
    set_last_error("plan_chunks memset", e);
    return DACSR_ERR_CUDA;
  }
  const int64_t nchunks = (re - rs + chunk_rows - 1) / chunk_rows;
  if (nchunks > 0) {
    const int g = static_cast<int>(std::min<int64_t>((nchunks + 255) / 256, 148 * 32));
    if (a->rowptr_dtype == DACSR_I64)
      classify_chunks_kernel<int64_t><<<g, 256, 0, st>>>(static_cast<const int64_t*>(a->rowptr), rs, re,
                                                         chunk_rows, vcap, align, last_aligned,
                                                         chunks_dev, count);
    else if (a->rowptr_dtype == DACSR_I32)
      classify_chunks_kernel<int32_t><<<g, 256, 0, st>>>(static_cast<const int32_t*>(a->rowptr), rs, re,
                                                         chunk_rows, vcap, align, last_aligned,
                                                         chunks_dev, count);
    else
      return DACSR_ERR_DTYPE;
    int rc = check_launch("classify_chunks_kernel");
    if (rc) return rc;
  }
  unsigned long long h = 0;
  e = cudaMemcpyAsync(&h, count, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    set_last_error("plan_chunks count", e);
    return DACSR_ERR_CUDA;
  }
  inout->chunk_vcap = vcap;
  inout->chunk_rows = chunk_rows;
  inout->n_complex = static_cast<int64_t>(h);
  inout->complex_chunks = chunks_dev;
  return DACSR_OK;
}

int dacsr_spmv(const dacsr_matrix_t* a, const dacsr_plan_t* plan, int32_t variant, int32_t order,
               const void* x, int64_t x_offset, void* y, double alpha, double beta,
               int64_t row_start, int64_t row_end, void* stream) {
  if (!a || !y || row_start < 0 || row_end < row_start || row_end > a->nrows) return DACSR_ERR_ARG;
  if (row_end == row_start) return DACSR_OK;
  if (!a->rowptr || (a->nnz > 0 && (!a->colids || !a->values || !x))) return DACSR_ERR_ARG;
  if (order < DACSR_ORDER_NAIVE || order > DACSR_ORDER_TREE) return DACSR_ERR_VARIANT;
  if (variant == DACSR_VARIANT_AUTO) variant = plan ? DACSR_VARIANT_ROWBLOCK : DACSR_VARIANT_STAGED;
  Req q{plan, variant, order, x, x_offset, y, alpha, beta, row_start, row_end,
        static_cast<cudaStream_t>(stream)};
  switch (a->values_dtype) {
    case DACSR_F64: return launch_values_f64(a, q);
    case DACSR_F32: return launch_values_f32(a, q);
    case DACSR_F16: return launch_values_f16(a, q);
    case DACSR_BF16: return launch_values_bf16(a, q);
    default: return DACSR_ERR_DTYPE;
  }
}

int dacsr_spmv_dev_alpha(const dacsr_matrix_t* a, const dacsr_plan_t* plan, int32_t variant,
                         int32_t order, const void* x, int64_t x_offset, void* y,
                         const double* alpha_dev, double beta, int64_t row_start, int64_t row_end,
                         void* stream) {
  if (!a || !y || !alpha_dev || row_start < 0 || row_end < row_start || row_end > a->nrows)
    return DACSR_ERR_ARG;
  if (row_end == row_start) return DACSR_OK;
  if (!a->rowptr || (a->nnz > 0 && (!a->colids || !a->values || !x))) return DACSR_ERR_ARG;
  if (order < DACSR_ORDER_NAIVE || order > DACSR_ORDER_TREE) return DACSR_ERR_VARIANT;
  if (variant == DACSR_VARIANT_AUTO) variant = plan ? DACSR_VARIANT_ROWBLOCK : DACSR_VARIANT_STAGED;
  Req q{plan, variant, order, x, x_offset, y, 0.0, beta, row_start, row_end,
        static_cast<cudaStream_t>(stream), alpha_dev};
  switch (a->values_dtype) {
    case DACSR_F64: return launch_values_f64(a, q);
    case DACSR_F32: return launch_values_f32(a, q);
    case DACSR_F16: return launch_values_f16(a, q);
    case DACSR_BF16: return launch_values_bf16(a, q);
    default: return DACSR_ERR_DTYPE;
  }
}

int dacsr_spmv_dev_alpha_sumsq(const dacsr_matrix_t* a, const dacsr_plan_t* plan, int32_t variant,
                               int32_t order, const void* x, int64_t x_offset, void* y,
                               const double* alpha_dev, double beta, int64_t row_start,
                               int64_t row_end, double* group_sumsq, void* stream) {
  if (!a || !y || !alpha_dev || !group_sumsq || row_start < 0 || row_end < row_start ||
      row_end > a->nrows)
    return DACSR_ERR_ARG;
  if (row_end == row_start) return DACSR_OK;
  if (!a->rowptr || (a->nnz > 0 && (!a->colids || !a->values || !x))) return DACSR_ERR_ARG;
  if (variant != DACSR_VARIANT_TILED) return DACSR_ERR_VARIANT;
  if (order < DACSR_ORDER_NAIVE || order > DACSR_ORDER_TREE) return DACSR_ERR_VARIANT;
  Req q{plan, variant, order, x, x_offset, y, 0.0, beta, row_start, row_end,
        static_cast<cudaStream_t>(stream), alpha_dev, group_sumsq};
  switch (a->values_dtype) {
    case DACSR_F64: return launch_values_f64(a, q);
    case DACSR_F32: return launch_values_f32(a, q);
    case DACSR_F16: return launch_values_f16(a, q);
    case DACSR_BF16: return launch_values_bf16(a, q);
    default: return DACSR_ERR_DTYPE;
  }
}

// Host-buffer SpMV with the copies overlapped (see hostpath.py): rows are
// split into the plans' row ranges; piece p needs x[0, min(ncols, r1_p + w))
// (w = bandwidth).  h2d: the x prefix not yet sent; comp: waits for it, runs
// the piece.  y: when y_host is page-locked and mapped (any cudaHostAlloc /
// registered buffer under UVA) the kernels store y straight into host
// memory over PCIe — the D2H copy disappears and with it the pipeline drain
// (and with beta != 0 they read the old y from there too).  Otherwise y goes
// through y_dev: the y piece in on h2d if beta != 0, out on d2h after the
// piece's kernel.  Blocks until y_host is complete.
int dacsr_spmv_host_streamed(const dacsr_matrix_t* a, const dacsr_plan_t* plans, int32_t npieces,
                             int32_t variant, int32_t order, const void* x_host, void* y_host,
                             void* x_dev, void* y_dev, double alpha, double beta, int64_t w,
                             void* s_h2d, void* s_comp, void* s_d2h, int32_t y_through_device) {
  if (!a || !plans || npieces <= 0 || npieces > 64 || !x_host || !y_host || !x_dev || !y_dev ||
      w < 0)
    return DACSR_ERR_ARG;
  static const int kBytes[8] = {1, 2, 4, 8, 4, 8, 2, 2};
  if (a->values_dtype < DACSR_F32 || a->values_dtype > DACSR_BF16) return DACSR_ERR_DTYPE;
  const size_t vb = kBytes[a->values_dtype];
  auto h2d = static_cast<cudaStream_t>(s_h2d), comp = static_cast<cudaStream_t>(s_comp),
       d2h = static_cast<cudaStream_t>(s_d2h);
  // y straight to host memory?
  void* y_mapped = nullptr;
  {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, y_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer)
      y_mapped = pa.devicePointer;
    else
      cudaGetLastError();  // pageable memory: not an error, take the copy path
    if (y_through_device) y_mapped = nullptr;
  }
  cudaEvent_t ev[128];
  int nev = 0;
  auto fail = [&](const char* what, cudaError_t e) {
    set_last_error(what, e);
    for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
    return DACSR_ERR_CUDA;
  };
  for (int i = 0; i < 2 * npieces; ++i) {
    cudaError_t e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return fail("streamed event", e);
    ++nev;
  }
  const char* xh = static_cast<const char*>(x_host);
  char* yh = static_cast<char*>(y_host);
  char* xd = static_cast<char*>(x_dev);
  char* yd = static_cast<char*>(y_dev);
  void* y_target = y_mapped ? y_mapped : y_dev;
  int64_t sent = 0;
  cudaError_t e;
  for (int p = 0; p < npieces; ++p) {
    const int64_t r0 = plans[p].row_start, r1 = plans[p].row_end;
    const int64_t hi = std::min<int64_t>(a->ncols, r1 + w);
    if (hi > sent) {
      e = cudaMemcpyAsync(xd + sent * vb, xh + sent * vb, (hi - sent) * vb,
                          cudaMemcpyHostToDevice, h2d);
      if (e != cudaSuccess) return fail("streamed x copy", e);
      sent = hi;
    }
    if (!y_mapped && beta != 0.0 && r1 > r0) {
      e = cudaMemcpyAsync(yd + r0 * vb, yh + r0 * vb, (r1 - r0) * vb, cudaMemcpyHostToDevice, h2d);
      if (e != cudaSuccess) return fail("streamed y copy in", e);
    }
    if ((e = cudaEventRecord(ev[2 * p], h2d)) != cudaSuccess) return fail("event", e);
    if ((e = cudaStreamWaitEvent(comp, ev[2 * p], 0)) != cudaSuccess) return fail("wait", e);
    if (r1 > r0) {
      const int rc = dacsr_spmv(a, &plans[p], variant, order, x_dev, 0, y_target, alpha, beta, r0,
                                r1, s_comp);
      if (rc) {
        for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
        return rc;
      }
    }
    if (y_mapped) continue;
    if ((e = cudaEventRecord(ev[2 * p + 1], comp)) != cudaSuccess) return fail("event", e);
    if ((e = cudaStreamWaitEvent(d2h, ev[2 * p + 1], 0)) != cudaSuccess) return fail("wait", e);
    if (r1 > r0) {
      e = cudaMemcpyAsync(yh + r0 * vb, yd + r0 * vb, (r1 - r0) * vb, cudaMemcpyDeviceToHost, d2h);
      if (e != cudaSuccess) return fail("streamed y copy out", e);
    }
  }
  e = cudaStreamSynchronize(y_mapped ? comp : d2h);
  for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
  if (e != cudaSuccess) {
    set_last_error("streamed sync", e);
    return DACSR_ERR_CUDA;
  }
  return DACSR_OK;
}

// Reference-named kernels: the paper's layout (int32 rowptr; DA int16
// offsets, CSR int32 colids), the named order, STAGED engine (no plan).
#define DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, NAME, ORDER, VT, VCODE, VN)                 \
  int dacsr_##KIND##_##NAME##_##VN(const int32_t* rowptr, const CI* colids, const VT* values,   \
                                   const VT* x, VT* y, double alpha, double beta,               \
                                   int64_t row_start, int64_t row_end, void* stream) {          \
    dacsr_matrix_t a{KCODE, DACSR_I32, CICODE, VCODE, row_end, 0, 0, rowptr, colids, values};  \
    return dacsr_spmv(&a, nullptr, DACSR_VARIANT_STAGED, ORDER, x, 0, y, alpha, beta,           \
                      row_start, row_end, stream);                                              \
  }
#define DACSR_DEFINE_KIND(KIND, KCODE, CI, CICODE)                                                  \
  DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, naive, DACSR_ORDER_NAIVE, double, DACSR_F64, f64)     \
  DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, shifted_base, DACSR_ORDER_NAIVE, double, DACSR_F64, f64) \
  DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, multi_acc3, DACSR_ORDER_MACC3, double, DACSR_F64, f64) \
  DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, strip_mined4, DACSR_ORDER_STRIP4, double, DACSR_F64, f64) \
  DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, naive, DACSR_ORDER_NAIVE, float, DACSR_F32, f32)      \
  DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, shifted_base, DACSR_ORDER_NAIVE, float, DACSR_F32, f32) \
  DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, multi_acc3, DACSR_ORDER_MACC3, float, DACSR_F32, f32) \
  DACSR_DEFINE_TYPED(KIND, KCODE, CI, CICODE, strip_mined4, DACSR_ORDER_STRIP4, float, DACSR_F32, f32)
DACSR_DEFINE_KIND(csr, DACSR_KIND_CSR, int32_t, DACSR_I32)
DACSR_DEFINE_KIND(da, DACSR_KIND_DA, int16_t, DACSR_I16)

}  // extern "C"
