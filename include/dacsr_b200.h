/*
 * dacsr_b200.h — C ABI of the B200 (sm_100a) DA-CSR / CSR SpMV library.
 *
 * The drop-in boundary for the reference's kernel plugin interface
 * (/root/reference/pkg/src/dacsr/spmv/__init__.py:88-101 resolves
 * `getattr(module, f"{kind}_{suffix}")` and calls
 * `kernel(rowptr, colids, values, x, y, alpha, beta, row_start, row_end)`,
 * _numba_kernels.py:13).  Everything here is plain pointers and sizes; all
 * array pointers are DEVICE pointers, `stream` is a cudaStream_t (NULL =
 * legacy default stream).  Launches are stream-ordered and the library
 * holds no global mutable state, so calls on different streams/devices may
 * run concurrently.  Functions never allocate device memory: buffers (the
 * plan's block table) are caller-owned.
 *
 * Arithmetic contract (identical to the reference's numba kernels):
 * y[r] = alpha * acc_r (+ beta * y[r] iff beta != 0), acc_r accumulated in
 * float64 from +0.0, products rounded separately (no FMA contraction); for
 * float32 data the product is rounded to float32 before the float64
 * accumulation and the result rounded once on the store.  beta == 0 never
 * reads y.  With an exact order (NAIVE/MACC3/STRIP4) the result is
 * bit-identical to the reference kernel of the same summation order.
 */
#ifndef DACSR_B200_H
#define DACSR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (0 = success) ---------------------------------------- */
enum {
  DACSR_OK = 0,
  DACSR_ERR_ARG = 1,     /* null pointer / bad row range / bad size        */
  DACSR_ERR_DTYPE = 2,   /* unsupported dtype or kind combination          */
  DACSR_ERR_VARIANT = 3, /* unknown variant or order                       */
  DACSR_ERR_CUDA = 4,    /* CUDA runtime/launch error: dacsr_last_error()  */
  DACSR_ERR_PLAN = 5     /* plan does not match the matrix / row range     */
};

/* ---- dtype, kind, order, variant codes ---------------------------------- */
enum { DACSR_I8 = 0, DACSR_I16 = 1, DACSR_I32 = 2, DACSR_I64 = 3, DACSR_F32 = 4, DACSR_F64 = 5 };
/* 16-bit values (extension along model.py:21-74's width lattice; the
 * reference kernels stop at f32): values, x and y in binary16 / bfloat16,
 * products exact in f32, f64 accumulation in the selected order, one
 * rounding on the store. */
enum { DACSR_F16 = 6, DACSR_BF16 = 7 };
enum { DACSR_KIND_CSR = 0, DACSR_KIND_DA = 1 };

/* Summation order inside a row.  NAIVE/MACC3/STRIP4 reproduce the
 * reference kernels naive|shifted_base / multi_acc3 / strip_mined4
 * (_numba_kernels.py:12-160) bit-for-bit.  TREE allows a lane-parallel
 * tree combine (not bit-exact; within 2^-40 relative in tests). */
enum { DACSR_ORDER_NAIVE = 0, DACSR_ORDER_MACC3 = 1, DACSR_ORDER_STRIP4 = 2, DACSR_ORDER_TREE = 3 };

enum {
  DACSR_VARIANT_AUTO = 0,     /* pick from the plan's row statistics             */
  DACSR_VARIANT_ROWBLOCK = 1, /* nnz-balanced entry chunks, TMA-bulk staged,      */
                              /* persistent; thread-per-row (exact orders),       */
                              /* long rows cooperatively; needs a plan           */
  DACSR_VARIANT_SCALAR = 2,   /* thread per row straight from global (exact)     */
  DACSR_VARIANT_VECTOR2 = 3,  /* 2/4/8/16/32 lanes per row + __shfl_xor (TREE)   */
  DACSR_VARIANT_VECTOR4 = 4,
  DACSR_VARIANT_VECTOR8 = 5,
  DACSR_VARIANT_VECTOR16 = 6,
  DACSR_VARIANT_WARP = 7,
  DACSR_VARIANT_STAGED = 8,   /* fixed rows per CTA, TMA-bulk staged (no plan)   */
  DACSR_VARIANT_WSTREAM = 9,  /* warp streams: 32-row chunks per warp, TMA bulk  */
                              /* double-buffered per warp, exact naive order;    */
                              /* staging window from the plan (chunk_vcap)       */
  DACSR_VARIANT_SLICED = 10,  /* sliced layout (plan->slices): lane per row,     */
                              /* coalesced column-major entries straight from    */
                              /* HBM, exact naive order; spill rows by side warps*/
  /* 11, 12, 13: retired round-1 sliced modes (TMA-staged, warp-specialised
   * ring, offset-predicted): exact but slower on every BASELINE config;
   * the codes now return DACSR_ERR_VARIANT */
  DACSR_VARIANT_SLICED_PIPE = 14, /* SLICED with the next slice's offsets loaded */
                              /* while this slice's gathers are in flight       */
  DACSR_VARIANT_TILED = 15    /* band-tiled layout (plan->tiles): x staged in    */
                              /* shared memory tile by tile (TMA bulk copies),  */
                              /* lane per 16 rows, exact naive order; for wide  */
                              /* random bands (C3, C5)                          */
};

/* A matrix in CSR (absolute colids) or DA-CSR (colids = col - row) layout.
 * rowptr: I32|I64, colids: CSR I32|I64, DA I8|I16|I32; values: F32|F64. */
typedef struct {
  int32_t kind;
  int32_t rowptr_dtype;
  int32_t colids_dtype;
  int32_t values_dtype;
  int64_t nrows;
  int64_t ncols;
  int64_t nnz;
  const void* rowptr;
  const void* colids;
  const void* values;
} dacsr_matrix_t;

/* Sliced device layout of rows [row_start, row_end) — a derived copy of the
 * entries in HBM (the CSR/DA-CSR arrays stay the reference layout).
 *
 * Main slices: slice s holds rows row_start + 32s + lane (lane 0..31);
 * entry j of that row sits at slot slice_ptr[s] + 32*j + lane of `inner` /
 * `values`, so the 32 lanes of a warp read entry j of their rows as one
 * contiguous 32-element run.  Width W_s = (slice_ptr[s+1] - slice_ptr[s]) /
 * 32 = the longest row of the slice with at most max_len entries; shorter
 * rows are zero-padded (never read), longer rows are not in main slices.
 *
 * Medium rows (max_len < len <= medium_len) are listed ascending in
 * medium_rows and packed 32 per "medium slice" the same way (lane l of
 * medium slice m = row medium_rows[32m + l]; slots in m_slice_ptr /
 * m_inner / m_values).  Long rows (len > medium_len) are listed ascending
 * in long_rows and reduced by a whole warp from the CSR arrays.
 *
 * row_len[r - row_start] = entries of row r, or 255 if the row has more
 * than 254.  max_len <= medium_len <= 254.  All buffers are device memory
 * owned by the caller; entries are bit-for-bit copies, in row order. */
typedef struct {
  int64_t row_start;
  int64_t row_end;
  int64_t nslices;          /* ceil((row_end - row_start) / 32)              */
  int64_t total;            /* main slots = slice_ptr[nslices]               */
  int32_t max_len;          /* main-slice rows: len <= max_len               */
  int32_t medium_len;       /* medium rows: max_len < len <= medium_len      */
  const int64_t* slice_ptr; /* nslices + 1                                   */
  const uint8_t* row_len;   /* row_end - row_start                           */
  const void* inner;        /* total, the matrix's colids dtype              */
  const void* values;       /* total, the matrix's values dtype              */
  int64_t n_medium;
  int64_t m_nslices;        /* ceil(n_medium / 32)                           */
  int64_t m_total;          /* m_slice_ptr[m_nslices]                        */
  const int64_t* medium_rows; /* n_medium, ascending                         */
  const int64_t* m_slice_ptr; /* m_nslices + 1                               */
  const void* m_inner;
  const void* m_values;
  int64_t n_long;
  const int64_t* long_rows; /* n_long, ascending                             */
} dacsr_slices_t;

/* Band-tiled device layout of rows [row_start, row_end) (TILED kernel) — a
 * derived copy of the entries for matrices whose rows spread over a wide
 * band (x gathers would miss L1 one sector per entry).
 *
 * Rows come in groups of 512 (row slot s = 32j + l, j = 0..15, l = 0..31:
 * row row_start + 512g + s).  Columns come in tiles of tile_cols: tile t =
 * [col0 + t*tile_cols, col0 + (t+1)*tile_cols).  Group g spans tiles
 * tile_lo[g] .. tile_lo[g] + (cnt_ptr[g+1] - cnt_ptr[g]) - 1; its k-th tile
 * is block b = cnt_ptr[g] + k.  In block b lane l folds, for j = 0..15, row
 * slot 32j + (l ^ m_j), m_j = nibble j of masks[b] (a per-tile lane remap
 * that evens out the lanes' list lengths), in the order order[b * 32 + l]
 * gives: nibble k = the row slot j of its k-th row (an order chosen to
 * spread the shared-memory banks); nibble k of counts[b * 32 + l] = the
 * entries of that row whose column falls in the tile (1..15; rows without
 * entries in the tile are not listed, their nibbles 0).
 * The group's entries start at ent_ptr[g], tile after tile.  Inside a tile,
 * lane l's entries (its rows in that order, each row's entries in
 * column order) form a list L_l, stored in steps of G = step_group
 * entries: entries Gq .. Gq+G-1 of L_l sit at tile_base + G * (sum_{q' < q}
 * |{l' : |L_l'| > Gq'}| + |{l' < l : |L_l'| > Gq}|) (a list whose length
 * is not a multiple of G ends in zero slots), so the lanes of a warp read
 * step q of their lists as one packed run of G-entry vectors.  Every tile
 * segment is a multiple of G long.  Entries are bit-for-bit copies; every row's entries keep
 * their order, so a lane folding its list in order reproduces the naive
 * sum.
 * Rows with more than 15 entries inside one tile are left out (counts 0,
 * bit j of skip[32g + l] set) and listed ascending in ovf_rows; the kernel
 * reduces them warp by warp from the CSR arrays.  inner / values carry 16
 * padding entries past `total` (bulk L2 prefetches may round up). */
typedef struct {
  int64_t row_start;
  int64_t row_end;
  int64_t ngroups;          /* ceil((row_end - row_start) / 512)            */
  int64_t col0;             /* first column of tile 0 (= cmin)              */
  int64_t cmax;             /* last column any entry uses                   */
  int32_t tile_cols;        /* columns per tile (x tile = tile_cols values) */
  int32_t step_group;       /* entries per lane per packed step: 2 or 4     */
  int64_t total;            /* slots in the layout (entries + padding)      */
  int64_t nblocks;          /* cnt_ptr[ngroups]                             */
  const int64_t* ent_ptr;   /* ngroups + 1                                  */
  const int64_t* cnt_ptr;   /* ngroups + 1                                  */
  const int32_t* tile_lo;   /* ngroups                                      */
  const uint64_t* counts;   /* nblocks * 32                                 */
  const uint16_t* skip;     /* ngroups * 32                                 */
  const void* inner;        /* total + 16, the matrix's colids dtype        */
  const void* values;       /* total + 16, the matrix's values dtype        */
  int64_t n_ovf;
  const int64_t* ovf_rows;  /* n_ovf, ascending                             */
  const uint64_t* masks;    /* nblocks: lane remap nibbles of each block     */
  const uint64_t* order;    /* nblocks * 32: row order nibbles               */
} dacsr_tiles_t;

/* dacsr_plan_t.flags: the SLICED kernels skip the L2 bulk prefetch of the
 * slice two steps ahead (measured per matrix by DeviceMatrix.autotune). */
enum { DACSR_PLAN_NO_L2_PREFETCH = 1 };

/* Row-length statistics of rows [row_start, row_end). */
typedef struct {
  int64_t rows;
  int64_t nnz;
  int64_t entry_start; /* rowptr[row_start] */
  int64_t entry_end;   /* rowptr[row_end]   */
  int64_t max_len;
  int64_t empty_rows;
  double mean_len;
  double cv_len; /* coefficient of variation of row lengths */
  /* gather locality: fraction of sampled adjacent row pairs whose middle
   * entries' columns are more than 16 apart (beyond the diagonal step) —
   * near 1 for random bands (C3, C5), near 0 for stencils / RCM orders */
  double scatter;
} dacsr_stats_t;

/* nnz-balanced partition: block b stages entries
 * [entry_base + b*cap, entry_base + (b+1)*cap) and owns the rows whose first
 * entry falls there (rows [block_rows[b], block_rows[b+1])). */
typedef struct {
  int64_t row_start;
  int64_t row_end;
  int64_t entry_base;  /* rowptr[row_start] rounded down to 16 entries       */
  int64_t entry_end;   /* rowptr[row_end]                                     */
  int64_t nblocks;
  int32_t cap;         /* entries per block (multiple of 16)                  */
  int32_t long_len;    /* rows longer than this are reduced by the whole CTA  */
  const int64_t* block_rows; /* device, nblocks + 1 entries (caller-owned)    */
  /* WSTREAM: 32-row chunks whose entries do not fit the staging window are
   * listed here and reduced by a side kernel (dacsr_plan_chunks).           */
  int32_t chunk_vcap;  /* staging window (entries, multiple of 16), 0 = none  */
  int32_t chunk_rows;  /* rows per warp chunk: 32 (1 per lane) or 64 (2)     */
  int64_t n_complex;
  const int64_t* complex_chunks; /* device, n_complex chunk indices          */
  int32_t ctas_per_sm; /* WSTREAM/SLICED resident CTAs per SM (0 = max)      */
  int32_t flags;       /* DACSR_PLAN_* bits                                  */
  /* SLICED: the layout (its row range must contain the launch's rows).     */
  const dacsr_slices_t* slices;
  /* TILED: the layout (its row range must contain the launch's rows).      */
  const dacsr_tiles_t* tiles;
} dacsr_plan_t;

const char* dacsr_version(void);
/* Text of the last CUDA error seen by this thread ("" if none). */
const char* dacsr_last_error(void);

/* Row statistics (reads rowptr on the device; synchronizes `stream`).
 * scratch_dev: caller-owned device buffer of DACSR_ANALYZE_SCRATCH bytes. */
#define DACSR_ANALYZE_SCRATCH 64
int dacsr_analyze(const dacsr_matrix_t* a, int64_t row_start, int64_t row_end,
                  void* scratch_dev, dacsr_stats_t* out, void* stream);

/* Default block capacity for a matrix with these statistics. */
int32_t dacsr_plan_default_cap(const dacsr_stats_t* stats, int32_t values_dtype,
                               int32_t colids_dtype);
/* Number of blocks a plan of capacity `cap` needs (size block_rows as +1). */
int64_t dacsr_plan_nblocks(const dacsr_matrix_t* a, int64_t entry_start, int64_t entry_end,
                           int32_t cap);
/* Fill `block_rows_dev` (nblocks + 1 int64) and `out`.  entry_start/end are
 * rowptr[row_start], rowptr[row_end] (known to the caller from analyze). */
int dacsr_plan_build(const dacsr_matrix_t* a, int64_t row_start, int64_t row_end,
                     int64_t entry_start, int64_t entry_end, int32_t cap, int32_t long_len,
                     int64_t* block_rows_dev, dacsr_plan_t* out, void* stream);

/* Classify the chunk_rows-row chunks (32 or 64) of [row_start, row_end)
 * for a WSTREAM window of `vcap` entries (multiple of 16, 64..16384): chunks
 * that do not fit go to chunks_dev (capacity ceil(rows/chunk_rows) int64);
 * count_scratch_dev is 8 device bytes.  Fills
 * inout->chunk_vcap / n_complex / complex_chunks; synchronizes `stream`. */
int dacsr_plan_chunks(const dacsr_matrix_t* a, int64_t row_start, int64_t row_end,
                      int32_t chunk_rows, int32_t vcap, int64_t* chunks_dev,
                      void* count_scratch_dev, dacsr_plan_t* inout, void* stream);

/* Sliced layout builder (warp per slice; scans with dacsr_counts_to_rowptr
 * into int64 between the passes; the caller sizes the buffers from the
 * scanned totals).
 * 1. dacsr_slices_count: row_len_dev[r - row_start]; per main slice
 *    slot_counts[s] = 32 * W_s, medium_counts[s], long_counts[s] (int32).
 * 2. dacsr_slices_fill: s->inner / s->values (padding zeroed), the medium
 *    and long row lists (medium_ptr / long_ptr: the scanned counts).
 * 3. dacsr_slices_medium_count: m_slot_counts[m] = 32 * width of medium
 *    slice m (needs s->medium_rows, s->row_len).
 * 4. dacsr_slices_medium_fill: s->m_inner / s->m_values.
 * 1 <= max_len <= medium_len <= 254. */
int dacsr_slices_count(const dacsr_matrix_t* a, int64_t row_start, int64_t row_end,
                       int32_t max_len, int32_t medium_len, uint8_t* row_len_dev,
                       int32_t* slot_counts_dev, int32_t* medium_counts_dev,
                       int32_t* long_counts_dev, void* stream);
int dacsr_slices_fill(const dacsr_matrix_t* a, const dacsr_slices_t* s,
                      const int64_t* medium_ptr_dev, const int64_t* long_ptr_dev, void* stream);
int dacsr_slices_medium_count(const dacsr_slices_t* s, int32_t* m_slot_counts_dev, void* stream);
int dacsr_slices_medium_fill(const dacsr_matrix_t* a, const dacsr_slices_t* s, void* stream);

/* Band-tiled layout builder (warp per 512-row group; the caller scans the
 * per-group counts into int64 prefixes between the passes and sizes the
 * buffers from the totals).
 * 1. dacsr_tiles_extent: out2_dev[0] = min column, out2_dev[1] = max column
 *    of the entries of rows [row_start, row_end) (INT64_MAX / INT64_MIN if
 *    none); stream-ordered.
 * 2. dacsr_tiles_count (t->row_start/row_end/ngroups/col0/tile_cols set):
 *    per group nt_counts[g] = tiles spanned, ent_counts[g] = entries kept,
 *    ovf_counts[g] = rows left out; t->tile_lo and t->skip filled.
 * 3. dacsr_tiles_fill (every t field set; ovf_ptr = scanned ovf_counts):
 *    counts, inner, values, ovf_rows.
 * 64 <= tile_cols <= 65536, a multiple of 16; the TILED kernel keeps its x
 * tiles in shared memory, so tile_cols <= dacsr_tiles_max_cols(values dtype)
 * (DACSR_ERR_PLAN otherwise). */
int dacsr_tiles_extent(const dacsr_matrix_t* a, int64_t row_start, int64_t row_end,
                       int64_t* out2_dev, void* stream);
int dacsr_tiles_count(const dacsr_matrix_t* a, const dacsr_tiles_t* t, int32_t* nt_counts_dev,
                      int32_t* ent_counts_dev, int32_t* ovf_counts_dev, void* stream);
int dacsr_tiles_fill(const dacsr_matrix_t* a, const dacsr_tiles_t* t, const int64_t* ovf_ptr_dev,
                     void* stream);
/* The step_group the TILED kernel of this build reads (layouts must match). */
int32_t dacsr_tiles_step_group(void);
/* Widest tile_cols whose x ring fits the TILED kernel's shared memory for
 * this value type (DeviceMatrix.build_tiles' default: fewer, larger tiles
 * cost less per entry). */
int32_t dacsr_tiles_max_cols(int32_t values_dtype);

/* Variant the library would run for DACSR_VARIANT_AUTO. */
int32_t dacsr_select_variant(const dacsr_stats_t* stats, int32_t order);

/* y[r] = alpha * sum_i values[i] * x[col_i + x_offset] (+ beta*y[r]) for
 * r in [row_start, row_end), col_i = colids[i] (CSR) or r + colids[i] (DA).
 * `plan` may be NULL except for DACSR_VARIANT_ROWBLOCK (AUTO falls back to
 * STAGED without a plan).  x_offset shifts x addressing (a rank-local halo
 * buffer); 0 for a plain SpMV. */
int dacsr_spmv(const dacsr_matrix_t* a, const dacsr_plan_t* plan, int32_t variant,
               int32_t order, const void* x, int64_t x_offset, void* y, double alpha,
               double beta, int64_t row_start, int64_t row_end, void* stream);

/* dacsr_spmv with alpha read from DEVICE memory by the kernel (at the
 * epilogue, after the previous grid on the stream completed): iterative
 * methods whose alpha comes from a device reduction (the power iteration's
 * 1 / ||y||) run without host round trips and can be graph-captured.  There
 * is no alpha == 0 short-cut here (the kernel always runs). */
int dacsr_spmv_dev_alpha(const dacsr_matrix_t* a, const dacsr_plan_t* plan, int32_t variant,
                         int32_t order, const void* x, int64_t x_offset, void* y,
                         const double* alpha_dev, double beta, int64_t row_start, int64_t row_end,
                         void* stream);

/* dacsr_spmv_dev_alpha on the TILED kernel that also returns ||y||^2 by
 * 512-row groups: group_sumsq[r / 512] = the sum of y[r]^2 (y as stored)
 * over the group's rows in the fixed group tree of dacsr_sumsq_chunks — the
 * power iteration's norm without a second pass over y.  Needs whole groups:
 * the layout's row_start, row_start and row_end (unless the layout's end)
 * multiples of 512, no rows left out of the layout, the naive order;
 * DACSR_ERR_PLAN / DACSR_ERR_VARIANT otherwise (run dacsr_sumsq_chunks
 * then).  dacsr_sumsq_from_groups folds the group sums into chunk partials
 * (chunk a multiple of 512) identical to dacsr_sumsq_chunks'. */
int dacsr_spmv_dev_alpha_sumsq(const dacsr_matrix_t* a, const dacsr_plan_t* plan, int32_t variant,
                               int32_t order, const void* x, int64_t x_offset, void* y,
                               const double* alpha_dev, double beta, int64_t row_start,
                               int64_t row_end, double* group_sumsq_dev, void* stream);
int dacsr_sumsq_from_groups(const double* group_sumsq_dev, int64_t n, int64_t chunk,
                            double* partial_dev, void* stream);

/* spmv with HOST x / y, copies overlapped with the kernels: rows split into
 * the row ranges of plans[0..npieces) (ascending, covering the rows); piece
 * p needs x[0, min(ncols, row_end_p + w)) with w the bandwidth (max |col -
 * row|).  x_dev / y_dev are caller-owned device buffers of ncols / nrows
 * values; s_h2d carries the x copies, s_comp the kernels.  If y_host is
 * page-locked and mapped (cudaHostAlloc / cudaHostRegister under UVA) the
 * kernels store y straight into it over PCIe and y_dev / s_d2h are unused;
 * otherwise (or with y_through_device != 0: the copy engine moves large
 * pieces a few per cent faster than the kernels' stores over the link) y
 * returns through y_dev with D2H copies on s_d2h.  Blocks until y_host is
 * complete. */
int dacsr_spmv_host_streamed(const dacsr_matrix_t* a, const dacsr_plan_t* plans, int32_t npieces,
                             int32_t variant, int32_t order, const void* x_host, void* y_host,
                             void* x_dev, void* y_dev, double alpha, double beta, int64_t w,
                             void* s_h2d, void* s_comp, void* s_d2h, int32_t y_through_device);

/* The reference's alpha == 0 short-cut (spmv/__init__.py:150-156):
 * y = 0 if beta == 0, y = (T)((double)beta * y) if beta not in {0, 1}. */
int dacsr_scale(void* y, int32_t values_dtype, int64_t n, double beta, void* stream);

/* Deterministic sum of squares: partial[c] = sum over rows [c*chunk,
 * (c+1)*chunk) ∩ [0, n) of y^2 in a fixed tree, independent of how rows are
 * spread over ranks when rank boundaries are chunk-aligned.  The tree: the
 * chunk is cut into groups of 512 values from its start; in a group lane l
 * (0..31) folds y[32j + l]^2 for j = 0..15 in order, a 5-step xor butterfly
 * (offsets 16, 8, 4, 2, 1) over the lanes gives the group's sum, and the
 * groups' sums are folded left to right. */
int dacsr_sumsq_chunks(const void* y, int32_t values_dtype, int64_t n, int64_t chunk,
                       double* partial, void* stream);
/* out[0] = sum of partial[0..m) in index order (one thread, exact order). */
int dacsr_sum_ordered(const double* partial, int64_t m, double* out, void* stream);
/* Power-iteration norm on the device: s = sqrt(sum of partial[0..m) in index
 * order), *norm_out = s (if norm_out), *alpha_out = 1 / s (IEEE sqrt and
 * division, round to nearest: Python's math.sqrt and 1.0 / s). */
int dacsr_norm_alpha(const double* partial, int64_t m, double* norm_out, double* alpha_out,
                     void* stream);
/* y = (T)(*beta_dev * (double)y) for f64 / f32 y, beta read from device memory. */
int dacsr_scale_dev(void* y, int32_t values_dtype, int64_t n, const double* beta_dev,
                    void* stream);

/* Reference-named kernel entry points (one per _numba_kernels.py function;
 * int32 rowptr, DA int16 offsets / CSR int32 colids, the paper's layout).
 * Exact order of the named reference kernel; no plan needed. */
#define DACSR_DECLARE_TYPED(KIND, CI, NAME, VT, VN)                                       \
  int dacsr_##KIND##_##NAME##_##VN(const int32_t* rowptr, const CI* colids,               \
                                   const VT* values, const VT* x, VT* y, double alpha,    \
                                   double beta, int64_t row_start, int64_t row_end,       \
                                   void* stream);
#define DACSR_DECLARE_KIND(KIND, CI)                          \
  DACSR_DECLARE_TYPED(KIND, CI, naive, double, f64)           \
  DACSR_DECLARE_TYPED(KIND, CI, shifted_base, double, f64)    \
  DACSR_DECLARE_TYPED(KIND, CI, multi_acc3, double, f64)      \
  DACSR_DECLARE_TYPED(KIND, CI, strip_mined4, double, f64)    \
  DACSR_DECLARE_TYPED(KIND, CI, naive, float, f32)            \
  DACSR_DECLARE_TYPED(KIND, CI, shifted_base, float, f32)     \
  DACSR_DECLARE_TYPED(KIND, CI, multi_acc3, float, f32)       \
  DACSR_DECLARE_TYPED(KIND, CI, strip_mined4, float, f32)
DACSR_DECLARE_KIND(csr, int32_t)
DACSR_DECLARE_KIND(da, int16_t)

/* ---- device-side conversion (reference core.py:320-355) ------------------ */
/* max |col - row| over the entries of a CSR or DA-CSR matrix into the
 * device int64 *out_dev (0 if empty); stream-ordered, no synchronization. */
int dacsr_bandwidth(const dacsr_matrix_t* a, int64_t* out_dev, void* stream);
/* offsets[i] = colids[i] - row(i) into an int8/int16/int32 array; caller
 * checks the bandwidth first (BandwidthExceedsIndexRange is host logic). */
int dacsr_csr_to_da(const dacsr_matrix_t* a, void* offsets, int32_t offsets_dtype,
                    void* stream);

/* ---- seeded C3/C5 generator (oracle: oracle/gen_oracle.c) ----------------- */
/* counts[r - r0] = entries of row r (diagonal included).  1 <= kmax <= 64
 * and kmax - 1 <= 2b (a row draws up to kmax - 1 distinct non-zero offsets
 * from [-b, b]); DACSR_ERR_ARG otherwise. */
int dacsr_gen_banded_counts(int64_t n, int64_t b, int32_t kmax, uint64_t seed,
                            const double* cdf_dev, int64_t r0, int64_t r1, int32_t* counts,
                            void* stream);
/* Fill rows [r0, r1) given their (local, from 0) rowptr; DA offsets and/or
 * CSR colids (either may be NULL), f64 or f32 values. */
int dacsr_gen_banded_fill(int64_t n, int64_t b, int32_t kmax, uint64_t seed,
                          const double* cdf_dev, const double* table_dev, int64_t r0,
                          int64_t r1, const void* rowptr, int32_t rowptr_dtype,
                          int16_t* offsets, int32_t* colids, void* values,
                          int32_t values_dtype, void* stream);
/* out[i - i0] = N(H(seed, i, 0)) for i in [i0, i1). */
int dacsr_gen_normal(uint64_t seed, int64_t i0, int64_t i1, const double* table_dev,
                     void* out, int32_t values_dtype, void* stream);
/* Inclusive-exclusive scan helper: rowptr[0] = 0, rowptr[k+1] = sum counts[0..k]
 * into int32 or int64 (uses a caller-provided temp buffer of temp_bytes;
 * query with temp == NULL). */
int dacsr_counts_to_rowptr(const int32_t* counts, int64_t m, void* rowptr,
                           int32_t rowptr_dtype, void* temp, size_t* temp_bytes,
                           void* stream);

/* ---- measurement ---------------------------------------------------------- */
/* Read-stream probe: warps stream `bytes` of `buf` into shared memory with
 * TMA bulk copies of `chunk` bytes (two slots per warp, 8 warps per CTA,
 * `ctas` CTAs) — the WSTREAM data path without compute.  `sink` is a device
 * double that is never written in practice. */
int dacsr_stream_probe(const void* buf, int64_t bytes, int32_t chunk, int32_t ctas, double* sink,
                       void* stream);

/* ---- host-side reordering (reference reorder.py:70-220), CPU only -------- */
/* Symmetrized adjacency of a square CSR pattern (pattern of A + A^T, no
 * self-loops, ascending, deduplicated).  Two calls: first with
 * indices == NULL to get indptr and the count; then with indices. */
int dacsr_host_adjacency(int64_t n, const int64_t* rowptr, const int64_t* colids,
                         int64_t* indptr, int64_t* indices);
/* Reverse Cuthill–McKee with the reference's tie-breaking; perm[new] = old. */
int dacsr_host_rcm(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t* perm);
/* P A P^T in canonical CSR: rows/cols relabelled through inv (old -> new),
 * values carried as raw bytes of width value_bytes; out arrays int64. */
int dacsr_host_permute(int64_t n, const int64_t* rowptr, const int64_t* colids,
                       const void* values, int32_t value_bytes, const int64_t* perm,
                       int64_t* out_rowptr, int64_t* out_colids, void* out_values);

#ifdef __cplusplus
}
#endif

#endif /* DACSR_B200_H */
