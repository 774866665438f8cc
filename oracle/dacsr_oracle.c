/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the DA-CSR SpMV hot path.
 *
 * A plain-C restatement of the reference's CPU algorithm, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * as the CHECKER and the timed CPU baseline.  The product path
 * (paper_2307_06305_b200/) never links or calls this file.
 *
 * Restated reference functions (/root/reference/pkg/src/dacsr/...):
 *   spmv/_numba_kernels.py:12-21    csr_naive      (csr_shifted_base alias :26)
 *   spmv/_numba_kernels.py:29-51    csr_multi_acc3
 *   spmv/_numba_kernels.py:54-79    csr_strip_mined4
 *   spmv/_numba_kernels.py:82-91    da_naive
 *   spmv/_numba_kernels.py:94-107   da_shifted_base  (same arithmetic as naive)
 *   spmv/_numba_kernels.py:110-132  da_multi_acc3
 *   spmv/_numba_kernels.py:135-160  da_strip_mined4
 *   spmv/__init__.py:71-85          row_blocks
 *   spmv/__init__.py:158-179        ParallelRowBlock dispatch (one thread/block)
 *   reorder.py:100-197              rcm (_level_structure, _min_degree_node,
 *                                   _pseudo_peripheral, CM BFS, reversal)
 *
 * Floating-point contract (numba default, no fastmath; verified against the
 * reference by tests/golden/): products and sums rounded separately (this
 * file MUST be compiled with -ffp-contract=off), accumulation from +0.0 in
 * float64; for float32 data the product is rounded to float32 and then
 * accumulated in float64; the epilogue alpha*acc (+ beta*y) is float64 with a
 * single rounding on the store.
 *
 * Pinned by tests/test_oracle.py against the fixtures in tests/golden, which the
 * reference itself generated (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_I8 = 0, ORC_I16 = 1, ORC_I32 = 2, ORC_I64 = 3, ORC_F32 = 4, ORC_F64 = 5, ORC_F16 = 6, ORC_BF16 = 7 };
enum { ORC_NAIVE = 0, ORC_MACC3 = 1, ORC_STRIP4 = 2 };
enum { ORC_CSR = 0, ORC_DA = 1 };

/* ------------------------------------------------------------------ SpMV */

#define COLUMN_CSR(r, c) ((int64_t)(c))
#define COLUMN_DA(r, c) ((int64_t)(r) + (int64_t)(c))

/* Per value type: storage type T, product P (as the double that is summed),
 * load-to-double L, store-with-one-rounding S.
 *   f64: product rounded in f64;  f32: product rounded to f32, widened
 *   (numba: f32*f32 -> f32, acc float64);  f16/bf16 (extension, no reference
 *   kernel): the f32 product of two 16-bit significands is exact, the sum is
 *   f64 in the same order, one rounding to 16 bits on the store. */
static float h16_to_f32(uint16_t h) {
  const int e = (h >> 10) & 31, m = h & 1023;
  float v;
  if (e == 0) v = ldexpf((float)m, -24);
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = ldexpf((float)(1024 + m), e - 25);
  return (h & 0x8000) ? -v : v;
}
static float b16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float v;
  memcpy(&v, &u, 4);
  return v;
}
/* round a double to a 16-bit binary format with p significand bits (incl.
 * the hidden one), exponent range [emin, emax] and bias ebias: round to
 * nearest even, directly from the double (no f32 detour) */
static uint16_t round_bits(double d, int p, int emin, int ebias, int emax) {
  const uint16_t sign = signbit(d) ? 0x8000 : 0;
  const int mbits = p - 1;
  if (isnan(d)) return sign | (uint16_t)(((2 * ebias + 1) << mbits) | (1 << (mbits - 1)));
  const double a = fabs(d);
  if (a == 0.0) return sign;
  if (isinf(a)) return sign | (uint16_t)((2 * ebias + 1) << mbits);
  int e2;
  frexp(a, &e2);
  int E = e2 - 1; /* a in [2^E, 2^(E+1)) */
  if (E < emin) E = emin;
  double q = rint(ldexp(a, mbits - E)); /* significand in units of 2^(E-mbits) */
  if (q >= ldexp(1.0, p)) { q = ldexp(q, -1); E += 1; } /* q == 2^p exactly: renormalise */
  if (E > emax) return sign | (uint16_t)((2 * ebias + 1) << mbits); /* inf */
  const uint32_t qi = (uint32_t)q;
  if (qi < (1u << mbits)) return sign | (uint16_t)qi; /* subnormal (E == emin) */
  return sign | (uint16_t)(((uint32_t)(E + ebias) << mbits) | (qi - (1u << mbits)));
}
static uint16_t f64_to_h16(double d) { return round_bits(d, 11, -14, 15, 15); }
static uint16_t f64_to_b16(double d) { return round_bits(d, 8, -126, 127, 127); }

#define f64_T double
#define f64_P(V, X) ((V) * (X))
#define f64_L(Y) ((double)(Y))
#define f64_S(D) (D)
#define f32_T float
#define f32_P(V, X) ((double)((V) * (X)))
#define f32_L(Y) ((double)(Y))
#define f32_S(D) ((float)(D))
#define f16_T uint16_t
#define f16_P(V, X) ((double)(h16_to_f32(V) * h16_to_f32(X)))
#define f16_L(Y) ((double)h16_to_f32(Y))
#define f16_S(D) f64_to_h16(D)
#define bf16_T uint16_t
#define bf16_P(V, X) ((double)(b16_to_f32(V) * b16_to_f32(X)))
#define bf16_L(Y) ((double)b16_to_f32(Y))
#define bf16_S(D) f64_to_b16(D)

#define EPI(VN, r, acc) \
  y[r] = VN##_S(beta == 0.0 ? alpha * (acc) : alpha * (acc) + beta * VN##_L(y[r]))

#define DEFINE_ROWS(NAME, RP, CI, VN, COLUMN)                                          \
  static void NAME##_naive(const RP* rp, const CI* ci, const VN##_T* v,                \
                           const VN##_T* x, VN##_T* y, double alpha, double beta,      \
                           int64_t rs, int64_t re) {                                   \
    for (int64_t r = rs; r < re; ++r) {                                                \
      double acc = 0.0;                                                                \
      for (int64_t i = (int64_t)rp[r]; i < (int64_t)rp[r + 1]; ++i)                    \
        acc += VN##_P(v[i], x[COLUMN(r, ci[i])]);                                      \
      EPI(VN, r, acc);                                                                 \
    }                                                                                  \
  }                                                                                    \
  static void NAME##_macc3(const RP* rp, const CI* ci, const VN##_T* v,                \
                           const VN##_T* x, VN##_T* y, double alpha, double beta,      \
                           int64_t rs, int64_t re) {                                   \
    for (int64_t r = rs; r < re; ++r) {                                                \
      int64_t i = (int64_t)rp[r], e = (int64_t)rp[r + 1];                              \
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;                                             \
      for (; i + 3 <= e; i += 3) {                                                     \
        a0 += VN##_P(v[i], x[COLUMN(r, ci[i])]);                                       \
        a1 += VN##_P(v[i + 1], x[COLUMN(r, ci[i + 1])]);                               \
        a2 += VN##_P(v[i + 2], x[COLUMN(r, ci[i + 2])]);                               \
      }                                                                                \
      if (i < e) a0 += VN##_P(v[i], x[COLUMN(r, ci[i])]);                              \
      if (i + 1 < e) a1 += VN##_P(v[i + 1], x[COLUMN(r, ci[i + 1])]);                  \
      double acc = (a0 + a1) + a2;                                                     \
      EPI(VN, r, acc);                                                                 \
    }                                                                                  \
  }                                                                                    \
  static void NAME##_strip4(const RP* rp, const CI* ci, const VN##_T* v,               \
                            const VN##_T* x, VN##_T* y, double alpha, double beta,     \
                            int64_t rs, int64_t re) {                                  \
    for (int64_t r = rs; r < re; ++r) {                                                \
      int64_t i = (int64_t)rp[r], e = (int64_t)rp[r + 1];                              \
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;                                   \
      for (; i + 4 <= e; i += 4) {                                                     \
        a0 += VN##_P(v[i], x[COLUMN(r, ci[i])]);                                       \
        a1 += VN##_P(v[i + 1], x[COLUMN(r, ci[i + 1])]);                               \
        a2 += VN##_P(v[i + 2], x[COLUMN(r, ci[i + 2])]);                               \
        a3 += VN##_P(v[i + 3], x[COLUMN(r, ci[i + 3])]);                               \
      }                                                                                \
      double acc = (a0 + a1) + (a2 + a3);                                              \
      double tail = 0.0;                                                               \
      for (; i < e; ++i) tail += VN##_P(v[i], x[COLUMN(r, ci[i])]);                    \
      acc = acc + tail;                                                                \
      EPI(VN, r, acc);                                                                 \
    }                                                                                  \
  }

typedef void (*rows_fn)(const void*, const void*, const void*, const void*, void*, double,
                        double, int64_t, int64_t);

#define DEFINE_KIND_VT(RPN, RP, CIN, CI)                                \
  DEFINE_ROWS(csr_##RPN##_##CIN##_f64, RP, CI, f64, COLUMN_CSR)        \
  DEFINE_ROWS(csr_##RPN##_##CIN##_f32, RP, CI, f32, COLUMN_CSR)        \
  DEFINE_ROWS(csr_##RPN##_##CIN##_f16, RP, CI, f16, COLUMN_CSR)        \
  DEFINE_ROWS(csr_##RPN##_##CIN##_bf16, RP, CI, bf16, COLUMN_CSR)      \
  DEFINE_ROWS(da_##RPN##_##CIN##_f64, RP, CI, f64, COLUMN_DA)          \
  DEFINE_ROWS(da_##RPN##_##CIN##_f32, RP, CI, f32, COLUMN_DA)          \
  DEFINE_ROWS(da_##RPN##_##CIN##_f16, RP, CI, f16, COLUMN_DA)          \
  DEFINE_ROWS(da_##RPN##_##CIN##_bf16, RP, CI, bf16, COLUMN_DA)

#define DEFINE_RP(RPN, RP)               \
  DEFINE_KIND_VT(RPN, RP, i8, int8_t)    \
  DEFINE_KIND_VT(RPN, RP, i16, int16_t)  \
  DEFINE_KIND_VT(RPN, RP, i32, int32_t)  \
  DEFINE_KIND_VT(RPN, RP, i64, int64_t)

DEFINE_RP(p32, int32_t)
DEFINE_RP(p64, int64_t)

/* table [kind][rp 0=i32,1=i64][ci 0..3][vt 0=f32,1=f64,2=f16,3=bf16][order] */
#define ENTRY(K, RPN, CIN, VTN) \
  {(rows_fn)K##_##RPN##_##CIN##_##VTN##_naive, (rows_fn)K##_##RPN##_##CIN##_##VTN##_macc3, \
   (rows_fn)K##_##RPN##_##CIN##_##VTN##_strip4}
#define ENTRY_VT(K, RPN, CIN) \
  {ENTRY(K, RPN, CIN, f32), ENTRY(K, RPN, CIN, f64), ENTRY(K, RPN, CIN, f16), ENTRY(K, RPN, CIN, bf16)}
#define ENTRY_CI(K, RPN) \
  {ENTRY_VT(K, RPN, i8), ENTRY_VT(K, RPN, i16), ENTRY_VT(K, RPN, i32), ENTRY_VT(K, RPN, i64)}
#define ENTRY_RP(K) {ENTRY_CI(K, p32), ENTRY_CI(K, p64)}

static const rows_fn TABLE[2][2][4][4][3] = {ENTRY_RP(csr), ENTRY_RP(da)};

static rows_fn lookup(int kind, int order, int rp_dt, int ci_dt, int val_dt) {
  if (kind < 0 || kind > 1 || order < 0 || order > 2) return NULL;
  if (rp_dt != ORC_I32 && rp_dt != ORC_I64) return NULL;
  if (ci_dt < ORC_I8 || ci_dt > ORC_I64) return NULL;
  if (val_dt < ORC_F32 || val_dt > ORC_BF16) return NULL;
  return TABLE[kind][rp_dt == ORC_I64][ci_dt][val_dt - ORC_F32][order];
}

int orc_spmv(int kind, int order, int rp_dt, int ci_dt, int val_dt, const void* rowptr,
             const void* colids, const void* values, const void* x, void* y, double alpha,
             double beta, int64_t row_start, int64_t row_end) {
  rows_fn f = lookup(kind, order, rp_dt, ci_dt, val_dt);
  if (!f) return 1;
  f(rowptr, colids, values, x, y, alpha, beta, row_start, row_end);
  return 0;
}

/* 16-bit conversions (tests): f64 -> bits with one RNE rounding, bits -> f64 */
void orc_to_half_bits(const double* in, uint16_t* out, int64_t n, int bf16) {
  for (int64_t i = 0; i < n; ++i) out[i] = bf16 ? f64_to_b16(in[i]) : f64_to_h16(in[i]);
}
void orc_from_half_bits(const uint16_t* in, double* out, int64_t n, int bf16) {
  for (int64_t i = 0; i < n; ++i) out[i] = bf16 ? b16_to_f32(in[i]) : h16_to_f32(in[i]);
}

/* ------------------------------------------------------------ row_blocks */

static int64_t rp_at(const void* rp, int rp_dt, int64_t i) {
  return rp_dt == ORC_I64 ? ((const int64_t*)rp)[i] : (int64_t)((const int32_t*)rp)[i];
}

/* searchsorted(rowptr, target, side="left") over rowptr[0..nrows] */
static int64_t lower_bound_rp(const void* rp, int rp_dt, int64_t nrows, int64_t target) {
  int64_t lo = 0, hi = nrows + 1;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (rp_at(rp, rp_dt, mid) < target) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* cuts[0..nblocks]: block k is [cuts[k], cuts[k+1]) (spmv/__init__.py:71-85) */
int orc_row_blocks(const void* rowptr, int rp_dt, int64_t nrows, int64_t nblocks,
                   int64_t* cuts) {
  if (nblocks < 1) return 1;
  int64_t nnz = rp_at(rowptr, rp_dt, nrows);
  cuts[0] = 0;
  for (int64_t k = 1; k < nblocks; ++k) {
    /* (k * nnz) // nblocks with Python floor semantics on non-negatives */
    __int128 prod = (__int128)k * (__int128)nnz;
    int64_t target = (int64_t)(prod / nblocks);
    int64_t b = lower_bound_rp(rowptr, rp_dt, nrows, target);
    if (b < cuts[k - 1]) b = cuts[k - 1];
    if (b > nrows) b = nrows;
    cuts[k] = b;
  }
  cuts[nblocks] = nrows;
  return 0;
}

/* -------------------------------------------------- ParallelRowBlock(T) */

typedef struct {
  rows_fn f;
  const void *rp, *ci, *v, *x;
  void* y;
  double alpha, beta;
  int64_t rs, re;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  j->f(j->rp, j->ci, j->v, j->x, j->y, j->alpha, j->beta, j->rs, j->re);
  return NULL;
}

/* Like the reference: threads==1 runs inline; otherwise one thread per
 * non-empty nnz-balanced block, spawned per call and joined. */
int orc_spmv_parallel(int kind, int order, int rp_dt, int ci_dt, int val_dt,
                      const void* rowptr, const void* colids, const void* values,
                      const void* x, void* y, double alpha, double beta, int64_t nrows,
                      int threads) {
  rows_fn f = lookup(kind, order, rp_dt, ci_dt, val_dt);
  if (!f || threads < 1) return 1;
  if (threads == 1) {
    f(rowptr, colids, values, x, y, alpha, beta, 0, nrows);
    return 0;
  }
  int64_t* cuts = (int64_t*)malloc(sizeof(int64_t) * (threads + 1));
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * threads);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  if (!cuts || !jobs || !tids) return 2;
  orc_row_blocks(rowptr, rp_dt, nrows, threads, cuts);
  int nj = 0;
  for (int k = 0; k < threads; ++k) {
    if (cuts[k] >= cuts[k + 1]) continue;
    jobs[nj] = (job_t){f, rowptr, colids, values, x, y, alpha, beta, cuts[k], cuts[k + 1]};
    ++nj;
  }
  int rc = 0;
  int started = 0;
  for (int k = 0; k < nj; ++k) {
    if (pthread_create(&tids[k], NULL, run_job, &jobs[k]) != 0) { rc = 3; break; }
    ++started;
  }
  for (int k = 0; k < started; ++k) pthread_join(tids[k], NULL);
  free(cuts);
  free(jobs);
  free(tids);
  return rc;
}

/* ------------------------------------------------------------------- RCM */

/* BFS from start (neighbours in stored ascending order); level[] must be -1
 * on entry for unvisited nodes.  Writes the visit order, returns its length
 * and the eccentricity through *ecc (reorder.py:100-118). */
static int64_t bfs_levels(const int64_t* indptr, const int64_t* indices, int64_t start,
                          int64_t* level, int64_t* order, int64_t* ecc) {
  int64_t tail = 0, head = 0, e = 0;
  order[tail++] = start;
  level[start] = 0;
  while (head < tail) {
    int64_t u = order[head++];
    int64_t d = level[u] + 1;
    for (int64_t k = indptr[u]; k < indptr[u + 1]; ++k) {
      int64_t w = indices[k];
      if (level[w] < 0) {
        level[w] = d;
        if (d > e) e = d;
        order[tail++] = w;
      }
    }
  }
  *ecc = e;
  return tail;
}

/* argmin over nodes of (degree, index) (reorder.py:121-123) */
static int64_t min_deg(const int64_t* nodes, int64_t cnt, const int64_t* deg) {
  int64_t best = nodes[0];
  for (int64_t k = 1; k < cnt; ++k) {
    int64_t u = nodes[k];
    if (deg[u] < deg[best] || (deg[u] == deg[best] && u < best)) best = u;
  }
  return best;
}

static const int64_t* g_deg;
static int cmp_deg_idx(const void* a, const void* b) {
  int64_t u = *(const int64_t*)a, w = *(const int64_t*)b;
  if (g_deg[u] != g_deg[w]) return g_deg[u] < g_deg[w] ? -1 : 1;
  return u < w ? -1 : (u > w);
}

/* perm[new] = old (reorder.py:146-197).  indptr/indices: symmetrized
 * adjacency (pattern of A+A^T, no self loops, sorted, deduplicated). */
int orc_rcm(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t* perm) {
  if (n == 0) return 0;
  int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* level = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* comp_nodes = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* comp_off = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  int64_t* starts = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* last = (int64_t*)malloc(sizeof(int64_t) * n);
  char* seen = (char*)calloc(n, 1);
  if (!deg || !level || !order || !comp_nodes || !comp_off || !starts || !last || !seen)
    return 2;
  for (int64_t u = 0; u < n; ++u) { deg[u] = indptr[u + 1] - indptr[u]; level[u] = -1; }

  /* components, discovered by BFS from the lowest unseen index */
  int64_t ncomp = 0, filled = 0;
  comp_off[0] = 0;
  for (int64_t s = 0; s < n; ++s) {
    if (seen[s]) continue;
    int64_t ecc;
    int64_t cnt = bfs_levels(indptr, indices, s, level, comp_nodes + filled, &ecc);
    for (int64_t k = 0; k < cnt; ++k) { level[comp_nodes[filled + k]] = -1; seen[comp_nodes[filled + k]] = 1; }
    filled += cnt;
    comp_off[++ncomp] = filled;
  }

  /* pseudo-peripheral start per component (reorder.py:126-143) */
  for (int64_t c = 0; c < ncomp; ++c) {
    const int64_t* nodes = comp_nodes + comp_off[c];
    int64_t cnt = comp_off[c + 1] - comp_off[c];
    int64_t r = min_deg(nodes, cnt, deg);
    int64_t ecc, ecc_c;
    int64_t len = bfs_levels(indptr, indices, r, level, order, &ecc);
    int64_t nlast = 0;
    for (int64_t k = 0; k < len; ++k) if (level[order[k]] == ecc) last[nlast++] = order[k];
    for (int64_t k = 0; k < len; ++k) level[order[k]] = -1;
    for (;;) {
      int64_t cand = min_deg(last, nlast, deg);
      len = bfs_levels(indptr, indices, cand, level, order, &ecc_c);
      if (ecc_c > ecc) {
        nlast = 0;
        for (int64_t k = 0; k < len; ++k) if (level[order[k]] == ecc_c) last[nlast++] = order[k];
        for (int64_t k = 0; k < len; ++k) level[order[k]] = -1;
        r = cand;
        ecc = ecc_c;
      } else {
        for (int64_t k = 0; k < len; ++k) level[order[k]] = -1;
        break;
      }
    }
    starts[c] = r;
  }

  /* components in ascending order of start node; CM BFS with neighbours
   * sorted by (degree, index); then reverse everything */
  int64_t* comp_ix = (int64_t*)malloc(sizeof(int64_t) * (ncomp ? ncomp : 1));
  for (int64_t c = 0; c < ncomp; ++c) comp_ix[c] = c;
  /* insertion sort of component ids by start (distinct starts) */
  for (int64_t a = 1; a < ncomp; ++a) {
    int64_t t = comp_ix[a], b = a - 1;
    while (b >= 0 && starts[comp_ix[b]] > starts[t]) { comp_ix[b + 1] = comp_ix[b]; --b; }
    comp_ix[b + 1] = t;
  }
  char* placed = seen;
  memset(placed, 0, n);
  int64_t qn = 0;
  g_deg = deg;
  for (int64_t a = 0; a < ncomp; ++a) {
    int64_t s = starts[comp_ix[a]];
    int64_t head = qn;
    order[qn++] = s;
    placed[s] = 1;
    while (head < qn) {
      int64_t u = order[head++];
      int64_t first = qn;
      for (int64_t k = indptr[u]; k < indptr[u + 1]; ++k) {
        int64_t w = indices[k];
        if (!placed[w]) order[qn++] = w;
      }
      if (qn - first > 1) qsort(order + first, qn - first, sizeof(int64_t), cmp_deg_idx);
      for (int64_t k = first; k < qn; ++k) placed[order[k]] = 1;
    }
  }
  for (int64_t k = 0; k < n; ++k) perm[k] = order[n - 1 - k];
  free(deg); free(level); free(order); free(comp_nodes); free(comp_off);
  free(starts); free(last); free(seen); free(comp_ix);
  return 0;
}
