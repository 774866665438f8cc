// Shared device helpers for the sm_100a DA-CSR library: PTX wrappers for
// mbarrier + cp.async.bulk (the TMA bulk-copy engine, SASS UBLKCP), the
// reference's rounding rules, and error plumbing for the C ABI.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dacsr_b200.h"

// Bounds-checked build (compute-sanitizer is unavailable on this pool):
// -DDACSR_CHECKED turns every DACSR_CHECK into a trap on violation.
#ifdef DACSR_CHECKED
#define DACSR_CHECK(cond) \
  do {                    \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define DACSR_CHECK(cond) ((void)0)
#endif

namespace dacsr {

// ---------------------------------------------------------------- errors
void set_last_error(const char* what, cudaError_t e);
int check_launch(const char* what);

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t arrivals) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(arrivals)
               : "memory");
}

// make the initialised barriers visible to the async (bulk copy) proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order earlier generic-proxy smem reads before later async-proxy writes
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> shared, completion signalled as tx bytes on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// --------------------------------------------------- reference arithmetic
// float64 data: product rounded in float64 (no FMA contraction).
__device__ __forceinline__ double product(double v, double x) { return __dmul_rn(v, x); }
// float32 data: product rounded to float32, then widened for the float64 sum
// (numba: f32*f32 -> f32; `acc += p` with acc float64).
__device__ __forceinline__ double product(float v, float x) {
  return static_cast<double>(__fmul_rn(v, x));
}

// 16-bit data: the f32 product of two 16-bit significands is exact
// (11+11 <= 24, 8+8 <= 24 bits), so the f64 sum sees the exact product.
__device__ __forceinline__ double product(__half v, __half x) {
  return static_cast<double>(__fmul_rn(__half2float(v), __half2float(x)));
}
__device__ __forceinline__ double product(__nv_bfloat16 v, __nv_bfloat16 x) {
  return static_cast<double>(__fmul_rn(__bfloat162float(v), __bfloat162float(x)));
}

__device__ __forceinline__ double to_f64(double v) { return v; }
__device__ __forceinline__ double to_f64(float v) { return static_cast<double>(v); }
__device__ __forceinline__ double to_f64(__half v) { return static_cast<double>(__half2float(v)); }
__device__ __forceinline__ double to_f64(__nv_bfloat16 v) {
  return static_cast<double>(__bfloat162float(v));
}
__device__ __forceinline__ void store_rounded(double* p, double v) { *p = v; }
__device__ __forceinline__ void store_rounded(float* p, double v) { *p = __double2float_rn(v); }
// one rounding f64 -> 16 bit (round to nearest even, no detour through f32)
__device__ __forceinline__ void store_rounded(__half* p, double v) { *p = __double2half(v); }
__device__ __forceinline__ void store_rounded(__nv_bfloat16* p, double v) {
  *p = __double2bfloat16(v);
}

// the value store_rounded leaves in memory, widened back (no reload)
template <class VT>
__device__ __forceinline__ double as_stored(double v);
template <> __device__ __forceinline__ double as_stored<double>(double v) { return v; }
template <> __device__ __forceinline__ double as_stored<float>(double v) {
  return static_cast<double>(__double2float_rn(v));
}
template <> __device__ __forceinline__ double as_stored<__half>(double v) {
  return static_cast<double>(__half2float(__double2half(v)));
}
template <> __device__ __forceinline__ double as_stored<__nv_bfloat16>(double v) {
  return static_cast<double>(__bfloat162float(__double2bfloat16(v)));
}

// y[r] = alpha*acc (+ beta*y[r] iff beta != 0); y is not read when beta == 0.
template <class VT>
__device__ __forceinline__ void epilogue(VT* y, int64_t r, double acc, double alpha,
                                         double beta) {
  double out = __dmul_rn(alpha, acc);
  if (beta != 0.0) out = __dadd_rn(out, __dmul_rn(beta, to_f64(y[r])));
  store_rounded(y + r, out);
}
// the same, returning y[r] as stored (rounded to VT) for a fused ||y||^2
template <class VT>
__device__ __forceinline__ double epilogue_stored(VT* y, int64_t r, double acc, double alpha,
                                                  double beta) {
  double out = __dmul_rn(alpha, acc);
  if (beta != 0.0) out = __dadd_rn(out, __dmul_rn(beta, to_f64(y[r])));
  store_rounded(y + r, out);
  return as_stored<VT>(out);
}

// Exact thread-sequential sums in the reference's three orders
// (_numba_kernels.py:82-91 naive, :110-132 multi_acc3, :135-160 strip_mined4).
// `get(i)` returns the rounded product of entry i.
template <class Get>
__device__ __forceinline__ double sum_naive(int64_t s, int64_t e, const Get& get) {
  double acc = 0.0;
  int64_t i = s;
  for (; i + 4 <= e; i += 4) {
    const double p0 = get(i), p1 = get(i + 1), p2 = get(i + 2), p3 = get(i + 3);
    acc = __dadd_rn(acc, p0);
    acc = __dadd_rn(acc, p1);
    acc = __dadd_rn(acc, p2);
    acc = __dadd_rn(acc, p3);
  }
  for (; i < e; ++i) acc = __dadd_rn(acc, get(i));
  return acc;
}

template <class Get>
__device__ __forceinline__ double sum_macc3(int64_t s, int64_t e, const Get& get) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  int64_t i = s;
  for (; i + 3 <= e; i += 3) {
    const double p0 = get(i), p1 = get(i + 1), p2 = get(i + 2);
    a0 = __dadd_rn(a0, p0);
    a1 = __dadd_rn(a1, p1);
    a2 = __dadd_rn(a2, p2);
  }
  if (i < e) a0 = __dadd_rn(a0, get(i));
  if (i + 1 < e) a1 = __dadd_rn(a1, get(i + 1));
  return __dadd_rn(__dadd_rn(a0, a1), a2);
}

template <class Get>
__device__ __forceinline__ double sum_strip4(int64_t s, int64_t e, const Get& get) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t i = s;
  for (; i + 4 <= e; i += 4) {
    const double p0 = get(i), p1 = get(i + 1), p2 = get(i + 2), p3 = get(i + 3);
    a0 = __dadd_rn(a0, p0);
    a1 = __dadd_rn(a1, p1);
    a2 = __dadd_rn(a2, p2);
    a3 = __dadd_rn(a3, p3);
  }
  double acc = __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3));
  double tail = 0.0;
  for (; i < e; ++i) tail = __dadd_rn(tail, get(i));
  return __dadd_rn(acc, tail);
}

template <class Get>
__device__ __forceinline__ double row_sum(int order, int64_t s, int64_t e, const Get& get) {
  if (order == DACSR_ORDER_MACC3) return sum_macc3(s, e, get);
  if (order == DACSR_ORDER_STRIP4) return sum_strip4(s, e, get);
  return sum_naive(s, e, get);  // NAIVE, and TREE for rows one thread owns
}

// Streaming form of the three orders for a row consumed in order by one
// thread (cooperative long rows): call add() once per product, in order.
struct OrderedAcc {
  int order, ph3;
  int64_t k, full4;
  double a0, a1, a2, a3, tail;
  __device__ void init(int o, int64_t n) {
    order = o;
    ph3 = 0;
    k = 0;
    full4 = n - (n & 3);
    a0 = a1 = a2 = a3 = tail = 0.0;
  }
  __device__ __forceinline__ void add(double p) {
    if (order == DACSR_ORDER_MACC3) {  // round robin a0, a1, a2 (tail lands on a0, a1)
      if (ph3 == 0) a0 = __dadd_rn(a0, p);
      else if (ph3 == 1) a1 = __dadd_rn(a1, p);
      else a2 = __dadd_rn(a2, p);
      ph3 = ph3 == 2 ? 0 : ph3 + 1;
    } else if (order == DACSR_ORDER_STRIP4) {  // full groups of 4, then a tail sum
      if (k >= full4) {
        tail = __dadd_rn(tail, p);
      } else {
        const int m = static_cast<int>(k & 3);
        if (m == 0) a0 = __dadd_rn(a0, p);
        else if (m == 1) a1 = __dadd_rn(a1, p);
        else if (m == 2) a2 = __dadd_rn(a2, p);
        else a3 = __dadd_rn(a3, p);
      }
    } else {
      a0 = __dadd_rn(a0, p);
    }
    ++k;
  }
  // n products in order, same result as n calls of add(): aligned blocks run
  // as bare addition chains (one per accumulator), add() does the alignment
  // and the remainder.  Through add() alone a fold ran at ~100 cycles per
  // entry on its one lane (the order's branches around every addition).
  __device__ __forceinline__ void add_many(const double* p, int n) {
    int i = 0;
    if (order == DACSR_ORDER_MACC3) {
      for (; i < n && ph3 != 0; ++i) add(p[i]);
      for (; i + 3 <= n; i += 3) {
        a0 = __dadd_rn(a0, p[i]);
        a1 = __dadd_rn(a1, p[i + 1]);
        a2 = __dadd_rn(a2, p[i + 2]);
        k += 3;
      }
      for (; i < n; ++i) add(p[i]);
      return;
    }
    if (order == DACSR_ORDER_STRIP4) {
      for (; i < n && (k & 3) != 0; ++i) add(p[i]);
      while (i + 4 <= n && k + 4 <= full4) {
        a0 = __dadd_rn(a0, p[i]);
        a1 = __dadd_rn(a1, p[i + 1]);
        a2 = __dadd_rn(a2, p[i + 2]);
        a3 = __dadd_rn(a3, p[i + 3]);
        i += 4;
        k += 4;
      }
      for (; i < n; ++i) add(p[i]);
      return;
    }
    double a = a0;
    for (; i + 4 <= n; i += 4) {
      const double q0 = p[i], q1 = p[i + 1], q2 = p[i + 2], q3 = p[i + 3];
      a = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(a, q0), q1), q2), q3);
    }
    for (; i < n; ++i) a = __dadd_rn(a, p[i]);
    a0 = a;
    k += n;
  }
  __device__ double result() const {
    if (order == DACSR_ORDER_MACC3) return __dadd_rn(__dadd_rn(a0, a1), a2);
    if (order == DACSR_ORDER_STRIP4)
      return __dadd_rn(__dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3)), tail);
    return a0;
  }
};

// read-only-path loads (LDG.E.CONSTANT); int64_t is `long` on LP64, which
// has no __ldg overload, so route it through long long.
template <class T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ int64_t ldg<int64_t>(const int64_t* p) {
  return static_cast<int64_t>(__ldg(reinterpret_cast<const long long*>(p)));
}

}  // namespace dacsr
