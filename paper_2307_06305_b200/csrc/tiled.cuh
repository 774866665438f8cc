// TILED: the band-tiled SpMV kernel (layout: csrc/tiles.cu, dacsr_tiles_t).
//
// Included by spmv_kernels.cuh inside namespace dacsr (needs Mat, Scal,
// warp_long_row, ldcs, prefetch_l2_bulk).
//
// One CTA per SM, persistent over chunks of kTileWarps 512-row groups
// (7680 rows).  Warp kTileWarps is the producer: it walks the chunk's
// column tiles in order and streams each tile of x into a ring of
// kTileXBufs shared-memory buffers with TMA bulk copies (cp.async.bulk,
// full/empty mbarriers; waiting warps sleep in mbarrier.try_wait).  Consumer warp w owns group w of the chunk: lane l holds rows
// 32j + l (j = 0..15) and, per tile, folds its list of entries (its rows in
// order, each row's entries of the tile in column order) with the x values
// read from shared memory — random 8-byte reads that cost a few bank
// wavefronts per warp instead of a 32-byte L2 sector each.  The row sums
// live in shared memory between tiles (a lane swaps its running sum when it
// moves to its next row), so each row is folded from +0.0 in column order:
// the reference's naive order, bit for bit (_numba_kernels.py:82-91).
//
// The operator is read once, step-major packed (coalesced runs), with
// evict-first loads; the next tile's segment is pulled into L2 by a bulk
// prefetch one tile ahead.  Rows the layout left out (more than 15 entries
// inside one tile) are reduced warp by warp from the CSR arrays at the end.
#pragma once


// 15 consumer warps + the producer = 16 warps, 4 per SM sub-partition: the
// register file is split per sub-partition, so a 17th warp would cap every
// thread at 96 registers (measured: spills) instead of 128
#ifndef DACSR_TILED_WARPS
#define DACSR_TILED_WARPS 15
#endif
constexpr int kTileWarps = DACSR_TILED_WARPS;  // consumer warps (groups) per CTA
constexpr int kTileRows = 16;   // rows per lane
#ifndef DACSR_TILED_G
#define DACSR_TILED_G 2  // entries per lane per packed step (layout step_group)
#endif
#ifndef DACSR_TILED_XBUFS
#define DACSR_TILED_XBUFS 2
#endif
constexpr int kTileXBufs = DACSR_TILED_XBUFS;  // x tile ring (producer runs kTileXBufs-1 ahead)
#ifndef DACSR_TILED_BATCH
#define DACSR_TILED_BATCH 6     // steps per batch (two batches in flight; measured 4/6/8 on C3: 6)
#endif

template <class CI, class VT>
struct TileArgs {
  const int64_t* __restrict__ ent_ptr;
  const int64_t* __restrict__ cnt_ptr;
  const int32_t* __restrict__ tile_lo;
  const uint64_t* __restrict__ counts;
  const uint64_t* __restrict__ order;
  const uint64_t* __restrict__ masks;
  const uint16_t* __restrict__ skip;
  const CI* __restrict__ ci;
  const VT* __restrict__ v;
  const int64_t* __restrict__ ovf;
  int64_t row0, col0, cmax, total, n_ovf;
  int T;
};

// shared memory: kTileXBufs x buffers of xbuf elements, the row sums, the mbarriers
template <class VT>
__host__ __device__ constexpr size_t tiled_xbuf_bytes(int xbuf) {
  return (static_cast<size_t>(xbuf) * sizeof(VT) + 127) & ~size_t(127);
}
template <class VT>
__host__ __device__ constexpr size_t tiled_smem_bytes(int xbuf) {
  return kTileXBufs * tiled_xbuf_bytes<VT>(xbuf) + size_t(kTileWarps) * (kTileRows + 1) * 32 * 8 +
         16 * kTileXBufs;
}

__device__ __forceinline__ int nibble_sum(uint64_t v) {
  const uint64_t s = (v & 0x0F0F0F0F0F0F0F0Full) + ((v >> 4) & 0x0F0F0F0F0F0F0F0Full);
  return static_cast<int>((s * 0x0101010101010101ull) >> 56);
}

// shared-memory loads / stores through 32-bit shared addresses
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
template <class VT>
__device__ __forceinline__ VT lds_val(uint32_t a);
template <>
__device__ __forceinline__ double lds_val<double>(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
template <>
__device__ __forceinline__ float lds_val<float>(uint32_t a) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
template <>
__device__ __forceinline__ __half lds_val<__half>(uint32_t a) {
  unsigned short v;
  asm("ld.shared.b16 %0, [%1];" : "=h"(v) : "r"(a));
  return __ushort_as_half(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 lds_val<__nv_bfloat16>(uint32_t a) {
  unsigned short v;
  asm("ld.shared.b16 %0, [%1];" : "=h"(v) : "r"(a));
  return __ushort_as_bfloat16(v);
}

// &base[o] for a 32-bit unsigned offset as one IMAD.WIDE.U32
template <class T>
__device__ __forceinline__ const T* elem_addr_u32(const T* base, uint32_t o) {
  const T* p;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(o), "n"(static_cast<int>(sizeof(T))), "l"(base));
  return p;
}

// Predicated evict-first load of a packed step's two consecutive elements
// (one vector load; p aligned to 2 * sizeof(T)), kept as loaded: two
// registers for 4- and 8-byte types, one 32-bit word for narrower ones.
// The loads are asm volatile, so a batch's loads issue in program order
// before the previous batch folds; narrow elements are unpacked in the fold
// by pair_elem, also volatile (unpacked at load time, nvcc placed the
// sign-extensions right behind the loads and every warp sat out the full
// load latency there).  Words are undefined when !pred (every use is
// predicated or selected away).
template <class T>
struct PairReg {
  static constexpr bool kPacked = sizeof(T) <= 2;
  using W = typename std::conditional<kPacked, uint32_t, T>::type;
  static constexpr int kWords = kPacked ? 1 : 2;
};
#define DACSR_PAIR_PRED "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q "
#define DACSR_ONE_PRED "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q "
__device__ __forceinline__ void pair_ld_cs(const double* p, bool pred, double* w) {
  asm volatile(DACSR_PAIR_PRED "ld.global.cs.v2.f64 {%0, %1}, [%2];\n\t}"
               : "=d"(w[0]), "=d"(w[1]) : "l"(p), "r"(static_cast<unsigned>(pred)));
}
__device__ __forceinline__ void pair_ld_cs(const float* p, bool pred, float* w) {
  asm volatile(DACSR_PAIR_PRED "ld.global.cs.v2.f32 {%0, %1}, [%2];\n\t}"
               : "=f"(w[0]), "=f"(w[1]) : "l"(p), "r"(static_cast<unsigned>(pred)));
}
__device__ __forceinline__ void pair_ld_cs(const int32_t* p, bool pred, int32_t* w) {
  asm volatile(DACSR_PAIR_PRED "ld.global.cs.v2.s32 {%0, %1}, [%2];\n\t}"
               : "=r"(w[0]), "=r"(w[1]) : "l"(p), "r"(static_cast<unsigned>(pred)));
}
__device__ __forceinline__ void pair_ld_cs(const int64_t* p, bool pred, int64_t* w) {
  long long x, y;
  asm volatile(DACSR_PAIR_PRED "ld.global.cs.v2.s64 {%0, %1}, [%2];\n\t}"
               : "=l"(x), "=l"(y) : "l"(p), "r"(static_cast<unsigned>(pred)));
  w[0] = x;
  w[1] = y;
}
template <class T>
__device__ __forceinline__ typename std::enable_if<sizeof(T) == 2>::type pair_ld_cs(
    const T* p, bool pred, uint32_t* w) {
  asm volatile(DACSR_ONE_PRED "ld.global.cs.b32 %0, [%1];\n\t}"
               : "=r"(w[0]) : "l"(p), "r"(static_cast<unsigned>(pred)));
}
__device__ __forceinline__ void pair_ld_cs(const int8_t* p, bool pred, uint32_t* w) {
  asm volatile(DACSR_ONE_PRED "ld.global.cs.u16 %0, [%1];\n\t}"
               : "=r"(w[0]) : "l"(p), "r"(static_cast<unsigned>(pred)));
}
#undef DACSR_PAIR_PRED
#undef DACSR_ONE_PRED

// element K (0 or 1) of a loaded pair, as the fold consumes it
template <class T, int K>
__device__ __forceinline__ auto pair_elem(const typename PairReg<T>::W* w) {
  if constexpr (!PairReg<T>::kPacked) {
    return w[K];
  } else if constexpr (std::is_same<T, int16_t>::value) {
    int v;
    if constexpr (K == 0)
      asm volatile("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(v) : "r"(w[0]));
    else
      asm volatile("shr.s32 %0, %1, 16;" : "=r"(v) : "r"(w[0]));
    return v;
  } else if constexpr (std::is_same<T, int8_t>::value) {
    int v;
    asm volatile("bfe.s32 %0, %1, %2, 8;" : "=r"(v) : "r"(w[0]), "n"(8 * K));
    return v;
  } else {  // __half / __nv_bfloat16 bits
    unsigned short h;
    if constexpr (K == 0)
      asm volatile("{\n\t.reg .b16 t;\n\tmov.b32 {%0, t}, %1;\n\t}" : "=h"(h) : "r"(w[0]));
    else
      asm volatile("{\n\t.reg .b16 t;\n\tmov.b32 {t, %0}, %1;\n\t}" : "=h"(h) : "r"(w[0]));
    if constexpr (std::is_same<T, __half>::value)
      return __ushort_as_half(h);
    else
      return __ushort_as_bfloat16(h);
  }
}

// acc += p (round to nearest) when pred, as one predicated DADD
__device__ __forceinline__ void dadd_if(double& acc, double p, bool pred) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q add.rn.f64 %0, %0, %1;\n\t}"
      : "+d"(acc) : "d"(p), "r"(static_cast<unsigned>(pred)));
}

// mbarrier waits that sleep instead of spinning (try_wait with a suspend
// time hint: the warp is descheduled until the phase completes)
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
}

// Group metadata of the chunk, one group per lane (lanes < kTileWarps),
// loaded a chunk ahead.
struct ChunkMeta {
  int64_t cnt0, cnt1, ent;
  int32_t tlo;
};

template <int KIND, class RP, class CI, class VT>
__global__ void __launch_bounds__(32 * (kTileWarps + 1), 1)
    tiled_kernel(Mat<KIND, RP, CI, VT> m, Scal s, TileArgs<CI, VT> ta, int64_t g_first,
                 int64_t g_last, int64_t rs, int64_t re, int xbuf) {
  using OT = typename std::conditional<sizeof(CI) == 8, int64_t, int>::type;
  constexpr int U = DACSR_TILED_BATCH;
  constexpr int G = DACSR_TILED_G;
  static_assert(G == 2 && U % G == 0, "the kernel folds pair steps, whole pairs per batch");
  extern __shared__ __align__(128) unsigned char dsm[];
  VT* const xs = reinterpret_cast<VT*>(dsm);
  const size_t xstride = tiled_xbuf_bytes<VT>(xbuf) / sizeof(VT);
  double* const accs = reinterpret_cast<double*>(dsm + kTileXBufs * tiled_xbuf_bytes<VT>(xbuf));
  uint64_t* const bars = reinterpret_cast<uint64_t*>(accs + kTileWarps * (kTileRows + 1) * 32);
  uint64_t* const full = bars;
  uint64_t* const empty = bars + kTileXBufs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kTileXBufs; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kTileWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t nchunks = (g_last - g_first + kTileWarps - 1) / kTileWarps;
  const VT* const xb = m.x + m.xoff;

  auto load_meta = [&](int64_t c) {
    ChunkMeta q{0, 0, 0, 0};
    const int64_t g = g_first + c * kTileWarps + lane;
    if (c < nchunks && lane < kTileWarps && g < g_last) {
      q.cnt0 = ldg(ta.cnt_ptr + g);
      q.cnt1 = ldg(ta.cnt_ptr + g + 1);
      q.ent = ldg(ta.ent_ptr + g);
      q.tlo = ldg(ta.tile_lo + g);
    }
    return q;
  };
  // tiles spanned by the chunk (empty: tlo > thi)
  auto chunk_range = [&](const ChunkMeta& q, int64_t& tlo, int64_t& thi) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    if (q.cnt1 > q.cnt0) {
      lo = q.tlo;
      hi = lo + (q.cnt1 - q.cnt0) - 1;
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    tlo = lo;
    thi = hi;
  };
  // x element i of a tile buffer holds column base + i, base = cs - shift
  // (the bulk copy starts at the 16-byte boundary at or below x[cs])
  auto tile_shift = [&](int64_t cs) {
    return static_cast<int>((reinterpret_cast<uintptr_t>(xb + cs) & 15) / sizeof(VT));
  };

  if (warp == kTileWarps) {  // ---------------------------------- producer
    int rb = 0;
    uint32_t rph = 0;
    bool wrapped = false;
    ChunkMeta nq = load_meta(blockIdx.x);
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      const ChunkMeta q = nq;
      nq = load_meta(c + gridDim.x);
      int64_t tlo, thi;
      chunk_range(q, tlo, thi);
      for (int64_t t = tlo; t <= thi; ++t) {
        if (lane == 0) {
          if (wrapped) mbar_wait_sleep(&empty[rb], rph ^ 1u);
          const int64_t cs = ta.col0 + t * ta.T;
          const int64_t ce = min64(cs + ta.T, ta.cmax + 1);
          const int shift = tile_shift(cs);
          const VT* src = xb + cs - shift;  // 16-byte aligned
          const int64_t n = ce - cs + shift;
          DACSR_CHECK(n > 0 && n <= xbuf);
          const uint32_t main = static_cast<uint32_t>((n * sizeof(VT)) & ~int64_t(15));
          VT* dst = xs + rb * xstride;
          // the last < 16 bytes with plain loads (the bulk copy must not
          // read past x's last element)
          for (int64_t q2 = main / sizeof(VT); q2 < n; ++q2) dst[q2] = src[q2];
          mbar_arrive_expect_tx(&full[rb], main);
          if (main) bulk_copy_g2s(dst, src, main, &full[rb]);
        }
        if (++rb == kTileXBufs) {
          rb = 0;
          rph ^= 1u;
          wrapped = true;
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  // row sums: lane l's row j at wacc + (32 j + l) * 8; row 16 is a dummy
  // slot (the first "switch" of a tile parks the empty running sum there)
  double* const wacc = accs + warp * (kTileRows + 1) * 32;
  const uint32_t wab = smem_addr(wacc);
  const uint32_t wa = wab + 8u * lane;
  const uint32_t xs0 = smem_addr(xs);
  // segment starts are multiples of G entries (every lane list is padded
  // to whole step groups) and inner / values carry 16 padding entries, so
  // rounding a segment out to 16-byte boundaries stays inside the arrays
  auto prefetch_segment = [&](int64_t p0, int n) {
    if (lane != 0 || n <= 0) return;
    const uintptr_t v0 = reinterpret_cast<uintptr_t>(ta.v + p0);
    const uintptr_t va = v0 & ~uintptr_t(15);
    prefetch_l2_bulk(reinterpret_cast<const void*>(va),
                     static_cast<uint32_t>(((v0 + n * sizeof(VT) + 15) & ~uintptr_t(15)) - va));
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(ta.ci + p0);
    const uintptr_t ia = i0 & ~uintptr_t(15);
    prefetch_l2_bulk(reinterpret_cast<const void*>(ia),
                     static_cast<uint32_t>(((i0 + n * sizeof(CI) + 15) & ~uintptr_t(15)) - ia));
  };
  int rb = 0;
  uint32_t rph = 0;
  ChunkMeta nq = load_meta(blockIdx.x);
  // this warp's group's first two count words, loaded a chunk ahead too
  // the operator segment of a tile: its lanes' lists rounded up to pairs
  auto seg_slots = [&](uint64_t w) {
    return static_cast<int>(
        __reduce_add_sync(0xffffffffu, static_cast<unsigned>((nibble_sum(w) + G - 1) / G * G)));
  };
  // count words and lane remap words of a block: (counts, masks)
  // and row order words (one tile ahead: the fold alone reads them)
  uint64_t ncn0 = 0, ncn1 = 0, nmw0 = 0, nmw1 = 0, now0 = 0;
  auto load_first_counts = [&](const ChunkMeta& q2) {
    const int64_t c0 = __shfl_sync(0xffffffffu, q2.cnt0, warp);
    const int64_t c1 = __shfl_sync(0xffffffffu, q2.cnt1, warp);
    ncn0 = c1 > c0 ? ldg(ta.counts + c0 * 32 + lane) : 0;
    now0 = c1 > c0 ? ldg(ta.order + c0 * 32 + lane) : 0;
    nmw0 = c1 > c0 ? ldg(ta.masks + c0) : 0;
    ncn1 = c1 > c0 + 1 ? ldg(ta.counts + (c0 + 1) * 32 + lane) : 0;
    nmw1 = c1 > c0 + 1 ? ldg(ta.masks + c0 + 1) : 0;
  };
  load_first_counts(nq);
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const ChunkMeta q = nq;
    nq = load_meta(c + gridDim.x);
    int64_t tlo, thi;
    chunk_range(q, tlo, thi);
    const int64_t g = g_first + c * kTileWarps + warp;
    const bool has = g < g_last;
    const int64_t cbase = __shfl_sync(0xffffffffu, q.cnt0, warp);
    const int64_t gnt = __shfl_sync(0xffffffffu, q.cnt1, warp) - cbase;
    const int64_t gtlo = __shfl_sync(0xffffffffu, q.tlo, warp);
    int64_t pos = __shfl_sync(0xffffffffu, q.ent, warp);
#pragma unroll
    for (int j = 0; j < kTileRows; ++j) sts_f64(wa + 256u * j, 0.0);
    uint64_t cn0 = ncn0, cn1 = ncn1, mw0 = nmw0, mw1 = nmw1, ow0 = now0;
    // the operator segment of the group's first tile into L2 now, every
    // later one a tile ahead of its fold (bulk prefetch; measured: without
    // it C3 runs 11 % slower, two tiles ahead 4 % slower)
    int64_t pf_pos = pos;
    if (gnt > 0) {
      const int n0 = seg_slots(cn0);
      prefetch_segment(pf_pos, n0);
      pf_pos += n0;
    }
    // rows of lane l: row0 + 512g + 32j + l
    const int64_t lrow = ta.row0 + 512 * g + lane;
    // byte offset of column 0 relative to x buffer element 0 of tile tlo
    // (32-bit wrap-around); tile starts advance by T columns and T is a
    // multiple of 16, so every tile shares tile col0's 16-byte shift
    uint32_t xoff = static_cast<uint32_t>((ta.col0 - tile_shift(ta.col0) + tlo * ta.T) *
                                          static_cast<int64_t>(sizeof(VT)));
    const uint32_t tstep = static_cast<uint32_t>(ta.T * sizeof(VT));
    const uint32_t grow_b =
        static_cast<uint32_t>((ta.row0 + 512 * g) * static_cast<int64_t>(sizeof(VT)));
    for (int64_t t = tlo; t <= thi; ++t) {
      const int64_t k = t - gtlo;
      const bool mine = has && k >= 0 && k < gnt;
      uint64_t cur = 0, mw = 0, ow = 0;
      int total = 0;
      if (mine) {
        cur = cn0;
        mw = mw0;
        ow = ow0;
        ow0 = k + 1 < gnt ? ldg(ta.order + (cbase + k + 1) * 32 + lane) : 0;
        cn0 = cn1;
        mw0 = mw1;
        cn1 = k + 2 < gnt ? ldg(ta.counts + (cbase + k + 2) * 32 + lane) : 0;
        mw1 = k + 2 < gnt ? ldg(ta.masks + cbase + k + 2) : 0;
        total = nibble_sum(cur);
        if (k + 1 < gnt) {
          const int n = seg_slots(cn0);
          prefetch_segment(pf_pos, n);
          pf_pos += n;
        }
      }
      if (t == thi) load_first_counts(nq);  // the next chunk's first count words
      mbar_wait_sleep(&full[rb], rph);
      if (mine) {
        DACSR_CHECK(xoff == static_cast<uint32_t>((ta.col0 + t * ta.T - tile_shift(ta.col0 + t * ta.T)) *
                                                  static_cast<int64_t>(sizeof(VT))));
        const uint32_t xsa = xs0 + static_cast<uint32_t>(rb * xstride * sizeof(VT));
        // d = column of x buffer element 0.  DA: x of entry (row, offset o)
        // at xr + o * sizeof(VT), xr = &xbuf[row - d]; CSR: at xc + c *
        // sizeof(VT), xc = &xbuf[-d] (32-bit wrap-around arithmetic).  Row
        // slot s of the group: xr = xg + s * sizeof(VT), its sum at wab + 8s.
        const uint32_t xc = xsa - xoff;
        const uint32_t xg = xc + grow_b;
        const int kmax = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(total)));
        // the lane's rows in fold order: nibble kq / 4 of ow (row slot j)
        // and of cur (its entries in the tile)
        uint32_t kq = 0;
        int rem = 0;
        uint32_t acc_a = wa + 32u * 8u * kTileRows;  // dummy slot
        uint32_t xr = xg;
        double acc = 0.0;
        const VT* vt = ta.v + pos;
        const CI* ct = ta.ci + pos;
        // opaque bases: each load address is then one IMAD.WIDE.U32 off the
        // 32-bit step offset (nvcc otherwise re-derives 64-bit index sums)
        asm("" : "+l"(vt));
        asm("" : "+l"(ct));
        uint32_t lp = 0;
        // batch of U steps = U/G packed steps: positions from the step
        // ballots, then every operator load of the batch issued (G-entry
        // vector loads, predicated asm, program order)
        constexpr int UP = U / G;
        using OW = typename PairReg<CI>::W;
        using VW = typename PairReg<VT>::W;
        constexpr int OK = PairReg<CI>::kWords, VK = PairReg<VT>::kWords;
        auto load_batch = [&](int q0, OW* off, VW* val) {
#pragma unroll
          for (int u = 0; u < UP; ++u) {
            const bool act = G * (q0 + u) < total;
            const unsigned msk = __ballot_sync(0xffffffffu, act);
            const uint32_t o = lp + G * __popc(msk & below);
            lp += G * __popc(msk);
            DACSR_CHECK(!act || pos + o + G - 1 < ta.total);
            pair_ld_cs(elem_addr_u32(ct, o), act, off + OK * u);
            pair_ld_cs(elem_addr_u32(vt, o), act, val + VK * u);
          }
        };
        // element u of a batch (u even: first of pair u / 2); u is a
        // constant after unrolling, so one branch remains
        auto off_at = [&](const OW* off, int u) -> OT {
          return static_cast<OT>(u & 1 ? pair_elem<CI, 1>(off + OK * (u / 2))
                                       : pair_elem<CI, 0>(off + OK * (u / 2)));
        };
        auto val_at = [&](const VW* val, int u) -> VT {
          return u & 1 ? pair_elem<VT, 1>(val + VK * (u / 2)) : pair_elem<VT, 0>(val + VK * (u / 2));
        };
        auto fold_batch = [&](int k0, const OW* off, const VW* val) {
          const int left = total - k0;  // steps of this lane left in the tile
          if constexpr (KIND == DACSR_KIND_DA) {
            // the row of each step from the counts alone (no dependence on
            // the sums), branch-free, so every x read of the batch can issue
            // before the first sum of the batch is formed
            uint32_t xrs[U];
            uint32_t swm = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const bool sw = u < left && rem == 0;
              const uint32_t sh = kq & 63u;  // 64 only once every row is done (sw false)
              const uint32_t jn = static_cast<uint32_t>(ow >> sh) & 15u;
              const int rem2 = static_cast<int>((cur >> sh) & 15u);
              const uint32_t slot = (jn << 5) | (lane ^ static_cast<uint32_t>((mw >> (4 * jn)) & 15u));
              kq = sw ? kq + 4u : kq;
              rem = (sw ? rem2 : rem) - 1;
              xr = sw ? xg + slot * static_cast<uint32_t>(sizeof(VT)) : xr;
              swm |= sw ? 1u << u : 0u;
              xrs[u] = xr;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if ((swm >> u) & 1u) {  // this lane's next row of the tile
                sts_f64(acc_a, acc);
                acc_a = wab + (xrs[u] - xg) * static_cast<uint32_t>(8 / sizeof(VT));
                acc = lds_f64(acc_a);
              }
              const uint32_t xa = xrs[u] + static_cast<uint32_t>(static_cast<int>(off_at(off, u)) * static_cast<int>(sizeof(VT)));
              DACSR_CHECK(!(u < left) || (xa >= xsa && xa < xsa + xbuf * sizeof(VT)));
              if (u < left) dadd_if(acc, product(val_at(val, u), lds_val<VT>(xa)), true);
            }
          } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const bool act = u < left;  // once false, false for the rest of the tile
              if (act && rem == 0) {  // this lane's next row of the tile
                sts_f64(acc_a, acc);
                const uint32_t j = static_cast<uint32_t>(ow >> kq) & 15u;
                rem = static_cast<int>((cur >> kq) & 15u);
                kq += 4u;
                acc_a = wab + 8u * ((j << 5) |
                                    (lane ^ static_cast<uint32_t>((mw >> (4 * j)) & 15u)));
                acc = lds_f64(acc_a);
              }
              const uint32_t xa = xc + static_cast<uint32_t>(off_at(off, u) * static_cast<OT>(sizeof(VT)));
              DACSR_CHECK(!act || (xa >= xsa && xa < xsa + xbuf * sizeof(VT)));
              if (act) dadd_if(acc, product(val_at(val, u), lds_val<VT>(xa)), true);
              --rem;
            }
          }
        };
        // two batches in flight: batch i+1's loads are issued before batch i folds
        OW offA[OK * U / 2], offB[OK * U / 2];
        VW valA[VK * U / 2], valB[VK * U / 2];
        // ptxas puts every operator load of this loop on one scoreboard, and
        // a scoreboard wait drains all of it: with batch i+1's loads issued
        // ahead of batch i's first use, that use waited for the loads just
        // issued (no lead at all; 18 % of the kernel's stall samples sat on
        // that one instruction).  touch() makes the next batch's load
        // addresses depend on a word of this batch (or-ed in under a zero
        // the compiler cannot see), so the wait comes first and covers only
        // loads issued a whole fold earlier.
#ifndef DACSR_TILED_TOUCH
#define DACSR_TILED_TOUCH 1
#endif
        const uint32_t zero = static_cast<uint32_t>(ta.T) & 1u;  // T is a multiple of 16
        auto touch = [&](const OW* off) {
          if (DACSR_TILED_TOUCH) lp |= static_cast<uint32_t>(off[0]) & zero;
        };
        int k0 = 0;
        if (kmax > 0) load_batch(0, offA, valA);
        while (k0 < kmax) {
          touch(offA);
          if (k0 + U < kmax) load_batch((k0 + U) / G, offB, valB);
          fold_batch(k0, offA, valA);
          k0 += U;
          if (k0 >= kmax) break;
          touch(offB);
          if (k0 + U < kmax) load_batch((k0 + U) / G, offA, valA);
          fold_batch(k0, offB, valB);
          k0 += U;
        }
        sts_f64(acc_a, acc);
        pos += lp;
      }
      xoff += tstep;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[rb]);
      if (++rb == kTileXBufs) {
        rb = 0;
        rph ^= 1u;
      }
    }
    // the chunk's rows: y = alpha * sum (+ beta * y)
    if (has) {
      const unsigned sk = ldg(ta.skip + 32 * g + lane);
      if (s.group_sumsq == nullptr) {
#pragma unroll 4
        for (int j = 0; j < kTileRows; ++j) {
          const int64_t r = lrow + 32 * j;
          if (r >= rs && r < re && !((sk >> j) & 1u))
            epilogue(m.y, r, lds_f64(wa + 256u * j), s.a(), s.beta);
        }
      } else {
        // ... and the group's sum of y^2 in the fixed group tree: lane l
        // folds its rows 32j + l in j order, then the xor butterfly
        // (aux.cu group_sumsq restates it for a y already in memory)
        double sq = 0.0;
#pragma unroll 4
        for (int j = 0; j < kTileRows; ++j) {
          const int64_t r = lrow + 32 * j;
          if (r >= rs && r < re) {
            const double v = epilogue_stored(m.y, r, lds_f64(wa + 256u * j), s.a(), s.beta);
            sq = __dadd_rn(sq, __dmul_rn(v, v));
          }
        }
        for (int o = 16; o > 0; o >>= 1) sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
        if (lane == 0) s.group_sumsq[(ta.row0 + 512 * g) >> 9] = sq;
      }
    }
    __syncwarp();
  }
  // rows left out of the layout: warp per row from the CSR arrays
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * kTileWarps + warp; w < ta.n_ovf;
       w += static_cast<int64_t>(gridDim.x) * kTileWarps) {
    const int64_t r = ldg(ta.ovf + w);
    if (r < rs || r >= re) continue;
    const int64_t b = ldg(m.rp + r), e = ldg(m.rp + r + 1);
    __syncwarp();
    warp_long_row(m, s, r, b, e, static_cast<const VT*>(nullptr), static_cast<const CI*>(nullptr),
                  0, 0, lane, wacc);
  }
}

