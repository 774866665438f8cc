// Builder of the band-tiled device layout (dacsr_tiles_t, include/dacsr_b200.h).
//
// For a wide random band (C3/C5: offsets uniform over +-32767) every x
// gather of the row-major kernels is its own 32-byte sector of L2, and the
// L1TEX pipe retires about one such gather per SM clock — the kernel then
// runs at a third of HBM speed.  The TILED kernel stages x in shared memory
// one column tile at a time (TMA bulk copies) and folds, for each tile, the
// entries of its rows that fall inside it; the layout built here is the same
// entries re-laid in exactly that consumption order:
//
//   group g (512 rows, row slot 32j + l)
//     tile t (tile_lo[g] ..):  mask        — 16 nibbles m_j: lane l folds
//                                           row slot 32j + (l ^ m_j)
//                              order[32]   — lane l: nibble k = j of the
//                                           k-th row it folds in the tile
//                              counts[32]  — lane l: nibble k = entries of
//                                           that row inside the tile
//                              entries     — lane lists L_l stored in pair
//                                           steps (pair step q: entries 2q,
//                                           2q + 1 of every lane whose list
//                                           is longer than 2q, lanes
//                                           ascending; a list of odd length
//                                           ends in one zero slot)
//
// A row's entries stay in column order (tiles ascend, and inside a tile its
// entries are consecutive in its lane's list), so each lane folds every row
// in the reference's naive order (_numba_kernels.py:82-91).  Entries are
// copied as raw bits.
//
// The lane remap evens out the lanes' list lengths: with a fixed row ->
// lane map a tile's lists are Poisson-ragged (C3: the longest list of a
// warp is ~1.4x the mean, and every lane of the warp steps through it); the
// masks, chosen greedily row slot by row slot, bring that near 1.1x.
//
// Passes (warp per group): extent (min / max column), count, fill.  Count
// and fill derive the masks from the same counts with the same function.

#include <algorithm>
#include <climits>

#include "device_common.cuh"

namespace dacsr {
namespace {

constexpr int kGroupRows = 512;
constexpr int kRowsPerLane = 16;

template <int KIND, class CI>
__device__ __forceinline__ int64_t entry_col(int64_t r, CI c) {
  return KIND == DACSR_KIND_DA ? r + static_cast<int64_t>(c) : static_cast<int64_t>(c);
}

__global__ void extent_init_kernel(long long* out) {
  out[0] = LLONG_MAX;
  out[1] = LLONG_MIN;
}

template <int KIND, class RP, class CI>
__global__ void extent_kernel(const RP* __restrict__ rp, const CI* __restrict__ ci, int64_t rs,
                              int64_t re, long long* out) {
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (int64_t r = rs + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < re;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = static_cast<int64_t>(rp[r]), e = static_cast<int64_t>(rp[r + 1]);
    if (e > b) {
      lo = min(lo, static_cast<long long>(entry_col<KIND>(r, ci[b])));
      hi = max(hi, static_cast<long long>(entry_col<KIND>(r, ci[e - 1])));
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}

// Lane remap of one tile: c[j] = entries of row slot 32j + lane in the
// tile.  For j = 0..15 in turn, m_j (0..15) minimises (longest list in
// steps of G, sum of squared list lengths) over the lists so far plus row
// slots 32j + (l ^ m_j); ties go to the smallest m_j.  Returns the mask
// word (the same in every lane) and this lane's list length.
__device__ __forceinline__ uint64_t balance_lanes(const int (&c)[kRowsPerLane], int G, int& total) {
  const int lane = threadIdx.x & 31;
  uint64_t mw = 0;
  int tot = 0;
#pragma unroll
  for (int j = 0; j < kRowsPerLane; ++j) {
    unsigned long long best = ~0ull;
    int bm = 0;
    if (__any_sync(0xffffffffu, c[j] != 0)) {
#pragma unroll 1
      for (int m = 0; m < 16; ++m) {
        const int t2 = tot + __shfl_sync(0xffffffffu, c[j], lane ^ m);
        const unsigned mx = __reduce_max_sync(0xffffffffu, static_cast<unsigned>((t2 + G - 1) / G));
        const unsigned sq = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(t2 * t2));
        const unsigned long long key = (static_cast<unsigned long long>(mx) << 32) | sq;
        if (key < best) {
          best = key;
          bm = m;
        }
      }
    }
    tot += __shfl_sync(0xffffffffu, c[j], lane ^ bm);
    mw |= static_cast<uint64_t>(bm) << (4 * j);
  }
  // refinement: each row slot's mask chosen again against all the others
  // (same key; a tie keeps the current mask).  Three sweeps take the lane
  // utilisation of a C3 tile from 0.88 to 0.90, of a C5 tile from 0.83 to
  // 0.86 (simulated on Poisson counts; every step saved is a step of the
  // whole warp).
#ifndef DACSR_TILES_SWEEPS
#define DACSR_TILES_SWEEPS 3
#endif
#pragma unroll 1
  for (int sweep = 0; sweep < DACSR_TILES_SWEEPS; ++sweep) {
    bool changed = false;
#pragma unroll
    for (int j = 0; j < kRowsPerLane; ++j) {
      if (!__any_sync(0xffffffffu, c[j] != 0)) continue;
      const int cur = static_cast<int>((mw >> (4 * j)) & 15u);
      const int base = tot - __shfl_sync(0xffffffffu, c[j], lane ^ cur);
      unsigned long long best = ~0ull;
      int bm = cur;
#pragma unroll 1
      for (int k = 0; k < 16; ++k) {
        const int m = k == 0 ? cur : (k <= cur ? k - 1 : k);  // the current mask first
        const int t2 = base + __shfl_sync(0xffffffffu, c[j], lane ^ m);
        const unsigned mx = __reduce_max_sync(0xffffffffu, static_cast<unsigned>((t2 + G - 1) / G));
        const unsigned sq = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(t2 * t2));
        const unsigned long long key = (static_cast<unsigned long long>(mx) << 32) | sq;
        if (key < best) {
          best = key;
          bm = m;
        }
      }
      if (bm != cur) {
        changed = true;
        mw = (mw & ~(15ull << (4 * j))) | (static_cast<uint64_t>(bm) << (4 * j));
      }
      tot = base + __shfl_sync(0xffffffffu, c[j], lane ^ bm);
    }
    if (!changed) break;
  }
  total = tot;
  return mw;
}

// Row order of one tile, chosen for the shared-memory banks.  At each step
// a lane either continues its row or starts its next one; the starting
// lanes pick, one lane per half warp at a time, the not yet started row
// whose bank pairs collide least with the rows already placed: its x
// gathers at this and the following steps, its accumulator load now and
// its accumulator store at the step its successor starts (cost = the
// number of lanes of the half warp already on each of those bank pairs;
// ties to the lowest j).  Returns the order word (nibble k = row slot j of
// the lane's k-th row) and the counts word in that order.  Every row's
// entries stay consecutive and in column order, so any order folds every
// row in the naive order.
constexpr int kOrderSteps = kRowsPerLane * 15 + 16;  // longest list + a row
struct OrderScratch {  // per warp: 4-bit counters per (half, step, bank pair)
  uint64_t x[2][kOrderSteps];   // x gathers
  uint64_t st[2][kOrderSteps];  // accumulator stores
};
__device__ __forceinline__ int occ_get(uint64_t w, int b) { return static_cast<int>((w >> (4 * b)) & 15u); }
__device__ __forceinline__ uint64_t occ_add(uint64_t w, int b) {  // saturating
  return occ_get(w, b) == 15 ? w : w + (1ull << (4 * b));
}
template <int KIND, class CI, class VB>
__device__ void order_rows(const CI* __restrict__ ci, const int64_t (&src)[kRowsPerLane],
                           const int (&nr)[kRowsPerLane], uint64_t mw, int64_t row_base,
                           int64_t tstart, int total, int kmax, OrderScratch& sc, uint64_t& ow,
                           uint64_t& cw) {
  const int lane = threadIdx.x & 31;
  const int h = lane >> 4;
  // bank pair (8-byte units, 16 per half warp) of a gather at column c
  auto xkey = [&](int64_t c) {
    return static_cast<int>(((c - tstart) * static_cast<int64_t>(sizeof(VB)) >> 3) & 15);
  };
  auto row_of = [&](int j) {
    return row_base + 32 * j + (lane ^ static_cast<int>((mw >> (4 * j)) & 15u));
  };
  for (int i = lane; i < 2 * (kmax + 16); i += 32) {
    sc.x[i & 1][i >> 1] = 0;
    sc.st[i & 1][i >> 1] = 0;
  }
  __syncwarp();
  unsigned left = 0;  // rows not started (bit j)
  for (int j = 0; j < kRowsPerLane; ++j)
    if (nr[j] > 0) left |= 1u << j;
  int rem = 0, k = 0;
  ow = cw = 0;
  for (int stp = 0; stp < kmax; ++stp) {
    const bool sw = stp < total && rem == 0;
    const unsigned swm = __ballot_sync(0xffffffffu, sw);
    uint64_t ao = 0;  // accumulator loads of this step (per half)
    for (unsigned qm = (swm | (swm >> 16)) & 0xffffu; qm; qm &= qm - 1) {
      const int q = __ffs(qm) - 1;
      const bool me = sw && (lane & 15) == q;
      uint64_t add_a = 0;
      if (me) {
        int best = INT_MAX, pick = 0;
        for (unsigned m = left; m; m &= m - 1) {
          const int j = __ffs(m) - 1;
          const int ak = (lane ^ static_cast<int>((mw >> (4 * j)) & 15u)) & 15;
          const int64_t r = row_of(j);
          int cost = occ_get(ao, ak) + occ_get(sc.st[h][stp + nr[j]], ak);
          for (int e = 0; e < nr[j]; ++e)
            cost += occ_get(sc.x[h][stp + e], xkey(entry_col<KIND>(r, ci[src[j] + e])));
          if (cost < best) {
            best = cost;
            pick = j;
          }
        }
        left &= ~(1u << pick);
        ow |= static_cast<uint64_t>(pick) << (4 * k);
        cw |= static_cast<uint64_t>(nr[pick]) << (4 * k);
        ++k;
        rem = nr[pick];
        const int ak = (lane ^ static_cast<int>((mw >> (4 * pick)) & 15u)) & 15;
        const int64_t r = row_of(pick);
        for (int e = 0; e < nr[pick]; ++e)
          sc.x[h][stp + e] = occ_add(sc.x[h][stp + e], xkey(entry_col<KIND>(r, ci[src[pick] + e])));
        sc.st[h][stp + nr[pick]] = occ_add(sc.st[h][stp + nr[pick]], ak);
        add_a = 1ull << (4 * ak);
      }
      ao += __shfl_sync(0xffffffffu, add_a, (lane & 16) | q);
      __syncwarp();
    }
    if (stp < total) --rem;
  }
  __syncwarp();
}

struct TileGeom {
  int64_t rs, re, col0;
  int T, G;
  __device__ __forceinline__ int64_t tile(int64_t c) const { return (c - col0) / T; }
};

// Per group: tiles spanned, entries kept, rows left out (some tile holds
// more than 15 of their entries); tile_lo and the skip masks.
template <int KIND, class RP, class CI>
__global__ void tiles_count_kernel(const RP* __restrict__ rp, const CI* __restrict__ ci,
                                   TileGeom geo, int64_t ngroups, int32_t* __restrict__ nt_counts,
                                   int32_t* __restrict__ ent_counts,
                                   int32_t* __restrict__ ovf_counts, int32_t* __restrict__ tile_lo,
                                   uint16_t* __restrict__ skip) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < ngroups;
       g += nw) {
    int64_t tmin = INT64_MAX, tmax = -1;
    int kept = 0, ovf = 0;
    unsigned sk = 0;
    for (int j = 0; j < kRowsPerLane; ++j) {
      const int64_t r = geo.rs + kGroupRows * g + 32 * j + lane;
      if (r >= geo.re) continue;
      const int64_t b = static_cast<int64_t>(rp[r]), e = static_cast<int64_t>(rp[r + 1]);
      if (e == b) continue;
      // longest run of entries inside one tile (columns ascend)
      int run = 0, worst = 0;
      int64_t cur = -1;
      for (int64_t i = b; i < e; ++i) {
        const int64_t t = geo.tile(entry_col<KIND>(r, ci[i]));
        run = t == cur ? run + 1 : 1;
        cur = t;
        worst = run > worst ? run : worst;
      }
      if (worst > 15) {
        sk |= 1u << j;
        ++ovf;
        continue;
      }
      kept += static_cast<int>(e - b);
      tmin = min(tmin, geo.tile(entry_col<KIND>(r, ci[b])));
      tmax = max(tmax, geo.tile(entry_col<KIND>(r, ci[e - 1])));
    }
    for (int o = 16; o > 0; o >>= 1) {
      tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
      tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      ovf += __shfl_xor_sync(0xffffffffu, ovf, o);
    }
    // slots: per tile, each lane's list rounded up to whole pairs
    int64_t slots = 0;
    if (tmax >= 0) {
      int64_t cur[kRowsPerLane], end[kRowsPerLane];
#pragma unroll
      for (int j = 0; j < kRowsPerLane; ++j) {
        const int64_t r = geo.rs + kGroupRows * g + 32 * j + lane;
        cur[j] = end[j] = 0;
        if (r < geo.re && !((sk >> j) & 1u)) {
          cur[j] = static_cast<int64_t>(rp[r]);
          end[j] = static_cast<int64_t>(rp[r + 1]);
        }
      }
      for (int64_t t = tmin; t <= tmax; ++t) {
        int c[kRowsPerLane];
#pragma unroll
        for (int j = 0; j < kRowsPerLane; ++j) {
          const int64_t r = geo.rs + kGroupRows * g + 32 * j + lane;
          c[j] = 0;
          while (cur[j] < end[j] && geo.tile(entry_col<KIND>(r, ci[cur[j]])) == t) {
            ++cur[j];
            ++c[j];
          }
        }
        int total;
        balance_lanes(c, geo.G, total);
        slots += (total + geo.G - 1) / geo.G * geo.G;
      }
    }
    for (int o = 16; o > 0; o >>= 1) slots += __shfl_xor_sync(0xffffffffu, slots, o);
    (void)kept;
    skip[32 * g + lane] = static_cast<uint16_t>(sk);
    if (lane == 0) {
      const bool any = tmax >= 0;
      nt_counts[g] = any ? static_cast<int32_t>(tmax - tmin + 1) : 0;
      tile_lo[g] = any ? static_cast<int32_t>(tmin) : 0;
      ent_counts[g] = static_cast<int32_t>(slots);
      ovf_counts[g] = ovf;
    }
  }
}

// IT / VB: raw element types of the inner / value widths (bit copies).
template <int KIND, class RP, class CI, class IT, class VB>
__global__ void __launch_bounds__(128) tiles_fill_kernel(
    const RP* __restrict__ rp, const CI* __restrict__ ci, const VB* __restrict__ v,
    TileGeom geo, int64_t ngroups, const int64_t* __restrict__ ent_ptr,
    const int64_t* __restrict__ cnt_ptr, const int32_t* __restrict__ tile_lo,
    const uint16_t* __restrict__ skip, const int64_t* __restrict__ ovf_ptr,
    uint64_t* __restrict__ counts, uint64_t* __restrict__ order, uint64_t* __restrict__ masks,
    IT* __restrict__ t_inner,
    VB* __restrict__ t_values, int64_t* __restrict__ ovf_rows) {
  __shared__ OrderScratch scratch[4];  // one per warp (128 threads)
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const IT* __restrict__ raw_ci = reinterpret_cast<const IT*>(ci);
  for (int64_t g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < ngroups;
       g += nw) {
    const unsigned sk = skip[32 * g + lane];
    // left-out rows, ascending (row order = j-major, lane-minor)
    int64_t op = ovf_ptr[g];
    for (int j = 0; j < kRowsPerLane; ++j) {
      const bool o = (sk >> j) & 1u;
      const unsigned m = __ballot_sync(0xffffffffu, o);
      if (o) ovf_rows[op + __popc(m & below)] = geo.rs + kGroupRows * g + 32 * j + lane;
      op += __popc(m);
    }
    int64_t cur[kRowsPerLane], end[kRowsPerLane];
#pragma unroll
    for (int j = 0; j < kRowsPerLane; ++j) {
      const int64_t r = geo.rs + kGroupRows * g + 32 * j + lane;
      cur[j] = end[j] = 0;
      if (r < geo.re && !((sk >> j) & 1u)) {
        cur[j] = static_cast<int64_t>(rp[r]);
        end[j] = static_cast<int64_t>(rp[r + 1]);
      }
    }
    const int64_t nt = cnt_ptr[g + 1] - cnt_ptr[g];
    const int64_t t0 = tile_lo[g];
    int64_t pos = ent_ptr[g];
    for (int64_t k = 0; k < nt; ++k) {
      const int64_t t = t0 + k;
      // this tile's entries of each own row: [cur[j], cur[j] + n[j])
      int n[kRowsPerLane];
#pragma unroll
      for (int j = 0; j < kRowsPerLane; ++j) {
        const int64_t r = geo.rs + kGroupRows * g + 32 * j + lane;
        int c = 0;
        while (cur[j] + c < end[j] && geo.tile(entry_col<KIND>(r, ci[cur[j] + c])) == t) ++c;
        n[j] = c;
      }
      int total;
      const uint64_t mw = balance_lanes(n, geo.G, total);
      // the rows this lane folds: slot 32j + (lane ^ m_j)
      int64_t src[kRowsPerLane];
      int nr[kRowsPerLane];
#pragma unroll
      for (int j = 0; j < kRowsPerLane; ++j) {
        const int from = lane ^ static_cast<int>((mw >> (4 * j)) & 15u);
        nr[j] = __shfl_sync(0xffffffffu, n[j], from);
        src[j] = __shfl_sync(0xffffffffu, cur[j], from);
      }
      const int kmax = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(total)));
      uint64_t ow, cw;
      order_rows<KIND, CI, VB>(ci, src, nr, mw, geo.rs + kGroupRows * g, geo.col0 + t * geo.T, total,
                               kmax, scratch[threadIdx.x >> 5], ow, cw);
      counts[(cnt_ptr[g] + k) * 32 + lane] = cw;
      order[(cnt_ptr[g] + k) * 32 + lane] = ow;
      if (lane == 0) masks[cnt_ptr[g] + k] = mw;
      int kk = 0, used = 0;
      auto next_src = [&]() {  // this lane's next list entry
        while (used == static_cast<int>((cw >> (4 * kk)) & 15u)) {
          ++kk;
          used = 0;
        }
        return src[(ow >> (4 * kk)) & 15u] + used++;
      };
      for (int s = 0; s < kmax; s += geo.G) {  // step group: list entries s .. s + G - 1
        const bool act = s < total;
        const unsigned m = __ballot_sync(0xffffffffu, act);
        if (act) {
          const int64_t dst = pos + geo.G * __popc(m & below);
          for (int e = 0; e < geo.G; ++e) {
            if (s + e < total) {
              const int64_t a = next_src();
              t_inner[dst + e] = raw_ci[a];
              t_values[dst + e] = v[a];
            } else {
              t_inner[dst + e] = IT(0);
              t_values[dst + e] = VB(0);
            }
          }
        }
        pos += geo.G * __popc(m);
      }
#pragma unroll
      for (int jj = 0; jj < kRowsPerLane; ++jj) cur[jj] += n[jj];
    }
  }
}

int grid_for_groups(int64_t ngroups, int warps_per_block) {
  const int64_t blocks = (ngroups + warps_per_block - 1) / warps_per_block;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 64)));
}

const int kBytes[8] = {1, 2, 4, 8, 4, 8, 2, 2};

template <int KIND, class RP, class CI, class F>
int with_value_raw(const dacsr_matrix_t* a, F&& f) {
  switch (kBytes[a->values_dtype]) {
    case 8: return f(std::integral_constant<int, KIND>(), RP(), CI(), uint64_t());
    case 4: return f(std::integral_constant<int, KIND>(), RP(), CI(), uint32_t());
    case 2: return f(std::integral_constant<int, KIND>(), RP(), CI(), uint16_t());
    default: return DACSR_ERR_DTYPE;
  }
}

template <int KIND, class RP, class F>
int with_inner(const dacsr_matrix_t* a, F&& f) {
  if (KIND == DACSR_KIND_DA) {
    switch (a->colids_dtype) {
      case DACSR_I8: return with_value_raw<KIND, RP, int8_t>(a, f);
      case DACSR_I16: return with_value_raw<KIND, RP, int16_t>(a, f);
      case DACSR_I32: return with_value_raw<KIND, RP, int32_t>(a, f);
      default: return DACSR_ERR_DTYPE;
    }
  }
  switch (a->colids_dtype) {
    case DACSR_I32: return with_value_raw<KIND, RP, int32_t>(a, f);
    case DACSR_I64: return with_value_raw<KIND, RP, int64_t>(a, f);
    default: return DACSR_ERR_DTYPE;
  }
}

// f(kind_constant, RP(), CI(), VB()) for the matrix's types
template <class F>
int by_matrix_types(const dacsr_matrix_t* a, F&& f) {
  if (a->values_dtype < DACSR_F32 || a->values_dtype > DACSR_BF16) return DACSR_ERR_DTYPE;
  const bool i64 = a->rowptr_dtype == DACSR_I64;
  if (!i64 && a->rowptr_dtype != DACSR_I32) return DACSR_ERR_DTYPE;
  if (a->kind == DACSR_KIND_DA)
    return i64 ? with_inner<DACSR_KIND_DA, int64_t>(a, f) : with_inner<DACSR_KIND_DA, int32_t>(a, f);
  if (a->kind == DACSR_KIND_CSR)
    return i64 ? with_inner<DACSR_KIND_CSR, int64_t>(a, f)
               : with_inner<DACSR_KIND_CSR, int32_t>(a, f);
  return DACSR_ERR_DTYPE;
}

template <class T>
struct RawOf;
template <> struct RawOf<int8_t> { using type = uint8_t; };
template <> struct RawOf<int16_t> { using type = uint16_t; };
template <> struct RawOf<int32_t> { using type = uint32_t; };
template <> struct RawOf<int64_t> { using type = uint64_t; };

bool geometry_ok(const dacsr_matrix_t* a, const dacsr_tiles_t* t) {
  return a && t && a->rowptr && t->row_start >= 0 && t->row_end >= t->row_start &&
         t->row_end <= a->nrows && t->ngroups == (t->row_end - t->row_start + 511) / 512 &&
         t->tile_cols >= 64 && t->tile_cols <= 65536 && (t->tile_cols & 15) == 0 &&
         (t->step_group == 2 || t->step_group == 4) &&
         (a->nnz == 0 || (a->colids && a->values));
}

}  // namespace
}  // namespace dacsr

using namespace dacsr;

extern "C" {

int dacsr_tiles_extent(const dacsr_matrix_t* a, int64_t rs, int64_t re, int64_t* out2, void* stream) {
  if (!a || !a->rowptr || !out2 || rs < 0 || re < rs || re > a->nrows ||
      (a->nnz > 0 && !a->colids))
    return DACSR_ERR_ARG;
  auto st = static_cast<cudaStream_t>(stream);
  auto* o = reinterpret_cast<long long*>(out2);
  extent_init_kernel<<<1, 1, 0, st>>>(o);
  int rc = check_launch("extent_init_kernel");
  if (rc || re == rs) return rc;
  const int g = static_cast<int>(std::min<int64_t>((re - rs + 255) / 256, 148 * 16));
  return by_matrix_types(a, [&](auto kc, auto rp0, auto ci0, auto) {
    constexpr int KIND = decltype(kc)::value;
    using RP = decltype(rp0);
    using CI = decltype(ci0);
    extent_kernel<KIND, RP, CI><<<g, 256, 0, st>>>(static_cast<const RP*>(a->rowptr),
                                                   static_cast<const CI*>(a->colids), rs, re, o);
    return check_launch("extent_kernel");
  });
}

int dacsr_tiles_count(const dacsr_matrix_t* a, const dacsr_tiles_t* t, int32_t* nt_counts,
                      int32_t* ent_counts, int32_t* ovf_counts, void* stream) {
  if (!geometry_ok(a, t) || (t->ngroups > 0 && (!nt_counts || !ent_counts || !ovf_counts ||
                                                !t->tile_lo || !t->skip)))
    return DACSR_ERR_ARG;
  if (t->ngroups == 0) return DACSR_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const TileGeom geo{t->row_start, t->row_end, t->col0, t->tile_cols, t->step_group};
  const int g = grid_for_groups(t->ngroups, 8);
  return by_matrix_types(a, [&](auto kc, auto rp0, auto ci0, auto) {
    constexpr int KIND = decltype(kc)::value;
    using RP = decltype(rp0);
    using CI = decltype(ci0);
    tiles_count_kernel<KIND, RP, CI><<<g, 256, 0, st>>>(
        static_cast<const RP*>(a->rowptr), static_cast<const CI*>(a->colids), geo, t->ngroups,
        nt_counts, ent_counts, ovf_counts, const_cast<int32_t*>(t->tile_lo),
        const_cast<uint16_t*>(t->skip));
    return check_launch("tiles_count_kernel");
  });
}

int dacsr_tiles_fill(const dacsr_matrix_t* a, const dacsr_tiles_t* t, const int64_t* ovf_ptr,
                     void* stream) {
  if (!geometry_ok(a, t) || !ovf_ptr ||
      (t->ngroups > 0 && (!t->ent_ptr || !t->cnt_ptr || !t->tile_lo || !t->skip)) ||
      (t->nblocks > 0 && (!t->counts || !t->order || !t->masks)) ||
      (t->total > 0 && (!t->inner || !t->values)) || (t->n_ovf > 0 && !t->ovf_rows))
    return DACSR_ERR_ARG;
  if (t->ngroups == 0) return DACSR_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const TileGeom geo{t->row_start, t->row_end, t->col0, t->tile_cols, t->step_group};
  const int g = grid_for_groups(t->ngroups, 4);
  return by_matrix_types(a, [&](auto kc, auto rp0, auto ci0, auto vb0) {
    constexpr int KIND = decltype(kc)::value;
    using RP = decltype(rp0);
    using CI = decltype(ci0);
    using VB = decltype(vb0);
    using IT = typename RawOf<CI>::type;
    tiles_fill_kernel<KIND, RP, CI, IT, VB><<<g, 128, 0, st>>>(
        static_cast<const RP*>(a->rowptr), static_cast<const CI*>(a->colids),
        static_cast<const VB*>(a->values), geo, t->ngroups, t->ent_ptr, t->cnt_ptr, t->tile_lo,
        t->skip, ovf_ptr, const_cast<uint64_t*>(t->counts), const_cast<uint64_t*>(t->order),
        const_cast<uint64_t*>(t->masks),
        static_cast<IT*>(const_cast<void*>(t->inner)), static_cast<VB*>(const_cast<void*>(t->values)),
        const_cast<int64_t*>(t->ovf_rows));
    return check_launch("tiles_fill_kernel");
  });
}

}  // extern "C"
