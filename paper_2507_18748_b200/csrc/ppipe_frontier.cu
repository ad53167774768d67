// ppipe_frontier.cu -- the frontier pass, hand-written for sm_100a.
//
// Input: n candidate records in any order (survivors of the score kernels' in-SM
// fold, or the union of per-rank frontiers in the merge). Output: per segment
// (model, K, k_1..k_K) the strict (E min, theta max) staircase in canonical order
// (E ascending, theta strictly ascending; among identical (E, theta) the smallest
// batch, then the smallest (c_1, c_2): readings A1 / A17), plus the CSR offsets.
// theta = b / Cmax is the bottleneck throughput x_l = min_d b / C_d
// (eqs. 1.10 / 1.13); E is the end-to-end latency of eq. 1.12
// (PAPER.md:2283). Frontier = the feasible candidates no other candidate of the
// segment beats in both objectives.
//
// Pipeline (no library sort / scan / select):
//   1. fp_count     segment id of every record; per-segment counts by warp-aggregated
//                   atomics (__match_any_sync); each record keeps its rank in its segment
//   2. scan         exclusive scan of the counts -> segment start offsets
//   3. fp_scatter   counting-sort scatter of a 16-byte sort item (E, Cmax, b, cuts) and
//                   the record index to start[segment] + rank
//   4. fp_small     warp per segment with <= kFpWarpMax items: rank sort in shared memory
//                   (every lane counts the items that precede each of its items under the
//                   total order), then a warp-shuffle prefix max of theta in sorted order;
//                   an item is kept iff its theta strictly exceeds every item before it
//                   (which is exactly "best of its E, and above every smaller E")
//   5. fp_large     CTA per segment with <= kFpCap items: bitonic sort of a permutation in
//                   shared memory, block-level prefix max and compaction
//   6. huge         (segments > kFpCap, rare) chunk sorts + merge-path rounds in global
//                   memory, then the same block-level staircase streamed with a carry
//   7. scan         exclusive scan of the kept counts -> the output CSR
//   8. fp_compact   warp per segment copies its kept records into place
// The same machinery (templated on the item traits) serves the per-stage batch
// frontier (ppipe_pb.cu) and the SLO truncation.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ppipe_internal.h"

namespace ppipe {

namespace {

constexpr int kFpThreads = 256;
constexpr int kFpWarpR = 4;                    // items per lane in the warp path
constexpr int kFpWarpMax = 32 * kFpWarpR;      // 128
constexpr int kFpMid = 1024;                   // medium CTA path
constexpr int kFpCap = 4096;                   // large CTA path: keys staged in shared memory
constexpr int kScanPerThread = 16;
constexpr int kScanTile = kFpThreads * kScanPerThread;  // 4096 counts per scan tile

__device__ __forceinline__ unsigned lanemask_lt_() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__host__ __device__ __forceinline__ uint32_t wt4(uint32_t wpack, int k) { return (wpack >> (4 * k)) & 15u; }

template <class Rec>
__device__ __forceinline__ uint64_t seg_of_rec(const Rec& p, const uint64_t* seg_base, int C) {
  uint64_t off = 0, pw = 1;
  for (int k = 1; k < p.K; ++k) {
    pw *= (uint64_t)C;
    off += pw;
  }
  uint64_t idx = 0;
  for (int d = 0; d < p.K; ++d) idx = idx * C + p.cls[d];
  return seg_base[p.model] + off + idx;
}

// ---------------------------------------------------------------------------
// Item traits. kMode selects what is kept after the per-segment sort:
//   kStaircase     theta strictly above every earlier item (the (E, theta) frontier)
//   kFirstOfGroup  the first item of each run of T::same items (F2 equal vectors)
//   kKeepAll       every item (a segmented sort into canonical order)
// ---------------------------------------------------------------------------
constexpr int kStaircase = 0, kFirstOfGroup = 1, kKeepAll = 2;
// Unified batch (ppipe_point): theta = b / Cmax, Cmax = max_d w_{k_d} C_d (w = 1
// unless ppipe_set_vgpu), compared exactly by cross-multiplication (Cmax = 0 reads
// as +inf; two +inf tie, reading R1).
struct UniTraits {
  static constexpr int kMode = kStaircase;
  using Rec = ppipe_point;
  struct Item {
    uint32_t E, c, b, cuts;
  };
  struct Th {
    uint32_t b, c;
  };
  struct Params {
    uint32_t wpack;
    const uint16_t* batches;
    int B;
  };
  static __device__ __forceinline__ Item item_of(const Rec& p, const Params& q) {
    uint32_t m;
    if (q.wpack == 0x11111111u) {
      m = p.stage_us[0];
      if (p.K >= 2) m = max(m, p.stage_us[1]);
      if (p.K >= 3) m = max(m, p.stage_us[2]);
    } else {
      m = wt4(q.wpack, p.cls[0]) * p.stage_us[0];
      if (p.K >= 2) m = max(m, wt4(q.wpack, p.cls[1]) * p.stage_us[1]);
      if (p.K >= 3) m = max(m, wt4(q.wpack, p.cls[2]) * p.stage_us[2]);
    }
    return Item{p.e2e_us, m, p.batch, (uint32_t)p.cut[0] << 16 | p.cut[1]};
  }
  // a strictly before b: E asc, theta desc, b asc, (c_1, c_2) asc -- a strict total
  // order on distinct candidates of one segment
  static __device__ __forceinline__ bool prec(const Item& a, const Item& b) {
    if (a.E != b.E) return a.E < b.E;
    const uint64_t l = (uint64_t)a.b * b.c, r = (uint64_t)b.b * a.c;
    if (l != r) return l > r;
    if (a.b != b.b) return a.b < b.b;
    return a.cuts < b.cuts;
  }
  static __device__ __forceinline__ uint32_t primary(const Item& a) { return a.E; }  // monotone under prec
  static __device__ __forceinline__ uint64_t key(const Item& a) { return a.E; }      // a prefix of prec
  // theta as the bits of the double b / Cmax: order-exact (b < 2^16, Cmax < 2^32: distinct
  // fractions differ by a relative >= 2^-48 > 2^-53; equal fractions give equal doubles)
  static __device__ __forceinline__ unsigned long long thkey(const Item& a) {
    return a.c ? (unsigned long long)__double_as_longlong((double)a.b / (double)a.c) : 0x7FF0000000000000ull;
  }
  static __device__ __forceinline__ Th theta(const Item& a) { return Th{a.b, a.c}; }
  static __device__ __forceinline__ bool gt(const Th& x, const Th& y) {
    return (uint64_t)x.b * y.c > (uint64_t)y.b * x.c;
  }
  static __device__ __forceinline__ Th zero() { return Th{0, 1}; }
  static __device__ __forceinline__ Th shfl_up(const Th& t, int d) {
    return Th{__shfl_up_sync(0xffffffffu, t.b, d), __shfl_up_sync(0xffffffffu, t.c, d)};
  }
  static __device__ __forceinline__ Th shfl(const Th& t, int src) {
    return Th{__shfl_sync(0xffffffffu, t.b, src), __shfl_sync(0xffffffffu, t.c, src)};
  }
  static __device__ __forceinline__ void finalize(Rec&) {}
};

// Per-stage batch (ppipe_point_pb, App. A.1): theta = min_d b_d / C_d compared as the
// bit pattern of the double (exact order for b < 2^16, C < 2^28: distinct fractions
// differ by a relative >= 2^-44 >> 2^-53; PB-3); ties by the batch indices
// (b_1..b_K) lexicographic, then (c_1, c_2) (reading PB-4).
struct PbTraits {
  static constexpr int kMode = kStaircase;
  using Rec = ppipe_point_pb;
  struct Item {
    uint32_t E, hi, lo, bidx, cuts;
  };
  using Th = unsigned long long;
  using Params = UniTraits::Params;
  static __device__ __forceinline__ double stage_th(uint32_t b, uint32_t Cd) {
    return Cd > 0 ? (double)b / (double)Cd : __longlong_as_double(0x7FF0000000000000ll);
  }
  static __device__ __forceinline__ Item item_of(const Rec& p, const Params& q) {
    const int K = min((int)p.K, 3);
    double th = stage_th(q.batches[min((int)p.bidx[0], q.B - 1)], p.stage_us[0]);
    for (int d = 1; d < K; ++d) th = fmin(th, stage_th(q.batches[min((int)p.bidx[d], q.B - 1)], p.stage_us[d]));
    const unsigned long long k = (unsigned long long)__double_as_longlong(th);
    return Item{p.e2e_us, (uint32_t)(k >> 32), (uint32_t)k,
                (uint32_t)p.bidx[0] << 16 | (uint32_t)p.bidx[1] << 8 | p.bidx[2],
                (uint32_t)p.cut[0] << 16 | p.cut[1]};
  }
  static __device__ __forceinline__ Th thkey(const Item& a) { return (unsigned long long)a.hi << 32 | a.lo; }
  static __device__ __forceinline__ uint64_t key(const Item& a) { return a.E; }
  static __device__ __forceinline__ bool prec(const Item& a, const Item& b) {
    if (a.E != b.E) return a.E < b.E;
    const Th ka = thkey(a), kb = thkey(b);
    if (ka != kb) return ka > kb;
    if (a.bidx != b.bidx) return a.bidx < b.bidx;
    return a.cuts < b.cuts;
  }
  static __device__ __forceinline__ uint32_t primary(const Item& a) { return a.E; }
  static __device__ __forceinline__ Th theta(const Item& a) { return thkey(a); }
  static __device__ __forceinline__ bool gt(const Th& x, const Th& y) { return x > y; }
  static __device__ __forceinline__ Th zero() { return 0ull; }
  static __device__ __forceinline__ Th shfl_up(const Th& t, int d) { return __shfl_up_sync(0xffffffffu, t, d); }
  static __device__ __forceinline__ Th shfl(const Th& t, int src) { return __shfl_sync(0xffffffffu, t, src); }
  static __device__ __forceinline__ void finalize(Rec&) {}
};

// F2 (MILP-lossless frontier, ppipe_pareto_f2) finalize, pass 1: candidates with an
// identical per-stage throughput vector x = (b / C_1, .., b / C_K) are the same point
// for the MILP (eqs. 1.10 / 1.13); of each such run the smallest
// (E, b, c_1, c_2) stays (reading F2-2). Identical vectors <=> proportional (b, C_1..C_K)
// <=> equal tuples after dividing by g = gcd(b, C_1..C_K) (C_d = 0 stays 0: +inf).
struct F2DedupTraits {
  static constexpr int kMode = kFirstOfGroup;
  using Rec = ppipe_point;
  struct Item {
    uint32_t h, vb, v1, v2, v3, E, b, cuts;
  };
  using Th = uint32_t;
  using Params = UniTraits::Params;
  static __device__ __forceinline__ uint32_t gcd32(uint32_t a, uint32_t b) {
    while (b) {
      const uint32_t t = a % b;
      a = b;
      b = t;
    }
    return a;
  }
  static __device__ __forceinline__ Item item_of(const Rec& p, const Params&) {
    uint32_t g = p.batch;
    for (int d = 0; d < p.K; ++d) g = gcd32(g, p.stage_us[d]);
    const uint32_t vb = p.batch / g, v1 = p.stage_us[0] / g, v2 = p.stage_us[1] / g, v3 = p.stage_us[2] / g;
    return Item{mix(vb, v1, v2, v3), vb, v1, v2, v3, p.e2e_us, p.batch, (uint32_t)p.cut[0] << 16 | p.cut[1]};
  }
  static __device__ __forceinline__ bool same(const Item& a, const Item& b) {
    return a.vb == b.vb && a.v1 == b.v1 && a.v2 == b.v2 && a.v3 == b.v3;
  }
  // a hash of the reduced vector, so that a large segment splits evenly by key ranges
  static __device__ __forceinline__ uint32_t mix(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    uint32_t h = a * 0x9E3779B1u;
    h = (h ^ (h >> 15) ^ b) * 0x85EBCA77u;
    h = (h ^ (h >> 13) ^ c) * 0xC2B2AE3Du;
    h = (h ^ (h >> 16) ^ d) * 0x27D4EB2Fu;
    return h ^ (h >> 15);
  }
  // runs of equal vectors are contiguous under any order that compares the vector
  // right after a function of it (the hash); pass 2 restores the canonical order
  static __device__ __forceinline__ uint32_t primary(const Item& a) { return a.h; }
  static __device__ __forceinline__ uint64_t key(const Item& a) { return a.h; }
  static __device__ __forceinline__ bool prec(const Item& a, const Item& b) {
    if (a.h != b.h) return a.h < b.h;
    if (a.v1 != b.v1) return a.v1 < b.v1;
    if (a.v2 != b.v2) return a.v2 < b.v2;
    if (a.v3 != b.v3) return a.v3 < b.v3;
    if (a.vb != b.vb) return a.vb < b.vb;
    if (a.E != b.E) return a.E < b.E;
    if (a.b != b.b) return a.b < b.b;
    return a.cuts < b.cuts;
  }
  static __device__ __forceinline__ Th zero() { return 0; }
  static __device__ __forceinline__ void finalize(Rec&) {}
};

// F2 finalize, pass 2: canonical output order (b, c_1, c_2) per segment (reading
// F2-3); the survivors' tie flag (reserved) is cleared.
struct F2OrderTraits {
  static constexpr int kMode = kKeepAll;
  using Rec = ppipe_point;
  struct Item {
    uint32_t b, cuts;
  };
  using Th = uint32_t;
  using Params = UniTraits::Params;
  static __device__ __forceinline__ Item item_of(const Rec& p, const Params&) {
    return Item{p.batch, (uint32_t)p.cut[0] << 16 | p.cut[1]};
  }
  static __device__ __forceinline__ uint32_t primary(const Item& a) { return a.b << 16 | a.cuts >> 16; }
  static __device__ __forceinline__ uint64_t key(const Item& a) {  // b, c_1, c_2 (M <= 4096 for F2)
    return (uint64_t)a.b << 24 | (a.cuts >> 16) << 12 | (a.cuts & 0xfffu);
  }
  static __device__ __forceinline__ bool prec(const Item& a, const Item& b) {
    return a.b != b.b ? a.b < b.b : a.cuts < b.cuts;
  }
  static __device__ __forceinline__ Th zero() { return 0; }
  static __device__ __forceinline__ void finalize(Rec& r) { r.reserved = 0; }
};

// ---------------------------------------------------------------------------
// exclusive scan of uint32 counts into uint64 offsets: out[i] = sum_{j<i} in[j],
// out[n] = total. Three launches: per-tile scan, scan of tile totals, add.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t block_excl_sum(uint64_t v, uint64_t* total, uint64_t* sh /* [32] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t t = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    if (lane < nw) sh[lane] = t;
  }
  __syncthreads();
  const uint64_t before = warp ? sh[warp - 1] : 0;
  *total = sh[nw - 1];
  __syncthreads();
  return before + x - v;
}

__global__ void __launch_bounds__(kFpThreads) scan_tile_kernel(const uint32_t* in, uint64_t n, uint64_t* out,
                                                                uint64_t* partial) {
  __shared__ uint64_t sh[32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanPerThread;
  uint32_t v[kScanPerThread];
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanPerThread; ++i) {
    v[i] = base + i < n ? in[base + i] : 0u;
    s += v[i];
  }
  uint64_t tot;
  uint64_t run = block_excl_sum(s, &tot, sh);
#pragma unroll
  for (int i = 0; i < kScanPerThread; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// single CTA: exclusive scan of the tile totals in place (chunks of blockDim with a
// carry); out[n] = the grand total
__global__ void __launch_bounds__(1024) scan_partials_kernel(uint64_t* partial, uint64_t n_tiles, uint64_t* out,
                                                              uint64_t n) {
  __shared__ uint64_t sh[32];
  uint64_t carry = 0;
  for (uint64_t b = 0; b < n_tiles; b += blockDim.x) {
    const uint64_t i = b + threadIdx.x;
    const uint64_t v = i < n_tiles ? partial[i] : 0;
    uint64_t tot;
    const uint64_t ex = block_excl_sum(v, &tot, sh);
    if (i < n_tiles) partial[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) out[n] = carry;
}

__global__ void scan_add_kernel(uint64_t* out, uint64_t n, const uint64_t* partial) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += partial[i / kScanTile];
}

// ---------------------------------------------------------------------------
// 1. count, 3. scatter
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kFpThreads) fp_count_kernel(const typename T::Rec* in, uint64_t n,
                                                               const uint64_t* seg_base, int C, uint32_t* cnt,
                                                               uint2* segrank) {
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); w0 < n; w0 += stride) {
    const uint64_t i = w0 + lane;
    const bool valid = i < n;
    const uint32_t seg = valid ? (uint32_t)seg_of_rec(in[i], seg_base, C) : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, seg);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader && valid) base = atomicAdd(&cnt[seg], (uint32_t)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (valid) segrank[i] = make_uint2(seg, base + (uint32_t)__popc(peers & lanemask_lt_()));
  }
}

template <class T>
__global__ void __launch_bounds__(kFpThreads) fp_scatter_kernel(const typename T::Rec* in, uint64_t n,
                                                                 const uint2* segrank, const uint64_t* start,
                                                                 typename T::Params q, typename T::Item* items,
                                                                 uint32_t* idx) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint2 sr = segrank[i];
    const uint64_t pos = start[sr.x] + sr.y;
    items[pos] = T::item_of(in[i], q);
    idx[pos] = (uint32_t)i;
  }
}

// ---------------------------------------------------------------------------
// block-level staircase over a sorted sequence: element p of the segment sits at
// position pos(p); keep it iff theta strictly exceeds the prefix maximum of every
// element before it (carried across tiles). Appends the record indices of the kept
// elements to kept[count..]; returns the new count. Every thread of the CTA calls it.
// ---------------------------------------------------------------------------
template <class T>
struct BlockStairSmem {
  typename T::Th warp_max[kFpThreads / 32];
  uint32_t warp_keep[kFpThreads / 32];
};

template <class T, class ItemAt>
__device__ uint32_t block_staircase(ItemAt item_at, uint32_t n, const uint32_t* idx_of_pos, uint32_t* kept,
                                    uint32_t count, typename T::Th& carry, BlockStairSmem<T>& sm) {
  using Th = typename T::Th;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint32_t t0 = 0; t0 < n; t0 += blockDim.x) {
    const uint32_t p = t0 + threadIdx.x;
    const bool valid = p < n;
    uint32_t pos = 0;
    Th th = T::zero();
    bool keep = false;
    if constexpr (T::kMode == kStaircase) {
      if (valid) th = T::theta(item_at(p, &pos));
      // inclusive warp max-scan
      Th incl = th;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const Th o = T::shfl_up(incl, d);
        if (lane >= d && T::gt(o, incl)) incl = o;
      }
      if (lane == 31) sm.warp_max[warp] = incl;
      __syncthreads();
      Th before = carry;  // max of everything before this warp's first element
      for (int w = 0; w < warp; ++w)
        if (T::gt(sm.warp_max[w], before)) before = sm.warp_max[w];
      Th excl = T::shfl_up(incl, 1);
      if (lane == 0 || T::gt(before, excl)) excl = before;
      keep = valid && T::gt(th, excl);
    } else {
      if (valid) {
        const auto it = item_at(p, &pos);
        keep = true;
        if constexpr (T::kMode == kFirstOfGroup) {
          uint32_t pp;
          if (p > 0) keep = !T::same(item_at(p - 1, &pp), it);
        }
      }
      __syncthreads();
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) sm.warp_keep[warp] = __popc(bal);
    __syncthreads();
    uint32_t off = count, tot = 0;
    for (int w = 0; w < nw; ++w) {
      const uint32_t k = sm.warp_keep[w];
      if (w < warp) off += k;
      tot += k;
    }
    if (keep) kept[off + __popc(bal & lanemask_lt_())] = idx_of_pos[pos];
    count += tot;
    if constexpr (T::kMode == kStaircase)
      for (int w = 0; w < nw; ++w)
        if (T::gt(sm.warp_max[w], carry)) carry = sm.warp_max[w];
    __syncthreads();
  }
  return count;
}

// ---------------------------------------------------------------------------
// bitonic sort of a permutation under the full order T::prec (positions >= n are
// +inf): the chunk sorts of the last-resort global-memory path
// ---------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ bool before_pos(const typename T::Item* it, uint32_t a, uint32_t b, uint32_t n) {
  if (a >= n) return false;
  if (b >= n) return true;
  return T::prec(it[a], it[b]);
}

template <class T>
__device__ void block_bitonic(const typename T::Item* it, uint16_t* perm, uint32_t n) {
  uint32_t P2 = 32;
  while (P2 < n) P2 <<= 1;
  for (uint32_t i = threadIdx.x; i < P2; i += blockDim.x) perm[i] = (uint16_t)i;
  __syncthreads();
  for (uint32_t k = 2; k <= P2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < P2 / 2; t += blockDim.x) {
        const uint32_t i = 2 * j * (t / j) + (t % j), l = i + j;
        const uint32_t a = perm[i], b = perm[l];
        const bool asc = (i & k) == 0;
        if (asc ? before_pos<T>(it, b, a, n) : before_pos<T>(it, a, b, n)) {
          perm[i] = (uint16_t)b;
          perm[l] = (uint16_t)a;
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// 4./5. sort by key, then select. Every item gets the unique 64-bit sort key
// T::key(item) << 12 | local index; T::key is a prefix of the total order T::prec
// (E for the staircase), so after the sort only runs of equal T::key ("groups",
// rare: equal E) need the full order. Selection at sorted position p:
//   staircase      p is the best of its group under T::prec, and its theta exceeds
//                  the maximum theta M[g - 1] of every position before its group
//                  (for a group of one: the plain exclusive prefix maximum)
//   first-of-group no earlier item (under T::prec) of its group is T::same
//   keep-all       always
// ---------------------------------------------------------------------------
constexpr int kFpWarpsPerCta = kFpThreads / 32;
template <class T>
__host__ __device__ constexpr size_t small_warp_bytes() {  // items, sorted keys, prefix maxima
  return (sizeof(typename T::Item) * kFpWarpMax + 8 * kFpWarpMax + sizeof(typename T::Th) * kFpWarpMax + 15) / 16 * 16;
}
constexpr int kIdxBits = 12;
constexpr uint32_t kFpBucketMax = 48;  // keys per bucket the insertion sort accepts
constexpr uint32_t kTierSample = 256;  // keys sampled per segment for the bucket splitters  // local index bits of a sort key (segments <= kFpCap = 4096 items)
static_assert((1 << kIdxBits) >= kFpCap, "sort keys carry the local index");

template <class T>
__device__ __forceinline__ uint64_t sort_key(const typename T::Item& it, uint32_t i) {
  return T::key(it) << kIdxBits | i;
}

// Group handling at sorted position p (tie with a neighbour). sk: sorted keys, item(i):
// the item of local index i. Returns whether p is selected among its group.
template <class T, class ItemOf>
__device__ bool group_pick(uint32_t p, uint32_t n, const uint64_t* sk, ItemOf item, uint32_t* g_out) {
  const uint64_t K = sk[p] >> kIdxBits;
  uint32_t g = p, e = p;
  while (g > 0 && (sk[g - 1] >> kIdxBits) == K) --g;
  while (e + 1 < n && (sk[e + 1] >> kIdxBits) == K) ++e;
  *g_out = g;
  const auto me = item((uint32_t)(sk[p] & ((1u << kIdxBits) - 1)));
  for (uint32_t q = g; q <= e; ++q) {
    if (q == p) continue;
    const auto o = item((uint32_t)(sk[q] & ((1u << kIdxBits) - 1)));
    if constexpr (T::kMode == kStaircase) {
      if (T::prec(o, me)) return false;  // not the best of its E
    } else {
      if (T::same(o, me) && T::prec(o, me)) return false;  // an earlier equal vector stays
    }
  }
  return true;
}

template <class T>
__global__ void __launch_bounds__(kFpThreads) fp_small_kernel(const typename T::Item* items, const uint32_t* idx,
                                                               const uint64_t* start, uint64_t n_seg,
                                                               uint32_t* kept, uint32_t* kc, typename T::Th* tmax,
                                                               uint32_t* large, uint4* huge, unsigned long long* ctr) {
  using Item = typename T::Item;
  using Th = typename T::Th;
  extern __shared__ __align__(16) unsigned char fp_dyn[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t s = (uint64_t)blockIdx.x * kFpWarpsPerCta + warp;
  if (s >= n_seg) return;
  const uint64_t lo = start[s];
  const uint32_t n = (uint32_t)(start[s + 1] - lo);
  if (n > (uint32_t)kFpWarpMax) {
    if (lane == 0) {
      if (n > (uint32_t)kFpCap) huge[atomicAdd(&ctr[1], 1ull)] = make_uint4((uint32_t)s, (uint32_t)lo, n, 0u);
      else if (n > (uint32_t)kFpMid) large[n_seg + atomicAdd(&ctr[4], 1ull)] = (uint32_t)s;
      else large[atomicAdd(&ctr[0], 1ull)] = (uint32_t)s;
      atomicMax(&ctr[2], (unsigned long long)n);
    }
    return;
  }
  if (n == 0) {
    if (lane == 0) {
      kc[s] = 0;
      if (tmax) tmax[s] = T::zero();
    }
    return;
  }
  unsigned char* base = fp_dyn + (size_t)warp * small_warp_bytes<T>();
  Item* it = reinterpret_cast<Item*>(base);
  uint64_t* sk = reinterpret_cast<uint64_t*>(base + sizeof(Item) * kFpWarpMax);
  uint32_t* k32 = reinterpret_cast<uint32_t*>(sk);  // the unsorted 32-bit keys share sk's space
  Th* Msm = reinterpret_cast<Th*>(base + sizeof(Item) * kFpWarpMax + 8 * kFpWarpMax);
  const int nr = (int)((n + 31) >> 5);
  uint64_t kmin = ~0ull, kmax = 0;
  for (uint32_t i = lane; i < n; i += 32) {
    const Item x = items[lo + i];
    it[i] = x;
    const uint64_t K = T::key(x);
    kmin = min(kmin, K);
    kmax = max(kmax, K);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    kmin = min(kmin, (uint64_t)__shfl_xor_sync(0xffffffffu, kmin, d));
    kmax = max(kmax, (uint64_t)__shfl_xor_sync(0xffffffffu, kmax, d));
  }
  __syncwarp();
  uint32_t rank[kFpWarpR];
#pragma unroll
  for (int r = 0; r < kFpWarpR; ++r) rank[r] = 0;
  if (kmax - kmin < (1ull << (32 - 7))) {
    // 32-bit keys (K - Kmin) << 7 | i: rank = how many keys are smaller
    uint32_t mine[kFpWarpR];
#pragma unroll
    for (int r = 0; r < kFpWarpR; ++r) {
      const uint32_t i = lane + 32 * r;
      mine[r] = (r < nr && i < n) ? (uint32_t)(T::key(it[i]) - kmin) << 7 | i : 0xffffffffu;
    }
    const uint32_t n4 = (n + 3) & ~3u;
    for (uint32_t i = n + lane; i < n4; i += 32) k32[i] = 0xffffffffu;
#pragma unroll
    for (int r = 0; r < kFpWarpR; ++r) {
      const uint32_t i = lane + 32 * r;
      if (r < nr && i < n) k32[i] = mine[r];
    }
    __syncwarp();
    for (uint32_t j = 0; j < n4; j += 4) {
      const uint4 y = *reinterpret_cast<const uint4*>(k32 + j);
#pragma unroll
      for (int r = 0; r < kFpWarpR; ++r)
        if (r < nr) rank[r] += (y.x < mine[r]) + (y.y < mine[r]) + (y.z < mine[r]) + (y.w < mine[r]);
    }
  } else {
    uint64_t mine[kFpWarpR];
#pragma unroll
    for (int r = 0; r < kFpWarpR; ++r) {
      const uint32_t i = lane + 32 * r;
      mine[r] = (r < nr && i < n) ? sort_key<T>(it[i], i) : ~0ull;
      if (r < nr && i < n) sk[i] = mine[r];
    }
    __syncwarp();
    for (uint32_t j = 0; j < n; ++j) {
      const uint64_t y = sk[j];
#pragma unroll
      for (int r = 0; r < kFpWarpR; ++r)
        if (r < nr) rank[r] += y < mine[r] ? 1u : 0u;
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < kFpWarpR; ++r) {
    const uint32_t i = lane + 32 * r;
    if (r < nr && i < n) sk[rank[r]] = sort_key<T>(it[i], i);
  }
  __syncwarp();
  auto item = [&](uint32_t i) { return it[i]; };
  Th carry = T::zero();
  uint32_t count = 0;
  for (int r = 0; r < nr; ++r) {
    const uint32_t p = lane + 32 * r;
    const bool valid = p < n;
    const uint64_t key = valid ? sk[p] : 0ull;
    const uint32_t i = (uint32_t)(key & ((1u << kIdxBits) - 1));
    const bool tie = valid && ((p > 0 && (sk[p - 1] >> kIdxBits) == (key >> kIdxBits)) ||
                               (p + 1 < n && (sk[p + 1] >> kIdxBits) == (key >> kIdxBits)));
    bool keep = valid;
    if constexpr (T::kMode == kStaircase) {
      const Th th = valid ? T::theta(it[i]) : T::zero();
      Th incl = th;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const Th o = T::shfl_up(incl, d);
        if (lane >= d && T::gt(o, incl)) incl = o;
      }
      Th excl = T::shfl_up(incl, 1);
      if (lane == 0 || T::gt(carry, excl)) excl = carry;
      Th m = incl;
      if (T::gt(carry, m)) m = carry;
      if (valid) Msm[p] = m;
      __syncwarp();
      if (tie) {
        uint32_t g;
        keep = group_pick<T>(p, n, sk, item, &g);
        if (keep) keep = T::gt(th, g > 0 ? Msm[g - 1] : T::zero());
      } else {
        keep = valid && T::gt(th, excl);
      }
      const Th last = T::shfl(m, 31);
      if (T::gt(last, carry)) carry = last;
    } else if constexpr (T::kMode == kFirstOfGroup) {
      if (tie) {
        uint32_t g;
        keep = group_pick<T>(p, n, sk, item, &g);
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) kept[lo + count + __popc(bal & lanemask_lt_())] = idx[lo + i];
    count += __popc(bal);
  }
  if (lane == 0) {
    kc[s] = count;
    if (tmax) tmax[s] = carry;
  }
}

// CTA path: bitonic sort of the 64-bit keys in shared memory, then the selection
// tile by tile (block prefix maximum with a carry, ballot compaction). Items are read
// from global memory at their sorted positions. Persistent CTAs over the list.
// Shared memory of a CTA-path kernel with capacity CAP: sorted keys, prefix maxima,
// bucket counts [CAP + 1], per-item bucket ranks and ids.
template <class T>
__host__ __device__ constexpr size_t tier_smem(int cap) {
  return sizeof(uint64_t) * cap + sizeof(typename T::Th) * cap + 4 * (cap + 4) + 4 * cap;
}

// Two tiers: (kFpWarpMax, kFpMid] with 128-thread CTAs (many per SM: the per-segment
// steps are latency-bound) and (kFpMid, kFpCap] with 256-thread CTAs.
// LIST 0: medium list, counters ctr[0] (count) / ctr[3] (work); LIST 1: large list,
// ctr[4] / ctr[5].
template <class T, int NT, int CAP, int LIST>
__global__ void __launch_bounds__(NT) fp_tier_kernel(const typename T::Item* items, const uint32_t* idx,
                                                     const uint64_t* start, const uint32_t* large,
                                                     unsigned long long* ctr, uint32_t* kept, uint32_t* kc,
                                                     typename T::Th* tmax) {
  using Th = typename T::Th;
  extern __shared__ __align__(16) unsigned char fp_dyn[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(fp_dyn);
  Th* Msm = reinterpret_cast<Th*>(fp_dyn + 8 * CAP);
  unsigned long long* fold = reinterpret_cast<unsigned long long*>(Msm);  // E-bucket fold (staircase), aliases Msm
  uint32_t* bcnt = reinterpret_cast<uint32_t*>(fp_dyn + 8 * CAP + sizeof(Th) * CAP);  // [CAP + 1]
  uint16_t* rk = reinterpret_cast<uint16_t*>(bcnt + CAP + 4);
  uint16_t* bid = rk + CAP;
  uint16_t* surv = reinterpret_cast<uint16_t*>(sk);  // fold survivors' local indices (before the key sort)
  __shared__ Th warp_max[NT / 32];
  __shared__ uint32_t warp_keep[NT / 32];
  __shared__ uint64_t red_max[NT / 32];
  __shared__ uint32_t cur, crowded, n_surv;
  __shared__ uint64_t smp[kTierSample], spl[kTierSample];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t n_large = (uint32_t)ctr[LIST ? 4 : 0];
  for (;;) {
    if (threadIdx.x == 0) cur = (uint32_t)atomicAdd(&ctr[LIST ? 5 : 3], 1ull);
    __syncthreads();
    const uint32_t q = cur;
    __syncthreads();
    if (q >= n_large) return;
    const uint32_t s = large[q];
    const uint64_t lo = start[s];
    const uint32_t n0 = (uint32_t)(start[s + 1] - lo);
    const typename T::Item* its = items + lo;
    // Buckets at the quantiles of a sorted sample of the keys (robust to clustered E:
    // the score kernels' folds leave survivors in narrow E bands). bucket(K) = number of
    // splitters <= K, monotone in K; nb buckets of about n0 / nb keys each.
    for (uint32_t t = threadIdx.x; t < kTierSample; t += blockDim.x)
      smp[t] = T::key(its[(uint32_t)((uint64_t)t * n0 / kTierSample)]);
    if (threadIdx.x == 0) {
      crowded = 0;
      n_surv = 0;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= kTierSample; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t t = threadIdx.x; t < kTierSample / 2; t += blockDim.x) {
          const uint32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), l = i + j;
          const uint64_t x = smp[i], y = smp[l];
          if (((i & k) == 0) ? (y < x) : (x < y)) {
            smp[i] = y;
            smp[l] = x;
          }
        }
        __syncthreads();
      }
    }
    const uint32_t nb = max(1u, min(kTierSample, n0 / 4));
    for (uint32_t t = threadIdx.x; t + 1 < nb; t += blockDim.x) spl[t] = smp[(t + 1) * kTierSample / nb];
    if constexpr (T::kMode == kStaircase)
      for (uint32_t t = threadIdx.x; t < nb; t += blockDim.x) fold[t] = 0ull;
    __syncthreads();
    auto bucket_of = [&](uint64_t K) {
      uint32_t lo2 = 0, hi2 = nb - 1;
      while (lo2 < hi2) {
        const uint32_t mid = (lo2 + hi2) >> 1;
        if (spl[mid] <= K) lo2 = mid + 1;
        else hi2 = mid;
      }
      return lo2;
    };
    uint32_t n = n0;
    if constexpr (T::kMode == kStaircase) {
      // E-bucket fold: an item whose theta does not exceed the best theta of a strictly
      // earlier E bucket is dominated (smaller E, theta at least as good); drop it.
      for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) {
        const uint32_t b = bucket_of(T::key(its[i]));
        bid[i] = (uint16_t)b;
        atomicMax(&fold[b], T::thkey(its[i]));
      }
      __syncthreads();
      {  // exclusive prefix maximum over the nb buckets (blocked)
        const uint32_t per = (nb + blockDim.x - 1) / blockDim.x, b0 = threadIdx.x * per;
        unsigned long long mx = 0ull;
        for (uint32_t b = b0; b < b0 + per && b < nb; ++b) mx = max(mx, fold[b]);
        unsigned long long x = mx;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x = max(x, y);
        }
        if (lane == 31) red_max[warp] = x;
        __syncthreads();
        unsigned long long run = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) run = 0ull;
        for (int w = 0; w < warp; ++w) run = max(run, (unsigned long long)red_max[w]);
        __syncthreads();
        for (uint32_t b = b0; b < b0 + per && b < nb; ++b) {
          const unsigned long long v = fold[b];
          fold[b] = run;
          run = max(run, v);
        }
      }
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) {
        const bool keep = T::thkey(its[i]) > fold[bid[i]];
        const unsigned bal = __ballot_sync(__activemask(), keep);
        uint32_t base = 0;
        const int leader = __ffs(__activemask()) - 1;
        if (lane == leader) base = atomicAdd(&n_surv, (uint32_t)__popc(bal));
        base = __shfl_sync(__activemask(), base, leader);
        if (keep) surv[base + __popc(bal & lanemask_lt_())] = (uint16_t)i;
      }
      __syncthreads();
      n = n_surv;
      // the survivors' local indices move from sk's space into rk's (sk is rebuilt below)
      for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) rk[j] = surv[j];
      __syncthreads();
    }
    auto local = [&](uint32_t j) -> uint32_t {
      if constexpr (T::kMode == kStaircase) return rk[j];
      else return j;
    };
    // counting sort of the (surviving) keys by key range, insertion sort per bucket;
    // a crowded bucket sends the segment to a bitonic sort instead
    for (uint32_t b = threadIdx.x; b <= nb; b += blockDim.x) bcnt[b] = 0;
    __syncthreads();
    uint32_t myb[CAP / NT], myr[CAP / NT];
#pragma unroll
    for (int r = 0; r < CAP / NT; ++r) {
      const uint32_t j = threadIdx.x + r * NT;
      if (j < n) {
        if constexpr (T::kMode == kStaircase) myb[r] = bid[local(j)];
        else myb[r] = bucket_of(T::key(its[j]));
        myr[r] = atomicAdd(&bcnt[myb[r]], 1u);
      }
    }
    __syncthreads();
    {  // exclusive scan of the nb bucket counts (blocked)
      const uint32_t per = (nb + blockDim.x - 1) / blockDim.x, b0 = threadIdx.x * per;
      uint32_t sum = 0;
      for (uint32_t b = b0; b < b0 + per && b < nb; ++b) sum += bcnt[b];
      uint32_t x = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (lane == 31) warp_keep[warp] = x;
      __syncthreads();
      uint32_t run = x - sum;
      for (int w = 0; w < warp; ++w) run += warp_keep[w];
      __syncthreads();
      for (uint32_t b = b0; b < b0 + per && b < nb; ++b) {
        const uint32_t c = bcnt[b];
        if (c > kFpBucketMax) crowded = 1;
        bcnt[b] = run;
        run += c;
      }
      if (threadIdx.x == blockDim.x - 1) bcnt[nb] = n;
    }
    __syncthreads();
    uint32_t P2 = 32;
    while (P2 < n) P2 <<= 1;
    if (!crowded) {
#pragma unroll
      for (int r = 0; r < CAP / NT; ++r) {
        const uint32_t j = threadIdx.x + r * NT;
        if (j < n) sk[bcnt[myb[r]] + myr[r]] = sort_key<T>(its[local(j)], local(j));
      }
      __syncthreads();
      for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
        const uint32_t b0 = bcnt[b], b1 = bcnt[b + 1];
        for (uint32_t x = b0 + 1; x < b1; ++x) {  // insertion sort of a few keys
          const uint64_t v = sk[x];
          uint32_t y = x;
          while (y > b0 && sk[y - 1] > v) {
            sk[y] = sk[y - 1];
            --y;
          }
          sk[y] = v;
        }
      }
      __syncthreads();
    } else {
      for (uint32_t j = threadIdx.x; j < P2; j += blockDim.x) sk[j] = j < n ? sort_key<T>(its[local(j)], local(j)) : ~0ull;
      __syncthreads();
      for (uint32_t k = 2; k <= P2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t t = threadIdx.x; t < P2 / 2; t += blockDim.x) {
            const uint32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), l = i + j;
            const uint64_t a = sk[i], b = sk[l];
            if (((i & k) == 0) ? (b < a) : (a < b)) {
              sk[i] = b;
              sk[l] = a;
            }
          }
          __syncthreads();
        }
      }
    }
    auto item = [&](uint32_t i) { return its[i]; };
    Th carry = T::zero();
    uint32_t count = 0;
    for (uint32_t t0 = 0; t0 < n; t0 += blockDim.x) {
      const uint32_t p = t0 + threadIdx.x;
      const bool valid = p < n;
      const uint64_t key = valid ? sk[p] : 0ull;
      const uint32_t i = (uint32_t)(key & ((1u << kIdxBits) - 1));
      const bool tie = valid && ((p > 0 && (sk[p - 1] >> kIdxBits) == (key >> kIdxBits)) ||
                                 (p + 1 < n && (sk[p + 1] >> kIdxBits) == (key >> kIdxBits)));
      bool keep = valid;
      if constexpr (T::kMode == kStaircase) {
        const Th th = valid ? T::theta(its[i]) : T::zero();
        Th incl = th;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const Th o = T::shfl_up(incl, d);
          if (lane >= d && T::gt(o, incl)) incl = o;
        }
        if (lane == 31) warp_max[warp] = incl;
        __syncthreads();
        Th before = carry;
        for (int w = 0; w < warp; ++w)
          if (T::gt(warp_max[w], before)) before = warp_max[w];
        Th excl = T::shfl_up(incl, 1);
        if (lane == 0 || T::gt(before, excl)) excl = before;
        Th m = incl;
        if (T::gt(before, m)) m = before;
        if (valid) Msm[p] = m;
        for (int w = 0; w < nw; ++w)
          if (T::gt(warp_max[w], carry)) carry = warp_max[w];
        __syncthreads();
        if (tie) {
          uint32_t g;
          keep = group_pick<T>(p, n, sk, item, &g);
          if (keep) keep = T::gt(th, g > 0 ? Msm[g - 1] : T::zero());
        } else {
          keep = valid && T::gt(th, excl);
        }
      } else if constexpr (T::kMode == kFirstOfGroup) {
        if (tie) {
          uint32_t g;
          keep = group_pick<T>(p, n, sk, item, &g);
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) warp_keep[warp] = __popc(bal);
      __syncthreads();
      uint32_t off = count, tot = 0;
      for (int w = 0; w < nw; ++w) {
        if (w < warp) off += warp_keep[w];
        tot += warp_keep[w];
      }
      if (keep) kept[lo + off + __popc(bal & lanemask_lt_())] = idx[lo + i];
      count += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      kc[s] = count;
      if (tmax) tmax[s] = carry;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// 6. huge segments (> kFpCap items): chunks sorted in shared memory, then merge
// rounds in global memory (each element finds its place in the partner run by a
// binary search: the order is strict and total), then the streamed staircase.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kFpThreads) fp_chunk_sort_kernel(const typename T::Item* items, uint32_t n,
                                                                    uint32_t* pos_out) {
  using Item = typename T::Item;
  extern __shared__ __align__(16) unsigned char fp_dyn[];
  Item* it = reinterpret_cast<Item*>(fp_dyn);
  uint16_t* perm = reinterpret_cast<uint16_t*>(fp_dyn + sizeof(Item) * kFpCap);
  const uint32_t c0 = blockIdx.x * (uint32_t)kFpCap;
  const uint32_t m = min((uint32_t)kFpCap, n - c0);
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) it[i] = items[c0 + i];
  __syncthreads();
  block_bitonic<T>(it, perm, m);
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) pos_out[c0 + i] = c0 + perm[i];
}

template <class T>
__global__ void fp_merge_kernel(const typename T::Item* items, uint32_t n, uint32_t width, const uint32_t* src,
                                uint32_t* dst) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t run = i / width, prun = run ^ 1u;
  const uint64_t p0 = (uint64_t)prun * width;
  if (p0 >= n) {
    dst[i] = src[i];
    return;
  }
  const uint32_t p1 = (uint32_t)min((uint64_t)n, p0 + width);
  const typename T::Item x = items[src[i]];
  uint32_t a = (uint32_t)p0, b = p1;  // first partner element not preceding x
  while (a < b) {
    const uint32_t mid = (a + b) >> 1;
    if (T::prec(items[src[mid]], x)) a = mid + 1;
    else b = mid;
  }
  const uint32_t ms = min(run, prun) * width;
  dst[ms + (i - run * width) + (a - (uint32_t)p0)] = src[i];
}

template <class T>
__global__ void __launch_bounds__(kFpThreads) fp_stream_kernel(const typename T::Item* items, const uint32_t* idx,
                                                                const uint32_t* sorted_pos, uint32_t n,
                                                                uint32_t* kept, uint32_t* kc_out,
                                                                typename T::Th* tmax_out) {
  __shared__ BlockStairSmem<T> sm;
  typename T::Th carry = T::zero();
  const uint32_t cnt = block_staircase<T>(
      [&](uint32_t p, uint32_t* pos) {
        *pos = sorted_pos[p];
        return items[*pos];
      },
      n, idx, kept, 0, carry, sm);
  if (threadIdx.x == 0) {
    *kc_out = cnt;
    if (tmax_out) *tmax_out = carry;
  }
}

// ---------------------------------------------------------------------------
// huge segments, batched: every segment with more than kFpCap items is split by
// ranges of its primary sort key (E for the staircase; monotone under the order)
// into nb sub-segments of about kHkTarget items (splitters at the quantiles of a
// sorted sample); the sub-segments run through the warp / CTA paths like segments;
// then (staircase) a locally kept item stays only if its theta also exceeds the
// maximum theta of every earlier sub-segment of its segment, and the sub-segments'
// kept lists are concatenated in order. Every step is spread over many CTAs:
// chunks of kHkChunk items for counting and scattering, a CTA per sub-segment for the
// filter and the gather.
// hdesc[2h] = {segment, lo, n, hoff}, hdesc[2h + 1] = {hbase, nb, 0, 0};
// hchunk[c] = {h, first item, end item, 0}.
// ---------------------------------------------------------------------------
constexpr uint32_t kHkSample = 2048;    // primary keys sampled per huge segment
constexpr uint32_t kHkTarget = 512;     // expected items per sub-segment (the medium path)
constexpr uint32_t kHkMaxSplit = 4096;  // sub-segments per huge segment
constexpr uint32_t kHkChunk = 4096;     // items per counting / scattering CTA

template <class T>
__global__ void __launch_bounds__(kFpThreads) hk_split_kernel(const typename T::Item* items, const uint4* hdesc,
                                                               uint32_t* spl, uint32_t* sub2h) {
  __shared__ uint32_t smp[kHkSample];
  const uint4 d0 = hdesc[2 * blockIdx.x], d1 = hdesc[2 * blockIdx.x + 1];
  const uint32_t lo = d0.y, n = d0.z, hbase = d1.x, nb = d1.y;
  for (uint32_t t = threadIdx.x; t < kHkSample; t += blockDim.x)
    smp[t] = T::primary(items[lo + (uint32_t)((uint64_t)t * n / kHkSample)]);
  __syncthreads();
  for (uint32_t k = 2; k <= kHkSample; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < kHkSample / 2; t += blockDim.x) {
        const uint32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), l = i + j;
        const uint32_t a = smp[i], b = smp[l];
        if (((i & k) == 0) ? (b < a) : (a < b)) {
          smp[i] = b;
          smp[l] = a;
        }
      }
      __syncthreads();
    }
  }
  // sub-segment b holds the keys with spl[b-1] <= key < spl[b] (equal keys share one)
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    if (b + 1 < nb) spl[hbase + b] = smp[(uint32_t)((uint64_t)(b + 1) * kHkSample / nb)];
    sub2h[hbase + b] = blockIdx.x;
  }
}

template <class T>
__global__ void __launch_bounds__(kFpThreads) hk_count_kernel(const typename T::Item* items, const uint4* hdesc,
                                                               const uint4* hchunk, const uint32_t* spl_g,
                                                               uint32_t* subcnt, uint2* hsr) {
  __shared__ uint32_t spl[kHkMaxSplit];
  const uint4 ch = hchunk[blockIdx.x];
  const uint4 d0 = hdesc[2 * ch.x], d1 = hdesc[2 * ch.x + 1];
  const uint32_t lo = d0.y, hoff = d0.w, hbase = d1.x, nb = d1.y;
  const int lane = threadIdx.x & 31;
  for (uint32_t b = threadIdx.x; b + 1 < nb; b += blockDim.x) spl[b] = spl_g[hbase + b];
  __syncthreads();
  for (uint32_t i0 = ch.y + (threadIdx.x & ~31u); i0 < ch.z; i0 += blockDim.x) {
    const uint32_t i = i0 + lane;
    const bool valid = i < ch.z;
    uint32_t sub = 0xffffffffu;
    if (valid) {
      const uint32_t key = T::primary(items[lo + i]);
      uint32_t a = 0, z = nb - 1;  // number of splitters <= key
      while (a < z) {
        const uint32_t mid = (a + z) >> 1;
        if (spl[mid] <= key) a = mid + 1;
        else z = mid;
      }
      sub = hbase + a;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, sub);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader && valid) base = atomicAdd(&subcnt[sub], (uint32_t)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (valid) hsr[hoff + i] = make_uint2(sub, base + (uint32_t)__popc(peers & lanemask_lt_()));
  }
}

template <class T>
__global__ void __launch_bounds__(kFpThreads) hk_scatter_kernel(const typename T::Item* items, const uint32_t* idx,
                                                                 const uint4* hdesc, const uint4* hchunk,
                                                                 const uint2* hsr, const uint64_t* substart,
                                                                 typename T::Item* hitems, uint32_t* hidx) {
  const uint4 ch = hchunk[blockIdx.x];
  const uint4 d0 = hdesc[2 * ch.x];
  const uint32_t lo = d0.y, hoff = d0.w;
  for (uint32_t i = ch.y + threadIdx.x; i < ch.z; i += blockDim.x) {
    const uint2 sr = hsr[hoff + i];
    const uint64_t pos = substart[sr.x] + sr.y;
    hitems[pos] = items[lo + i];
    hidx[pos] = idx[lo + i];
  }
}

// thread per huge segment, over its sub-segments in order: pre[sub] = the maximum theta
// of every earlier sub-segment of the segment (staircase only)
template <class T>
__global__ void hk_pre_kernel(const uint4* hdesc, uint32_t nh, const typename T::Th* tmax_sub,
                              typename T::Th* pre) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= nh) return;
  const uint4 d1 = hdesc[2 * h + 1];
  typename T::Th run = T::zero();
  for (uint32_t b = 0; b < d1.y; ++b) {
    pre[d1.x + b] = run;
    const typename T::Th t = tmax_sub[d1.x + b];
    if (T::gt(t, run)) run = t;
  }
}

// CTA per sub-segment: keep the locally kept items whose theta exceeds pre[sub]
// (staircase; other modes keep all), compacted in place; fcnt[sub] = how many
template <class T>
__global__ void __launch_bounds__(128) hk_filter_kernel(const typename T::Rec* in, typename T::Params q,
                                                        const uint64_t* substart, uint32_t* hkept,
                                                        const uint32_t* kc_sub, const typename T::Th* pre,
                                                        uint32_t* fcnt) {
  __shared__ uint32_t wk[4];
  const uint32_t sub = blockIdx.x, k = kc_sub[sub];
  const uint64_t base = substart[sub];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t count = 0;
  for (uint32_t t0 = 0; t0 < k; t0 += blockDim.x) {
    const uint32_t j = t0 + threadIdx.x;
    const bool valid = j < k;
    const uint32_t r = valid ? hkept[base + j] : 0u;
    bool keep = valid;
    if constexpr (T::kMode == kStaircase)
      if (valid) keep = T::gt(T::theta(T::item_of(in[r], q)), pre[sub]);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wk[warp] = __popc(bal);
    __syncthreads();  // every read of this tile precedes its writes (write index <= read index)
    uint32_t off = count, tot = 0;
    for (int w = 0; w < 4; ++w) {
      if (w < warp) off += wk[w];
      tot += wk[w];
    }
    if (keep) hkept[base + off + __popc(bal & lanemask_lt_())] = r;
    count += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) fcnt[sub] = count;
}

// thread per huge segment: output offsets of its sub-segments and the segment's count
__global__ void hk_offsets_kernel(const uint4* hdesc, uint32_t nh, const uint32_t* fcnt, uint32_t* suboff,
                                  uint32_t* kc) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= nh) return;
  const uint4 d0 = hdesc[2 * h], d1 = hdesc[2 * h + 1];
  uint32_t run = 0;
  for (uint32_t b = 0; b < d1.y; ++b) {
    suboff[d1.x + b] = run;
    run += fcnt[d1.x + b];
  }
  kc[d0.x] = run;
}

// CTA per sub-segment: its filtered list into the segment's kept range
__global__ void __launch_bounds__(128) hk_gather_kernel(const uint4* hdesc, const uint32_t* sub2h,
                                                        const uint64_t* substart, const uint32_t* hkept,
                                                        const uint32_t* fcnt, const uint32_t* suboff,
                                                        uint32_t* kept) {
  const uint32_t sub = blockIdx.x;
  const uint32_t lo = hdesc[2 * sub2h[sub]].y, n = fcnt[sub];
  const uint64_t src = substart[sub];
  uint32_t* dst = kept + lo + suboff[sub];
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = hkept[src + i];
}

// ---------------------------------------------------------------------------
// 8. compaction: CTA per chunk of kFpThreads output records (thread per record), so a
// few very large segments do not serialise; the chunk's first segment comes from one
// binary search over the output CSR, each thread walks forward from it
// ---------------------------------------------------------------------------
template <class T, class Rec = typename T::Rec>
__global__ void __launch_bounds__(kFpThreads) fp_compact_kernel(const Rec* in, const uint32_t* kept,
                                                                 const uint64_t* start, const uint64_t* out_off,
                                                                 uint64_t n_seg, Rec* out) {
  __shared__ uint64_t s0;
  const uint64_t total = out_off[n_seg];
  for (uint64_t c0 = (uint64_t)blockIdx.x * blockDim.x; c0 < total; c0 += (uint64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x == 0) {
      uint64_t lo = 0, hi = n_seg;  // last segment with out_off[s] <= c0
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (out_off[mid] <= c0) lo = mid;
        else hi = mid;
      }
      s0 = lo;
    }
    __syncthreads();
    const uint64_t i = c0 + threadIdx.x;
    if (i < total) {
      // galloping search from s0 for the segment holding i: a few steps for the usual
      // short distance, log steps across long runs of empty segments
      uint64_t sg = s0, step = 1;
      while (sg + step < n_seg && out_off[sg + step + 1] <= i) {
        sg += step;
        step <<= 1;
      }
      uint64_t hi = min(sg + step, n_seg - 1);  // out_off[hi + 1] > i
      while (sg < hi) {  // last s in [sg, hi] with out_off[s] <= i
        const uint64_t mid = (sg + hi + 1) >> 1;
        if (out_off[mid] <= i) sg = mid;
        else hi = mid - 1;
      }
      Rec r = in[kept[start[sg] + (i - out_off[sg])]];
      T::finalize(r);
      out[i] = r;
    }
    __syncthreads();
  }
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Scratch {
  char* base;
  size_t off;
  template <class X>
  X* take(size_t count) {
    X* p = reinterpret_cast<X*>(base ? base + off : nullptr);
    off = align_up(off + sizeof(X) * (count ? count : 1), 256);
    return p;
  }
};

cudaError_t ensure(FrontierScratch* s, size_t bytes) {
  if (s->bytes >= bytes) return cudaSuccess;
  if (s->buf) cudaFree(s->buf);
  s->buf = nullptr;
  s->bytes = 0;
  cudaError_t e = cudaMalloc(&s->buf, bytes);
  if (e != cudaSuccess) return e;
  s->bytes = bytes;
  return cudaSuccess;
}

// exclusive scan of n uint32 counts into out[0..n] (uint64); partial holds
// ceil(n / kScanTile) entries
cudaError_t scan_counts(const uint32_t* in, uint64_t n, uint64_t* out, uint64_t* partial, cudaStream_t s,
                        int* n_launches) {
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles) scan_tile_kernel<<<(unsigned)tiles, kFpThreads, 0, s>>>(in, n, out, partial);
  scan_partials_kernel<<<1, 1024, 0, s>>>(partial, tiles, out, n);
  if (tiles > 1) scan_add_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(out, n, partial);
  *n_launches += (tiles ? 1 : 0) + 1 + (tiles > 1 ? 1 : 0);
  return cudaGetLastError();
}

template <class T>
size_t small_smem() {
  return small_warp_bytes<T>() * kFpWarpsPerCta;
}

template <class T>
size_t large_smem() {  // fp_tier (large) and fp_chunk_sort (items + permutation)
  return std::max(tier_smem<T>(kFpCap), sizeof(typename T::Item) * kFpCap + sizeof(uint16_t) * kFpCap);
}

template <class T>
struct Level {  // one reduction level: segments (or sub-segments) of sorted-by-key items
  const typename T::Item* items;
  const uint32_t* idx;
  const uint64_t* start;
  uint64_t n_seg;
  uint32_t* kept;
  uint32_t* kc;
  typename T::Th* tmax;
  uint32_t* large;
  uint4* huge;
  unsigned long long* ctr;  // [0] large, [1] huge, [2] max size, [3] CTA-path work counter
};

template <class T>
cudaError_t launch_level(const Level<T>& L, cudaStream_t s, int* n_launches) {
  cudaError_t e = cudaMemsetAsync(L.ctr, 0, sizeof(unsigned long long) * 8, s);
  if (e != cudaSuccess || L.n_seg == 0) return e;
  const unsigned gs = (unsigned)((L.n_seg + kFpWarpsPerCta - 1) / kFpWarpsPerCta);
  fp_small_kernel<T><<<gs, kFpThreads, small_smem<T>(), s>>>(L.items, L.idx, L.start, L.n_seg, L.kept, L.kc, L.tmax,
                                                             L.large, L.huge, L.ctr);
  fp_tier_kernel<T, 128, kFpMid, 0><<<148 * 8, 128, tier_smem<T>(kFpMid), s>>>(L.items, L.idx, L.start, L.large,
                                                                                 L.ctr, L.kept, L.kc, L.tmax);
  fp_tier_kernel<T, kFpThreads, kFpCap, 1><<<148 * 2, kFpThreads, large_smem<T>(), s>>>(
      L.items, L.idx, L.start, L.large + L.n_seg, L.ctr, L.kept, L.kc, L.tmax);
  *n_launches += 3;
  return cudaGetLastError();
}

// The rare last resort for a (sub-)segment of more than kFpCap items that the key
// ranges could not split: chunk sorts, merge rounds in global memory, streamed
// staircase. items / idx / pos point at the segment's own range.
template <class T>
cudaError_t sort_reduce_one(const typename T::Item* items, const uint32_t* idx, uint32_t m, uint32_t* posA,
                            uint32_t* posB, uint32_t* kept, uint32_t* kc_out, typename T::Th* tmax_out,
                            cudaStream_t s, int* n_launches) {
  const unsigned chunks = (m + kFpCap - 1) / kFpCap;
  fp_chunk_sort_kernel<T><<<chunks, kFpThreads, large_smem<T>(), s>>>(items, m, posA);
  ++*n_launches;
  uint32_t *a = posA, *b = posB;
  for (uint32_t w = kFpCap; w < m; w *= 2) {
    fp_merge_kernel<T><<<(m + 255) / 256, 256, 0, s>>>(items, m, w, a, b);
    ++*n_launches;
    std::swap(a, b);
  }
  fp_stream_kernel<T><<<1, kFpThreads, 0, s>>>(items, idx, a, m, kept, kc_out, tmax_out);
  ++*n_launches;
  return cudaGetLastError();
}

template <class T>
cudaError_t frontier_generic(const typename T::Rec* in, uint64_t n, const uint64_t* seg_base, int C, uint64_t n_seg,
                             typename T::Params q, typename T::Rec* out, uint64_t* seg_offsets, uint64_t* n_out_host,
                             FrontierScratch* scratch, cudaStream_t s, int* n_launches) {
  using Item = typename T::Item;
  using Th = typename T::Th;
  if (n_seg >= 0xffffffffull || n >= 0xffffffffull) return cudaErrorInvalidValue;
  const uint64_t tiles = (n_seg + kScanTile - 1) / kScanTile + 1;
  const uint64_t max_huge = n / (kFpCap + 1) + 1, max_sub = n / kHkTarget + max_huge + 2;
  const uint64_t sub_tiles = (max_sub + kScanTile - 1) / kScanTile + 1;
  struct Arrays {
    uint32_t *cnt, *idx, *kept, *kc, *large, *posA, *posB, *hidx, *hkept, *subcnt, *kc_sub, *large2;
    uint32_t *spl, *sub2h, *fcnt, *suboff;
    uint64_t *start, *partial, *substart;
    uint2 *segrank, *hsr;
    Item *items, *hitems;
    unsigned long long *ctr, *ctr2;
    uint4 *huge, *huge2, *hdesc, *hchunk;
    Th *tmax_sub, *pre_sub;
  } A;
  auto layout = [&](Scratch& sc) {
    A.cnt = sc.take<uint32_t>(n_seg + 1);
    A.start = sc.take<uint64_t>(n_seg + 1);
    A.partial = sc.take<uint64_t>(std::max(tiles, sub_tiles));
    A.segrank = sc.take<uint2>(n);
    A.items = sc.take<Item>(n);
    A.idx = sc.take<uint32_t>(n);
    A.kept = sc.take<uint32_t>(n);
    A.kc = sc.take<uint32_t>(n_seg + 1);
    A.large = sc.take<uint32_t>(2 * n_seg);
    A.huge = sc.take<uint4>(max_huge);
    A.ctr = sc.take<unsigned long long>(8);
    A.ctr2 = sc.take<unsigned long long>(8);
    A.hdesc = sc.take<uint4>(2 * max_huge);
    A.subcnt = sc.take<uint32_t>(max_sub + 1);
    A.substart = sc.take<uint64_t>(max_sub + 1);
    A.kc_sub = sc.take<uint32_t>(max_sub + 1);
    A.tmax_sub = sc.take<Th>(max_sub + 1);
    A.pre_sub = sc.take<Th>(max_sub + 1);
    A.spl = sc.take<uint32_t>(max_sub + 1);
    A.sub2h = sc.take<uint32_t>(max_sub + 1);
    A.fcnt = sc.take<uint32_t>(max_sub + 1);
    A.suboff = sc.take<uint32_t>(max_sub + 1);
    A.hchunk = sc.take<uint4>(n / kHkChunk + max_huge + 1);
    A.large2 = sc.take<uint32_t>(2 * (max_sub + 1));
    A.huge2 = sc.take<uint4>(max_sub + 1);
    A.hsr = sc.take<uint2>(n);
    A.hitems = sc.take<Item>(n);
    A.hidx = sc.take<uint32_t>(n);
    A.hkept = sc.take<uint32_t>(n);
    A.posA = sc.take<uint32_t>(n);
    A.posB = sc.take<uint32_t>(n);
  };
  Scratch plan{nullptr, 0};
  layout(plan);
  cudaError_t e = ensure(scratch, plan.off);
  if (e != cudaSuccess) return e;
  Scratch sc{(char*)scratch->buf, 0};
  layout(sc);

  if ((e = cudaFuncSetAttribute(fp_tier_kernel<T, kFpThreads, kFpCap, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)large_smem<T>())) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(fp_tier_kernel<T, 128, kFpMid, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)tier_smem<T>(kFpMid))) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(fp_small_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)small_smem<T>())) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(fp_chunk_sort_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)large_smem<T>())) != cudaSuccess)
    return e;
  const char* dbgs = getenv("PPIPE_DEBUG_FLAGS");
  const bool dbg = dbgs && (atoi(dbgs) & 16);
  cudaEvent_t ev[6] = {};
  if (dbg)
    for (auto& x : ev) cudaEventCreate(&x);
  auto mark = [&](int i) {
    if (dbg) cudaEventRecord(ev[i], s);
  };
  mark(0);
  if ((e = cudaMemsetAsync(A.cnt, 0, sizeof(uint32_t) * (n_seg + 1), s)) != cudaSuccess) return e;
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + kFpThreads - 1) / kFpThreads, 148 * 8));
  if (n) {
    fp_count_kernel<T><<<g, kFpThreads, 0, s>>>(in, n, seg_base, C, A.cnt, A.segrank);
    ++*n_launches;
  }
  if ((e = scan_counts(A.cnt, n_seg, A.start, A.partial, s, n_launches)) != cudaSuccess) return e;
  unsigned long long h_ctr[3] = {0, 0, 0};
  if (n && n_seg) {
    fp_scatter_kernel<T><<<g, kFpThreads, 0, s>>>(in, n, A.segrank, A.start, q, A.items, A.idx);
    ++*n_launches;
    mark(1);
    const Level<T> L1{A.items, A.idx, A.start, n_seg, A.kept, A.kc, nullptr, A.large, A.huge, A.ctr};
    if ((e = launch_level(L1, s, n_launches)) != cudaSuccess) return e;
    mark(2);
    // the huge-segment count decides whether the batched split path runs
    if ((e = cudaMemcpyAsync(h_ctr, A.ctr, sizeof h_ctr, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  } else {
    if ((e = cudaMemsetAsync(A.kc, 0, sizeof(uint32_t) * (n_seg + 1), s)) != cudaSuccess) return e;
  }
  if (dbg)
      fprintf(stderr, "ppipe frontier: %llu records, %llu segments, large %llu, huge %llu, max %llu\n",
              (unsigned long long)n, (unsigned long long)n_seg, h_ctr[0], h_ctr[1], h_ctr[2]);
  mark(3);
  if (h_ctr[1]) {
    const uint32_t nh = (uint32_t)h_ctr[1];
    std::vector<uint4> hl(nh), hd(2 * (size_t)nh);
    if ((e = cudaMemcpyAsync(hl.data(), A.huge, sizeof(uint4) * nh, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    // PPIPE_FP_SPLIT (tests only): a fixed number of sub-segments per huge segment;
    // 1 sends every huge segment through the global-memory sort (sort_reduce_one)
    uint32_t split = 0;
    if (const char* v = getenv("PPIPE_FP_SPLIT")) split = (uint32_t)atoi(v);
    uint32_t hoff = 0, hbase = 0;
    std::vector<uint4> hc;
    for (uint32_t h = 0; h < nh; ++h) {
      const uint32_t m = hl[h].z, nb = std::min<uint32_t>(kHkMaxSplit, split ? split : (m + kHkTarget - 1) / kHkTarget);
      hd[2 * h] = make_uint4(hl[h].x, hl[h].y, m, hoff);
      hd[2 * h + 1] = make_uint4(hbase, nb, 0, 0);
      for (uint32_t i0 = 0; i0 < m; i0 += kHkChunk) hc.push_back(make_uint4(h, i0, std::min(m, i0 + kHkChunk), 0));
      hoff += m;
      hbase += nb;
    }
    const uint64_t S = hbase;
    const unsigned nchunk = (unsigned)hc.size();
    if ((e = cudaMemcpyAsync(A.hdesc, hd.data(), sizeof(uint4) * hd.size(), cudaMemcpyHostToDevice, s)) !=
        cudaSuccess)
      return e;
    if ((e = cudaMemcpyAsync(A.hchunk, hc.data(), sizeof(uint4) * hc.size(), cudaMemcpyHostToDevice, s)) !=
        cudaSuccess)
      return e;
    if ((e = cudaMemsetAsync(A.subcnt, 0, sizeof(uint32_t) * (S + 1), s)) != cudaSuccess) return e;
    hk_split_kernel<T><<<nh, kFpThreads, 0, s>>>(A.items, A.hdesc, A.spl, A.sub2h);
    hk_count_kernel<T><<<nchunk, kFpThreads, 0, s>>>(A.items, A.hdesc, A.hchunk, A.spl, A.subcnt, A.hsr);
    *n_launches += 2;
    if ((e = scan_counts(A.subcnt, S, A.substart, A.partial, s, n_launches)) != cudaSuccess) return e;
    hk_scatter_kernel<T><<<nchunk, kFpThreads, 0, s>>>(A.items, A.idx, A.hdesc, A.hchunk, A.hsr, A.substart,
                                                       A.hitems, A.hidx);
    ++*n_launches;
    const Level<T> L2{A.hitems, A.hidx, A.substart, S, A.hkept, A.kc_sub, A.tmax_sub, A.large2, A.huge2, A.ctr2};
    if ((e = launch_level(L2, s, n_launches)) != cudaSuccess) return e;
    unsigned long long c2[3] = {0, 0, 0};
    if ((e = cudaMemcpyAsync(c2, A.ctr2, sizeof c2, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if (dbg)
        fprintf(stderr, "ppipe frontier split: %u huge -> %llu sub-segments, large %llu, huge %llu, max %llu\n", nh,
                (unsigned long long)S, c2[0], c2[1], c2[2]);
    if (c2[1]) {
      std::vector<uint4> h2(c2[1]);
      if ((e = cudaMemcpyAsync(h2.data(), A.huge2, sizeof(uint4) * h2.size(), cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess)
        return e;
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      for (const uint4& d : h2)
        if ((e = sort_reduce_one<T>(A.hitems + d.y, A.hidx + d.y, d.z, A.posA + d.y, A.posB + d.y, A.hkept + d.y,
                                    A.kc_sub + d.x, A.tmax_sub + d.x, s, n_launches)) != cudaSuccess)
          return e;
    }
    if constexpr (T::kMode == kStaircase) {
      hk_pre_kernel<T><<<(nh + 127) / 128, 128, 0, s>>>(A.hdesc, nh, A.tmax_sub, A.pre_sub);
      ++*n_launches;
    }
    hk_filter_kernel<T><<<(unsigned)S, 128, 0, s>>>(in, q, A.substart, A.hkept, A.kc_sub, A.pre_sub, A.fcnt);
    hk_offsets_kernel<<<(nh + 127) / 128, 128, 0, s>>>(A.hdesc, nh, A.fcnt, A.suboff, A.kc);
    hk_gather_kernel<<<(unsigned)S, 128, 0, s>>>(A.hdesc, A.sub2h, A.substart, A.hkept, A.fcnt, A.suboff, A.kept);
    *n_launches += 3;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  mark(4);
  if ((e = scan_counts(A.kc, n_seg, seg_offsets, A.partial, s, n_launches)) != cudaSuccess) return e;
  if (n && n_seg) {
    fp_compact_kernel<T><<<(unsigned)std::min<uint64_t>((n + kFpThreads - 1) / kFpThreads, 148 * 16), kFpThreads, 0,
                           s>>>(in, A.kept, A.start, seg_offsets, n_seg, out);
    ++*n_launches;
  }
  uint64_t nk = 0;
  if ((e = cudaMemcpyAsync(&nk, seg_offsets + n_seg, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  mark(5);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  *n_out_host = nk;
  if (dbg) {
    float t[5] = {0, 0, 0, 0, 0};
    if (n && n_seg)
      for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    fprintf(stderr, "ppipe frontier ms: count+scan+scatter %.3f, level 1 %.3f, sync %.3f, split %.3f, tail %.3f\n",
            t[0], t[1], t[2], t[3], t[4]);
    for (auto& x : ev) cudaEventDestroy(x);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// SLO truncation (ppipe_frontier_at): per segment the prefix with E <= T_new[model]
// ---------------------------------------------------------------------------
__global__ void trunc_count_kernel(const ppipe_point* in, const uint64_t* off, uint64_t n_seg, const uint32_t* T_new,
                                   uint32_t* cnt) {
  const uint64_t sg = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (sg >= n_seg) return;
  uint64_t lo = off[sg], hi = off[sg + 1];
  if (lo == hi) {
    cnt[sg] = 0;
    return;
  }
  const uint32_t T = T_new[in[lo].model];
  const uint64_t base = lo;
  while (lo < hi) {  // first point with E > T (E ascends along a segment)
    const uint64_t mid = (lo + hi) >> 1;
    if (in[mid].e2e_us <= T) lo = mid + 1;
    else hi = mid;
  }
  cnt[sg] = (uint32_t)(lo - base);
}

__global__ void __launch_bounds__(kFpThreads) trunc_copy_kernel(const ppipe_point* in, const uint64_t* off_in,
                                                                 const uint64_t* off_out, uint64_t n_seg,
                                                                 ppipe_point* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t s = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_seg) return;
  const uint64_t src = off_in[s], dst = off_out[s], n = off_out[s + 1] - dst;
  for (uint64_t k = lane; k < n; k += 32) out[dst + k] = in[src + k];
}

}  // namespace

cudaError_t frontier_pass(const ppipe_point* in, uint64_t n, const uint64_t* seg_base_by_model, int C,
                          uint64_t n_seg, ppipe_point* out, uint64_t* seg_offsets, uint64_t* n_out_host,
                          FrontierScratch* scratch, cudaStream_t s, int* n_launches, uint32_t wpack) {
  return frontier_generic<UniTraits>(in, n, seg_base_by_model, C, n_seg, UniTraits::Params{wpack, nullptr, 1}, out,
                                     seg_offsets, n_out_host, scratch, s, n_launches);
}

cudaError_t pb_frontier_pass(const ppipe_point_pb* in, uint64_t n, const uint64_t* seg_base, int C, uint64_t n_seg,
                             const uint16_t* batches, int B, ppipe_point_pb* out, uint64_t* seg_offsets,
                             uint64_t* n_out_host, FrontierScratch* scratch, cudaStream_t s, int* n_launches) {
  return frontier_generic<PbTraits>(in, n, seg_base, C, n_seg, PbTraits::Params{0x11111111u, batches, B}, out,
                                    seg_offsets, n_out_host, scratch, s, n_launches);
}

// F2 survivors the query kernels could not rule out from having an identical vector carry
// a flag (reserved != 0); only those need the equal-vector pass. Split: flagged -> fl,
// unflagged -> un (two atomically advanced cursors; order is restored by the final sort).
__global__ void f2_split_kernel(const ppipe_point* in, uint64_t n, ppipe_point* fl, ppipe_point* un,
                                unsigned long long* cur) {
  const int lane = threadIdx.x & 31;
  for (uint64_t w0 = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); w0 < n;
       w0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = w0 + lane;
    const bool valid = i < n;
    ppipe_point p{};
    if (valid) p = in[i];
    const bool f = valid && p.reserved != 0;
    const unsigned bf = __ballot_sync(0xffffffffu, f), bu = __ballot_sync(0xffffffffu, valid && !f);
    unsigned long long bF = 0, bU = 0;
    if (lane == 0) {
      if (bf) bF = atomicAdd(&cur[0], (unsigned long long)__popc(bf));
      if (bu) bU = atomicAdd(&cur[1], (unsigned long long)__popc(bu));
    }
    bF = __shfl_sync(0xffffffffu, bF, 0);
    bU = __shfl_sync(0xffffffffu, bU, 0);
    if (f) fl[bF + __popc(bf & lanemask_lt_())] = p;
    else if (valid) un[bU + __popc(bu & lanemask_lt_())] = p;
  }
}

cudaError_t f2_finalize(const ppipe_point* in, uint64_t n, const uint64_t* seg_base, int C, uint64_t n_seg,
                        ppipe_point* out, ppipe_point* tmp_pts, uint64_t* seg_offsets, uint64_t* seg_tmp,
                        uint64_t* n_out_host, FrontierScratch* scratch, cudaStream_t s, int* n_launches) {
  const UniTraits::Params q{0x11111111u, nullptr, 1};
  // 1) split: flagged survivors to `out` (scratch here), unflagged straight to tmp_pts
  cudaError_t e = cudaMemsetAsync(seg_tmp, 0, 16, s);
  if (e != cudaSuccess) return e;
  unsigned long long* cur = reinterpret_cast<unsigned long long*>(seg_tmp);
  if (n) {
    f2_split_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(in, n, out, tmp_pts, cur);
    ++*n_launches;
  }
  unsigned long long hc[2] = {0, 0};
  if ((e = cudaMemcpyAsync(hc, cur, 16, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  const uint64_t nf = hc[0], nu = hc[1];
  // 2) equal-vector runs among the flagged ones, appended after the unflagged
  uint64_t n1 = 0;
  if ((e = frontier_generic<F2DedupTraits>(out, nf, seg_base, C, n_seg, q, tmp_pts + nu, seg_offsets, &n1, scratch, s,
                                           n_launches)) != cudaSuccess)
    return e;
  // 3) canonical order (segment, b, c_1, c_2) and the CSR
  return frontier_generic<F2OrderTraits>(tmp_pts, nu + n1, seg_base, C, n_seg, q, out, seg_offsets, n_out_host,
                                         scratch, s, n_launches);
}

cudaError_t truncate_frontier(const ppipe_point* in, const uint64_t* seg_offsets_in, uint64_t n_in, uint64_t n_seg,
                              const uint32_t* T_new, ppipe_point* out, uint64_t* seg_offsets_out,
                              uint64_t* n_out_host, FrontierScratch* scratch, cudaStream_t s, int* n_launches) {
  (void)n_in;
  const uint64_t tiles = (n_seg + kScanTile - 1) / kScanTile + 1;
  Scratch plan{nullptr, 0};
  plan.take<uint32_t>(n_seg + 1);
  plan.take<uint64_t>(tiles);
  cudaError_t e = ensure(scratch, plan.off);
  if (e != cudaSuccess) return e;
  Scratch sc{(char*)scratch->buf, 0};
  uint32_t* cnt = sc.take<uint32_t>(n_seg + 1);
  uint64_t* partial = sc.take<uint64_t>(tiles);
  if (n_seg) trunc_count_kernel<<<(unsigned)((n_seg + 255) / 256), 256, 0, s>>>(in, seg_offsets_in, n_seg, T_new, cnt);
  if ((e = scan_counts(cnt, n_seg, seg_offsets_out, partial, s, n_launches)) != cudaSuccess) return e;
  if (n_seg)
    trunc_copy_kernel<<<(unsigned)((n_seg * 32 + kFpThreads - 1) / kFpThreads), kFpThreads, 0, s>>>(
        in, seg_offsets_in, seg_offsets_out, n_seg, out);
  *n_launches += n_seg ? 2 : 0;
  uint64_t nk = 0;
  if ((e = cudaMemcpyAsync(&nk, seg_offsets_out + n_seg, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  *n_out_host = nk;
  return cudaGetLastError();
}

}  // namespace ppipe
