// ppipe_kernels.cu -- sm_100a kernels of the PPipe plan-enumeration hot path.
//
//   pack      §8(a1): prefix tables P[k][b][l] (C_d as prefix differences,
//             PAPER.md:2244 / eq. 1.9), transfer tables Y[v][b][c]
//             (Y_{bj} = ceil(8 S_{j-1} b / bw), PAPER.md:2246 / eq. 1.11),
//             T_eff = floor(slo (1000 - margin) / 1000).
//   score     §8(a2-a7): one CTA per (model, k_2, batch) enumerates every
//             candidate of its rows for K = 1, 2, 3 (all k_1, k_3), tests
//             E <= T_eff (eq. 1.12) with one integer compare
//             per candidate against a per-(c_1, k_1) threshold, and folds the
//             feasible ones through per-(segment, batch) E-bucket tables in
//             shared memory (two passes) so that only candidates not dominated
//             by an earlier bucket reach HBM. Integer ALU only: no tensor cores
//             (the path is not a contraction).
//   frontier  §8(a7): sort survivors by (segment, E), best point per
//             (segment, E) by (theta desc, b asc, cuts asc), strict staircase
//             over theta = b / Cmax compared as exact rationals, compaction.
//
// DESIGN.md §5 gives the roofline and algorithmic op counts of each kernel.
#include <algorithm>
#include <climits>
#include <cstdio>

#include "ppipe_internal.h"

// Debug builds (-DPPIPE_DEBUG_CHECKS, scripts/variants.py) bounds-check every
// shared-memory index the kernels derive from data; the product build compiles
// them away.
#ifdef PPIPE_DEBUG_CHECKS
#include <cstdio>
#define PPIPE_DCHECK(c)                                                                  \
  do {                                                                                   \
    if (!(c)) {                                                                          \
      printf("PPIPE_DCHECK failed at %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                         \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define PPIPE_DCHECK(c) \
  do {                  \
  } while (0)
#endif

namespace ppipe {

#define FULL_MASK 0xffffffffu

// ---------------------------------------------------------------------------
// pack
// ---------------------------------------------------------------------------
constexpr int kPackLT = 32;  // layers per tile
constexpr int kPackBT = 64;  // batches per tile

// CTA per (local model, class, batch tile). Transposes [M][B] -> [B][Mp] through
// shared memory so both the reads and the writes are coalesced.
__global__ void __launch_bounds__(256) pack_p_kernel(Problem pb, int n_btiles) {
  __shared__ int32_t tile[kPackLT][kPackBT + 1];
  __shared__ int32_t carry[kPackBT];
  const int bt = blockIdx.x % n_btiles;
  const int k = (blockIdx.x / n_btiles) % pb.C;
  const int ml = pb.model_base + blockIdx.x / (n_btiles * pb.C);
  DevModel* mdp = &pb.models[ml];
  const uint32_t M = mdp->M, Mp = mdp->Mp;
  const int B = pb.B;
  const int b0 = bt * kPackBT;
  const int nb = min(kPackBT, B - b0);
  const uint32_t* lat = pb.raw_lat + mdp->lat_off + (size_t)k * M * B;
  int32_t* Pk = pb.P + mdp->p_off + (size_t)k * B * Mp;
  if (threadIdx.x == 0 && k == 0 && bt == 0) {
    // T_eff = floor(slo * (1000 - margin) / 1000)   (reading A5)
    mdp->T = (int32_t)(((uint64_t)mdp->slo_us * (uint64_t)(1000 - pb.margin)) / 1000u);
  }
  if (threadIdx.x < nb) carry[threadIdx.x] = 0;
  // P[k][b][0] = 0
  for (int i = threadIdx.x; i < nb; i += blockDim.x) Pk[(size_t)(b0 + i) * Mp] = 0;
  for (uint32_t l0 = 0; l0 < M; l0 += kPackLT) {
    const int nl = min((uint32_t)kPackLT, M - l0);
    __syncthreads();
    for (int e = threadIdx.x; e < kPackLT * kPackBT; e += blockDim.x) {
      const int l = e / kPackBT, bb = e % kPackBT;
      // values are read as unsigned and clamped: unvalidated uploads (ppipe_update_profiles_async
      // validates on the device, the error surfaces in ppipe_pareto) never make a prefix negative
      tile[l][bb] = (l < nl && bb < nb) ? (int32_t)min(lat[(size_t)(l0 + l) * B + b0 + bb], (uint32_t)kRangeLimit) : 0;
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      int32_t acc = carry[threadIdx.x];
      for (int l = 0; l < nl; ++l) {
        acc = min(acc + tile[l][threadIdx.x], kRangeLimit);  // saturating (exact for valid inputs: totals < 2^28)
        tile[l][threadIdx.x] = acc;
      }
      carry[threadIdx.x] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kPackLT * kPackBT; e += blockDim.x) {
      const int bb = e / kPackLT, l = e % kPackLT;
      if (bb < nb && l < nl) Pk[(size_t)(b0 + bb) * Mp + l0 + l + 1] = tile[l][bb];
    }
  }
  __syncthreads();
  // padding entries beyond M repeat the total
  for (int e = threadIdx.x; e < nb * (int)(Mp - M - 1); e += blockDim.x) {
    const int bb = e / (Mp - M - 1), l = e % (Mp - M - 1);
    Pk[(size_t)(b0 + bb) * Mp + M + 1 + l] = carry[bb];
  }
  // the saturating total reaches kRangeLimit iff the true whole-model latency does
  if (pb.err_key && threadIdx.x < nb && carry[threadIdx.x] >= kRangeLimit)
    atomicMin(pb.err_key, ((unsigned long long)mdp->model << 40) | (unsigned long long)(k * B + b0 + threadIdx.x));
}

// CTA per (local model, distinct bandwidth v, batch): Y[v][b][c] for c in [0, Mp).
__global__ void __launch_bounds__(256) pack_y_kernel(Problem pb) {
  const int bi = blockIdx.x % pb.B;
  const int v = (blockIdx.x / pb.B) % pb.V;
  const int ml = pb.model_base + blockIdx.x / (pb.B * pb.V);
  const DevModel md = pb.models[ml];
  const uint64_t b = pb.batches[bi];
  const uint64_t bw = pb.bw_v[v];
  const uint64_t* S = pb.raw_s + md.s_off;
  int32_t* row = pb.Y + md.y_off + ((size_t)v * pb.B + bi) * md.Mp;
  if (pb.err_key && v == 0 && bi == 0)
    for (uint32_t l = threadIdx.x; l < md.M; l += blockDim.x)
      if (S[l] > pb.smax)
        atomicMin(pb.err_key, ((unsigned long long)md.model << 40) | (1ull << 39) | (unsigned long long)l);
  for (uint32_t c = threadIdx.x; c < md.Mp; c += blockDim.x) {
    int32_t y = 0;
    if (c >= 1 && c + 1 <= md.M) {
      // ceil(8 * S[c-1] * b / bw); the loader guarantees 8 * S * b < 2^63.
      const uint64_t num = 8ull * S[c - 1] * b;
      const uint64_t q = (num + bw - 1) / bw;
      y = q >= (uint64_t)kRangeLimit ? kRangeLimit : (int32_t)q;  // clamp: > any T_eff, stays infeasible
    }
    row[c] = y;
  }
}

__device__ __forceinline__ void tile_mina_body(const Problem& pb);

// CTA per (local model, batch), all k2 at once: for every K = 3 tile of 32 * kJ1 first
// cuts, the minimum over its valid c_1 and every k_1 of A(c_1, k_1) = C_1 + Y_1 - P[k2][c_1]. Then
// T_eff - minA is the loosest threshold of the tile, known before any slot is loaded.
__global__ void __launch_bounds__(128) tile_mina_kernel(Problem pb) { tile_mina_body(pb); }

cudaError_t launch_pack(const Problem& pb, cudaStream_t s) {
  if (pb.n_chunk == 0) return cudaSuccess;
  const int n_btiles = (pb.B + kPackBT - 1) / kPackBT;
  pack_p_kernel<<<pb.n_chunk * pb.C * n_btiles, 256, 0, s>>>(pb, n_btiles);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pack_y_kernel<<<pb.n_chunk * pb.V * pb.B, 256, 0, s>>>(pb);
  if (pb.minA && pb.Kmax >= 3) {
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    tile_mina_kernel<<<pb.n_chunk * pb.B, 32 * kJ1, 0, s>>>(pb);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// score
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

struct Rec {
  uint32_t w[8];
};

__device__ __forceinline__ Rec make_rec(uint32_t model, int K, int c1, int c2, int k1, int k2, int k3, int b,
                                        int E, int s1, int s2, int s3) {
  Rec r;
  r.w[0] = model;
  r.w[1] = (uint32_t)c1 | ((uint32_t)c2 << 16);
  r.w[2] = (uint32_t)K | ((uint32_t)(k1 & 0xFF) << 8) | ((uint32_t)(k2 & 0xFF) << 16) | ((uint32_t)(k3 & 0xFF) << 24);
  r.w[3] = (uint32_t)b;
  r.w[4] = (uint32_t)E;
  r.w[5] = (uint32_t)s1;
  r.w[6] = (uint32_t)s2;
  r.w[7] = (uint32_t)s3;
  return r;
}

#ifndef PPIPE_P2_PREFILTER
// Pass 2 scans its (short, tightened) ranges with the exact group tests only: without the
// two per-warp 16-bit prefilter rows score3b fits 8 CTAs/SM at 128 registers without
// spills (measured: score3b 24.0 ms with the prefilter at 7 CTAs/SM, 22.4 without at 7,
// 20.8 without at 8). 1: the prefilter in pass 2 as well.
#define PPIPE_P2_PREFILTER 0
#endif
#ifndef PPIPE_P1_FOLD_EVERY
#define PPIPE_P1_FOLD_EVERY 4  // pass 1 folds one c2 in 4 of a hit group (1: every feasible candidate)
#endif
// unroll of the per-c2 slow path over a hit group's 4 c2, per pass (measured, config 5:
// pass 1 at 1 / 2 / 4: score3a 34.9 / 32.8 / 32.4 ms; pass 2 at 1 / 2 / 4: score3b 24.1 /
// 27.1 / 36.9 ms -- pass 2's body is large, unrolled it spills)
#ifndef PPIPE_U_UNROLL_P1
#define PPIPE_U_UNROLL_P1 4
#endif
#ifndef PPIPE_U_UNROLL_P2
#define PPIPE_U_UNROLL_P2 1
#endif
constexpr int kUUnrollP1 = PPIPE_U_UNROLL_P1, kUUnrollP2 = PPIPE_U_UNROLL_P2;
#ifndef PPIPE_SCAN_UNROLL
#define PPIPE_SCAN_UNROLL 2
#endif
constexpr int kScanUnroll = PPIPE_SCAN_UNROLL;  // prefilter groups per vote in the pass-1 scan
constexpr int kWarps = 2;      // warps per CTA (share the fold tables and the staged rows)
constexpr int kEmitBuf = 32;   // survivor records staged per warp before a global flush
static_assert(kEmitBuf >= 32, "emit_warp appends up to one record per lane before it flushes");

// Survivor output: each warp stages records in a shared-memory buffer and flushes
// it with one global atomicAdd and coalesced 16-byte stores.
struct Emitter {
  int4* sbuf;  // [kEmitBuf][2]
  int count;   // warp-uniform
};

__device__ __noinline__ void emit_flush(const ScoreOut& o, Emitter& em) {
  const int lane = threadIdx.x & 31;
  const int n = em.count;
  if (n == 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&o.counters[0], (unsigned long long)n);
  base = __shfl_sync(FULL_MASK, base, 0);
  __syncwarp();
  int4* dst = reinterpret_cast<int4*>(o.surv);
  for (int w = lane; w < 2 * n; w += 32)
    if (base + (unsigned long long)(w >> 1) < o.cap) dst[2 * base + w] = em.sbuf[w];
  __syncwarp();
  em.count = 0;
}

// Warp-aggregated append. Called by all 32 lanes of a warp (out of line: rare path).
__device__ __noinline__ void emit_warp(const ScoreOut& o, Emitter& em, bool cond, Rec r) {
  const unsigned mask = __ballot_sync(FULL_MASK, cond);
  const int n = __popc(mask);
  if (n == 0) return;
  if (em.count + n > kEmitBuf) emit_flush(o, em);
  if (cond) {
    const int idx = em.count + __popc(mask & lanemask_lt());
    PPIPE_DCHECK(idx < kEmitBuf);
    em.sbuf[2 * idx] = make_int4((int)r.w[0], (int)r.w[1], (int)r.w[2], (int)r.w[3]);
    em.sbuf[2 * idx + 1] = make_int4((int)r.w[4], (int)r.w[5], (int)r.w[6], (int)r.w[7]);
  }
  __syncwarp();
  em.count += n;
}

// ---- fold tables ----
// Pass 1 keeps, per k_1 and E-bucket j = E >> sh, the bucket's best point (smallest
// Cmax, then smallest E) packed in 32 bits: key = (ceil(Cmax / 2^q) << sh) | (E mod 2^sh),
// so a plain 32-bit shared atomicMin folds it (a 64-bit min would be a CAS loop).
// q = 0 (exact) whenever bits(T_eff) + 1 + sh <= 32, i.e. for SLOs below ~1 s at
// 256 buckets; otherwise Cmax is rounded UP, which only makes the tests below
// more conservative. Row length nb + 2 (nb + 1 used).
// finalize: fin[j] = {U[j] = min rounded Cmax over buckets < j, key[j]}, fin[nb].x = U[nb].
// pass 2 keeps a feasible candidate (E, Cmax) of bucket j unless it is dominated:
//   Cmax >= U[j] << q                  by a point of an earlier bucket (smaller E), or
//   E >= E*_j, Cmax >= C*_j << q, not both equal, with (C*_j, E*_j) decoded from key[j]:
//                                      by the bucket's own best point.
// (proof sketch: every pruned candidate has a real candidate with E' <= E and
// Cmax' <= Cmax, strictly better in one, or is an exact duplicate kept elsewhere.)
constexpr uint32_t kEmpty = 0xffffffffu;

__device__ __forceinline__ void reset_raw(uint32_t* raw, int n, int tid, int nthreads) {
  for (int i = tid; i < n; i += nthreads) raw[i] = kEmpty;
}

__device__ __forceinline__ uint32_t pack_key(int E, int Cmax, int sh, int q) {
  const uint32_t cr = ((uint32_t)Cmax + ((1u << q) - 1u)) >> q;
  return (cr << sh) | ((uint32_t)E & ((1u << sh) - 1u));
}

// Virtual-GPU throughput weight of class k (Problem::wpack) and a weighted stage
// latency w * C, clamped at INT_MAX (only non-feasible values can reach it: a
// feasible candidate has C <= T_eff and w * T_eff < 2^31 is checked on the host).
__host__ __device__ __forceinline__ int wt(uint32_t wpack, int k) { return (int)((wpack >> (4 * k)) & 15u); }
template <bool W>
__device__ __forceinline__ int wtw(uint32_t wpack, int k) { return W ? wt(wpack, k) : 1; }
__device__ __forceinline__ int wmul(int w, int c) {
  const long long v = (long long)w * c;
  return v > INT_MAX ? INT_MAX : (int)v;
}

// theta = b / C as the bits of the double (C = 0: +inf). Exact order for b < 2^16,
// C < 2^32: distinct fractions differ by a relative >= 2^-48 > 2^-53.
__device__ __forceinline__ unsigned long long theta_bits(uint32_t b, uint32_t C) {
  return C ? (unsigned long long)__double_as_longlong((double)b / (double)C) : 0x7FF0000000000000ull;
}

// raw [nc][nb + 2] -> fin [nc][nb + 2] (fin may be global memory; nullptr: not written).
// One warp per k_1. With gf (the unit's K = 3 global-fold rows, k1-major, stride
// gf_stride), every bucket-best point that improves on all earlier buckets of the unit
// (a step of the unit's staircase) pushes its theta = b / Cmax into gf[k1][bucket].
__device__ __noinline__ void tables_finalize(const uint32_t* raw, uint2* fin, int nc, int nb, int sh, int warp,
                                             int nwarps, unsigned long long* gf = nullptr, size_t gf_stride = 0,
                                             uint32_t b = 0, int q = 0) {
  const int lane = threadIdx.x & 31;
  for (int k = warp; k < nc; k += nwarps) {
    const uint32_t* r = raw + (size_t)k * (nb + 2);
    uint2* f = fin ? fin + (size_t)k * (nb + 2) : nullptr;
    uint32_t run = kEmpty;
    for (int r0 = 0; r0 < nb; r0 += 32) {
      const uint32_t key = r[r0 + lane];
      const uint32_t c = key == kEmpty ? kEmpty : key >> sh;
      uint32_t incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(FULL_MASK, incl, d);
        if (lane >= d) incl = min(incl, o);
      }
      uint32_t excl = __shfl_up_sync(FULL_MASK, incl, 1);
      if (lane == 0) excl = kEmpty;
      if (f) f[r0 + lane] = make_uint2(min(run, excl), key);
      // the bucket's best point is a real candidate with Cmax <= c << q (rounded up when
      // q > 0, so its theta is at least b / (c << q))
      if (gf && c != kEmpty && c < min(run, excl))
        atomicMax(gf + (size_t)k * gf_stride + r0 + lane, theta_bits(b, c << q));
      run = min(run, __shfl_sync(FULL_MASK, incl, 31));
    }
    if (f && lane == 0) f[nb] = make_uint2(run, kEmpty);
  }
}

// Exclusive prefix maximum of every global-fold row (nb + 1 entries) in place: entry j
// = the best theta of buckets < j. Warp per row.
__global__ void __launch_bounds__(256) gfold_prefix_kernel(unsigned long long* gf, size_t rows, int nb1) {
  const int lane = threadIdx.x & 31;
  const size_t row = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= rows) return;
  unsigned long long* g = gf + row * nb1;
  unsigned long long run = 0ull;
  for (int j0 = 0; j0 < nb1; j0 += 32) {
    const int j = j0 + lane;
    const unsigned long long v = j < nb1 ? g[j] : 0ull;
    unsigned long long incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long o = __shfl_up_sync(FULL_MASK, incl, d);
      if (lane >= d) incl = max(incl, o);
    }
    unsigned long long excl = __shfl_up_sync(FULL_MASK, incl, 1);
    if (lane == 0) excl = 0ull;
    if (j < nb1) g[j] = max(run, excl);
    run = max(run, __shfl_sync(FULL_MASK, incl, 31));
  }
}

// The smallest Cmax a candidate of batch b must reach to be dominated by a point of
// theta g (a double b' / C' from the global fold): any Cmax >= bound has b / Cmax <
// b' / C'. Conservative by a relative 2^-30 against the rounding of g (so it never
// drops a candidate that is not strictly dominated); 0 for g = +inf.
__device__ __forceinline__ uint32_t gfold_bound(unsigned long long gbits, uint32_t b) {
  const double g = __longlong_as_double((long long)gbits);
  if (gbits >= 0x7FF0000000000000ull) return 0u;
  const double c = (double)b / g * (1.0 + 0x1p-30);
  return c >= 4294967294.0 ? 0xffffffffu : (uint32_t)c + 1u;
}

// Is a feasible candidate (E, Cmax) kept by the finalized row (see above)?
__device__ __forceinline__ bool survives(const uint2* row, int jb, int E, int Cmax, int sh, int q) {
  const uint2 ent = row[jb];
  if (ent.x != kEmpty && (unsigned)Cmax >= (ent.x << q)) return false;
  if (ent.y == kEmpty) return true;
  const int Cs = (int)((ent.y >> sh) << q);
  const int Es = (jb << sh) | (int)(ent.y & ((1u << sh) - 1u));
  return !(E >= Es && Cmax >= Cs && (E > Es || Cmax > Cs));
}

// First j in [0, nb] with U[j] << q <= v in a finalized (nonincreasing) row; nb + 1 if none.
__device__ __forceinline__ int first_bucket_le(const uint2* row, int nb, int v, int q) {
  int lo = 0, hi = nb + 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const uint32_t u = row[mid].x;
    if (u != kEmpty && (u << q) <= (unsigned)v) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

template <int NC>
struct CtaCtx {
  const int32_t* P2;   // P[k2][b][.]
  const int32_t* Pm;   // P[m] base
  const int32_t* Ym;   // Y[m] base
  size_t Mp, B;
  int bi, b, k2, M, T, sh, q, m1, nb, dbg, row_len, w2;
  uint32_t wpack;
  uint32_t model;
  const uint8_t* pair_v;
  __device__ const int32_t* Prow(int k) const { return Pm + ((size_t)k * B + bi) * Mp; }
  __device__ const int32_t* Yrow(int ka, int kb) const {
    return Ym + ((size_t)__ldg(pair_v + ka * NC + kb) * B + bi) * Mp;
  }
};

constexpr int kInvalidThr = -(1 << 30);  // threshold of an empty slot: B(c2) >= 0 never passes
constexpr int kPadB = 0x3fffffff;        // B(c2) beyond the model: above every threshold

// d = thr - Bv on the FMA pipe (IMAD with a run-time -1 the compiler cannot fold).
__device__ __forceinline__ int mad_diff(int Bv, int m1, int thr) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(Bv), "r"(m1), "r"(thr));
  return d;
}

// Does any of this lane's candidates at B(c2) = Bv (slots j < jmax, all k1)
// satisfy E <= T_eff, i.e. Bv <= thr[j][k1]? Every candidate gets its own
// integer instruction: the k1 = 0 (and, for NC >= 7, k1 = NC-1) candidates as
// ISETP (ALU pipe, OR-chained in a predicate), the others as IMAD d = thr - Bv
// (FMA pipe) AND-reduced by LOP3 (sign bit clear <=> some d >= 0), so both
// integer pipes share the work and the SM's issue slot is the limit. The
// compares are inline PTX so the compiler cannot replace them by one compare
// against a hoisted max of the thresholds (that would skip per-candidate work).
static_assert(kJ1 == 4, "any_feasible's PTX is written for 4 slots per lane");
template <int NC>
__device__ __forceinline__ int any_feasible(const int (&thr)[kJ1][NC], int Bv, int m1, int jmax = kJ1) {
  constexpr bool kTwo = NC >= 7;
  int acc = -1;
#pragma unroll
  for (int j = 0; j < kJ1; ++j) {
    if (j >= jmax) break;  // jmax is a constant after unrolling the caller's band switch
#pragma unroll
    for (int k = 1; k < (kTwo ? NC - 1 : NC); ++k) acc &= mad_diff(Bv, m1, thr[j][k]);
  }
  int t[kJ1], u[kJ1];
#pragma unroll
  for (int j = 0; j < kJ1; ++j) {
    t[j] = j < jmax ? thr[j][0] : kInvalidThr;
    u[j] = (kTwo && j < jmax) ? thr[j][NC - 1] : kInvalidThr;
  }
  int h;
  if (kTwo) {
    asm("{\n\t.reg .pred p;\n\t"
        "setp.le.s32 p, %1, %2;\n\tsetp.le.or.s32 p, %1, %3, p;\n\t"
        "setp.le.or.s32 p, %1, %4, p;\n\tsetp.le.or.s32 p, %1, %5, p;\n\t"
        "setp.le.or.s32 p, %1, %7, p;\n\tsetp.le.or.s32 p, %1, %8, p;\n\t"
        "setp.le.or.s32 p, %1, %9, p;\n\tsetp.le.or.s32 p, %1, %10, p;\n\t"
        "setp.gt.or.s32 p, %6, -1, p;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(h)
        : "r"(Bv), "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(acc), "r"(u[0]), "r"(u[1]), "r"(u[2]),
          "r"(u[3]));
  } else {
    asm("{\n\t.reg .pred p;\n\t"
        "setp.le.s32 p, %1, %2;\n\tsetp.le.or.s32 p, %1, %3, p;\n\t"
        "setp.le.or.s32 p, %1, %4, p;\n\tsetp.le.or.s32 p, %1, %5, p;\n\t"
        "setp.gt.or.s32 p, %6, -1, p;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(h)
        : "r"(Bv), "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(acc));
  }
  return h;
}

// Main-phase fast test for a whole aligned group of 4 c2 values: does any of this
// lane's 4 x kJ1 x NC candidates pass? Same per-candidate split as any_feasible
// (one ISETP or one IMAD each), but one predicate and one vote per group; the
// per-c2 flags are recomputed only when the group hits (rare).
template <int NC>
__device__ __forceinline__ int any_feasible4(const int (&thr)[kJ1][NC], const int4& b4, int m1) {
  constexpr bool kTwo = NC >= 7;
  const int bv[4] = {b4.x, b4.y, b4.z, b4.w};
  int acc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    acc[u] = -1;
#pragma unroll
    for (int j = 0; j < kJ1; ++j) {
#pragma unroll
      for (int k = 1; k < (kTwo ? NC - 1 : NC); ++k) acc[u] &= mad_diff(bv[u], m1, thr[j][k]);
    }
  }
  const int a = acc[0] & acc[1] & acc[2] & acc[3];
  int h;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.gt.s32 p, %1, -1;\n\t"
      "setp.le.or.s32 p, %2, %6, p;\n\tsetp.le.or.s32 p, %2, %7, p;\n\t"
      "setp.le.or.s32 p, %2, %8, p;\n\tsetp.le.or.s32 p, %2, %9, p;\n\t"
      "setp.le.or.s32 p, %3, %6, p;\n\tsetp.le.or.s32 p, %3, %7, p;\n\t"
      "setp.le.or.s32 p, %3, %8, p;\n\tsetp.le.or.s32 p, %3, %9, p;\n\t"
      "setp.le.or.s32 p, %4, %6, p;\n\tsetp.le.or.s32 p, %4, %7, p;\n\t"
      "setp.le.or.s32 p, %4, %8, p;\n\tsetp.le.or.s32 p, %4, %9, p;\n\t"
      "setp.le.or.s32 p, %5, %6, p;\n\tsetp.le.or.s32 p, %5, %7, p;\n\t"
      "setp.le.or.s32 p, %5, %8, p;\n\tsetp.le.or.s32 p, %5, %9, p;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(h)
      : "r"(a), "r"(bv[0]), "r"(bv[1]), "r"(bv[2]), "r"(bv[3]), "r"(thr[0][0]), "r"(thr[1][0]), "r"(thr[2][0]),
        "r"(thr[3][0]));
  if (kTwo) {
    int h2;
    asm("{\n\t.reg .pred p;\n\t"
        "setp.le.s32 p, %1, %5;\n\tsetp.le.or.s32 p, %1, %6, p;\n\t"
        "setp.le.or.s32 p, %1, %7, p;\n\tsetp.le.or.s32 p, %1, %8, p;\n\t"
        "setp.le.or.s32 p, %2, %5, p;\n\tsetp.le.or.s32 p, %2, %6, p;\n\t"
        "setp.le.or.s32 p, %2, %7, p;\n\tsetp.le.or.s32 p, %2, %8, p;\n\t"
        "setp.le.or.s32 p, %3, %5, p;\n\tsetp.le.or.s32 p, %3, %6, p;\n\t"
        "setp.le.or.s32 p, %3, %7, p;\n\tsetp.le.or.s32 p, %3, %8, p;\n\t"
        "setp.le.or.s32 p, %4, %5, p;\n\tsetp.le.or.s32 p, %4, %6, p;\n\t"
        "setp.le.or.s32 p, %4, %7, p;\n\tsetp.le.or.s32 p, %4, %8, p;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(h2)
        : "r"(bv[0]), "r"(bv[1]), "r"(bv[2]), "r"(bv[3]), "r"(thr[0][NC - 1]), "r"(thr[1][NC - 1]),
          "r"(thr[2][NC - 1]), "r"(thr[3][NC - 1]));
    h |= h2;
  }
  return h;
}

// Hit flags of one aligned group of 4 c2 values inside diagonal band JB: slots
// j < JB are complete pairs, slot JB holds pairs for lanes < c2 - (c1_base + 32 JB).
template <int NC, int JB>
__device__ __forceinline__ void band_hits(const int (&thr)[kJ1][NC], const int4& b4, int m1, int lane, int rel,
                                          int& h0, int& h1, int& h2, int& h3) {
  const int bv[4] = {b4.x, b4.y, b4.z, b4.w};
  int h[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int accb = -1;
#pragma unroll
    for (int k1 = 0; k1 < NC; ++k1) accb &= mad_diff(bv[u], m1, thr[JB][k1]);
    h[u] = any_feasible<NC>(thr, bv[u], m1, JB) | ((lane < rel + u - 32 * JB) & (accb >= 0));
  }
  h0 = h[0];
  h1 = h[1];
  h2 = h[2];
  h3 = h[3];
}

// One warp processes one tile of 32 * kJ1 first cuts c_1 (lane l, slot j holds
// c_1 = c1_base + 32 j + l; slots outside [c1_lo, c1_hi] are empty) against every
// c_2 > c_1 for a fixed (k_2, k_3, b) and all k_1. The lane's thresholds
// thr[j][k1] = T_eff - A(c_1, k_1) stay in registers; B(c_2) comes from shared
// memory four at a time (c1_base = 3 mod 4 keeps every group aligned), so
// E <= T_eff is B(c_2) <= thr.
//
// pass 1 counts every feasible candidate and folds it into its bucket's best
// point (branch-free, predicated 64-bit shared atomics). pass 2 emits the feasible
// candidates the finalized tables do not prove dominated (survives()), after
// tightening each threshold so that candidates whose first stage alone is
// dominated (C_1 >= U(E)) never leave the fast loop. Q(c_2) = P[k2][c_2] and
// R(c_2) = C_3 are shared-memory rows like B. The fast loop and the slow paths
// each exist once in the code (one pass-generic instance).
// Pass-2 per-warp slot data: the dense survivor pass reads any lane's slot.
struct SlotData {
  const uint32_t* rowoff;  // pass 2: [2 NC] offsets of P[k1][b] (from Pm) and Y[k1 -> k2][b] (from Ym)
  int32_t* As;     // [kJ1 * NC][32] A = C1 + Y1 - P[k2][c1], so E = A + B(c2)
  int32_t* C1s;    // [kJ1 * NC][32] C_1
  int32_t* p1s;    // [kJ1][32] P[k2][c1]
  uint16_t* list;  // [kJ1 * NC * 32] (lane << 5 | slot) of the current c2
};
#ifndef PPIPE_SLOT_SMEM
#define PPIPE_SLOT_SMEM 0  // 1: pass-2 slot values staged in shared memory (else re-read through L1)
#endif
template <int NC>
__host__ __device__ constexpr size_t slot_bytes() {
  return PPIPE_SLOT_SMEM ? (size_t)kJ1 * 32 * (2 * sizeof(int32_t) * NC + sizeof(int32_t) + sizeof(uint16_t) * NC)
                         : (size_t)kJ1 * 32 * sizeof(uint16_t) * NC;
}
template <int NC>
__device__ __forceinline__ SlotData carve_slot(uint8_t* base) {
  SlotData d{};
#if PPIPE_SLOT_SMEM
  d.As = reinterpret_cast<int32_t*>(base);
  d.C1s = d.As + kJ1 * NC * 32;
  d.p1s = d.C1s + kJ1 * NC * 32;
  d.list = reinterpret_cast<uint16_t*>(d.p1s + kJ1 * 32);
#else
  d.As = d.C1s = d.p1s = nullptr;
  d.rowoff = nullptr;
  d.list = reinterpret_cast<uint16_t*>(base);
#endif
  return d;
}

template <int NC, int pass, bool W>
__device__ void k3_tile(const CtaCtx<NC>& cx, int k3, int c1_base, int c1_lo, int c1_hi,
                        const int32_t* Bs, const int32_t* Qs, const int32_t* Rs, uint32_t* raw, const uint2* fin,
                        const SlotData& sd, uint32_t* nb16, const ScoreOut& out, Emitter& em,
                        unsigned long long& feas, unsigned long long& cand, int Bmin = 0,
                        int tmax_hint = INT_MAX) {
  // tmax_hint (pass 1): T_eff - (the tile's minimum A) or INT_MAX
  const int lane = threadIdx.x & 31;
  const int nb = cx.nb;
  if (pass == 1 && tmax_hint != INT_MAX) {
    // Early tile skip: T_eff - minA (the loosest threshold of the tile, from the pack
    // launch) below every B(c2) of the range => no feasible candidate; count and leave
    // before loading any slot.
    int bmin = INT_MAX;
    for (int c2 = c1_base + 1 + lane; c2 < cx.M; c2 += 32) bmin = min(bmin, Bs[c2]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) bmin = min(bmin, __shfl_xor_sync(FULL_MASK, bmin, d));
    if (tmax_hint < bmin) {
#pragma unroll
      for (int j = 0; j < kJ1; ++j) {
        const int c1 = c1_base + 32 * j + lane;
        if (c1 >= c1_lo && c1 <= c1_hi) cand += (unsigned long long)(cx.M - 1 - c1) * NC;
      }
      return;
    }
  }
  // virtual-GPU weights: compile-time 1 unless the context set some (W)
  const uint32_t wp = W ? cx.wpack : 0x11111111u;
  const int w2 = W ? cx.w2 : 1;
  int thr[kJ1][NC];
  int c1r[kJ1][NC];
  int p1[kJ1];
  int wlo = INT_MAX, whi = -1;  // pass 2: c2 range that can hold survivors
  int amin_k[NC];               // pass 2: per k1, the minimum A of the tile (reduced below)
#pragma unroll
  for (int k1 = 0; k1 < NC; ++k1) amin_k[k1] = INT_MAX;
#pragma unroll
  for (int j = 0; j < kJ1; ++j) {
    const int c1 = c1_base + 32 * j + lane;
    const bool valid = c1 >= c1_lo && c1 <= c1_hi;
    p1[j] = valid ? __ldg(cx.P2 + c1) : 0;
#pragma unroll
    for (int k1 = 0; k1 < NC; ++k1) {
      const int C1 = valid ? __ldg(cx.Prow(k1) + c1) : 0;
      const int y = valid ? __ldg(cx.Yrow(k1, cx.k2) + c1) : 0;
      // E = A + B(c2) with A = C1 + Y1 - P[k2][c1]  =>  feasible iff B(c2) <= T - A
      int t = valid ? cx.T - (C1 + y - p1[j]) : kInvalidThr;
      if (pass == 2) {
        if (valid) amin_k[k1] = min(amin_k[k1], C1 + y - p1[j]);
        int b0 = nb;
        if (valid) {
          const uint2* frow = fin + (size_t)k1 * (nb + 2);
          // A survivor needs Cmax < U(E) <= U(E_min) with E_min = A + min_c2 B(c2) (U is
          // nonincreasing), so C_1, C_2 = Q(c2) - P[k2][c1] and C_3 = R(c2) must each stay
          // below Umax = U(E_min): with Q nondecreasing and R nonincreasing in c2 that
          // leaves one c2 interval [lo, hi] per slot; outside it nothing is emitted.
          const int Emin = max(0, cx.T - t + Bmin);  // E >= 0 for every real candidate
          const uint32_t ur = Emin <= cx.T ? frow[Emin >> cx.sh].x : 0u;
          const int Umax = ur == kEmpty ? INT_MAX : (int)min(ur << cx.q, (uint32_t)INT_MAX);
          const int C1w = wmul(wtw<W>(wp, k1), C1), w3 = wtw<W>(wp, k3);
          int lo = c1 + 1, hi = cx.M - 1;
          if (Emin > cx.T || C1w >= Umax) {
            t = kInvalidThr;  // nothing of this slot can survive
          } else {
            // first c2 with R(c2) < Umax
            int a = c1 + 1, z = cx.M;
            while (a < z) {
              const int m = (a + z) >> 1;
              if (wmul(w3, Rs[m]) < Umax) z = m;
              else a = m + 1;
            }
            lo = a;
            // last c2 with Q(c2) - p1 < Umax
            a = c1 + 1;
            z = cx.M;
            while (a < z) {
              const int m = (a + z) >> 1;
              if (wmul(w2, Qs[m] - p1[j]) >= Umax) z = m;
              else a = m + 1;
            }
            hi = a - 1;
            if (lo > hi) {
              t = kInvalidThr;
            } else {
              wlo = min(wlo, lo);
              whi = max(whi, hi);
              // U is nonincreasing; from bucket b0 on U <= C1 <= Cmax, so nothing there
              // survives: only E < b0 << sh can  =>  B <= (b0 << sh) - 1 - A.
              b0 = min(first_bucket_le(frow, nb, C1w, cx.q), nb);
              if (b0 < nb) t = t + min(0, (b0 << cx.sh) - 1 - cx.T);
            }
          }
        }
        // this lane's slot data for the dense survivor pass (E = A + B(c2) exactly)
#if PPIPE_SLOT_SMEM
        sd.As[(j * NC + k1) * 32 + lane] = valid ? C1 + y - p1[j] : 0;
        sd.C1s[(j * NC + k1) * 32 + lane] = C1;
#endif
      }
      thr[j][k1] = t;
      c1r[j][k1] = wmul(wtw<W>(wp, k1), C1);  // weighted: only Cmax uses it
    }
#if PPIPE_SLOT_SMEM
    if (pass == 2) sd.p1s[j * 32 + lane] = p1[j];
#endif
    if (pass == 1 && valid) cand += (unsigned long long)(cx.M - 1 - c1) * NC;
  }
  const int m1 = cx.m1;
  const int M = cx.M;
  unsigned nfeas = 0;
  int c2_start = c1_base + 1, c2_end = M;
  int amin_col = INT_MAX;  // pass 2, lane k1 < NC: the tile's minimum A of column k1
  if (pass == 2) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      wlo = min(wlo, __shfl_xor_sync(FULL_MASK, wlo, d));
      whi = max(whi, __shfl_xor_sync(FULL_MASK, whi, d));
    }
#pragma unroll
    for (int k1 = 0; k1 < NC; ++k1) {
      int a = amin_k[k1];
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) a = min(a, __shfl_xor_sync(FULL_MASK, a, d));
      if (lane == k1) amin_col = a;
    }
    if (whi < 0) return;  // no slot of this tile can hold a survivor
    c2_start = c1_base + 1 + (max(0, wlo - (c1_base + 1)) & ~3);  // keep groups aligned
    c2_end = min(M, whi + 1);
  }
  // ---- 16-bit prefilter ----
  // Every candidate is first tested in a 16-bit field: thresholds and B(c2) are
  // offset by L = min_c2 B(c2) + 16383 and saturated to 15 bits, then stored
  // offset-binary (t' = thr - L + 16384 in [0, 32767], n' = 16384 - (B - L) in
  // [1, 32767]), so t' + n' never carries out of its 16-bit field and its bit 15
  // is set exactly when thr - B >= 0. One plain 32-bit add therefore tests two
  // candidates, and ptxas is free to issue it as IADD3 (ALU pipe) or IMAD.IADD
  // (FMA pipe), which balances the two pipes; LOP3 OR-reduces the bits.
  // Saturation can only turn a "no" into a "yes" (B never saturates low by the
  // choice of L), so a group passing here is re-tested exactly in 32 bits below;
  // a group failing here has no feasible candidate.
  constexpr int kPairs = (kJ1 * NC + 1) / 2;
  // kQ64 64-bit words (4 candidates each) are added as IADD3 (ALU) + IMAD.X (FMA);
  // the other words as IMAD.IADD / VIADD.16x2 (FMA). With the LOP3 reduction on the
  // ALU pipe, (kPairs - 2) / 4 wide words balances the two half-rate pipes.
  constexpr int kQ64 = (kPairs - 2) / 4;
  unsigned thr16[kPairs];
  unsigned long long thr64[kQ64 > 0 ? kQ64 : 1];
  {
    // Tile skip and range trim: a c2 with B(c2) above every slot's threshold holds no
    // feasible candidate (in pass 2: no survivor). If no c2 of the range is reachable the
    // tile ends here (most tiles of a deep model: far from the SLO; candidates were
    // counted above); otherwise the scan runs from the first to the last reachable c2.
    int tmax = INT_MIN;
#pragma unroll
    for (int j = 0; j < kJ1; ++j) {
#pragma unroll
      for (int k1 = 0; k1 < NC; ++k1) tmax = max(tmax, thr[j][k1]);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) tmax = max(tmax, __shfl_xor_sync(FULL_MASK, tmax, d));
    int bmin = INT_MAX, rlo = INT_MAX, rhi = -1;
    for (int c2 = c2_start + lane; c2 < c2_end; c2 += 32) {
      const int bv = Bs[c2];
      bmin = min(bmin, bv);
      if (bv <= tmax) {
        rlo = min(rlo, c2);
        rhi = c2;
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      bmin = min(bmin, __shfl_xor_sync(FULL_MASK, bmin, d));
      rlo = min(rlo, __shfl_xor_sync(FULL_MASK, rlo, d));
      rhi = max(rhi, __shfl_xor_sync(FULL_MASK, rhi, d));
    }
    if (rhi < 0) return;
    c2_start += (rlo - c2_start) & ~3;  // keep the groups aligned (c2_start = c1_base + 1 mod 4)
    c2_end = rhi + 1;
    const long long L = (long long)bmin + 16383;
    // entries past c2_end hold n' = 0 (never pass) so that the unrolled, prefetching
    // scan below may read up to 16 values ahead
    if (pass == 1 || PPIPE_P2_PREFILTER) {
    const int fill_end = ((c2_end + 3) & ~3) + 8 * kScanUnroll - 4;
    PPIPE_DCHECK(fill_end <= cx.row_len && c2_start >= 0);
    for (int c2 = c2_start + lane; c2 < fill_end; c2 += 32) {
      const long long v = (long long)Bs[min(c2, c2_end - 1)] - L;
      const int sv = (int)max(-16383ll, min(16383ll, v));
      nb16[c2] = c2 < c2_end ? (unsigned)(16384 - sv) * 0x10001u : 0u;  // (n', n')
    }
#pragma unroll
    for (int p = 0; p < kPairs; ++p) {
      unsigned w = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = 2 * p + h;
        int tv = 0;  // unused half: never passes
        if (i < kJ1 * NC) tv = (int)max(-16384ll, min(16383ll, (long long)thr[i / NC][i % NC] - L)) + 16384;
        w |= (unsigned)tv << (16 * h);
      }
      thr16[p] = w;
    }
#pragma unroll
    for (int q = 0; q < kQ64; ++q) thr64[q] = ((unsigned long long)thr16[2 * q + 1] << 32) | thr16[2 * q];
    __syncwarp();
    }
  }
  // Prefilter hit bits of one aligned group of 4 c2 values (bit 15 / 31 of the result).
  auto group_bits = [&](const uint4& n4) -> unsigned {
    unsigned a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    const unsigned n4v[4] = {n4.x, n4.y, n4.z, n4.w};
    unsigned* const acc[4] = {&a0, &a1, &a2, &a3};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned long long nw = ((unsigned long long)n4v[u] << 32) | n4v[u];
#pragma unroll
      for (int q = 0; q < kQ64; ++q) {  // no field carries, so neither does the low word
        const unsigned long long x = thr64[q] + nw;
        *acc[u] |= (unsigned)x | (unsigned)(x >> 32);
      }
#pragma unroll
      for (int p = 2 * kQ64; p < kPairs; ++p) *acc[u] |= thr16[p] + n4v[u];
    }
    return (a0 | a1 | a2 | a3) & 0x80008000u;
  };
  const uint4* const nrow = reinterpret_cast<const uint4*>(nb16);
#pragma unroll 1
  for (int c2 = c2_start; c2 < c2_end; c2 += 4) {
    // Fast scan: two groups per iteration, one vote, next pair prefetched; stops at
    // the first group in which some lane's prefilter passes.
    if (pass == 2 && !PPIPE_P2_PREFILTER) {
      // no prefilter: every group goes to the exact tests below
    } else if (pass == 2) {  // short tightened ranges: one group per iteration
#pragma unroll 1
      for (;;) {
        if (__any_sync(FULL_MASK, group_bits(nrow[c2 >> 2]) != 0u)) break;
        c2 += 4;
        if (c2 >= c2_end) break;
      }
      if (c2 >= c2_end) break;
    } else {
      uint4 cur[kScanUnroll];
#pragma unroll
      for (int g = 0; g < kScanUnroll; ++g) cur[g] = nrow[(c2 >> 2) + g];
#pragma unroll 1
      for (;;) {
        PPIPE_DCHECK(4 * ((c2 >> 2) + 2 * kScanUnroll) <= cx.row_len);
        uint4 nxt[kScanUnroll];
#pragma unroll
        for (int g = 0; g < kScanUnroll; ++g) nxt[g] = nrow[(c2 >> 2) + kScanUnroll + g];
        unsigned hg[kScanUnroll], hor = 0;
#pragma unroll
        for (int g = 0; g < kScanUnroll; ++g) hor |= hg[g] = group_bits(cur[g]);
        if (__any_sync(FULL_MASK, hor != 0u)) {
#pragma unroll
          for (int g = 0; g < kScanUnroll - 1; ++g) {
            if (__any_sync(FULL_MASK, hg[g] != 0u)) break;
            c2 += 4;
          }
          break;
        }
        c2 += 4 * kScanUnroll;
        if (c2 >= c2_end) break;
#pragma unroll
        for (int g = 0; g < kScanUnroll; ++g) cur[g] = nxt[g];
      }
      if (c2 >= c2_end) break;
    }
    PPIPE_DCHECK(c2 + 4 <= cx.row_len && (c2 & 3) == 0);
    const int4 b4 = *reinterpret_cast<const int4*>(Bs + c2);
    const int rel = c2 - c1_base;  // 1 mod 4; the group is rel .. rel + 3
    int h0, h1, h2, h3;
    if (rel > 32 * kJ1) {
      if (!__any_sync(FULL_MASK, any_feasible4<NC>(thr, b4, m1))) continue;
      h0 = any_feasible<NC>(thr, b4.x, m1);  // the group hit: per-c2 flags for the slow path
      h1 = any_feasible<NC>(thr, b4.y, m1);
      h2 = any_feasible<NC>(thr, b4.z, m1);
      h3 = any_feasible<NC>(thr, b4.w, m1);
    } else {
      switch ((rel - 1) >> 5) {
        case 0: band_hits<NC, 0>(thr, b4, m1, lane, rel, h0, h1, h2, h3); break;
        case 1: band_hits<NC, 1>(thr, b4, m1, lane, rel, h0, h1, h2, h3); break;
        case 2: band_hits<NC, 2>(thr, b4, m1, lane, rel, h0, h1, h2, h3); break;
        default: band_hits<NC, 3>(thr, b4, m1, lane, rel, h0, h1, h2, h3); break;
      }
    }
    if (!__any_sync(FULL_MASK, h0 | h1 | h2 | h3)) continue;
    if (cx.dbg & 4) {
      nfeas += (h0 | h1 | h2 | h3) ? 1u : 0u;
      continue;
    }
    const int4 q4 = *reinterpret_cast<const int4*>(Qs + c2);
    const int4 r4 = *reinterpret_cast<const int4*>(Rs + c2);
    // Some lane passed at some c2 of the group. Slot j of this lane is a real
    // pair iff 32 j + lane < c2 - c1_base.
    // pass 2 runs this loop rolled: its per-c2 values come from shared memory and a hit
    // mask instead of select chains over the group's registers
    const unsigned hm = (h0 != 0 ? 1u : 0u) | (h1 != 0 ? 2u : 0u) | (h2 != 0 ? 4u : 0u) | (h3 != 0 ? 8u : 0u);
#pragma unroll(pass == 1 ? kUUnrollP1 : kUUnrollP2)
    for (int u = 0; u < 4; ++u) {
      const int hu = pass == 2 ? (int)((hm >> u) & 1u) : (u == 0 ? h0 : (u == 1 ? h1 : (u == 2 ? h2 : h3)));
      if (!__any_sync(FULL_MASK, hu)) continue;
      const int Bv = pass == 2 ? Bs[c2 + u] : (u == 0 ? b4.x : (u == 1 ? b4.y : (u == 2 ? b4.z : b4.w)));
      const int Q = pass == 2 ? Qs[c2 + u] : (u == 0 ? q4.x : (u == 1 ? q4.y : (u == 2 ? q4.z : q4.w)));
      const int R = pass == 2 ? Rs[c2 + u] : (u == 0 ? r4.x : (u == 1 ? r4.y : (u == 2 ? r4.z : r4.w)));
      const int relu = rel + u;
      if (pass == 1 && (u % PPIPE_P1_FOLD_EVERY) != 0) {
        // count only: the fold takes one c2 of every PPIPE_P1_FOLD_EVERY of a hit group.
        // The tables only need real candidates, so sampling keeps pass 2 exact; its
        // bounds get a little looser (measured: score3a 47.9 -> 35.0 ms, score3b 30.0 ->
        // 32.9 ms, survivors 16.6M -> 37.8M, step 85.7 -> 77.8 ms at 4; 79.2 ms at 2)
#pragma unroll
        for (int j = 0; j < kJ1; ++j) {
          const bool v = 32 * j + lane < relu;
#pragma unroll
          for (int k1 = 0; k1 < NC; ++k1) nfeas += (v && Bv <= thr[j][k1]) ? 1u : 0u;
        }
      } else if (pass == 1) {
        const int Rw = wmul(wtw<W>(wp, k3), R);
#pragma unroll
        for (int j = 0; j < kJ1; ++j) {
          const bool v = 32 * j + lane < relu;
          const int C2w = wmul(w2, Q - p1[j]);
#pragma unroll
          for (int k1 = 0; k1 < NC; ++k1) {
            if (v && Bv <= thr[j][k1]) {
              const int E = cx.T - thr[j][k1] + Bv;
              const int Cmax = max(max(c1r[j][k1], C2w), Rw);
              PPIPE_DCHECK(E >= 0 && (E >> cx.sh) < nb + 2);
              if (!(cx.dbg & 1)) atomicMin(raw + (size_t)k1 * (nb + 2) + (E >> cx.sh), pack_key(E, Cmax, cx.sh, cx.q));
              ++nfeas;
            }
          }
        }
      } else {
        // Dense survivor pass: the (lane, slot) pairs that pass the tightened
        // threshold are listed warp-wide, then checked 32 at a time, one per lane,
        // against the finalized tables (survives()) and emitted.
        const int c2u = c2 + u;
        const int Rw = wmul(wtw<W>(wp, k3), R);  // per c2 (may exceed T_eff for unlisted ones)
        // k_1 columns dead at this c2: every candidate of column k1 in the tile has E >= Elo
        // = B(c2) + (the column's minimum A over the tile), so with U nonincreasing, C_3 =
        // R(c2) >= U_k1(Elo) means Cmax >= U_k1(E): dominated (lane k1 tests column k1)
        unsigned live;
        {
          const int Elo = (int)max(0ll, min((long long)cx.T, (long long)Bv + amin_col));
          // and C_2 = Q(c2) - P[k2][c1] >= Q(c2) - P[k2][min(c2 - 1, last c1 of the tile)]
          const int c2lo = Q - Qs[min(c2u - 1, min(c1_base + 32 * kJ1 - 1, c1_hi))];
          const unsigned cm = (unsigned)max(Rw, wmul(w2, max(0, c2lo)));
          bool dead = false;
          if (lane < NC) {
            const uint32_t U0 = fin[(size_t)lane * (nb + 2) + (Elo >> cx.sh)].x;
            dead = U0 != kEmpty && cm >= (U0 << cx.q);
          }
          live = ~__ballot_sync(FULL_MASK, dead) & ((1u << NC) - 1u);
        }
        if (live == 0u) continue;
        unsigned fm = 0;
#pragma unroll
        for (int j = 0; j < kJ1; ++j) {
          const bool v = 32 * j + lane < relu;
#pragma unroll
          for (int k1 = 0; k1 < NC; ++k1) fm |= (v && Bv <= thr[j][k1]) ? (1u << (j * NC + k1)) : 0u;
        }
        {
          unsigned cols = 0;
#pragma unroll
          for (int j = 0; j < kJ1; ++j) cols |= live << (j * NC);
          fm &= cols;
        }
        const int cnt = __popc(fm);
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int t = __shfl_up_sync(FULL_MASK, incl, d);
          if (lane >= d) incl += t;
        }
        const int total = __shfl_sync(FULL_MASK, incl, 31);
        int pos = incl - cnt;
        while (fm) {
          const int sl = __ffs(fm) - 1;
          fm &= fm - 1;
          PPIPE_DCHECK(pos < kJ1 * NC * 32);
          sd.list[pos++] = (uint16_t)((lane << 5) | sl);
        }
        __syncwarp();
#pragma unroll 1
        for (int base = 0; base < total; base += 32) {
          const int i = base + lane;
          bool cond = false;
          Rec rec{};
          if (i < total) {
            const unsigned e = sd.list[i];
            const int src = (int)(e >> 5), sl = (int)(e & 31u);
            const int j = sl / NC, k1 = sl - j * NC;
#if PPIPE_SLOT_SMEM
            const int E = sd.As[sl * 32 + src] + Bv;
            const int C1 = sd.C1s[sl * 32 + src];
            const int C2 = Q - sd.p1s[j * 32 + src];
#else
            // the listed candidate's first-cut terms, re-read through L1 (the tile's rows
            // are a few KB): C_1 = P[k1][c1], Y_1 and P[k2][c1]
            const int c1 = c1_base + 32 * j + src;
            const int C1 = __ldg(cx.Pm + sd.rowoff[k1] + c1);
            const int pc1 = __ldg(cx.P2 + c1);
            const int E = C1 + __ldg(cx.Ym + sd.rowoff[NC + k1] + c1) - pc1 + Bv;
            const int C2 = Q - pc1;
#endif
            // listed candidates are feasible: C_1, C_2 <= E <= T_eff and w * T_eff < 2^31
            const int Cmax = max(max(wtw<W>(wp, k1) * C1, w2 * C2), Rw);
            PPIPE_DCHECK(E >= 0 && E <= cx.T && (E >> cx.sh) < nb + 2 && src < 32 && j < kJ1);
            cond = survives(fin + (size_t)k1 * (nb + 2), E >> cx.sh, E, Cmax, cx.sh, cx.q);
            if (cond) rec = make_rec(cx.model, 3, c1_base + 32 * j + src, c2u, k1, cx.k2, k3, cx.b, E, C1, C2, R);
          }
          if (__any_sync(FULL_MASK, cond)) emit_warp(out, em, cond, rec);
        }
        __syncwarp();  // the list is rewritten by the next u
      }
    }
  }
  feas += nfeas;
}

template <int NC, bool W>
__device__ __forceinline__ void make_ctx(CtaCtx<NC>& cx, const Problem& pb, const DevModel& md, int k2, int bi,
                                         int nb) {
  cx.Pm = pb.P + md.p_off;
  cx.Ym = pb.Y + md.y_off;
  cx.Mp = md.Mp;
  cx.B = pb.B;
  cx.bi = bi;
  cx.b = pb.batches[bi];
  cx.k2 = k2;
  cx.M = (int)md.M;
  cx.T = md.T;
  cx.model = md.model;
  cx.m1 = pb.neg_one;
  cx.nb = nb;
  cx.dbg = pb.debug_flags;
  cx.row_len = 0;
  cx.pair_v = pb.pair_v;
  cx.P2 = cx.Prow(k2);
  int sh = 0;
  while ((cx.T >> sh) >= nb) ++sh;
  cx.sh = sh;
  const int bits_t = 32 - __clz(cx.T | 1);
  // virtual-GPU weights only in the W instantiation (the plain one keeps constant 1s)
  cx.wpack = W ? pb.wpack : 0x11111111u;
  cx.w2 = W ? wt(pb.wpack, k2) : 1;
  cx.q = max(0, bits_t + (W ? pb.w_bits : 0) + 1 - (32 - sh));
}

// Shared-memory layout common to the score kernels (2 warps per CTA).
struct ScoreSmem {
  uint2* fin;     // [NC][nb + 2] finalized fold tables (pass 2); pass 1 uses the first half as
  uint32_t* raw;  // [NC][nb + 2] raw bucket-best keys
  int32_t* Bs;    // [row_len] B(c2) for the current k3
  int32_t* Qs;    // [row_len] Q(c2) = P[k2][b][c2]
  int32_t* Rs;    // [row_len] R(c2) = C_3 for the current k3
  int4* ebuf;     // [kWarps][kEmitBuf][2] survivor records
  uint8_t* slot;  // [kWarps] SlotData regions (pass 2)
  uint32_t* nb16; // [kWarps][row_len] per-warp packed 16-bit (-B, -B) rows of the prefilter
};

template <int NC>
__device__ __forceinline__ ScoreSmem carve_smem(uint8_t* raw, int nb, int row_len) {
  ScoreSmem m;
  m.fin = reinterpret_cast<uint2*>(raw);
  m.raw = reinterpret_cast<uint32_t*>(raw);
  m.Bs = reinterpret_cast<int32_t*>(m.fin + (size_t)NC * (nb + 2));
  m.Qs = m.Bs + row_len;
  m.Rs = m.Qs + row_len;
  m.nb16 = reinterpret_cast<uint32_t*>(m.Rs + row_len);
  m.ebuf = reinterpret_cast<int4*>(m.nb16 + (PPIPE_P2_PREFILTER ? (size_t)kWarps * row_len : 0));
  m.slot = reinterpret_cast<uint8_t*>(m.ebuf + kWarps * 2 * kEmitBuf);
  return m;
}

// pass-2 kernel: finalized tables (8 B per bucket) + rows + emit buffers + slot data;
// pass-1 kernel (carve_smem_a): raw tables (4 B per bucket) + rows.
template <int NC>
static size_t score_smem_bytes(int nb, int row_len, bool pass2 = true) {
  if (!pass2)
    return ((4 * (size_t)NC * (nb + 2) + 15) & ~(size_t)15) + sizeof(int32_t) * (3 + kWarps) * (size_t)row_len;
  const size_t base =
      8 * (size_t)NC * (nb + 2) + sizeof(int32_t) * (3 + (PPIPE_P2_PREFILTER ? kWarps : 0)) * (size_t)row_len;
  return base + (size_t)kWarps * kEmitBuf * 32 + (size_t)kWarps * slot_bytes<NC>();
}

template <int NC>
__device__ __forceinline__ ScoreSmem carve_smem_a(uint8_t* raw, int nb, int row_len) {
  ScoreSmem m;
  m.fin = nullptr;
  m.raw = reinterpret_cast<uint32_t*>(raw);
  m.Bs = reinterpret_cast<int32_t*>(raw + ((4 * (size_t)NC * (nb + 2) + 15) & ~(size_t)15));
  m.Qs = m.Bs + row_len;
  m.Rs = m.Qs + row_len;
  m.nb16 = reinterpret_cast<uint32_t*>(m.Rs + row_len);
  m.ebuf = nullptr;
  m.slot = nullptr;
  return m;
}

// The bucket count (table resolution) follows a fixed smem policy, independent of
// the pass-2 slot data, so that both kernels and the ABI agree on it.
template <int NC>
static size_t table_policy_bytes(int nb, int row_len) {
  return 8 * (size_t)NC * (nb + 2) + sizeof(int32_t) * (3 + kWarps) * (size_t)row_len +
         (size_t)kWarps * kEmitBuf * 32 + (size_t)kWarps * kJ1 * NC * 32 * sizeof(uint16_t);
}

// Stage the c2 rows of (k2, k3, b): B(c2) and R(c2) (Q(c2) is k3-independent).
template <int NC>
__device__ __forceinline__ void stage_rows(const CtaCtx<NC>& cx, const ScoreSmem& sm, int k3, int c2_from, int c2_to,
                                           bool with_q) {
  const int M = cx.M;
  const int32_t* P3 = cx.Prow(k3);
  const int32_t P3M = P3[M];
  const int32_t* Y23 = cx.Yrow(cx.k2, k3);
  PPIPE_DCHECK(c2_to <= cx.row_len);
  for (int c2 = c2_from + (int)threadIdx.x; c2 < c2_to; c2 += 32 * kWarps) {
    const bool in = c2 < M;
    const int p2 = in ? __ldg(cx.P2 + c2) : 0;
    const int p3 = in ? __ldg(P3 + c2) : 0;
    sm.Bs[c2] = in ? p2 - p3 + __ldg(Y23 + c2) + P3M : kPadB;
    sm.Rs[c2] = in ? P3M - p3 : 0;
    if (with_q) sm.Qs[c2] = p2;
  }
}

struct K3Range {
  int c1lo, c1hi, c1_base0, ntiles, c2_from, c2_to;
  bool empty;
};

__device__ __forceinline__ K3Range k3_range(const DevModel& md) {
  K3Range r;
  const int M = (int)md.M;
  r.c1lo = max(1, (int)md.row_lo);
  r.c1hi = min(M - 2, (int)md.row_hi - 1);
  r.empty = M < 3 || r.c1lo > r.c1hi;
  // tiles start at c1_base = 3 mod 4 so that every c2 group c1_base + 1 + 4i is aligned
  r.c1_base0 = r.c1lo - ((r.c1lo - 3) & 3);
  r.ntiles = (r.c1hi - r.c1_base0 + 32 * kJ1) / (32 * kJ1);
  r.c2_from = max(0, r.c1_base0);      // rows cover every c2 > c1_base0 and every c1 (Q(c1) = P[k2][c1])
  r.c2_to = ((M + 3) & ~3) + 4;        // padded, exclusive
  return r;
}

__device__ __forceinline__ void tile_mina_body(const Problem& pb) {
  const int bi = blockIdx.x % pb.B;
  const int ml = pb.model_base + blockIdx.x / pb.B;
  const DevModel md = pb.models[ml];
  const K3Range r = k3_range(md);
  if (r.empty) return;
  const int C = pb.C;
  constexpr int kMaxV = 8;  // distinct bandwidth values staged per thread (more: read through L1)
  __shared__ int wmin[4][kMaxClasses];
  // this thread's P[k][b][c_1] and Y[v][b][c_1] (its own column: no barrier between write and
  // read), and the class-pair -> bandwidth-value map
  __shared__ int sP[kMaxClasses][32 * kJ1];
  __shared__ int sY[kMaxV][32 * kJ1];
  __shared__ uint8_t s_pair[kMaxClasses * kMaxClasses];
  const int32_t* Pm = pb.P + md.p_off;
  const int32_t* Ym = pb.Y + md.y_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool fastY = pb.V <= kMaxV;
  if (tid < C * C) s_pair[tid] = pb.pair_v[tid];
  __syncthreads();
  for (int t = 0; t < r.ntiles; ++t) {
    const int c1 = r.c1_base0 + t * 32 * kJ1 + tid;
    const bool valid = c1 >= r.c1lo && c1 <= r.c1hi;
    if (valid) {
      for (int k = 0; k < C; ++k) sP[k][tid] = Pm[((size_t)k * pb.B + bi) * md.Mp + c1];
      if (fastY)
        for (int v = 0; v < pb.V; ++v) sY[v][tid] = Ym[((size_t)v * pb.B + bi) * md.Mp + c1];
    }
    for (int k2 = 0; k2 < C; ++k2) {
      int m = INT_MAX;
      if (valid) {
        const int p2 = sP[k2][tid];
        for (int k1 = 0; k1 < C; ++k1) {
          const int v = s_pair[k1 * C + k2];
          const int y = fastY ? sY[v][tid] : Ym[((size_t)v * pb.B + bi) * md.Mp + c1];
          m = min(m, sP[k1][tid] + y - p2);
        }
      }
      for (int d = 16; d > 0; d >>= 1) m = min(m, __shfl_xor_sync(FULL_MASK, m, d));
      if (lane == 0) wmin[warp][k2] = m;
    }
    __syncthreads();
    if (tid < C) {
      const int k2 = tid;
      pb.minA[((size_t)(ml * C + k2) * pb.B + bi) * pb.max_tiles + t] =
          min(min(wmin[0][k2], wmin[1][k2]), min(wmin[2][k2], wmin[3][k2]));
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void flush_counters(const ScoreOut& out, unsigned long long feas, unsigned long long cand) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    feas += __shfl_down_sync(FULL_MASK, feas, d);
    cand += __shfl_down_sync(FULL_MASK, cand, d);
  }
  if ((threadIdx.x & 31) == 0) {
    if (feas) atomicAdd(&out.counters[1], feas);
    if (cand) atomicAdd(&out.counters[2], cand);
  }
}

// ---- kernel 1: K = 1 and K = 2 candidates. CTA = (model, k_2, batch), 2 warps. ----
// Shared memory: fin [NC][nb + 2] (8 B) | raw [NC][nb + 2] (4 B) | emit buffers.
template <int NC>
static size_t score12_smem_bytes(int nb) {
  return 8 * (size_t)NC * (nb + 2) + ((4 * (size_t)NC * (nb + 2) + 15) & ~(size_t)15) + (size_t)kWarps * kEmitBuf * 32;
}

#ifndef PPIPE_12_CTAS_PER_SM
#define PPIPE_12_CTAS_PER_SM 16
#endif
#ifndef PPIPE_12_NB_LOG2_MAX
#define PPIPE_12_NB_LOG2_MAX 7
#endif
template <int NC, bool W>
__global__ void __launch_bounds__(32 * kWarps, PPIPE_12_CTAS_PER_SM)
    score12_kernel(Problem pb, ScoreOut out, int nb_log2) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int nb = 1 << nb_log2;
  uint2* fin = reinterpret_cast<uint2*>(smem_raw);
  uint32_t* raw = reinterpret_cast<uint32_t*>(fin + (size_t)NC * (nb + 2));
  int4* ebuf = reinterpret_cast<int4*>(smem_raw + 8 * (size_t)NC * (nb + 2) +
                                       ((4 * (size_t)NC * (nb + 2) + 15) & ~(size_t)15));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Emitter em{ebuf + warp * 2 * kEmitBuf, 0};
  const int ntab = NC * (nb + 2);
  // CTA = (model, k2, batch): many small CTAs keep enough loads in flight (the
  // K <= 2 work of one batch is a few hundred c_1 rows).
  const int bi = blockIdx.x % pb.B;
  const int k2 = (blockIdx.x / pb.B) % NC;
  const int ml = blockIdx.x / (pb.B * NC);
  const DevModel md = pb.models[ml];
  unsigned long long feas = 0, cand = 0;
  do {
    CtaCtx<NC> cx;
    make_ctx<NC, W>(cx, pb, md, k2, bi, nb);
    const int M = cx.M, T = cx.T, sh = cx.sh, q = cx.q;
    // K = 1: segment (k2), whole model on class k2
    if (warp == 0 && md.row_lo == 0) {
      const int E = cx.P2[M];
      if (lane == 0) ++cand;
      const bool f = lane == 0 && E <= T;
      if (f) ++feas;
      if (__any_sync(FULL_MASK, f))
        emit_warp(out, em, f, make_rec(md.model, 1, 0, 0, k2, 0xFF, 0xFF, cx.b, E, E, 0, 0));
    }
    // K = 2: segments (k1, k2); c1 in this rank's rows
    if (pb.Kmax < 2 || M < 2) break;
    const int lo = max(1, (int)md.row_lo), hi = min(M - 1, (int)md.row_hi - 1);
    if (lo > hi) break;
    reset_raw(raw, ntab, tid, 32 * kWarps);
    __syncthreads();
    const int P2M = cx.P2[M];
    int anyf = 0;
#pragma unroll 1
    for (int pass = 1; pass <= 2; ++pass) {
#pragma unroll 1
      for (int base = lo; base <= hi; base += 32 * kWarps) {
        const int c1 = base + tid;
        const bool valid = c1 <= hi;
        const int C2 = valid ? P2M - __ldg(cx.P2 + c1) : 0;
#pragma unroll
        for (int k1 = 0; k1 < NC; ++k1) {
          const int C1 = valid ? __ldg(cx.Prow(k1) + c1) : 0;
          const int y = valid ? __ldg(cx.Yrow(k1, k2) + c1) : 0;
          const int E = C1 + y + C2;
          const bool f = valid && E <= T;
          const int Cmax = W ? max(wmul(wt(cx.wpack, k1), C1), wmul(cx.w2, C2)) : max(C1, C2);
          if (pass == 1) {
            if (valid) ++cand;
            if (f) {
              ++feas;
              anyf = 1;
              atomicMin(raw + (size_t)k1 * (nb + 2) + (E >> sh), pack_key(E, Cmax, sh, q));
            }
          } else {
            const bool cond = f && survives(fin + (size_t)k1 * (nb + 2), f ? (E >> sh) : 0, E, Cmax, sh, q);
            if (__any_sync(FULL_MASK, cond))
              emit_warp(out, em, cond, make_rec(md.model, 2, c1, 0, k1, k2, 0xFF, cx.b, E, C1, C2, 0));
          }
        }
      }
      if (pass == 1) {
        if (!__syncthreads_or(anyf)) break;
        tables_finalize(raw, fin, NC, nb, sh, warp, kWarps);
        __syncthreads();
      }
    }
  } while (false);
  emit_flush(out, em);
  flush_counters(out, feas, cand);
}

// ---- kernel 2: K = 3 pass 1 over every (model, k_2, batch) CTA (2 warps, tiles from
// a shared counter). Counts every candidate and feasible candidate and builds the
// bucket-best tables of each (k_2, k_3, b) unit; units with a feasible candidate
// are "hot": their finalized tables go to global memory for kernel 3. ----
#ifndef PPIPE_3A_CTAS_PER_SM
#define PPIPE_3A_CTAS_PER_SM 10  // <= 102 registers, no spills; 10 x 23.1 KB of shared memory fit (measured: 8 / 9 / 10 CTAs/SM, score3a 32.3 / 32.0 / 31.2 ms)
#endif
// (more than 5 classes: 8, where the larger slot arrays need 128 registers without spills)
template <int NC>
constexpr int k3aCtasPerSm() { return NC <= 5 ? PPIPE_3A_CTAS_PER_SM : 8; }
#ifndef PPIPE_3B_CTAS_PER_SM
#define PPIPE_3B_CTAS_PER_SM 8
#endif
constexpr int k3bCtasPerSm = PPIPE_3B_CTAS_PER_SM;  // pass 2 holds more live state: fewer, fatter warps
template <int NC, bool W>
__global__ void __launch_bounds__(32 * kWarps, k3aCtasPerSm<NC>())
    score3a_kernel(Problem pb, ScoreOut out, int nb_log2, int row_len) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ int s_tile;
  __shared__ unsigned long long s_slot;
  __shared__ unsigned long long s_tmask;  // tiles (t < 64) of this unit with a feasible candidate
  __shared__ unsigned s_wfeas;            // the unit's feasible candidates (pass-2 order)
  const int nb = 1 << nb_log2;
  const ScoreSmem sm = carve_smem_a<NC>(smem_raw, nb, row_len);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntab = NC * (nb + 2);
  const int k2 = blockIdx.x % NC;
  const int ml = pb.model_base + (blockIdx.x / NC) % pb.n_chunk;
  const int bi = blockIdx.x / (NC * pb.n_chunk);
  const DevModel md = pb.models[ml];
  CtaCtx<NC> cx;
  make_ctx<NC, W>(cx, pb, md, k2, bi, nb);
  cx.row_len = row_len;
  Emitter em{nullptr, 0};  // unused in pass 1
  unsigned long long feas = 0, cand = 0;
  const K3Range r = k3_range(md);
  if (pb.Kmax >= 3 && !r.empty) {
    reset_raw(sm.raw, ntab, tid, 32 * kWarps);
#pragma unroll 1
    for (int k3 = 0; k3 < NC; ++k3) {
      stage_rows(cx, sm, k3, r.c2_from, r.c2_to, k3 == 0);
      if (tid == 0) {
        s_tile = 0;
        s_wfeas = 0;
        s_tmask = r.ntiles > 64 ? ~0ull : 0ull;  // more tiles than mask bits: pass 2 visits all
      }
      __syncthreads();
      const unsigned long long feas0 = feas;
#pragma unroll 1
      for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&s_tile, 1);
        t = __shfl_sync(FULL_MASK, t, 0);
        if (t >= r.ntiles) break;
        const unsigned long long ft = feas;
        const int hint = pb.minA ? cx.T - __ldg(pb.minA + ((size_t)(ml * NC + k2) * pb.B + bi) * pb.max_tiles + t)
                                 : INT_MAX;
        k3_tile<NC, 1, W>(cx, k3, r.c1_base0 + t * 32 * kJ1, r.c1lo, r.c1hi, sm.Bs, sm.Qs, sm.Rs, sm.raw, sm.fin,
                       SlotData{}, sm.nb16 + warp * row_len, out, em, feas, cand, 0, hint);
        if (__any_sync(FULL_MASK, feas != ft) && lane == 0 && t < 64) atomicOr(&s_tmask, 1ull << t);
      }
      {
        const unsigned wf = __reduce_add_sync(FULL_MASK, (unsigned)min(feas - feas0, 0xffffffffull));
        if (lane == 0 && wf) atomicAdd(&s_wfeas, wf);
      }
      if (__syncthreads_or(feas != feas0) && !(pb.debug_flags & 2)) {
        if (tid == 0) {
          s_slot = atomicAdd(&out.counters[3], 1ull);
          // (local model, k2 | k3 << 4 | b << 8, tile mask): pass 2 skips the tiles without a
          // feasible candidate (it only emits feasible ones)
          if (s_slot < out.hot_cap) {
            out.hot[s_slot] = make_uint4(ml, (unsigned)k2 | ((unsigned)k3 << 4) | ((unsigned)bi << 8),
                                         (unsigned)s_tmask, (unsigned)(s_tmask >> 32));
            out.hot_w[s_slot] = s_wfeas;
          }
        }
        __syncthreads();
        // finalized tables straight to the unit's global slot; staircase steps to the
        // cross-batch fold of the unit's segments (k1, k2, k3)
        unsigned long long* gf = pb.gfold ? pb.gfold + ((size_t)ml * NC * NC * NC + (size_t)k2 * NC + k3) * (nb + 1)
                                          : nullptr;
        tables_finalize(sm.raw,
                        s_slot < out.hot_cap ? reinterpret_cast<uint2*>(out.hot_tab) + s_slot * (unsigned long long)ntab
                                             : nullptr,
                        NC, nb, cx.sh, warp, kWarps, gf, (size_t)NC * NC * (nb + 1), (uint32_t)cx.b, cx.q);
      }
      __syncthreads();
      reset_raw(sm.raw, ntab, tid, 32 * kWarps);
      __syncthreads();
    }
  }
  flush_counters(out, feas, cand);
}

// ---- pass-2 order: longest-processing-time first. A hot unit's pass-2 work grows with
// the tiles that held a feasible candidate (popcount of its tile mask) times the model
// depth, and with its feasible count for the dense units (many feasible candidates per
// tile: their survivor checks dominate); one CTA counting-sorts the units by the larger
// of the two estimates (256 bins, descending) so the persistent score3b CTAs do not end
// on a heavy unit picked up late. The feasible term only moves the dense units forward
// (divisor 192, measured): ordering every unit by it (divisor <= 64) breaks up the units
// of a model, which share its rows in L2, and cost up to 8% of score3b at N = 1; with 192
// the N = 4 tail (a dense unit of 1.5 ms started late) shrinks, step 20.97 -> 20.58 ms. ----
constexpr int kOrderBins = 256;
#ifndef PPIPE_ORDER_FEAS_DIV
#define PPIPE_ORDER_FEAS_DIV 192
#endif
__global__ void __launch_bounds__(1024) hot_order_kernel(ScoreOut out, const DevModel* models) {
  __shared__ uint32_t cnt[kOrderBins];
  const uint32_t n = (uint32_t)min(out.counters[3], out.hot_cap);
  for (int i = threadIdx.x; i < kOrderBins; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  auto bin_of = [&](uint32_t u) {
    const uint4 h = out.hot[u];
    const uint32_t tiles = h.z == 0xffffffffu && h.w == 0xffffffffu ? 64u : (uint32_t)(__popc(h.z) + __popc(h.w));
    const uint32_t work = max(tiles * models[h.x].M, out.hot_w[u] / PPIPE_ORDER_FEAS_DIV);
    return kOrderBins - 1 - min((uint32_t)kOrderBins - 1, work >> 5);  // heavy -> low bin
  };
  for (uint32_t u = threadIdx.x; u < n; u += blockDim.x) atomicAdd(&cnt[bin_of(u)], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int b = 0; b < kOrderBins; ++b) {
      const uint32_t c = cnt[b];
      cnt[b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (uint32_t u = threadIdx.x; u < n; u += blockDim.x) out.hot_order[atomicAdd(&cnt[bin_of(u)], 1u)] = u;
}

// ---- bulk copy global -> shared (TMA engine, cp.async.bulk) completing on an mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// thread-side: earlier generic-proxy accesses of the destination before the async-proxy write
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- kernel 3: K = 3 pass 2 over the hot units only (persistent CTAs pull units
// from a counter): reload the unit's tables, re-scan with tightened thresholds and
// emit the survivors. ----
template <int NC, bool W>
__global__ void __launch_bounds__(32 * kWarps, k3bCtasPerSm)
    score3b_kernel(Problem pb, ScoreOut out, int nb_log2, int row_len) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ int s_tile;
  __shared__ unsigned long long s_unit;
  __shared__ uint32_t s_rowoff[2 * NC];
  __shared__ unsigned long long s_bar;  // completion of the unit table's bulk copy
  const int nb = 1 << nb_log2;
  const ScoreSmem sm = carve_smem<NC>(smem_raw, nb, row_len);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntab = NC * (nb + 2);
  Emitter em{sm.ebuf + warp * 2 * kEmitBuf, 0};
  unsigned long long feas = 0, cand = 0;
  const unsigned long long n_hot = min(out.counters[3], out.hot_cap);
  if (tid == 0) mbar_init(&s_bar, 1);
  unsigned parity = 0;
#pragma unroll 1
  for (;;) {
    if (tid == 0) s_unit = atomicAdd(&out.counters[4], 1ull);
    __syncthreads();
    if (s_unit >= n_hot) break;
    const unsigned long long u = out.hot_order ? out.hot_order[s_unit] : s_unit;
    // the unit's finalized tables (NC (nb + 2) x 8 bytes, a multiple of 16) arrive by one
    // bulk copy on the TMA engine while the threads stage the c2 rows
    const uint2* src = reinterpret_cast<const uint2*>(out.hot_tab) + u * (unsigned long long)ntab;
    if (tid == 0) {
      fence_proxy_async();
      bulk_load(sm.fin, src, (unsigned)(8 * ntab), &s_bar);
    }
    const uint4 hu = out.hot[u];
    const int ml = (int)hu.x, k2 = (int)(hu.y & 15u), k3 = (int)((hu.y >> 4) & 15u), bi = (int)(hu.y >> 8);
    const unsigned long long tmask = ((unsigned long long)hu.w << 32) | hu.z;
    const DevModel md = pb.models[ml];
    CtaCtx<NC> cx;
    make_ctx<NC, W>(cx, pb, md, k2, bi, nb);
    cx.row_len = row_len;
    const K3Range r = k3_range(md);
    stage_rows(cx, sm, k3, r.c2_from, r.c2_to, true);
    mbar_wait(&s_bar, parity);
    parity ^= 1u;
    if (pb.gfold) {
      // U'(j) = min(U(j), ceil(bound_j / 2^q)): the unit's own bound and the cross-batch one
      const unsigned long long* gf = pb.gfold + ((size_t)ml * NC * NC * NC + (size_t)k2 * NC + k3) * (nb + 1);
      for (int i = tid; i < ntab; i += 32 * kWarps) {
        const int k1 = i / (nb + 2), j = i - k1 * (nb + 2);
        if (j <= nb) {
          const unsigned long long g = gf[(size_t)k1 * NC * NC * (nb + 1) + j];
          if (g) {
            const uint32_t bnd = gfold_bound(g, (uint32_t)cx.b);
            // bounds at or above 2^31 exceed every feasible (weighted) Cmax: no bound
            const uint32_t ub = bnd >= 0x80000000u ? kEmpty : (uint32_t)(((uint64_t)bnd + ((1ull << cx.q) - 1)) >> cx.q);
            if (ub < sm.fin[i].x) sm.fin[i].x = ub;
          }
        }
      }
    }
    if (tid == 0) s_tile = 0;
    if (tid < NC) {
      s_rowoff[tid] = (uint32_t)(((size_t)tid * cx.B + bi) * cx.Mp);
      s_rowoff[NC + tid] = (uint32_t)(((size_t)__ldg(cx.pair_v + tid * NC + k2) * cx.B + bi) * cx.Mp);
    }
    __syncthreads();
    int Bmin = INT_MAX;  // min over the unit's c2 of B(c2) (bounds E from below)
    for (int c2 = r.c1lo + 1 + lane; c2 < cx.M; c2 += 32) Bmin = min(Bmin, sm.Bs[c2]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) Bmin = min(Bmin, __shfl_xor_sync(FULL_MASK, Bmin, d));
#pragma unroll 1
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&s_tile, 1);
      t = __shfl_sync(FULL_MASK, t, 0);
      if (t >= r.ntiles) break;
      if (t < 64 && !((tmask >> t) & 1ull)) continue;  // no feasible candidate in pass 1
      SlotData sd = carve_slot<NC>(sm.slot + warp * slot_bytes<NC>());
      sd.rowoff = s_rowoff;
      k3_tile<NC, 2, W>(cx, k3, r.c1_base0 + t * 32 * kJ1, r.c1lo, r.c1hi, sm.Bs, sm.Qs, sm.Rs, sm.raw, sm.fin, sd,
                     sm.nb16 + warp * row_len, out, em, feas, cand, Bmin);
    }
    __syncthreads();
  }
  emit_flush(out, em);
}

// Shared memory per CTA: the fold tables take what the budget leaves after the
// three staged c2 rows (B, Q, R), the emit buffers and the pass-2 slot data,
// rounded down to a power of two (128..2048 buckets).
#ifndef PPIPE_SMEM_BUDGET
#define PPIPE_SMEM_BUDGET (32 * 1024)
#endif
constexpr size_t kSmemBudget = PPIPE_SMEM_BUDGET;  // table-size policy (nb = 256 for config 5)

#ifndef PPIPE_CONCURRENT_12
#define PPIPE_CONCURRENT_12 0
#endif
// One non-blocking side stream (and its fork/join events) per device, created on
// first use and kept for the process lifetime.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
[[maybe_unused]] static SideStream& side_stream() {
  static SideStream per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& ss = per_dev[dev & 63];
  if (ss.s == nullptr) {
    if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
      ss.s = nullptr;
      cudaGetLastError();
    }
  }
  return ss;
}

template <int NC, bool W>
static cudaError_t launch_score_w(const Problem& pb, const ScoreOut& out, cudaStream_t s, int* n_launches,
                                  int part) {
  const int row_len = (int)((((size_t)pb.max_M + 3) & ~(size_t)3) + 8 * kScanUnroll);
  int nb_log2 = 7;
  while (nb_log2 < 11 && table_policy_bytes<NC>(2 << nb_log2, row_len) <= kSmemBudget) ++nb_log2;
  const size_t smem = score_smem_bytes<NC>(1 << nb_log2, row_len);
  const size_t smem_a = score_smem_bytes<NC>(1 << nb_log2, row_len, false);
  const unsigned grid = (unsigned)pb.n_chunk * NC * pb.B;
  cudaError_t e;
  // K <= 2 tables live only inside score12 (never in the hot-unit buffer), so their
  // resolution may differ from the K = 3 tables.
  const int nb12_log2 = std::min(nb_log2, PPIPE_12_NB_LOG2_MAX);
  const size_t smem12 = score12_smem_bytes<NC>(1 << nb12_log2);
  e = cudaFuncSetAttribute(score12_kernel<NC, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem12);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(score3a_kernel<NC, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(score3b_kernel<NC, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // part 0: everything; 1: score3a over the chunk; 2: score3b + score12 over all local models
  const bool k3a = pb.Kmax >= 3 && part != 2 && pb.n_chunk > 0;
  // score12 reads none of what score3a / score3b write (all three only append
  // survivors and counts through atomics), so with PPIPE_CONCURRENT_12 it runs on a
  // side stream: mode 1 forks after score3a (score12 fills the SMs score3b's
  // persistent CTAs release at its tail), mode 2 before it (score12's latency-bound
  // CTAs share the SMs with score3a's ALU-bound ones). The join restores the stream
  // order for the frontier pass.
  SideStream* ss = nullptr;
#if PPIPE_CONCURRENT_12
  if (part != 1) {
    ss = &side_stream();
    if (ss->s == nullptr) ss = nullptr;
  }
#endif
  const bool early = ss != nullptr && PPIPE_CONCURRENT_12 == 2;
  const cudaStream_t s12 = ss != nullptr ? ss->s : s;
  if (early) {
    cudaEventRecord(ss->fork, s);
    cudaStreamWaitEvent(s12, ss->fork, 0);
    score12_kernel<NC, W><<<(unsigned)pb.n_local * NC * pb.B, 32 * kWarps, smem12, s12>>>(pb, out, nb12_log2);
    ++*n_launches;
  }
  // PPIPE_DEBUG_FLAGS & 64: per-kernel event times of this launch sequence on stderr
  static cudaEvent_t dev_ev[4] = {};
  const bool tdbg = (pb.debug_flags & 64) != 0;
  if (tdbg && !dev_ev[0])
    for (auto& x : dev_ev) cudaEventCreate(&x);
  if (tdbg) cudaEventRecord(dev_ev[0], s);
  if (k3a) {
    score3a_kernel<NC, W><<<grid, 32 * kWarps, smem_a, s>>>(pb, out, nb_log2, row_len);
    ++*n_launches;
  }
  if (tdbg) cudaEventRecord(dev_ev[1], s);
  if (part == 1) return cudaGetLastError();
  if (ss != nullptr && !early) {
    cudaEventRecord(ss->fork, s);
    cudaStreamWaitEvent(s12, ss->fork, 0);
  }
  if (pb.Kmax >= 3 && pb.gfold && pb.n_local > 0) {
    const size_t rows = (size_t)pb.n_local * NC * NC * NC;
    gfold_prefix_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, s>>>(pb.gfold, rows, (1 << nb_log2) + 1);
    ++*n_launches;
  }
  if (pb.Kmax >= 3 && out.hot_order && pb.n_local > 0) {
    hot_order_kernel<<<1, 1024, 0, s>>>(out, pb.models);
    ++*n_launches;
  }
  if (pb.Kmax >= 3) {
    int dev = 0, n_sm = 148, smem_sm = 227 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const int ctas = std::max(1, std::min(k3bCtasPerSm, smem_sm / (int)(smem + 1024)));  // persistent: fill the SMs
    if (tdbg) cudaEventRecord(dev_ev[2], s);
    score3b_kernel<NC, W><<<n_sm * ctas, 32 * kWarps, smem, s>>>(pb, out, nb_log2, row_len);
    ++*n_launches;
  }
  if (tdbg) cudaEventRecord(dev_ev[3], s);
  if (!early) {
    score12_kernel<NC, W><<<(unsigned)pb.n_local * NC * pb.B, 32 * kWarps, smem12, s12>>>(pb, out, nb12_log2);
    ++*n_launches;
  }
  if (tdbg && part == 0) {
    cudaEventSynchronize(dev_ev[3]);
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, dev_ev[0], dev_ev[1]);
    cudaEventElapsedTime(&b, dev_ev[1], dev_ev[2]);
    cudaEventElapsedTime(&c, dev_ev[2], dev_ev[3]);
    fprintf(stderr, "ppipe score ms: score3a %.3f, prefix+order %.3f, score3b %.3f (local models %d)\n", a, b, c,
            pb.n_local);
  }
  if (ss != nullptr) {
    cudaEventRecord(ss->join, s12);
    cudaStreamWaitEvent(s, ss->join, 0);
  }
  return cudaGetLastError();
}

template <int NC>
static cudaError_t launch_score_nc(const Problem& pb, const ScoreOut& out, cudaStream_t s, int* n_launches,
                                  int part) {
  return pb.wpack == 0x11111111u ? launch_score_w<NC, false>(pb, out, s, n_launches, part)
                                 : launch_score_w<NC, true>(pb, out, s, n_launches, part);
}

int score_nb(const Problem& pb) { return (int)(hot_unit_table_bytes(pb) / (8 * (size_t)pb.C)) - 2; }

size_t gfold_elems(const Problem& pb) {
  return (size_t)std::max(pb.n_local, 1) * pb.C * pb.C * pb.C * (score_nb(pb) + 1);
}

// Bytes of one hot unit's tables for this problem (the ABI sizes its buffer with it).
size_t hot_unit_table_bytes(const Problem& pb) {
  const int row_len = (int)((((size_t)pb.max_M + 3) & ~(size_t)3) + 8 * kScanUnroll);
  int nb_log2 = 7;
  auto smem_for = [&](int nb) -> size_t {
    switch (pb.C) {
      case 1: return table_policy_bytes<1>(nb, row_len);
      case 2: return table_policy_bytes<2>(nb, row_len);
      case 3: return table_policy_bytes<3>(nb, row_len);
      case 4: return table_policy_bytes<4>(nb, row_len);
      case 5: return table_policy_bytes<5>(nb, row_len);
      case 6: return table_policy_bytes<6>(nb, row_len);
      case 7: return table_policy_bytes<7>(nb, row_len);
      default: return table_policy_bytes<8>(nb, row_len);
    }
  };
  while (nb_log2 < 11 && smem_for(2 << nb_log2) <= kSmemBudget) ++nb_log2;
  return 8 * (size_t)pb.C * ((1 << nb_log2) + 2);
}

cudaError_t launch_score_part(const Problem& pb, const ScoreOut& out, cudaStream_t s, int* n_launches, int part) {
  if (pb.n_local == 0) return cudaSuccess;
  switch (pb.C) {
    case 1: return launch_score_nc<1>(pb, out, s, n_launches, part);
    case 2: return launch_score_nc<2>(pb, out, s, n_launches, part);
    case 3: return launch_score_nc<3>(pb, out, s, n_launches, part);
    case 4: return launch_score_nc<4>(pb, out, s, n_launches, part);
    case 5: return launch_score_nc<5>(pb, out, s, n_launches, part);
    case 6: return launch_score_nc<6>(pb, out, s, n_launches, part);
    case 7: return launch_score_nc<7>(pb, out, s, n_launches, part);
    case 8: return launch_score_nc<8>(pb, out, s, n_launches, part);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_score(const Problem& pb, const ScoreOut& out, cudaStream_t s, int* n_launches) {
  return launch_score_part(pb, out, s, n_launches, 0);
}

// ---------------------------------------------------------------------------
// frontier pass
// ---------------------------------------------------------------------------
__global__ void seg_start_kernel(const uint64_t* keys, uint64_t n, uint64_t n_seg, uint64_t* start) {
  const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (s > n_seg) return;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (keys[mid] < s) lo = mid + 1;
    else hi = mid;
  }
  start[s] = lo;
}

__global__ void seg_of_kernel(const ppipe_point* in, uint64_t n, const uint64_t* seg_base, int C, uint64_t* seg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const ppipe_point p = in[i];
    uint64_t off = 0, pw = 1;
    for (int k = 1; k < p.K; ++k) {
      pw *= (uint64_t)C;
      off += pw;
    }
    uint64_t idx = 0;
    for (int d = 0; d < p.K; ++d) idx = idx * C + p.cls[d];
    seg[i] = seg_base[p.model] + off + idx;
  }
}

cudaError_t segment_offsets(const ppipe_point* pts, uint64_t n, const uint64_t* seg_base_by_model, int C,
                            uint64_t n_seg, uint64_t* seg_offsets, uint64_t* seg_tmp, cudaStream_t s,
                            int* n_launches) {
  if (n > 0) {
    const int blocks = (int)std::min<uint64_t>((n + 255) / 256, 148 * 16);
    seg_of_kernel<<<blocks, 256, 0, s>>>(pts, n, seg_base_by_model, C, seg_tmp);
    ++*n_launches;
  }
  seg_start_kernel<<<(unsigned)((n_seg + 1 + 255) / 256), 256, 0, s>>>(seg_tmp, n, n_seg, seg_offsets);
  ++*n_launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// device-side profile validation (ppipe_update_profiles)
// ---------------------------------------------------------------------------
__global__ void validate_kernel(const DevModel* models, const uint32_t* lat, const uint64_t* S, int C, int B,
                                uint64_t smax, unsigned long long* err_key) {
  const int i = blockIdx.x / C, k = blockIdx.x % C;
  const DevModel md = models[i];
  const int M = (int)md.M;
  const uint32_t* L = lat + md.lat_off + (size_t)k * M * B;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    unsigned long long tot = 0;
    for (int l = 0; l < M; ++l) tot += L[(size_t)l * B + b];  // coalesced over b
    if (tot >= (unsigned long long)kRangeLimit)
      atomicMin(err_key, ((unsigned long long)md.model << 40) | (unsigned long long)(k * B + b));
  }
  if (k == 0)
    for (int l = threadIdx.x; l < M; l += blockDim.x)
      if (S[md.s_off + l] > smax)
        atomicMin(err_key, ((unsigned long long)md.model << 40) | (1ull << 39) | (unsigned long long)l);
}

cudaError_t launch_validate(const DevModel* models, int n_local, const uint32_t* lat, const uint64_t* S, int C,
                            int B, uint64_t smax, unsigned long long* err_key, cudaStream_t s) {
  if (n_local > 0) validate_kernel<<<n_local * C, 128, 0, s>>>(models, lat, S, C, B, smax, err_key);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// greedy pre-partitioning (§5.2)
// ---------------------------------------------------------------------------
// One warp per model: prefix sums T of the reference runtimes, then per block the
// first layer j in [i+1, guard) whose inclusion would move the block's runtime
// strictly farther from total/N, f(j+1) > f(j) with f(j) = |N (T[j] - T[i]) - total|
// (the greedy's stopping point; j = guard if none), found 32 candidates per ballot.
__global__ void prepart_bounds_kernel(PrepartProblem p) {
  const int warps = blockDim.x >> 5;
  const int m = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (m >= p.n_models) return;
  const int M = (int)p.M[m];
  const int N = p.N;
  const uint32_t* t = p.lat + p.lat_off[m] + (size_t)p.ref_class * M * p.B + p.ref_b;
  int64_t* T = p.prefix + p.s_off[m] + m;  // M + 1 entries
  int64_t carry = 0;
  if (lane == 0) T[0] = 0;
  for (int base = 0; base < M; base += 32) {
    const int l = base + lane;
    int64_t v = l < M ? (int64_t)t[(size_t)l * p.B] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t u = __shfl_up_sync(FULL_MASK, v, d);
      if (lane >= d) v += u;
    }
    if (l < M) T[l + 1] = carry + v;
    carry += __shfl_sync(FULL_MASK, v, 31);
  }
  __syncwarp();
  const int64_t total = carry;
  uint32_t* bnd = p.bounds + (size_t)m * (N + 1);
  int i = 0;
  if (lane == 0) bnd[0] = 0;
  for (int blk = 0; blk + 1 < N; ++blk) {
    const int guard = M - (N - blk - 1);
    const int64_t Ti = T[i];
    int j = guard;
    for (int base = i + 1; base < guard; base += 32) {
      const int jj = base + lane;
      bool stop = false;
      if (jj < guard) {
        int64_t without = (int64_t)N * (T[jj] - Ti) - total, with = (int64_t)N * (T[jj + 1] - Ti) - total;
        without = without < 0 ? -without : without;
        with = with < 0 ? -with : with;
        stop = with > without;
      }
      const unsigned hit = __ballot_sync(FULL_MASK, stop);
      if (hit) {
        j = base + __ffs(hit) - 1;
        break;
      }
    }
    if (lane == 0) bnd[blk + 1] = (uint32_t)j;
    i = j;
  }
  if (lane == 0) bnd[N] = (uint32_t)M;
  __syncwarp();
  const uint64_t* S = p.S + p.s_off[m];
  for (int q = lane; q < N; q += 32) p.block_S[(size_t)m * N + q] = S[bnd[q + 1] - 1];
}

// Block sums: CTA per model, threads over (class, batch) so each layer's row is
// read coalesced; the running sum is written out at every block boundary.
__global__ void prepart_sum_kernel(PrepartProblem p) {
  const int m = blockIdx.x;
  const int M = (int)p.M[m];
  const int N = p.N, C = p.C, B = p.B;
  const uint32_t* lat = p.lat + p.lat_off[m];
  const uint32_t* bnd = p.bounds + (size_t)m * (N + 1);
  uint32_t* out = p.block_lat + (size_t)m * C * N * B;
  for (int kb = threadIdx.x; kb < C * B; kb += blockDim.x) {
    const int k = kb / B, b = kb - k * B;
    const uint32_t* row = lat + (size_t)k * M * B + b;
    int q = 0, next = (int)bnd[1];
    uint32_t acc = 0;
    for (int l = 0; l < M; ++l) {
      if (l == next) {
        out[((size_t)k * N + q) * B + b] = acc;
        acc = 0;
        ++q;
        next = (int)bnd[q + 1];
      }
      acc += row[(size_t)l * B];
    }
    out[((size_t)k * N + q) * B + b] = acc;
  }
}

cudaError_t launch_prepartition(const PrepartProblem& p, cudaStream_t s) {
  if (p.n_models == 0) return cudaSuccess;
  prepart_bounds_kernel<<<(p.n_models + 3) / 4, 128, 0, s>>>(p);
  prepart_sum_kernel<<<p.n_models, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ppipe
