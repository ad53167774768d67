// ppipe_pb.cu -- per-stage batch sizes (App. A.1).
//
// The basic MILP of App. A.1 lets every partition run its own batch size: eq. 1.1
// sums p_{ldbij} over (b, i, j) per partition d. A candidate is
// (cuts, classes, b_1..b_K) with
//   C_d = sum of lat[k_d][l][b_d] over partition d              (eq. 1.9)
//   Y_d = ceil(8 S[c_d - 1] b_d / bw[k_d][k_{d+1}]), d < K       (eq. 1.11: the sender's batch)
//   E = sum C_d + sum Y_d <= T_eff                               (eq. 1.12)
//   theta = min_d b_d / C_d                                      (x_l = min_d x_ld)
// reduced per segment to the (E min, theta max) staircase; ties on identical
// (E, theta) keep the smallest (b_1..b_K) (lexicographic batch indices), then the
// smallest (c_1, c_2) (PB-1..PB-4). B^K times the unified candidates.
//
// pb_score_kernel<K>: one CTA per unit (K = 3: segment, c_1, b_2; K = 2: segment, b_1;
// K = 1: segment) enumerates the unit's candidates twice. Pass 1 folds each feasible
// candidate's theta into its E-bucket (atomicMax on an order-preserving 64-bit key,
// see theta_key); an exclusive prefix maximum over the buckets then gives, per bucket,
// the best theta of every smaller E. Pass 2 emits only the candidates above it -- a
// candidate at or below it is beaten by a feasible candidate with strictly smaller E,
// so the drop is exact and the survivors' frontier is the unit's. pb_frontier_pass
// reduces all survivors: sort by (segment, E), best per (segment, E), strict
// staircase over theta, CSR.
#include <climits>

#include "ppipe_block.cuh"
#include "ppipe_internal.h"

namespace ppipe {

namespace {

constexpr int kPbThreads = 256;
constexpr int kPbBuckets = 1024;  // E-buckets per unit (4 per thread in the prefix scan)

__device__ __forceinline__ const int32_t* prow_pb(const Problem& pb, const DevModel& md, int k, int bi) {
  return pb.P + md.p_off + ((size_t)k * pb.B + bi) * md.Mp;
}
__device__ __forceinline__ const int32_t* yrow_pb(const Problem& pb, const DevModel& md, int k, int k2, int bi) {
  return pb.Y + md.y_off + ((size_t)pb.pair_v[k * pb.C + k2] * pb.B + bi) * md.Mp;
}

// theta = b / C as a double is exact-order-preserving for b < 2^16, C < 2^28: two distinct
// fractions differ by a relative 1 / (b s) >= 2^-44, far above the 2^-53 rounding of each,
// and equal fractions round alike. Positive doubles (and +inf for C = 0) order as their
// bit patterns, so theta compares as one 64-bit integer.
__device__ __forceinline__ double stage_theta(uint32_t b, int32_t Cd) {
  return Cd > 0 ? (double)b / (double)Cd : __longlong_as_double(0x7FF0000000000000ll);
}
__device__ __forceinline__ unsigned long long theta_key(double th) {
  return (unsigned long long)__double_as_longlong(th);
}

struct PbCand {
  int32_t E, C1, C2, C3;
  int c1, c2, b1, b2, b3;  // cuts and batch indices
};

// Candidate t of unit `unit` (see pb_score_kernel); returns false past the unit's end.
template <int K>
__device__ __forceinline__ void pb_candidate(const Problem& pb, const DevModel& md, int M, int k1, int k2, int k3,
                                             int c1u, int b2u, int b1u, int t, PbCand& c) {
  const int B = pb.B;
  if constexpr (K == 3) {
    c.b3 = t % B;
    c.b1 = (t / B) % B;
    c.b2 = b2u;
    c.c1 = c1u;
    c.c2 = c1u + 1 + t / (B * B);
    const int32_t *P1 = prow_pb(pb, md, k1, c.b1), *P2 = prow_pb(pb, md, k2, c.b2), *P3 = prow_pb(pb, md, k3, c.b3);
    c.C1 = P1[c.c1];
    c.C2 = P2[c.c2] - P2[c.c1];
    c.C3 = P3[M] - P3[c.c2];
    c.E = c.C1 + c.C2 + c.C3 + yrow_pb(pb, md, k1, k2, c.b1)[c.c1] + yrow_pb(pb, md, k2, k3, c.b2)[c.c2];
  } else if constexpr (K == 2) {
    c.b2 = t % B;
    c.b1 = b1u;
    c.b3 = 0xFF;
    c.c1 = 1 + t / B;
    c.c2 = 0;
    const int32_t *P1 = prow_pb(pb, md, k1, c.b1), *P2 = prow_pb(pb, md, k2, c.b2);
    c.C1 = P1[c.c1];
    c.C2 = P2[M] - P2[c.c1];
    c.C3 = 0;
    c.E = c.C1 + c.C2 + yrow_pb(pb, md, k1, k2, c.b1)[c.c1];
  } else {
    c.b1 = t;
    c.b2 = c.b3 = 0xFF;
    c.c1 = c.c2 = 0;
    c.C1 = prow_pb(pb, md, k1, c.b1)[M];
    c.C2 = c.C3 = 0;
    c.E = c.C1;
  }
}

template <int K>
__device__ __forceinline__ unsigned long long pb_key(const Problem& pb, const PbCand& c) {
  double th = stage_theta(pb.batches[c.b1], c.C1);
  if constexpr (K >= 2) th = fmin(th, stage_theta(pb.batches[c.b2], c.C2));
  if constexpr (K >= 3) th = fmin(th, stage_theta(pb.batches[c.b3], c.C3));
  return theta_key(th);
}

template <int K>
__global__ void __launch_bounds__(kPbThreads) pb_score_kernel(Problem pb, int ml, PbOut out) {
  __shared__ unsigned long long tab[kPbBuckets];
  __shared__ unsigned long long scan_sh[kPbThreads / 32];
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, C = pb.C, B = pb.B;
  const int32_t T = md.T;
  int seg, c1u = 0, b2u = 0, b1u = 0, n;
  if constexpr (K == 3) {
    b2u = blockIdx.x % B;
    c1u = 1 + (blockIdx.x / B) % (M - 2);
    seg = blockIdx.x / (B * (M - 2));
    n = (M - 1 - c1u) * B * B;
  } else if constexpr (K == 2) {
    b1u = blockIdx.x % B;
    seg = blockIdx.x / B;
    n = (M - 1) * B;
  } else {
    seg = blockIdx.x;
    n = B;
  }
  int k1, k2 = 0, k3 = 0;
  if constexpr (K == 3) {
    k1 = seg / (C * C);
    k2 = (seg / C) % C;
    k3 = seg % C;
  } else if constexpr (K == 2) {
    k1 = seg / C;
    k2 = seg % C;
  } else {
    k1 = seg;
  }
  for (int i = threadIdx.x; i < kPbBuckets; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  const uint64_t span = (uint64_t)T + 1;
  unsigned long long feas = 0;
  // pass 1: best theta per E-bucket
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    PbCand c;
    pb_candidate<K>(pb, md, M, k1, k2, k3, c1u, b2u, b1u, t, c);
    if (c.E <= T) {
      ++feas;
      atomicMax(&tab[(uint64_t)c.E * kPbBuckets / span], pb_key<K>(pb, c));
    }
  }
  __syncthreads();
  // exclusive prefix maximum: the best theta at any strictly smaller bucket
  {
    unsigned long long v[kPbBuckets / kPbThreads];
#pragma unroll
    for (int i = 0; i < kPbBuckets / kPbThreads; ++i) v[i] = tab[threadIdx.x * (kPbBuckets / kPbThreads) + i];
    {  // exclusive prefix maximum over the blocked arrangement
      unsigned long long agg = 0ull;
#pragma unroll
      for (int i = 0; i < kPbBuckets / kPbThreads; ++i) agg = max(agg, v[i]);
      unsigned long long pre = block_exclusive_scan<kPbThreads>(agg, 0ull, OpMax(), scan_sh);
#pragma unroll
      for (int i = 0; i < kPbBuckets / kPbThreads; ++i) {
        const unsigned long long t = v[i];
        v[i] = pre;
        pre = max(pre, t);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPbBuckets / kPbThreads; ++i) tab[threadIdx.x * (kPbBuckets / kPbThreads) + i] = v[i];
  }
  __syncthreads();
  // pass 2: emit what no smaller-E bucket beats (warp-uniform trip count for the ballot)
  const int lane = threadIdx.x & 31;
  for (int t0 = 0; t0 < n; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    bool want = false;
    PbCand c;
    if (t < n) {
      pb_candidate<K>(pb, md, M, k1, k2, k3, c1u, b2u, b1u, t, c);
      want = c.E <= T && pb_key<K>(pb, c) > tab[(uint64_t)c.E * kPbBuckets / span];
    }
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(&out.counters[0], (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (want) {
        const unsigned long long i = base + __popc(m & ((1u << lane) - 1));
        if (i < out.cap) {
          ppipe_point_pb p;
          p.model = md.model;
          p.cut[0] = (uint16_t)c.c1;
          p.cut[1] = (uint16_t)c.c2;
          p.K = (uint8_t)K;
          p.cls[0] = (uint8_t)k1;
          p.cls[1] = K >= 2 ? (uint8_t)k2 : (uint8_t)0xFF;
          p.cls[2] = K >= 3 ? (uint8_t)k3 : (uint8_t)0xFF;
          p.bidx[0] = (uint8_t)c.b1;
          p.bidx[1] = K >= 2 ? (uint8_t)c.b2 : (uint8_t)0xFF;
          p.bidx[2] = K >= 3 ? (uint8_t)c.b3 : (uint8_t)0xFF;
          p.reserved = 0;
          p.e2e_us = (uint32_t)c.E;
          p.stage_us[0] = (uint32_t)c.C1;
          p.stage_us[1] = (uint32_t)c.C2;
          p.stage_us[2] = (uint32_t)c.C3;
          out.surv[i] = p;
        }
      }
    }
  }
  for (int off = 16; off; off >>= 1) feas += __shfl_down_sync(0xffffffffu, feas, off);
  if (lane == 0 && feas) atomicAdd(&out.counters[1], feas);
}

// K = 3, separable form. In a unit (segment, c_1, b_2) a candidate (c_2, b_1, b_3) has
//   E = A1[b_1] + A2[c_2] + C3[c_2][b_3],   A1 = C_1 + Y_1 (depends on b_1 only),
//   A2 = C_2 + Y_2 (c_2 only), theta = min(th1[b_1], th2[c_2], th3[c_2][b_3]),
// so the CTA stages A1 / th1 for every b_1 sorted by A1 and, per (c_2, b_3) pair, visits
// only the prefix of b_1 with A1 <= T - A2 - C3 (the feasible ones): the work is
// O(pairs + feasible candidates) instead of O(candidates), with no division or global
// load per candidate.
__global__ void __launch_bounds__(kPbThreads, 4) pb_score3_kernel(Problem pb, int ml, PbOut out) {
  __shared__ unsigned long long tab[kPbBuckets];
  __shared__ unsigned long long scan_sh[kPbThreads / 32];
  __shared__ int32_t sA1[256];
  __shared__ unsigned long long sTh1[256];
  __shared__ uint8_t sIdx1[256];
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, C = pb.C, B = pb.B;
  const int32_t T = md.T;
  const int b2 = blockIdx.x % B;
  const int c1 = 1 + (blockIdx.x / B) % (M - 2);
  const int seg = blockIdx.x / (B * (M - 2));
  const int k1 = seg / (C * C), k2 = (seg / C) % C, k3 = seg % C;
  __shared__ uint8_t sB3[256];  // batches b_3 some pair of this unit can make feasible
  __shared__ int nB3;
  // stage A1 / th1 per b_1, then sort them by (A1, b_1) through ranks
  __shared__ int32_t uA1[256];
  __shared__ int32_t uC1[256];
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    uC1[b] = prow_pb(pb, md, k1, b)[c1];
    uA1[b] = uC1[b] + yrow_pb(pb, md, k1, k2, b)[c1];
  }
  for (int i = threadIdx.x; i < kPbBuckets; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int32_t a = uA1[b];
    int rank = 0;
    for (int q = 0; q < B; ++q) rank += (uA1[q] < a || (uA1[q] == a && q < b)) ? 1 : 0;
    sA1[rank] = a;
    sTh1[rank] = theta_key(stage_theta(pb.batches[b], uC1[b]));
    sIdx1[rank] = (uint8_t)b;
  }
  if (threadIdx.x == 0) nB3 = 0;
  __syncthreads();
  const int32_t *P2 = prow_pb(pb, md, k2, b2), *Y23 = yrow_pb(pb, md, k2, k3, b2);
  const int32_t p2c1 = P2[c1];
  // Unit bound: E >= min A1 - P2[c1] + P3_{b3}[M] + min_{c2 > c1} (P2[c2] + Y23[c2] - P3_{b3}[c2]),
  // the last term from the suffix-minimum rows SD (when the context built them). A b_3
  // whose bound exceeds T_eff has no feasible pair; most units of a deep model have none.
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    bool keep = true;
    if (out.SD) {
      const int32_t* P3 = prow_pb(pb, md, k3, b);
      const int64_t bound = (int64_t)sA1[0] - p2c1 + P3[M] +
                            out.SD[((((size_t)k2 * C + k3) * B + b2) * B + b) * M + c1 + 1];
      keep = bound <= T;
    }
    if (keep) sB3[atomicAdd(&nB3, 1)] = (uint8_t)b;
  }
  __syncthreads();
  const int nb3 = nB3;
  const int n_pairs = (M - 1 - c1) * nb3;
  const uint32_t bv2 = pb.batches[b2];
  const uint64_t span = (uint64_t)T + 1;
  unsigned long long feas = 0;
  // pass 1: best theta per E-bucket
  for (int t = threadIdx.x; t < n_pairs; t += blockDim.x) {
    const int b3 = sB3[t % nb3], c2 = c1 + 1 + t / nb3;
    const int32_t C2 = P2[c2] - p2c1, A2 = C2 + Y23[c2];
    const int32_t* P3 = prow_pb(pb, md, k3, b3);
    const int32_t C3 = P3[M] - P3[c2];
    const int32_t rem = T - A2 - C3;
    if (rem < sA1[0]) continue;
    const unsigned long long th23 =
        min(theta_key(stage_theta(bv2, C2)), theta_key(stage_theta(pb.batches[b3], C3)));
    for (int j = 0; j < B && sA1[j] <= rem; ++j) {
      const int32_t E = sA1[j] + A2 + C3;
      ++feas;
      atomicMax(&tab[(uint64_t)E * kPbBuckets / span], min(sTh1[j], th23));
    }
  }
  __syncthreads();
  {
    unsigned long long v[kPbBuckets / kPbThreads];
#pragma unroll
    for (int i = 0; i < kPbBuckets / kPbThreads; ++i) v[i] = tab[threadIdx.x * (kPbBuckets / kPbThreads) + i];
    {  // exclusive prefix maximum over the blocked arrangement
      unsigned long long agg = 0ull;
#pragma unroll
      for (int i = 0; i < kPbBuckets / kPbThreads; ++i) agg = max(agg, v[i]);
      unsigned long long pre = block_exclusive_scan<kPbThreads>(agg, 0ull, OpMax(), scan_sh);
#pragma unroll
      for (int i = 0; i < kPbBuckets / kPbThreads; ++i) {
        const unsigned long long t = v[i];
        v[i] = pre;
        pre = max(pre, t);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPbBuckets / kPbThreads; ++i) tab[threadIdx.x * (kPbBuckets / kPbThreads) + i] = v[i];
  }
  __syncthreads();
  // pass 2: emit the candidates no smaller-E bucket beats (rare: a plain atomic per record)
  for (int t = threadIdx.x; t < n_pairs; t += blockDim.x) {
    const int b3 = sB3[t % nb3], c2 = c1 + 1 + t / nb3;
    const int32_t C2 = P2[c2] - p2c1, A2 = C2 + Y23[c2];
    const int32_t* P3 = prow_pb(pb, md, k3, b3);
    const int32_t C3 = P3[M] - P3[c2];
    const int32_t rem = T - A2 - C3;
    if (rem < sA1[0]) continue;
    const unsigned long long th23 =
        min(theta_key(stage_theta(bv2, C2)), theta_key(stage_theta(pb.batches[b3], C3)));
    for (int j = 0; j < B && sA1[j] <= rem; ++j) {
      const int32_t E = sA1[j] + A2 + C3;
      if (min(sTh1[j], th23) <= tab[(uint64_t)E * kPbBuckets / span]) continue;
      const unsigned long long i = atomicAdd(&out.counters[0], 1ull);
      if (i < out.cap) {
        const int b1 = sIdx1[j];
        ppipe_point_pb p;
        p.model = md.model;
        p.cut[0] = (uint16_t)c1;
        p.cut[1] = (uint16_t)c2;
        p.K = 3;
        p.cls[0] = (uint8_t)k1;
        p.cls[1] = (uint8_t)k2;
        p.cls[2] = (uint8_t)k3;
        p.bidx[0] = (uint8_t)b1;
        p.bidx[1] = (uint8_t)b2;
        p.bidx[2] = (uint8_t)b3;
        p.reserved = 0;
        p.e2e_us = (uint32_t)E;
        p.stage_us[0] = (uint32_t)uC1[b1];
        p.stage_us[1] = (uint32_t)C2;
        p.stage_us[2] = (uint32_t)C3;
        out.surv[i] = p;
      }
    }
  }
  for (int off = 16; off; off >>= 1) feas += __shfl_down_sync(0xffffffffu, feas, off);
  if ((threadIdx.x & 31) == 0 && feas) atomicAdd(&out.counters[1], feas);
}

// ---------------------------------------------------------------------------
// frontier pass over per-stage-batch survivors
// ---------------------------------------------------------------------------
}  // namespace

// SD[k2][k3][b2][b3][c] = min_{c <= c' <= M - 1} (P_{k2,b2}[c'] + Y_{k2->k3,b2}[c'] - P_{k3,b3}[c'])
// for c in [1, M - 1]: one thread per (class pair, batch pair) row, a reverse running minimum.
__global__ void __launch_bounds__(kPbThreads) pb_sd_kernel(Problem pb, int ml, int32_t* SD) {
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, C = pb.C, B = pb.B;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= C * C * B * B) return;
  const int b3 = r % B, b2 = (r / B) % B, k3 = (r / (B * B)) % C, k2 = r / (B * B * C);
  const int32_t *P2 = prow_pb(pb, md, k2, b2), *Y23 = yrow_pb(pb, md, k2, k3, b2), *P3 = prow_pb(pb, md, k3, b3);
  int32_t* row = SD + (size_t)r * M;
  int32_t m = INT32_MAX;
  for (int c = M - 1; c >= 1; --c) {
    m = min(m, P2[c] + Y23[c] - P3[c]);
    row[c] = m;
  }
  row[0] = m;
}

cudaError_t launch_pb_model(const Problem& pb, int ml, uint32_t M, int Kmax, const PbOut& out, cudaStream_t s,
                            int* n_launches) {
  const int C = pb.C, B = pb.B;
  pb_score_kernel<1><<<C, kPbThreads, 0, s>>>(pb, ml, out);
  ++*n_launches;
  if (Kmax >= 2 && M >= 2) {
    pb_score_kernel<2><<<C * C * B, kPbThreads, 0, s>>>(pb, ml, out);
    ++*n_launches;
  }
  if (Kmax >= 3 && M >= 3) {
    if (out.SD) {
      pb_sd_kernel<<<(C * C * B * B + kPbThreads - 1) / kPbThreads, kPbThreads, 0, s>>>(pb, ml, out.SD);
      ++*n_launches;
    }
    pb_score3_kernel<<<C * C * C * (int)(M - 2) * B, kPbThreads, 0, s>>>(pb, ml, out);
    ++*n_launches;
  }
  return cudaGetLastError();
}

}  // namespace ppipe
