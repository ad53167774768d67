// ppipe_f2.cu -- F2, the MILP-lossless frontier.
//
// PPipe's pooled MILP gives a chosen pipeline g_d GPUs in stage d; its
// throughput is min_d g_d X_d with X_d = b / C_d the per-GPU throughput of stage
// d (X_{ldbij}, eqs. 1.10 / 1.13), and E only has to
// meet the SLO (eq. 1.12). So per segment (model, K, class tuple)
// the candidates the MILP can need are those whose vector x = (X_1 .. X_K) is not
// dominated by another feasible candidate's; among equal vectors the smallest
// (E, b, c_1, c_2) stays (readings F2-1..F2-4). Virtual-GPU weights
// scale one stage of every candidate of a segment alike, so they do not change F2.
//
// At one batch no two cut sets of a segment are comparable (moving a cut grows one
// stage and shrinks its neighbour), so dominance comes from other batches b'. For a
// feasible candidate p = (c_1, c_2, b) and a batch b', "some feasible q at b' has
// C'_d b <= C_d b' in every stage d, one of them strictly" is a range query:
//   C'_1 = P1'[c'_1] is non-decreasing in c'_1   ->  c'_1 <= u   (u by binary search)
//   C'_3 = P3'[M] - P3'[c'_2] non-increasing      ->  c'_2 >= l
//   C'_2 = P2'[c'_2] - P2'[c'_1]                   ->  G_{b'}[u][l] = min C'_2 over the
//        feasible (c'_1 <= u, c'_2 >= l) pairs -- a 2-D prefix/suffix minimum table
//        built per (segment, b') by f2_g3_kernel.
// Strict dominance = OR over the stage that is strict (three lookups per b').
// K = 2 uses prefix counts of feasible cuts (f2_g2_kernel), K = 1 compares batches
// directly. Equal vectors are resolved afterwards (f2_finalize): sort by
// (segment, vector reduced by gcd(b, C_1, .., C_K)), keep the best of each run,
// sort into the canonical (segment, b, c_1, c_2) order.
//
// Bound: the G tables are written once and read by the queries (HBM / L2); the
// enumeration itself is the same integer work as score3a. DESIGN.md §5.
#include <climits>

#include "ppipe_block.cuh"
#include "ppipe_internal.h"

namespace ppipe {

namespace {

constexpr int kF2Threads = 256;
constexpr int32_t kInf = INT32_MAX;

__device__ __forceinline__ const int32_t* prow(const Problem& pb, const DevModel& md, int k, int bi) {
  return pb.P + md.p_off + ((size_t)k * pb.B + bi) * md.Mp;
}
__device__ __forceinline__ const int32_t* yrow(const Problem& pb, const DevModel& md, int k, int k2, int bi) {
  return pb.Y + md.y_off + ((size_t)pb.pair_v[k * pb.C + k2] * pb.B + bi) * md.Mp;
}

// Warp-aggregated append of one record per lane that wants it.
__device__ __forceinline__ void emit_point(bool want, const ppipe_point& p, const F2Out& out) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&out.counters[0], (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (want) {
    const unsigned long long i = base + __popc(m & ((1u << lane) - 1));
    if (i < out.cap) out.surv[i] = p;
  }
}

__device__ __forceinline__ ppipe_point make_point(const DevModel& md, int K, int k1, int k2, int k3, int c1, int c2,
                                                  uint32_t b, int32_t E, int32_t C1, int32_t C2, int32_t C3) {
  ppipe_point p;
  p.model = md.model;
  p.cut[0] = (uint16_t)c1;
  p.cut[1] = (uint16_t)c2;
  p.K = (uint8_t)K;
  p.cls[0] = (uint8_t)k1;
  p.cls[1] = K >= 2 ? (uint8_t)k2 : (uint8_t)0xFF;
  p.cls[2] = K >= 3 ? (uint8_t)k3 : (uint8_t)0xFF;
  p.batch = (uint16_t)b;
  p.reserved = 0;
  p.e2e_us = (uint32_t)E;
  p.stage_us[0] = (uint32_t)C1;
  p.stage_us[1] = (uint32_t)C2;
  p.stage_us[2] = (uint32_t)C3;
  return p;
}

// ---------------------------------------------------------------------------
// K = 3: G tables. CTA per (segment in chunk, batch b'). Row u = c'_1 in 1..M-2,
// column l = c'_2 in 2..M-1 (n = M - 2 of each; rows padded to g_pitch(n)). Thread t
// holds columns j = 16 t + i (blocked); G[u][l] = min(G[u-1][l], min_{l' >= l} H[u][l'])
// with H[u][l] = C'_2 if (u < l and feasible) else +inf, and
// E' = (P1[u] - P2[u] + Y12[u]) + (P2[l] + P3[M] - P3[l] + Y23[l]) = a(u) + e(l).
// Warp w owns columns [512 w, 512 w + 512), 16 per lane: the row's suffix minimum is a
// thread-local pass, one warp scan and (W > 1 warps) one exchange through shared
// memory (double-buffered: one barrier per row). Each lane stores its 16 columns of a
// row as four 16-byte stores into the padded row pitch.
__host__ __device__ __forceinline__ int g_pitch(int n) { return (n + 15) & ~15; }

constexpr int kG3Cols = 16;  // columns per lane

template <int W>
__global__ void __launch_bounds__(32 * W) f2_g3_kernel(Problem pb, int ml, int seg_lo, int32_t* G) {
  constexpr int IT = kG3Cols;
  __shared__ int32_t sh[2][W];
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, n = M - 2, pitch = g_pitch(n), C = pb.C, B = pb.B;
  const int bq = blockIdx.x % B, seg = seg_lo + blockIdx.x / B;
  const int k1 = seg / (C * C), k2 = (seg / C) % C, k3 = seg % C;
  const int32_t *P1 = prow(pb, md, k1, bq), *P2 = prow(pb, md, k2, bq), *P3 = prow(pb, md, k3, bq);
  const int32_t *Y12 = yrow(pb, md, k1, k2, bq), *Y23 = yrow(pb, md, k2, k3, bq);
  const int32_t T = md.T, P3M = P3[M];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = threadIdx.x * IT;
  const bool writer = j0 < pitch;
  int32_t* Gs = G + (size_t)blockIdx.x * n * pitch + j0;
  int32_t e[IT], p2l[IT], prev[IT];
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const int j = j0 + i, l = j + 2;
    e[i] = j < n ? P2[l] + (P3M - P3[l]) + Y23[l] : 0;
    p2l[i] = j < n ? P2[l] : 0;
    prev[i] = kInf;
  }
  int par = 0;
  for (int u = 1; u <= M - 2; ++u, par ^= 1) {
    const int32_t a = P1[u] - P2[u] + Y12[u], p2u = P2[u];
    int32_t h[IT], run = kInf;
#pragma unroll
    for (int i = IT - 1; i >= 0; --i) {
      const int j = j0 + i;
      const bool ok = j < n && j + 2 > u && a + e[i] <= T;
      run = min(run, ok ? p2l[i] - p2u : kInf);
      h[i] = run;
    }
    int32_t inc = run;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t o = __shfl_down_sync(0xffffffffu, inc, off);
      if (lane + off < 32) inc = min(inc, o);
    }
    int32_t later = __shfl_down_sync(0xffffffffu, inc, 1);
    if (lane == 31) later = kInf;
    if constexpr (W > 1) {
      if (lane == 0) sh[par][warp] = inc;
      __syncthreads();
#pragma unroll
      for (int w = 1; w < W; ++w)
        if (w > warp) later = min(later, sh[par][w]);
    }
#pragma unroll
    for (int i = 0; i < IT; ++i) prev[i] = min(prev[i], min(h[i], later));
    if (writer) {
      int32_t* dst = Gs + (size_t)(u - 1) * pitch;
#pragma unroll
      for (int i = 0; i < IT; i += 4)
        if (j0 + i < pitch) *reinterpret_cast<int4*>(dst + i) = make_int4(prev[i], prev[i + 1], prev[i + 2], prev[i + 3]);
    }
  }
}

// Inverse stage tables (per model, u16, c in [1, M-1]; layout [k][b][c][b'] with b'
// padded to Bp = 4 * ceil(B / 4), so the four tables' entries for 4 consecutive b'
// are one 8-byte load):
//   PF[k][b][c][b']  = last c' in [1, M-1] with P_{k,b'}[c'] * b <= P_{k,b}[c] * b'  (0 = none)
//   SF[k][b][c][b']  = first c' in [1, M-1] with (P_{k,b'}[M] - P_{k,b'}[c']) * b
//                      <= (P_{k,b}[M] - P_{k,b}[c]) * b'                              (M = none)
// and the strict (<) versions PFs / SFs. A first stage [0, c) at batch b is matched or
// beaten at b' exactly by the cuts c' <= PF (C'_1 non-decreasing in c'); a last stage
// [c, M) by the cuts c' >= SF. K = 3 clamps them to [1, M-2] / [2, M-1].
__host__ __device__ __forceinline__ int b_pad(int B) { return (B + 3) & ~3; }

__device__ __forceinline__ size_t inv_at(int k, int bi, int c, int B, int M) {
  return (((size_t)k * B + bi) * M + c) * b_pad(B);
}

constexpr int kInvSplit = 8;  // CTAs per (class, batch)

__global__ void __launch_bounds__(kF2Threads) f2_inv_kernel(Problem pb, int ml, F2Out out) {
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, B = pb.B, Bp = b_pad(B);
  const int part = blockIdx.x % kInvSplit, bi = (blockIdx.x / kInvSplit) % B, k = blockIdx.x / (kInvSplit * B);
  const int32_t* P = prow(pb, md, k, bi);
  const uint64_t b = pb.batches[bi];
  const int64_t PM = P[M];
  const size_t base = inv_at(k, bi, 0, B, M);
  for (int t = part * kF2Threads + threadIdx.x; t < (M - 1) * Bp; t += kInvSplit * kF2Threads) {
    const int c = 1 + t / Bp, bq = t % Bp;
    int pf = 0, pfs = 0, sf = M, sfs = M;
    if (bq < B) {
      const int32_t* Q = prow(pb, md, k, bq);
      const uint64_t bv = pb.batches[bq];
      const int64_t QM = Q[M];
      const uint64_t r1 = (uint64_t)P[c] * bv, r2 = (uint64_t)(PM - P[c]) * bv;
      // prefix stage: largest c' with Q[c'] * b <= r1 (resp. < r1)
      int lo = 1, hi = M;  // first c' failing, in [1, M]
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((uint64_t)Q[mid] * b <= r1) lo = mid + 1;
        else hi = mid;
      }
      pf = lo - 1;
      lo = 1;
      hi = pf + 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((uint64_t)Q[mid] * b < r1) lo = mid + 1;
        else hi = mid;
      }
      pfs = lo - 1;
      // suffix stage: smallest c' with (QM - Q[c']) * b <= r2 (resp. < r2); non-increasing in c'
      lo = 1;
      hi = M;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((uint64_t)(QM - Q[mid]) * b <= r2) hi = mid;
        else lo = mid + 1;
      }
      sf = lo;
      hi = M;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((uint64_t)(QM - Q[mid]) * b < r2) hi = mid;
        else lo = mid + 1;
      }
      sfs = lo;
    }
    const size_t at = base + (size_t)c * Bp + bq;
    out.PF[at] = (uint16_t)pf;
    out.PFs[at] = (uint16_t)pfs;
    out.SF[at] = (uint16_t)sf;
    out.SFs[at] = (uint16_t)sfs;
  }
}

// K = 3 queries. Persistent warps pull rows (segment, b, c_1) from a counter in
// segment-major order (the rows in flight share one segment's G tables in L2). A
// warp scans its row 32 c_2 at a time, appends the feasible c_2 to a per-warp list
// and, whenever 32 are queued, runs one candidate per lane through the batches b'
// (largest first, four at a time, exit on the first dominator):
//   u = PF_{k1}[c_1], l = SF_{k3}[c_2]; G[u][l] * b > C_2 b'  => nothing at b' (the
//   strict variants read G at (us, l) / (u, ls), which are >= G[u][l]);
//   G[u][l] * b < C_2 b' => dominated (strict in stage 2); equal => check
//   G[us][l] * b <= C_2 b' (strict in stage 1) and G[u][ls] * b <= C_2 b' (stage 3).
constexpr int kQ3Warps = kF2Threads / 32;
constexpr int kQ3Rows = 4;  // c_1 rows per work unit

__device__ __forceinline__ int u16_at(const uint2& v, int i) {
  return (int)(((i < 2 ? v.x : v.y) >> (16 * (i & 1))) & 0xFFFFu);
}

// 1: some feasible candidate beats p in every stage (strictly in one); 0: none matches
// it in every stage at another batch; 2: not dominated, but one may match it exactly at
// another batch (G[u][l] * b == C_2 b'), so f2_finalize resolves it by its vector.
__device__ __forceinline__ int f2_dominated3(const Problem& pb, const F2Out& out, int M, int B, int k1, int k3,
                                             int bi, int c1, int c2, uint32_t b, int32_t C2, const int32_t* Gseg) {
  int res = 0;
  const int n = M - 2, pitch = g_pitch(n), Bp = b_pad(B);
  const size_t at1 = inv_at(k1, bi, c1, B, M), at3 = inv_at(k3, bi, c2, B, M);
  const size_t gstride = (size_t)n * pitch;
  for (int q = Bp / 4 - 1; q >= 0; --q) {
    const uint2 pf4 = *reinterpret_cast<const uint2*>(out.PF + at1 + 4 * q);
    const uint2 sf4 = *reinterpret_cast<const uint2*>(out.SF + at3 + 4 * q);
    int32_t g[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int bq = 4 * q + i, u = min(u16_at(pf4, i), M - 2), l = max(u16_at(sf4, i), 2);
      g[i] = (bq < B && u >= 1 && l <= M - 1) ? Gseg[bq * gstride + (size_t)(u - 1) * pitch + (l - 2)] : kInf;
    }
#pragma unroll
    for (int i = 3; i >= 0; --i) {
      if (g[i] == kInf) continue;
      const int bq = 4 * q + i;
      const uint64_t r2 = (uint64_t)C2 * pb.batches[bq], gb = (uint64_t)g[i] * b;
      if (gb > r2) continue;
      if (gb < r2) return 1;
      // G[u][l] * b == C_2 b': a pair strictly better in stage 1 or stage 3 decides
      const int u = min(u16_at(pf4, i), M - 2), l = max(u16_at(sf4, i), 2);
      const int32_t* Gb = Gseg + bq * gstride;
      const int us = min((int)out.PFs[at1 + bq], M - 2);
      if (us >= 1) {
        const int32_t g1 = Gb[(size_t)(us - 1) * pitch + (l - 2)];
        if (g1 != kInf && (uint64_t)g1 * b <= r2) return 1;
      }
      const int ls = max((int)out.SFs[at3 + bq], 2);
      if (ls <= M - 1) {
        const int32_t g3 = Gb[(size_t)(u - 1) * pitch + (ls - 2)];
        if (g3 != kInf && (uint64_t)g3 * b <= r2) return 1;
      }
      if (bq != bi) res = 2;  // at b' = b the pair found is p itself (same-batch twins: caller)
    }
  }
  return res;
}

__global__ void __launch_bounds__(kF2Threads, 4) f2_q3_kernel(Problem pb, int ml, int seg_lo, int nseg,
                                                           const int32_t* G, F2Out out) {
  __shared__ int32_t list[kQ3Warps][64];
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, n = M - 2, C = pb.C, B = pb.B;
  const int32_t T = md.T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* L = list[warp];
  const int nq = (n + kQ3Rows - 1) / kQ3Rows;
  const unsigned long long n_units = (unsigned long long)nseg * B * nq;
  unsigned long long feas = 0;
  for (;;) {
    unsigned long long unit = 0;
    if (lane == 0) unit = atomicAdd(&out.counters[2], 1ull);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit >= n_units) break;
    const int bi = (int)((unit / nq) % B);
    const int segc = (int)(unit / ((unsigned long long)nq * B));
    const int seg = seg_lo + segc;
    const int k1 = seg / (C * C), k2 = (seg / C) % C, k3 = seg % C;
    const int32_t *P1 = prow(pb, md, k1, bi), *P2 = prow(pb, md, k2, bi), *P3 = prow(pb, md, k3, bi);
    const int32_t *Y12 = yrow(pb, md, k1, k2, bi), *Y23 = yrow(pb, md, k2, k3, bi);
    const int32_t* E23 = out.E23 + ((size_t)(k2 * C + k3) * B + bi) * M;
    const int32_t* E23min = E23 + (size_t)C * C * B * M;
    const int32_t P3M = P3[M];
    const uint32_t b = pb.batches[bi];
    const int32_t* Gseg = G + (size_t)segc * B * n * g_pitch(n);
    const int c1_lo = 1 + kQ3Rows * (int)(unit % nq), c1_hi = min(c1_lo + kQ3Rows - 1, M - 2);
    for (int c1 = c1_lo; c1 <= c1_hi; ++c1) {
    const int32_t C1 = P1[c1], p2c1 = P2[c1], a = C1 - p2c1 + Y12[c1];
    if (a + E23min[c1 + 1] > T) continue;  // no feasible c_2 in this row (warp-uniform)
    int cnt = 0;
    for (int base = c1 + 1; base <= M - 1 || cnt > 0; base += 32) {
      if (base <= M - 1) {
        const int c2 = base + lane;
        bool f = false;
        if (c2 <= M - 1) f = a + E23[c2] <= T;
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (f) L[cnt + __popc(m & ((1u << lane) - 1))] = c2;
        cnt += __popc(m);
        feas += f;
        __syncwarp();
        if (cnt < 32 && base + 32 <= M - 1) continue;  // keep filling
      }
      // process up to 32 queued candidates, one per lane
      const bool act = lane < cnt;
      bool keep = false, tie = false;
      int32_t c2 = 0, E = 0, C2 = 0, C3 = 0;
      if (act) {
        c2 = L[lane];
        C2 = P2[c2] - p2c1;
        C3 = P3M - P3[c2];
        E = a + P2[c2] + C3 + Y23[c2];
        const int r = f2_dominated3(pb, out, M, B, k1, k3, bi, c1, c2, b, C2, Gseg);
        keep = r != 1;
        // a twin at the same batch has equal P1 at its first cut or equal P3 at its second:
        // a zero-latency layer next to c_1 (class k1) or c_2 (class k3)
        tie = r == 2 || (c1 > 1 && P1[c1 - 1] == C1) || (c1 < M - 2 && P1[c1 + 1] == C1) ||
              (c2 > 2 && P3[c2 - 1] == P3[c2]) || (c2 < M - 1 && P3[c2 + 1] == P3[c2]);
      }
      ppipe_point pt = make_point(md, 3, k1, k2, k3, c1, c2, b, E, C1, C2, C3);
      pt.reserved = tie ? 1 : 0;
      emit_point(keep, pt, out);
      __syncwarp();
      const int rest = cnt > 32 ? cnt - 32 : 0;
      if (lane < rest) L[lane] = L[32 + lane];
      __syncwarp();
      cnt = rest;
    }
    }
  }
  for (int off = 16; off; off >>= 1) feas += __shfl_down_sync(0xffffffffu, feas, off);
  if (lane == 0 && feas) atomicAdd(&out.counters[1], feas);
}

// E23[k2][k3][b][c] = P_{k2,b}[c] + (P_{k3,b}[M] - P_{k3,b}[c]) + Y_{k2->k3,b}[c]: the part of a
// K = 3 candidate's E that depends on its second cut (per class pair and batch).
__global__ void __launch_bounds__(kF2Threads) f2_e23_kernel(Problem pb, int ml, int32_t* E23) {
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, C = pb.C, B = pb.B;
  const int bi = blockIdx.x % B, k3 = (blockIdx.x / B) % C, k2 = blockIdx.x / (B * C);
  const int32_t *P2 = prow(pb, md, k2, bi), *P3 = prow(pb, md, k3, bi), *Y23 = yrow(pb, md, k2, k3, bi);
  const int32_t P3M = P3[M];
  int32_t* row = E23 + (size_t)blockIdx.x * M;
  for (int c = threadIdx.x; c < M; c += blockDim.x) row[c] = P2[c] + (P3M - P3[c]) + Y23[c];
  __syncthreads();
  // suffix minimum over c_2 in [c, M - 1] (E23min, at E23 + C*C*B*M): a row (c_1) with
  // a(c_1) + E23min[c_1 + 1] > T_eff has no feasible c_2 and is skipped whole
  if (threadIdx.x == 0) {
    int32_t* mrow = E23 + (size_t)C * C * B * M + (size_t)blockIdx.x * M;
    int32_t m = INT32_MAX;
    for (int c = M - 1; c >= 0; --c) {
      m = min(m, row[c]);
      mrow[c] = m;
    }
  }
}

// K = 2: per (segment, b') prefix counts F[c] = #feasible c'_1 in [1, c], c = 0..M-1.
__global__ void __launch_bounds__(kF2Threads) f2_g2_kernel(Problem pb, int ml, int32_t* F) {
  __shared__ int32_t scan_sh[kF2Threads / 32];
  __shared__ int32_t carry;
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, C = pb.C, B = pb.B;
  const int bq = blockIdx.x % B, seg = blockIdx.x / B;
  const int k1 = seg / C, k2 = seg % C;
  const int32_t *P1 = prow(pb, md, k1, bq), *P2 = prow(pb, md, k2, bq), *Y12 = yrow(pb, md, k1, k2, bq);
  const int32_t T = md.T, P2M = P2[M];
  int32_t* Fs = F + (size_t)blockIdx.x * M;
  if (threadIdx.x == 0) {
    carry = 0;
    Fs[0] = 0;
  }
  __syncthreads();
  for (int c0 = 1; c0 <= M - 1; c0 += kF2Threads) {
    const int c = c0 + threadIdx.x;
    const int32_t f = (c <= M - 1 && P1[c] + (P2M - P2[c]) + Y12[c] <= T) ? 1 : 0;
    int32_t inc, tot;
    inc = block_inclusive_scan<kF2Threads>(f, 0, OpSum(), &tot, scan_sh);
    if (c <= M - 1) Fs[c] = carry + inc;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// K = 2 queries: CTA per (segment, batch b), thread per c_1. Some feasible c' at b'
// beats p in stage 1 strictly (others <=) iff one lies in [SF_{k2}, PFs_{k1}], etc.
__global__ void __launch_bounds__(kF2Threads) f2_q2_kernel(Problem pb, int ml, const int32_t* F, F2Out out) {
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, C = pb.C, B = pb.B;
  const int bi = blockIdx.x % B, seg = blockIdx.x / B;
  const int k1 = seg / C, k2 = seg % C;
  const int32_t *P1 = prow(pb, md, k1, bi), *P2 = prow(pb, md, k2, bi), *Y12 = yrow(pb, md, k1, k2, bi);
  const int32_t T = md.T, P2M = P2[M];
  const uint32_t b = pb.batches[bi];
  unsigned long long feas = 0;
  for (int c0 = 1; c0 <= M - 1; c0 += blockDim.x) {
    const int c = c0 + threadIdx.x;
    bool keep = false, tie = false;
    int32_t E = 0, C1 = 0, C2 = 0;
    if (c <= M - 1) {
      C1 = P1[c];
      C2 = P2M - P2[c];
      E = C1 + C2 + Y12[c];
      if (E <= T) {
        ++feas;
        bool dom = false;
        for (int bq = B - 1; bq >= 0 && !dom; --bq) {
          const size_t a1 = inv_at(k1, bi, c, B, M) + bq, a2 = inv_at(k2, bi, c, B, M) + bq;
          const int u = out.PF[a1], l = out.SF[a2];
          if (u < l) continue;
          const int us = out.PFs[a1], ls = out.SFs[a2];
          const int32_t* Fb = F + ((size_t)seg * B + bq) * M;
          dom = (us >= l && Fb[us] - Fb[l - 1] > 0) || (ls <= u && Fb[u] - Fb[ls - 1] > 0);
          // not strictly beaten: any other feasible c' in [l, u] equals p in both stages
          tie = tie || Fb[u] - Fb[l - 1] > (bq == bi ? 1 : 0);
        }
        keep = !dom;
      }
    }
    ppipe_point pt = make_point(md, 2, k1, k2, 0, c, 0, b, E, C1, C2, 0);
    pt.reserved = tie ? 1 : 0;
    emit_point(keep, pt, out);
  }
  for (int off = 16; off; off >>= 1) feas += __shfl_down_sync(0xffffffffu, feas, off);
  if ((threadIdx.x & 31) == 0 && feas) atomicAdd(&out.counters[1], feas);
}

// K = 1: CTA per class, threads over batches (strict dominance only; ties in f2_finalize).
__global__ void __launch_bounds__(kF2Threads) f2_q1_kernel(Problem pb, int ml, F2Out out) {
  const DevModel md = pb.models[ml];
  const int M = (int)md.M, B = pb.B;
  const int k = blockIdx.x;
  const int32_t T = md.T;
  unsigned long long feas = 0;
  for (int b0 = 0; b0 < B; b0 += blockDim.x) {
    const int bi = b0 + threadIdx.x;
    bool keep = false, tie = false;
    int32_t C1 = 0;
    uint32_t b = 0;
    if (bi < B) {
      C1 = prow(pb, md, k, bi)[M];
      b = pb.batches[bi];
      if (C1 <= T) {
        ++feas;
        bool dom = false;
        for (int bq = 0; bq < B && !dom; ++bq) {
          const int32_t Cq = prow(pb, md, k, bq)[M];
          dom = Cq <= T && (uint64_t)Cq * b < (uint64_t)C1 * pb.batches[bq];
          tie = tie || (bq != bi && Cq <= T && (uint64_t)Cq * b == (uint64_t)C1 * pb.batches[bq]);
        }
        keep = !dom;
      }
    }
    ppipe_point pt = make_point(md, 1, k, 0, 0, 0, 0, b, C1, C1, 0, 0);
    pt.reserved = tie ? 1 : 0;
    emit_point(keep, pt, out);
  }
  for (int off = 16; off; off >>= 1) feas += __shfl_down_sync(0xffffffffu, feas, off);
  if ((threadIdx.x & 31) == 0 && feas) atomicAdd(&out.counters[1], feas);
}

template <int W>
cudaError_t launch_g3(const Problem& pb, int ml, int seg_lo, int nseg, int32_t* G, cudaStream_t s) {
  f2_g3_kernel<W><<<nseg * pb.B, 32 * W, 0, s>>>(pb, ml, seg_lo, G);
  return cudaGetLastError();
}

}  // namespace

int f2_q3_grid(int device) {
  int sms = 148, per_sm = 4;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f2_q3_kernel, kF2Threads, 0);
  return sms * std::max(per_sm, 1);
}

size_t f2_g3_elems_per_segment(int B, uint32_t M) {
  const size_t n = M >= 3 ? M - 2 : 0;
  return (size_t)B * n * g_pitch((int)n);
}

cudaError_t launch_f2_model(const Problem& pb, int ml, uint32_t M, int Kmax, const F2Out& out, cudaStream_t s,
                            int* n_launches) {
  cudaError_t e;
  const int C = pb.C;
  f2_q1_kernel<<<C, 64, 0, s>>>(pb, ml, out);
  ++*n_launches;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (Kmax >= 2 && M >= 2) {
    f2_inv_kernel<<<C * pb.B * kInvSplit, kF2Threads, 0, s>>>(pb, ml, out);
    ++*n_launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (Kmax >= 2 && M >= 2) {
    f2_g2_kernel<<<C * C * pb.B, kF2Threads, 0, s>>>(pb, ml, out.F);
    f2_q2_kernel<<<C * C * pb.B, kF2Threads, 0, s>>>(pb, ml, out.F, out);
    *n_launches += 2;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (Kmax >= 3 && M >= 3) {
    const size_t per_seg = f2_g3_elems_per_segment(pb.B, M);
    const int nseg_all = C * C * C;
    int chunk = (int)std::min<size_t>((size_t)nseg_all, std::max<size_t>(1, out.g_cap / per_seg));
    const int n = (int)M - 2, warps = (n + 32 * kG3Cols - 1) / (32 * kG3Cols);
    for (int lo = 0; lo < nseg_all; lo += chunk) {
      const int ns = std::min(chunk, nseg_all - lo);
      if (warps <= 1) e = launch_g3<1>(pb, ml, lo, ns, out.G, s);
      else if (warps <= 2) e = launch_g3<2>(pb, ml, lo, ns, out.G, s);
      else if (warps <= 4) e = launch_g3<4>(pb, ml, lo, ns, out.G, s);
      else e = launch_g3<8>(pb, ml, lo, ns, out.G, s);
      if (e != cudaSuccess) return e;
      if (lo == 0) {
        f2_e23_kernel<<<C * C * pb.B, kF2Threads, 0, s>>>(pb, ml, out.E23);
        ++*n_launches;
      }
      if ((e = cudaMemsetAsync(out.counters + 2, 0, sizeof(unsigned long long), s)) != cudaSuccess) return e;
      f2_q3_kernel<<<out.q3_grid, kF2Threads, 0, s>>>(pb, ml, lo, ns, out.G, out);
      *n_launches += 2;
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// finalize: equal-vector runs, canonical order, CSR
// ---------------------------------------------------------------------------
}  // namespace ppipe
