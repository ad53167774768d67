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
#include <cub/cub.cuh>
#include <climits>

#include "ppipe_internal.h"

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
  const int ml = blockIdx.x / (n_btiles * pb.C);
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
      tile[l][bb] = (l < nl && bb < nb) ? (int32_t)lat[(size_t)(l0 + l) * B + b0 + bb] : 0;
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      int32_t acc = carry[threadIdx.x];
      for (int l = 0; l < nl; ++l) {
        acc += tile[l][threadIdx.x];
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
}

// CTA per (local model, distinct bandwidth v, batch): Y[v][b][c] for c in [0, Mp).
__global__ void __launch_bounds__(256) pack_y_kernel(Problem pb) {
  const int bi = blockIdx.x % pb.B;
  const int v = (blockIdx.x / pb.B) % pb.V;
  const int ml = blockIdx.x / (pb.B * pb.V);
  const DevModel md = pb.models[ml];
  const uint64_t b = pb.batches[bi];
  const uint64_t bw = pb.bw_v[v];
  const uint64_t* S = pb.raw_s + md.s_off;
  int32_t* row = pb.Y + md.y_off + ((size_t)v * pb.B + bi) * md.Mp;
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

cudaError_t launch_pack(const Problem& pb, cudaStream_t s) {
  if (pb.n_local == 0) return cudaSuccess;
  const int n_btiles = (pb.B + kPackBT - 1) / kPackBT;
  pack_p_kernel<<<pb.n_local * pb.C * n_btiles, 256, 0, s>>>(pb, n_btiles);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pack_y_kernel<<<pb.n_local * pb.V * pb.B, 256, 0, s>>>(pb);
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

__device__ __forceinline__ void store_rec(ppipe_point* dst, const Rec& r) {
  int4* d = reinterpret_cast<int4*>(dst);
  d[0] = make_int4((int)r.w[0], (int)r.w[1], (int)r.w[2], (int)r.w[3]);
  d[1] = make_int4((int)r.w[4], (int)r.w[5], (int)r.w[6], (int)r.w[7]);
}

// Warp-aggregated append to the survivor buffer. Must be called by all 32 lanes.
__device__ __forceinline__ void emit_warp(const ScoreOut& o, bool cond, const Rec& r) {
  const unsigned mask = __ballot_sync(FULL_MASK, cond);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&o.counters[0], (unsigned long long)__popc(mask));
  base = __shfl_sync(FULL_MASK, base, leader);
  if (cond) {
    const unsigned long long idx = base + __popc(mask & lanemask_lt());
    if (idx < o.cap) store_rec(o.surv + idx, r);
  }
}

__device__ __forceinline__ void emit_one(const ScoreOut& o, const Rec& r) {
  const unsigned long long idx = atomicAdd(&o.counters[0], 1ull);
  if (idx < o.cap) store_rec(o.surv + idx, r);
}

// Exclusive prefix-min over each class's bucket row (strict "earlier buckets"),
// in place: U[j] = min_{j' < j} tab[j'].
template <int NC>
__device__ void tables_to_thresholds(int32_t* tab) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < NC; k += kScoreThreads / 32) {
    int32_t* row = tab + k * kNumBuckets;
    int32_t run = INT_MAX;
    for (int r0 = 0; r0 < kNumBuckets; r0 += 32) {
      const int32_t v = row[r0 + lane];
      int32_t incl = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t o = __shfl_up_sync(FULL_MASK, incl, d);
        if (lane >= d) incl = min(incl, o);
      }
      int32_t excl = __shfl_up_sync(FULL_MASK, incl, 1);
      if (lane == 0) excl = INT_MAX;
      row[r0 + lane] = min(run, excl);
      run = min(run, __shfl_sync(FULL_MASK, incl, 31));
    }
  }
}

__device__ __forceinline__ void reset_tables(int32_t* tab, int n) {
  for (int i = threadIdx.x; i < n; i += kScoreThreads) tab[i] = INT_MAX;
}

template <int NC>
struct CtaCtx {
  const int32_t* P2;   // P[k2][b][.]
  const int32_t* Pm;   // P[m] base
  const int32_t* Ym;   // Y[m] base
  size_t Mp, B;
  int bi, b, k2, M, T, sh;
  uint32_t model;
  const uint8_t* pair_v;
  __device__ const int32_t* Prow(int k) const { return Pm + ((size_t)k * B + bi) * Mp; }
  __device__ const int32_t* Yrow(int ka, int kb) const {
    return Ym + ((size_t)__ldg(pair_v + ka * NC + kb) * B + bi) * Mp;
  }
};

// One warp processes one tile of 32 * kJ1 first cuts c_1 against every c_2 > c_1
// for a fixed (k_2, k_3, b) and all k_1. PASS 1 builds the per-(k_1) bucket
// minima of Cmax over feasible candidates; PASS 2 emits feasible candidates
// strictly better than every earlier bucket.
template <int NC, int PASS, bool SMEM_B>
__device__ void k3_tile(const CtaCtx<NC>& cx, int k3, int c1_base, int c1_hi, const int32_t* Bs,
                        const int32_t* P3, int32_t P3M, const int32_t* Y23, int32_t* tab, const ScoreOut& out,
                        unsigned long long& feas, unsigned long long& cand, int& any_flag) {
  const int lane = threadIdx.x & 31;
  // Only the thresholds live in registers across the c2 loop; the slow path
  // reloads C_1 and P[k2][c1] (L1-resident rows) when a candidate is feasible.
  int thr[kJ1][NC];
#pragma unroll
  for (int j = 0; j < kJ1; ++j) {
    const int c1 = c1_base + 32 * j + lane;
    const bool valid = c1 <= c1_hi;
    const int p1 = valid ? __ldg(cx.P2 + c1) : 0;
#pragma unroll
    for (int k1 = 0; k1 < NC; ++k1) {
      const int C1 = valid ? __ldg(cx.Prow(k1) + c1) : 0;
      const int y = valid ? __ldg(cx.Yrow(k1, cx.k2) + c1) : 0;
      // E = A + B(c2) with A = C1 + Y1 - P[k2][c1]  =>  feasible iff B(c2) <= T - A
      thr[j][k1] = valid ? cx.T - (C1 + y - p1) : INT_MIN;
    }
    if (PASS == 1 && valid) cand += (unsigned long long)(cx.M - 1 - c1) * NC;
  }
  auto Bat = [&](int c2) -> int {
    if (SMEM_B) return Bs[c2];
    return __ldg(cx.P2 + c2) - __ldg(P3 + c2) + __ldg(Y23 + c2) + P3M;
  };
  // Slow path: some lane has a feasible candidate at this c2.
  auto slow = [&](int c2, int Bv, int rel, bool diag) {
    const int Q = __ldg(cx.P2 + c2);
    const int R = P3M - __ldg(P3 + c2);
#pragma unroll
    for (int j = 0; j < kJ1; ++j) {
      const int c1 = c1_base + 32 * j + lane;
      const bool v = (!diag || (32 * j + lane < rel)) && c1 <= c1_hi;
      bool fj = false;
#pragma unroll
      for (int k1 = 0; k1 < NC; ++k1) fj |= v && (Bv <= thr[j][k1]);
      if (!__any_sync(FULL_MASK, fj)) continue;
      const int p1 = v ? __ldg(cx.P2 + c1) : 0;
      const int C2 = Q - p1;
#pragma unroll
      for (int k1 = 0; k1 < NC; ++k1) {
        const bool f = v && (Bv <= thr[j][k1]);
        const int C1 = f ? __ldg(cx.Prow(k1) + c1) : 0;
        const int Cmax = max(max(C1, C2), R);
        const int E = cx.T - thr[j][k1] + Bv;
        if (PASS == 1) {
          if (f) {
            atomicMin(&tab[k1 * kNumBuckets + (E >> cx.sh)], Cmax);
            ++feas;
            any_flag = 1;
          }
        } else {
          const bool cond = f && (Cmax < tab[k1 * kNumBuckets + (f ? (E >> cx.sh) : 0)]);
          emit_warp(out, cond, make_rec(cx.model, 3, c1, c2, k1, cx.k2, k3, cx.b, E, C1, C2, R));
        }
      }
    }
  };
  const int c2_main = c1_base + 32 * kJ1;  // from here on every slot has c_1 < c_2
  const int diag_end = min(c2_main, cx.M);  // exclusive
  for (int c2 = c1_base + 1; c2 < diag_end; ++c2) {
    const int Bv = Bat(c2);
    const int rel = c2 - c1_base;
    bool any = false;
#pragma unroll
    for (int j = 0; j < kJ1; ++j) {
      if (32 * j < rel) {
        const bool v = 32 * j + lane < rel;
#pragma unroll
        for (int k1 = 0; k1 < NC; ++k1) any |= v && (Bv <= thr[j][k1]);
      }
    }
    if (__any_sync(FULL_MASK, any)) slow(c2, Bv, rel, true);
  }
  for (int c2 = c2_main; c2 < cx.M; ++c2) {
    const int Bv = Bat(c2);
    bool a0 = false, a1 = false;
#pragma unroll
    for (int j = 0; j < kJ1; ++j) {
#pragma unroll
      for (int k1 = 0; k1 < NC; ++k1) {
        if ((j * NC + k1) & 1) a1 |= (Bv <= thr[j][k1]);
        else a0 |= (Bv <= thr[j][k1]);
      }
    }
    if (__any_sync(FULL_MASK, a0 | a1)) slow(c2, Bv, 0, false);
  }
}

template <int NC, bool SMEM_B>
__global__ void __launch_bounds__(kScoreThreads, 4) score_kernel(Problem pb, ScoreOut out) {
  extern __shared__ int32_t smem[];
  int32_t* tab = smem;                    // [NC][kNumBuckets]
  int32_t* Bs = smem + NC * kNumBuckets;  // [max_M] when SMEM_B
  __shared__ int s_tile, s_any;
  __shared__ unsigned long long s_feas, s_cand;

  const int B = pb.B;
  const int bi = blockIdx.x % B;
  const int k2 = (blockIdx.x / B) % NC;
  const int ml = blockIdx.x / (B * NC);
  const DevModel md = pb.models[ml];
  const int tid = threadIdx.x;
  const int lane = tid & 31;

  CtaCtx<NC> cx;
  cx.Pm = pb.P + md.p_off;
  cx.Ym = pb.Y + md.y_off;
  cx.Mp = md.Mp;
  cx.B = B;
  cx.bi = bi;
  cx.b = pb.batches[bi];
  cx.k2 = k2;
  cx.M = (int)md.M;
  cx.T = md.T;
  cx.model = md.model;
  cx.pair_v = pb.pair_v;
  cx.P2 = cx.Prow(k2);
  int sh = 0;
  while ((cx.T >> sh) >= kNumBuckets) ++sh;
  cx.sh = sh;
  const int M = cx.M, T = cx.T;

  unsigned long long feas = 0, cand = 0;
  if (tid == 0) {
    s_feas = 0;
    s_cand = 0;
  }
  reset_tables(tab, NC * kNumBuckets);

  // ---- K = 1: segment (k2), whole model on class k2 ----
  if (tid == 0 && md.row_lo == 0) {
    const int E = cx.P2[M];
    ++cand;
    if (E <= T) {
      ++feas;
      emit_one(out, make_rec(md.model, 1, 0, 0, k2, 0xFF, 0xFF, cx.b, E, E, 0, 0));
    }
  }

  // ---- K = 2: segments (k1, k2); c1 in this rank's rows ----
  if (pb.Kmax >= 2 && M >= 2) {
    const int lo = max(1, (int)md.row_lo), hi = min(M - 1, (int)md.row_hi - 1);
    if (lo <= hi) {
      const int P2M = cx.P2[M];
      if (tid == 0) s_any = 0;
      __syncthreads();
      int anyf = 0;
      for (int pass = 1; pass <= 2; ++pass) {
        for (int base = lo; base <= hi; base += kScoreThreads) {
          const int c1 = base + tid;
          const bool valid = c1 <= hi;
          const int C2 = valid ? P2M - __ldg(cx.P2 + c1) : 0;
#pragma unroll
          for (int k1 = 0; k1 < NC; ++k1) {
            const int C1 = valid ? __ldg(cx.Prow(k1) + c1) : 0;
            const int y = valid ? __ldg(cx.Yrow(k1, k2) + c1) : 0;
            const int E = C1 + y + C2;
            const bool f = valid && E <= T;
            const int Cmax = max(C1, C2);
            if (pass == 1) {
              if (valid) ++cand;
              if (f) {
                ++feas;
                anyf = 1;
                atomicMin(&tab[k1 * kNumBuckets + (E >> sh)], Cmax);
              }
            } else {
              const bool cond = f && Cmax < tab[k1 * kNumBuckets + (f ? (E >> sh) : 0)];
              emit_warp(out, cond, make_rec(md.model, 2, c1, 0, k1, k2, 0xFF, cx.b, E, C1, C2, 0));
            }
          }
        }
        if (pass == 1) {
          if (anyf) s_any = 1;
          __syncthreads();
          if (!s_any) break;
          tables_to_thresholds<NC>(tab);
          __syncthreads();
        } else {
          __syncthreads();
          reset_tables(tab, NC * kNumBuckets);
        }
      }
    }
  }

  // ---- K = 3: for each k3, segments (k1, k2, k3) ----
  if (pb.Kmax >= 3 && M >= 3) {
    const int c1lo = max(1, (int)md.row_lo), c1hi = min(M - 2, (int)md.row_hi - 1);
    if (c1lo <= c1hi) {
      const int ntiles = (c1hi - c1lo + 1 + 32 * kJ1 - 1) / (32 * kJ1);
      for (int k3 = 0; k3 < NC; ++k3) {
        const int32_t* P3 = cx.Prow(k3);
        const int32_t P3M = P3[M];
        const int32_t* Y23 = cx.Yrow(k2, k3);
        __syncthreads();
        if (SMEM_B) {
          for (int c2 = c1lo + 1 + tid; c2 <= M - 1; c2 += kScoreThreads)
            Bs[c2] = __ldg(cx.P2 + c2) - __ldg(P3 + c2) + __ldg(Y23 + c2) + P3M;
        }
        if (tid == 0) {
          s_tile = 0;
          s_any = 0;
        }
        __syncthreads();
        int anyf = 0;
        for (;;) {
          int t = 0;
          if (lane == 0) t = atomicAdd(&s_tile, 1);
          t = __shfl_sync(FULL_MASK, t, 0);
          if (t >= ntiles) break;
          k3_tile<NC, 1, SMEM_B>(cx, k3, c1lo + t * 32 * kJ1, c1hi, Bs, P3, P3M, Y23, tab, out, feas, cand, anyf);
        }
        if (anyf) s_any = 1;
        __syncthreads();
        if (s_any) {
          tables_to_thresholds<NC>(tab);
          if (tid == 0) s_tile = 0;
          __syncthreads();
          for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(&s_tile, 1);
            t = __shfl_sync(FULL_MASK, t, 0);
            if (t >= ntiles) break;
            k3_tile<NC, 2, SMEM_B>(cx, k3, c1lo + t * 32 * kJ1, c1hi, Bs, P3, P3M, Y23, tab, out, feas, cand,
                                   anyf);
          }
          __syncthreads();
          reset_tables(tab, NC * kNumBuckets);
        }
      }
    }
  }

  // ---- counters ----
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    feas += __shfl_down_sync(FULL_MASK, feas, d);
    cand += __shfl_down_sync(FULL_MASK, cand, d);
  }
  if (lane == 0) {
    atomicAdd(&s_feas, feas);
    atomicAdd(&s_cand, cand);
  }
  __syncthreads();
  if (tid == 0) {
    atomicAdd(&out.counters[1], s_feas);
    atomicAdd(&out.counters[2], s_cand);
  }
}

template <int NC>
static cudaError_t launch_score_nc(const Problem& pb, const ScoreOut& out, cudaStream_t s) {
  const bool smem_b = pb.max_M <= (uint32_t)kMaxMSmem;
  const size_t smem = sizeof(int32_t) * ((size_t)NC * kNumBuckets + (smem_b ? pb.max_M : 0));
  const unsigned grid = (unsigned)pb.n_local * NC * pb.B;
  if (smem_b) {
    auto kfn = score_kernel<NC, true>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, kScoreThreads, smem, s>>>(pb, out);
  } else {
    auto kfn = score_kernel<NC, false>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kfn<<<grid, kScoreThreads, smem, s>>>(pb, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_score(const Problem& pb, const ScoreOut& out, cudaStream_t s, int* n_launches) {
  if (pb.n_local == 0) return cudaSuccess;
  ++*n_launches;
  switch (pb.C) {
    case 1: return launch_score_nc<1>(pb, out, s);
    case 2: return launch_score_nc<2>(pb, out, s);
    case 3: return launch_score_nc<3>(pb, out, s);
    case 4: return launch_score_nc<4>(pb, out, s);
    case 5: return launch_score_nc<5>(pb, out, s);
    case 6: return launch_score_nc<6>(pb, out, s);
    case 7: return launch_score_nc<7>(pb, out, s);
    case 8: return launch_score_nc<8>(pb, out, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// frontier pass
// ---------------------------------------------------------------------------
constexpr int kEBits = 28;

__global__ void make_keys_kernel(const ppipe_point* in, uint64_t n, const uint64_t* seg_base, int C,
                                 uint64_t* keys, uint32_t* vals) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const ppipe_point p = in[i];
    // segment offset within the model: sum_{K' < K} C^K'
    uint64_t off = 0, pw = 1;
    for (int k = 1; k < p.K; ++k) {
      pw *= (uint64_t)C;
      off += pw;
    }
    uint64_t idx = 0;
    for (int d = 0; d < p.K; ++d) idx = idx * C + p.cls[d];
    const uint64_t seg = seg_base[p.model] + off + idx;
    keys[i] = (seg << kEBits) | (uint64_t)p.e2e_us;
    vals[i] = (uint32_t)i;
  }
}

__global__ void seg_start_kernel(const uint64_t* keys, uint64_t n, uint64_t n_seg, uint64_t* start) {
  const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (s > n_seg) return;
  const uint64_t target = s << kEBits;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (keys[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  start[s] = lo;
}

__device__ __forceinline__ uint32_t cmax_of(const ppipe_point& p) {
  uint32_t m = p.stage_us[0];
  if (p.K >= 2) m = max(m, p.stage_us[1]);
  if (p.K >= 3) m = max(m, p.stage_us[2]);
  return m;
}

// theta_p > theta_q  <=>  b_p * Cmax_q > b_q * Cmax_p (exact; Cmax = 0 reads as +inf)
__device__ __forceinline__ bool theta_gt(uint64_t bp, uint64_t cp, uint64_t bq, uint64_t cq) {
  return bp * cq > bq * cp;
}

// Is p canonically better than q among records with the same (segment, E)?
__device__ __forceinline__ bool better(const ppipe_point& p, const ppipe_point& q) {
  const uint64_t cp = cmax_of(p), cq = cmax_of(q);
  if (theta_gt(p.batch, cp, q.batch, cq)) return true;
  if (theta_gt(q.batch, cq, p.batch, cp)) return false;
  if (p.batch != q.batch) return p.batch < q.batch;
  if (p.cut[0] != q.cut[0]) return p.cut[0] < q.cut[0];
  return p.cut[1] < q.cut[1];
}

// One thread per segment: walk its (E-sorted) records in equal-E groups, keep the
// group's best if its theta strictly exceeds every earlier kept theta.
template <bool WRITE>
__global__ void staircase_kernel(const ppipe_point* in, const uint64_t* keys, const uint32_t* vals,
                                 const uint64_t* start, uint64_t n_seg, uint64_t* counts,
                                 const uint64_t* offsets, ppipe_point* out) {
  const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  const uint64_t lo = start[s], hi = start[s + 1];
  uint64_t best_b = 0, best_c = 1;  // theta = 0
  uint64_t cnt = 0;
  const uint64_t emask = (1ull << kEBits) - 1;
  uint64_t i = lo;
  while (i < hi) {
    const uint64_t E = keys[i] & emask;
    ppipe_point g = in[vals[i]];
    uint64_t j = i + 1;
    for (; j < hi && (keys[j] & emask) == E; ++j) {
      const ppipe_point q = in[vals[j]];
      if (better(q, g)) g = q;
    }
    const uint64_t gc = cmax_of(g);
    if (theta_gt(g.batch, gc, best_b, best_c)) {
      if (WRITE) out[offsets[s] + cnt] = g;
      ++cnt;
      best_b = g.batch;
      best_c = gc;
    }
    i = j;
  }
  if (!WRITE) counts[s] = cnt;
}

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

cudaError_t frontier_pass(const ppipe_point* in, uint64_t n, const uint64_t* seg_base_by_model, int C,
                          uint64_t n_seg, ppipe_point* out, uint64_t* seg_offsets, uint64_t* n_out_host,
                          FrontierScratch* scratch, cudaStream_t s, int* n_launches) {
  // key bits: E (28) + segment id
  int seg_bits = 1;
  while ((1ull << seg_bits) <= n_seg) ++seg_bits;
  const int end_bit = kEBits + seg_bits;
  size_t sort_bytes = 0, scan_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                                  (uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)n, 0,
                                                  end_bit, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (int64_t)(n_seg + 1), s);
  if (e != cudaSuccess) return e;
  const size_t nn = n > 0 ? n : 1;
  size_t off = 0;
  const size_t o_keys = off; off = align_up(off + nn * 8, 256);
  const size_t o_keys2 = off; off = align_up(off + nn * 8, 256);
  const size_t o_vals = off; off = align_up(off + nn * 4, 256);
  const size_t o_vals2 = off; off = align_up(off + nn * 4, 256);
  const size_t o_start = off; off = align_up(off + (n_seg + 1) * 8, 256);
  const size_t o_counts = off; off = align_up(off + (n_seg + 1) * 8, 256);
  const size_t o_tmp = off; off = align_up(off + std::max(sort_bytes, scan_bytes), 256);
  if (scratch->bytes < off) {
    if (scratch->buf) cudaFree(scratch->buf);
    scratch->buf = nullptr;
    scratch->bytes = 0;
    e = cudaMalloc(&scratch->buf, off);
    if (e != cudaSuccess) return e;
    scratch->bytes = off;
  }
  char* base = (char*)scratch->buf;
  uint64_t* keys = (uint64_t*)(base + o_keys);
  uint64_t* keys2 = (uint64_t*)(base + o_keys2);
  uint32_t* vals = (uint32_t*)(base + o_vals);
  uint32_t* vals2 = (uint32_t*)(base + o_vals2);
  uint64_t* start = (uint64_t*)(base + o_start);
  uint64_t* counts = (uint64_t*)(base + o_counts);
  void* tmp = base + o_tmp;

  if (n > 0) {
    const int blocks = (int)std::min<uint64_t>((n + 255) / 256, 148 * 16);
    make_keys_kernel<<<blocks, 256, 0, s>>>(in, n, seg_base_by_model, C, keys, vals);
    ++*n_launches;
    e = cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, keys, keys2, vals, vals2, (int64_t)n, 0, end_bit, s);
    if (e != cudaSuccess) return e;
    *n_launches += 2 * ((end_bit + 7) / 8);
  }
  const unsigned sb = (unsigned)((n_seg + 1 + 255) / 256);
  seg_start_kernel<<<sb, 256, 0, s>>>(keys2, n, n_seg, start);
  ++*n_launches;
  e = cudaMemsetAsync(counts + n_seg, 0, 8, s);
  if (e != cudaSuccess) return e;
  const unsigned gb = (unsigned)((n_seg + 127) / 128);
  staircase_kernel<false><<<gb, 128, 0, s>>>(in, keys2, vals2, start, n_seg, counts, nullptr, nullptr);
  ++*n_launches;
  e = cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, counts, seg_offsets, (int64_t)(n_seg + 1), s);
  if (e != cudaSuccess) return e;
  *n_launches += 2;
  staircase_kernel<true><<<gb, 128, 0, s>>>(in, keys2, vals2, start, n_seg, nullptr, seg_offsets, out);
  ++*n_launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(n_out_host, seg_offsets + n_seg, 8, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

}  // namespace ppipe
