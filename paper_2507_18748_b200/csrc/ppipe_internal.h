// Internal declarations shared by the C-ABI shim (ppipe_abi.cpp) and the
// kernels (ppipe_kernels.cu). Not part of the public ABI (include/ppipe.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ppipe.h"

namespace ppipe {

constexpr int kMaxClasses = 8;
constexpr int kMaxPartitions = 3;
constexpr int32_t kRangeLimit = 1 << 28;  // exact-int32 envelope
constexpr int kJ1 = 4;                    // first-cut slots per lane (tile = 32 * kJ1 first cuts)
constexpr int kMaxLayers = 16384;         // c2 rows (B, Q, R) of a model are staged in shared memory

// Per-model device metadata. Row layouts (int32):
//   P[k][bi][l], l = 0..M   prefix sums sum_{l' < l} lat[k][l'][bi]           (row length Mp)
//   Y[v][bi][c], c = 1..M-1 ceil(8 * S[c-1] * b / bw_v) clamped to kRangeLimit (row length Mp)
struct DevModel {
  uint32_t M;          // layers
  uint32_t Mp;         // padded row length (>= M + 1, multiple of 4)
  uint64_t lat_off;    // u32 offset of raw lat [C][M][B] in the raw upload buffer
  uint64_t s_off;      // u64 offset of act bytes [M]
  uint64_t p_off;      // int32 offset of P[m]
  uint64_t y_off;      // int32 offset of Y[m]
  uint32_t model;      // index in the caller's model array
  uint32_t row_lo;     // this rank's first-cut rows [row_lo, row_hi)
  uint32_t row_hi;
  uint32_t slo_us;     // raw SLO (set per enumerate)
  int32_t T;           // T_eff, written by the pack kernel
  uint32_t pad;
};

struct Problem {
  int C, B, V, Kmax, margin;
  const uint16_t* batches;   // [B] values (device)
  const uint32_t* bw_v;      // [V] distinct bandwidth values (device)
  const uint8_t* pair_v;     // [C][C] -> index into bw_v (device)
  DevModel* models;          // [n_local] (device)
  int n_local;
  int model_base, n_chunk;    // pack / score3a launches cover local models [base, base + n_chunk)
  const uint32_t* raw_lat;   // device
  const uint64_t* raw_s;     // device
  int32_t* P;                // device
  int32_t* Y;                // device
  const uint64_t* seg_base;  // [n_models_total] global segment id base per model (device)
  uint32_t max_M;
  int neg_one;                // -1, passed at run time (keeps IMAD on the FMA pipe)
  // Virtual GPUs (ppipe_set_vgpu): 4-bit throughput weight w_k = L / v_k per class
  // (L = lcm of the v's in use); theta = b / max_d(w_{k_d} C_d). All 1 by default.
  uint32_t wpack;
  int w_bits;                 // bits of max_k w_k (widens the fold keys' Cmax)
  int debug_flags;            // timing experiments only (PPIPE_DEBUG_FLAGS); 0 in production
  // per (local model, k2, batch, K = 3 tile): min over the tile's first cuts and k1 of
  // A = C_1 + Y_1 - P[k2][c_1] (written by the pack launch; nullptr = not kept)
  int32_t* minA;
  int max_tiles;
  // Cross-batch fold of the K = 3 segments (nullptr = off): per (local model, k1, k2, k3)
  // row of nb + 1 entries, the best theta = b / Cmax (bits of the double) of any unit's
  // bucket-best point per E-bucket, pushed by score3a; turned into an exclusive prefix
  // maximum by gfold_prefix before score3b, which folds it into every hot unit's bound
  // U(E) (a candidate at or below the best theta of a strictly smaller E-bucket of any
  // batch is dominated).
  unsigned long long* gfold;
  // Device validation inside the pack launch (ppipe_update_profiles_async; nullptr: the
  // profiles were validated before): pack_p flags a whole-model latency >= 2^28, pack_y an
  // act_bytes value above smax, by atomicMin of the key validate_kernel would write.
  unsigned long long* err_key;
  uint64_t smax;
};

struct ScoreOut {
  ppipe_point* surv;
  unsigned long long* counters;  // [0] survivors, [1] feasible, [2] candidates, [3] hot units, [4] pass-2 progress
  unsigned long long cap;
  uint4* hot;                    // [hot_cap] (local model, k2 | k3 << 4 | b << 8, tile mask lo, hi) of hot units
  uint64_t* hot_tab;             // [hot_cap][table words] their finalized fold tables
  unsigned long long hot_cap;
  uint32_t* hot_order;           // [hot_cap] pass-2 processing order, heaviest units first (nullptr: slot order)
  uint32_t* hot_w;               // [hot_cap] feasible candidates of each hot unit (pass 1; for the order)
};

size_t hot_unit_table_bytes(const Problem& pb);
// E-buckets of the K = 3 fold tables (the same for every unit of a problem)
int score_nb(const Problem& pb);
// Problem::gfold elements: n_local * C^3 * (nb + 1)
size_t gfold_elems(const Problem& pb);

// F2 (ppipe_f2.cu): per-model strict-dominance queries append the candidates no
// other feasible candidate beats in every stage (ties left in) to surv.
struct F2Out {
  ppipe_point* surv;
  unsigned long long* counters;  // [0] survivors appended, [1] feasible
  unsigned long long cap;
  int32_t* G;                    // K = 3 quadrant-minimum tables, g_cap elements
  size_t g_cap;                  // >= f2_g3_elems_per_segment(B, M) for every model
  int32_t* F;                    // K = 2 prefix counts, >= C * C * B * M elements
  uint16_t *PF, *PFs, *SF, *SFs;  // inverse stage tables, >= C * B * 4 ceil(B / 4) * M elements each
  int32_t* E23;                   // K = 3 second-cut part of E and its suffix minimum, 2 * C * C * B * M
  int q3_grid;                    // persistent K = 3 query CTAs
};
constexpr uint32_t kF2MaxLayers = 4096;  // a G row (M - 2 values) is staged in shared memory
size_t f2_g3_elems_per_segment(int B, uint32_t M);
int f2_q3_grid(int device);  // persistent grid of the K = 3 query kernel
cudaError_t launch_f2_model(const Problem& pb, int local_model, uint32_t M, int Kmax, const F2Out& out,
                            cudaStream_t s, int* n_launches);

// Launchers (stream-ordered). Return cudaError_t of the launch.
cudaError_t launch_pack(const Problem& pb, cudaStream_t s);
cudaError_t launch_score(const Problem& pb, const ScoreOut& out, cudaStream_t s, int* n_launches);
// The same work in parts: score3a over the chunk [model_base, model_base + n_chunk)
// (part 1), then score3b and score12 over all local models (part 2).
cudaError_t launch_score_part(const Problem& pb, const ScoreOut& out, cudaStream_t s, int* n_launches, int part);

// Frontier pass over n records: sort by (segment, E), per-(segment, E) best,
// strict staircase over theta, compaction. seg_base_by_model gives each model's
// first global segment id; n_seg is the total number of segments.
struct FrontierScratch {
  void* buf = nullptr;
  size_t bytes = 0;
};
cudaError_t frontier_pass(const ppipe_point* in, uint64_t n, const uint64_t* seg_base_by_model, int C,
                          uint64_t n_seg, ppipe_point* out, uint64_t* seg_offsets /* [n_seg+1] device */,
                          uint64_t* n_out_host, FrontierScratch* scratch, cudaStream_t s, int* n_launches,
                          uint32_t wpack /* Problem::wpack */);

// CSR offsets [n_seg + 1] of n records already in canonical (segment-sorted)
// order; seg_tmp holds n uint64 scratch entries.
cudaError_t segment_offsets(const ppipe_point* pts, uint64_t n, const uint64_t* seg_base_by_model, int C,
                            uint64_t n_seg, uint64_t* seg_offsets, uint64_t* seg_tmp, cudaStream_t s,
                            int* n_launches);

// SLO truncation of a canonical frontier: per segment keep the points with
// E <= T_new[model] (a prefix of the segment). Writes out / seg_offsets_out and the
// kept count (host). scratch is grown as needed.
cudaError_t truncate_frontier(const ppipe_point* in, const uint64_t* seg_offsets_in, uint64_t n_in, uint64_t n_seg,
                              const uint32_t* T_new, ppipe_point* out, uint64_t* seg_offsets_out,
                              uint64_t* n_out_host, FrontierScratch* scratch, cudaStream_t s, int* n_launches);

// Per-stage batch sizes (ppipe_pb.cu).
struct PbOut {
  ppipe_point_pb* surv;
  unsigned long long* counters;  // [0] survivors appended, [1] feasible
  unsigned long long cap;
  int32_t* SD;                   // K = 3 suffix-minimum rows, C * C * B * B * M (nullptr: no unit bound)
};
cudaError_t launch_pb_model(const Problem& pb, int local_model, uint32_t M, int Kmax, const PbOut& out,
                            cudaStream_t s, int* n_launches);
cudaError_t pb_frontier_pass(const ppipe_point_pb* in, uint64_t n, const uint64_t* seg_base, int C, uint64_t n_seg,
                             const uint16_t* batches, int B, ppipe_point_pb* out, uint64_t* seg_offsets,
                             uint64_t* n_out_host, FrontierScratch* scratch, cudaStream_t s, int* n_launches);

// F2 tail: resolve equal vectors (keep the smallest (E, b, c_1, c_2) of each run),
// sort into (segment, b, c_1, c_2) order and build the CSR. tmp_pts holds n records.
cudaError_t f2_finalize(const ppipe_point* in, uint64_t n, const uint64_t* seg_base, int C, uint64_t n_seg,
                        ppipe_point* out, ppipe_point* tmp_pts, uint64_t* seg_offsets, uint64_t* seg_tmp,
                        uint64_t* n_out_host, FrontierScratch* scratch, cudaStream_t s, int* n_launches);

// Device-side profile validation for ppipe_update_profiles (the same envelope as
// the host check of ppipe_load_profiles): per local model, every whole-model
// latency sum_l lat[k][l][b] < 2^28 and every act_bytes <= smax. The first failure
// in (model, kind, index) order is folded into *err_key by atomicMin:
// model << 40 | kind << 39 | index, kind 0 = latency (index = k * B + b), 1 = bytes
// (index = layer); UINT64_MAX = none.
cudaError_t launch_validate(const DevModel* models, int n_local, const uint32_t* lat, const uint64_t* S, int C,
                            int B, uint64_t smax, unsigned long long* err_key, cudaStream_t s);

// Greedy pre-partitioning (ppipe_prepartition). Device arrays: lat/S of all models
// concatenated at lat_off/s_off, M per model; outputs bounds [n][N+1], block_lat
// [n][C][N][B] at n*C*N*B stride, block_S [n][N]; prefix scratch of sum(M+1) int64 at
// s_off + model index (one extra entry per model).
struct PrepartProblem {
  const uint32_t* lat;
  const uint64_t* S;
  const uint64_t* lat_off;
  const uint64_t* s_off;
  const uint32_t* M;
  int64_t* prefix;
  uint32_t* bounds;
  uint32_t* block_lat;
  uint64_t* block_S;
  int n_models, C, B, N, ref_class, ref_b;
};
cudaError_t launch_prepartition(const PrepartProblem& p, cudaStream_t s);

}  // namespace ppipe
