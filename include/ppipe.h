/*
 * ppipe.h -- C ABI of the B200-native PPipe plan-enumeration library
 * (libppipe_b200.so, built from paper_2507_18748_b200/csrc/).
 *
 * The library computes the data-parallel hot path of PPipe's control plane
 * (arXiv 2507.18748, "PPipe: Efficient Video Analytics Serving on Heterogeneous
 * GPU Clusters via Pool-Based Pipeline Parallelism"): for every model, every
 * well-formed split into K <= 3 contiguous partitions, every assignment of a GPU
 * class to each partition and every unified batch size, it scores the pooled
 * pipeline candidate and reduces the feasible ones to a per-(model, K, class
 * tuple) latency/throughput Pareto frontier -- the candidate set PPipe's MILP
 * picks from (its p_{ldbij} = 1 configurations, App. A.1;
 * PAPER.md:2365-2391, App. A.2).
 *
 * Definitions (all integer; DESIGN.md §2 lists every reading of the paper):
 *   partitions      c_0 = 0 < c_1 < ... < c_{K-1} < c_K = M; partition d covers
 *                   layers [c_{d-1}, c_d)           eqs. 1.1-1.5
 *   stage latency   C_d = sum_{l in partition d} lat_us[k_d][l][b]
 *                                                   C_{ldbij}, eq. 1.9
 *   transfer        Y_d = ceil(8 * act_bytes[c_d - 1] * b / bw[k_d][k_{d+1}])  for d < K
 *                                                   Y_{bj}, eq. 1.11
 *   E2E latency     E = sum_d C_d + sum_d Y_d        eq. 1.12
 *   feasible        E <= T_eff = floor(slo_us * (1000 - margin_permille) / 1000)
 *                                                   PAPER.md:1386-1394 (§5.4), 1690-1693 (§7.1)
 *   throughput      theta = b / max_d C_d (exact rational; max = 0 reads as +inf)
 *                                                   X = b / C, x_l = min_d x_ld
 *   frontier        per segment (model, K, k_1..k_K): feasible points not
 *                   dominated in (E min, theta max); among identical (E, theta)
 *                   the smallest batch, then the smallest (c_1, c_2) is kept.
 *
 * Conventions: every function returns PPIPE_OK (0) or a negative PPIPE_E*
 * code; nothing aborts and no C++ exception crosses the ABI. On error,
 * ppipe_last_error() returns a message naming the offending item. All input
 * pointers are host pointers owned by the caller and only read during the call.
 * Output arrays are owned by the context and stay valid until the next
 * ppipe_enumerate / ppipe_pareto on it or ppipe_free. One context per rank
 * (one process per GPU); calls on one context are not thread-safe. There is no
 * CPU fallback: without a usable sm_100 device every compute call returns
 * PPIPE_ECUDA.
 */
#ifndef PPIPE_H
#define PPIPE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PPIPE_OK = 0,
  PPIPE_EINVAL = -1, /* malformed input (sizes, ordering, zero bandwidth, bad K, margin >= 1000, NULL) */
  PPIPE_ERANGE = -2, /* input outside the exact-int32 envelope (see ppipe_load_profiles) */
  PPIPE_ENOMEM = -3, /* host or device allocation failed */
  PPIPE_ECUDA = -4,  /* CUDA runtime error, or no sm_100 device */
  PPIPE_ENCCL = -5,  /* NCCL unavailable or failed (world > 1 only) */
  PPIPE_ESTATE = -6  /* call out of order, e.g. ppipe_pareto before ppipe_enumerate */
};

typedef struct ppipe_ctx ppipe_ctx; /* opaque; owns all host and device memory it returns */

/* One model's profile (Table "Inputs to the MILP").
 * lat_us    [n_classes][n_layers][n_batches], row-major, integer microseconds, >= 0
 *           (L_{kbi}: latency of layer i at batch b on class k).
 * act_bytes [n_layers]: bytes ON THE WIRE of layer l's output at batch 1 (S_l;
 *           the caller halves fp32 sizes when quantising to fp16). */
typedef struct {
  uint32_t n_layers; /* M, 1..16384 (a model's c2 rows are staged in shared memory) */
  const uint32_t *lat_us;
  const uint64_t *act_bytes;
} ppipe_model;

/* Multi-GPU placement: one process per GPU. The enumeration space is split by
 * first-cut rows (contiguous (model, c_1) ranges of equal candidate weight);
 * local frontiers are merged with an NCCL all-gather and one final frontier pass. */
typedef struct {
  int32_t rank;           /* 0..world-1 */
  int32_t world;          /* >= 1 */
  int32_t device;         /* CUDA device ordinal for this rank; -1 = current device */
  const void *nccl_id;    /* 128-byte ncclUniqueId from ppipe_nccl_unique_id() on rank 0. NULL with
                             world > 1 = shard mode: no NCCL, ppipe_pareto returns this rank's LOCAL
                             frontier (exact over its rows; the union of all ranks' local frontiers
                             reduces to the global one by one more frontier pass) */
} ppipe_dist;

/* Validate, copy and upload the profiles this rank needs (host -> device).
 *   n_classes        1..8
 *   batches          [n_batches] batch VALUES, strictly increasing, 1..65535 (n_batches 1..65535)
 *   bw_bits_per_us   [n_classes][n_classes] effective bandwidth sender -> receiver in
 *                    bits/us (= Mbit/s), every entry >= 1 (1/5 of NIC rate)
 *   dist             NULL => single GPU, current device
 * Errors: PPIPE_EINVAL (NULLs, M = 0 or > 16384, n_classes, batch list, bw = 0);
 *         PPIPE_ERANGE (any whole-model latency sum at (class, batch) >= 2^28 us, or
 *         8 * act_bytes * max batch >= 2^63); PPIPE_ECUDA / PPIPE_ENOMEM / PPIPE_ENCCL.
 * On error *out is NULL and ppipe_last_error(NULL) holds the message. */
int ppipe_load_profiles(ppipe_ctx **out, uint32_t n_models, const ppipe_model *models, uint32_t n_classes,
                        uint32_t n_batches, const uint32_t *batches, const uint32_t *bw_bits_per_us,
                        const ppipe_dist *dist);

typedef struct {
  uint32_t max_partitions;  /* Kmax, 1..3 */
  const uint32_t *slo_us;   /* [n_models] raw latency SLO T per model, microseconds */
  uint32_t margin_permille; /* 0..999 deducted from the SLO; paper default 400 */
} ppipe_enum_params;

/* Replace the profile values of an existing context (same model count and
 * layer counts, same classes and batches): validate and copy host -> device.
 * Profiles change as workloads drift and the planner re-runs;
 * this keeps the device buffers and the NCCL communicator. The values are
 * validated on the device right after the host -> device copy (same envelope and
 * messages as ppipe_load_profiles; ranks with NCCL agree on the first failing
 * model; in shard mode a rank checks its own models). The call returns after
 * both, so the caller may reuse its buffers at once (page-locked buffers copy
 * fastest).
 * Errors as for ppipe_load_profiles; after a failed update the context has no
 * usable profiles and ppipe_enumerate returns PPIPE_ESTATE until an update
 * succeeds. Invalidates the last ppipe_enumerate. */
int ppipe_update_profiles(ppipe_ctx *ctx, uint32_t n_models, const ppipe_model *models);

/* Like ppipe_update_profiles, but returns at once after the shape checks: the
 * next ppipe_enumerate uploads the values itself, in up to 7 chunks of models on a
 * copy stream, and validates, packs and scores (K = 3 pass 1) each chunk as soon as
 * it has arrived, so the host -> device copy overlaps the scoring of earlier
 * chunks. The host buffers must stay valid and unchanged until the next
 * ppipe_pareto returns. Value errors (the ppipe_load_profiles envelope, same
 * messages) are returned by that ppipe_pareto (PPIPE_ERANGE; the context then has
 * no usable profiles until a successful update). Best with page-locked buffers.
 * Errors here: PPIPE_EINVAL. */
int ppipe_update_profiles_async(ppipe_ctx *ctx, uint32_t n_models, const ppipe_model *models);

/* Enqueue the whole enumeration on the context's stream: pack (prefix sums,
 * transfer tables, T_eff), then score every candidate of this rank's range and
 * fold feasible ones into per-(segment, batch) survivor sets. Asynchronous;
 * results are read through ppipe_pareto. Errors: PPIPE_EINVAL (Kmax, margin),
 * PPIPE_ERANGE (T_eff >= 2^28), PPIPE_ECUDA. */
int ppipe_enumerate(ppipe_ctx *ctx, const ppipe_enum_params *params);

/* One frontier point: 32 bytes, 4-byte aligned, little-endian. */
typedef struct {
  uint32_t model;       /* model index in the ppipe_load_profiles array */
  uint16_t cut[2];      /* c_1, c_2; 0 when unused */
  uint8_t K;            /* number of partitions, 1..3 */
  uint8_t cls[3];       /* k_d for d < K; 0xFF when unused */
  uint16_t batch;       /* batch VALUE b */
  uint16_t reserved;    /* 0 */
  uint32_t e2e_us;      /* E */
  uint32_t stage_us[3]; /* C_1..C_K; 0 when unused. max = bottleneck latency; E - sum = transfers */
} ppipe_point;

typedef struct {
  uint64_t n_candidates;  /* all ranks: sum_m sum_K C(M-1, K-1) * C^K * B */
  uint64_t n_feasible;    /* all ranks: candidates with E <= T_eff */
  uint64_t n_points;      /* frontier points */
  uint64_t n_segments;    /* sum_m sum_{K <= min(Kmax, M)} C^K, canonical order (m, K, tuple lexicographic) */
  const ppipe_point *points;     /* host copy in a page-locked buffer owned by ctx, valid until the
                                    next ppipe_pareto / ppipe_free; NULL unless copy_to_host */
  const uint64_t *seg_offsets;   /* host [n_segments + 1] CSR, same ownership; NULL unless copy_to_host */
  const ppipe_point *d_points;   /* device (this rank's GPU), same content */
  const uint64_t *d_seg_offsets; /* device [n_segments + 1] */
  uint64_t n_survivors;   /* diagnostics: this rank's pre-frontier survivor count */
  uint64_t n_candidates_local; /* this rank's share of n_candidates */
  uint64_t n_feasible_local;   /* this rank's share of n_feasible */
} ppipe_frontier;

/* Reduce the survivors to the exact frontier on device (sort + staircase
 * scan), merge across ranks (world > 1: NCCL all-gather + final pass; the
 * result is replicated on every rank), optionally copy to host, and block until
 * done. Errors: PPIPE_ESTATE (no prior ppipe_enumerate), PPIPE_ECUDA, PPIPE_ENCCL. */
int ppipe_pareto(ppipe_ctx *ctx, int copy_to_host, ppipe_frontier *out);

/* Merge the LOCAL frontiers of n_shards shard-mode contexts into the global frontier
 * (the decomposability F(A u B) = F(F(A) u F(B)) of the (E, theta)
 * staircase). shards[r] must be rank r of world n_shards loaded WITHOUT an NCCL id (shard
 * mode), on the same device, with the same models / classes / batches, each after a
 * successful ppipe_enumerate (same max_partitions, slo_us, margin_permille, vGPU
 * weights) and ppipe_pareto. This runs the same merge the NCCL path runs after its two
 * all-gathers -- counters and padded local frontiers in rank order, re-reduction of the
 * models that straddle a rank boundary, rank-ordered assembly, CSR -- with the
 * all-gathers replaced by device-to-device copies, so one GPU can check the multi-GPU
 * merge. The result (byte-identical to a one-rank ppipe_pareto of the same workload) is
 * owned by shards[0] like a ppipe_pareto result and replaces its local result; the other
 * shards are unchanged. n_candidates / n_feasible are summed over the shards. Errors:
 * EINVAL (NULL, ranks / shapes / parameters that do not match), ESTATE (a shard without a
 * local result), ECUDA / ENOMEM. */
int ppipe_merge_shards(ppipe_ctx *const *shards, int n_shards, int copy_to_host, ppipe_frontier *out);

/* F2, the MILP-lossless frontier (DESIGN.md §3 F2-1..F2-4).
 * PPipe's pooled MILP gives a chosen pipeline g_d GPUs in stage d and gets
 * throughput min_d g_d X_d, X_d = b / C_d the per-GPU throughput of stage d
 * (eqs. 1.10, 1.13); E only has to meet the SLO
 * (eq. 1.12). The (E, theta) frontier of ppipe_pareto can drop a
 * candidate the MILP needs for some g; F2 keeps, per segment, every feasible
 * candidate whose vector x = (X_1 .. X_K) no other feasible candidate of the segment
 * matches or beats in every stage (x_q >= x_p componentwise with x_q != x_p), and of
 * several with an identical vector the smallest (E, b, c_1, c_2). Virtual-GPU
 * weights scale a stage of every candidate alike and do not change F2.
 * One blocking call: pack, enumerate every candidate of params (as ppipe_enumerate),
 * reduce, and (world > 1 with NCCL) all-gather the per-rank frontiers; each model is
 * computed whole by the rank holding its K = 1 row (ppipe_partition_rows row 0), so
 * in shard mode a rank returns the F2 points of those models only.
 * out: as ppipe_pareto, except that points are ordered by (segment, b, c_1, c_2)
 * and n_survivors counts the candidates left after the strict-dominance pass
 * (before equal vectors are resolved). The result shares ppipe_pareto's buffers
 * (it invalidates the last ppipe_enumerate / ppipe_pareto) and cannot be swept by
 * ppipe_frontier_at (F2 frontiers are not SLO prefixes).
 * Device memory: K = 3 keeps a table of (M - 2)^2 int32 per (segment, batch) for a
 * group of segments at a time, at most PPIPE_F2_G_BYTES (environment; default
 * 8 GiB) or one segment's worth if that is larger.
 * Errors: as ppipe_enumerate; PPIPE_ERANGE for a model with more than 4096 layers;
 * PPIPE_ESTATE after ppipe_update_profiles_async (use ppipe_update_profiles);
 * PPIPE_ENOMEM, PPIPE_ECUDA, PPIPE_ENCCL. */
int ppipe_pareto_f2(ppipe_ctx *ctx, const ppipe_enum_params *params, int copy_to_host, ppipe_frontier *out);

/* Per-stage batch sizes (DESIGN.md §3 PB-1..PB-4). App. A.1's
 * basic MILP lets each partition run its own batch: eq. 1.1 sums p_{ldbij} over
 * (b, i, j) per partition d. A candidate is (cuts, classes, b_1..b_K):
 *   C_d = sum_{l in partition d} lat_us[k_d][l][b_d]                     eq. 1.9
 *   Y_d = ceil(8 * act_bytes[c_d - 1] * b_d / bw[k_d][k_{d+1}]), d < K   eq. 1.11 (the sender's batch)
 *   E   = sum C_d + sum Y_d <= T_eff                                     eq. 1.12
 *   theta = min_d b_d / C_d (exact rational; C_d = 0 reads as +inf)
 * and the frontier per segment (model, K, k_1..k_K) is the (E min, theta max)
 * staircase; among identical (E, theta) the smallest (b_1, .., b_K) (lexicographic),
 * then the smallest (c_1, c_2) stays. With one batch size this is ppipe_pareto's frontier.
 * B^K times the unified candidates: meant for block-level profiles.
 * Records carry batch INDICES per stage (bidx[d] into the batch list, 0xFF unused).
 * Virtual-GPU weights (ppipe_set_vgpu, an A.2 feature) do not apply: theta uses v = 1. */
typedef struct {
  uint32_t model;       /* model index */
  uint16_t cut[2];      /* c_1, c_2; 0 when unused */
  uint8_t K;            /* 1..3 */
  uint8_t cls[3];       /* k_d for d < K; 0xFF when unused */
  uint8_t bidx[3];      /* batch index of stage d for d < K; 0xFF when unused */
  uint8_t reserved;     /* 0 */
  uint32_t e2e_us;      /* E */
  uint32_t stage_us[3]; /* C_1..C_K */
} ppipe_point_pb;

typedef struct {
  uint64_t n_candidates;  /* all ranks: sum_m sum_K C(M-1, K-1) * C^K * B^K */
  uint64_t n_feasible;
  uint64_t n_points;
  uint64_t n_segments;
  const ppipe_point_pb *points;   /* host (page-locked, ctx-owned) if copy_to_host, else NULL; per segment E-ascending */
  const uint64_t *seg_offsets;    /* host [n_segments + 1] if copy_to_host */
  const ppipe_point_pb *d_points; /* device */
  const uint64_t *d_seg_offsets;  /* device */
  uint64_t n_survivors;           /* this rank's survivors of the in-CTA E-bucket fold */
} ppipe_frontier_pb;

/* One blocking call: pack, enumerate every per-stage-batch candidate, reduce, and
 * (world > 1 with NCCL) all-gather the per-rank frontiers; like ppipe_pareto_f2, each
 * model is computed whole by the rank holding its K = 1 row. The result shares the
 * context's result buffers (invalidates the last ppipe_enumerate / ppipe_pareto /
 * ppipe_pareto_f2 result) and is valid until the next such call or ppipe_free.
 * Errors: as ppipe_enumerate; PPIPE_ERANGE if n_batches > 255; PPIPE_ESTATE after
 * ppipe_update_profiles_async; PPIPE_ENOMEM, PPIPE_ECUDA, PPIPE_ENCCL. */
int ppipe_pareto_pb(ppipe_ctx *ctx, const ppipe_enum_params *params, int copy_to_host, ppipe_frontier_pb *out);

/* Virtual GPUs (§5.1; App. A.2 L_{kvbi}): declare
 * class k a pseudo-class that runs on 1/vgpu[k] of a physical GPU (MPS), vgpu[k] in
 * 1..4 (NULL = all 1, the default). Its profile is the caller's lat_us for that
 * fraction; a stage on it then delivers vgpu[k] * b / C_d per physical GPU, and a
 * plan's throughput is the minimum over its stages: theta = min_d v_{k_d} b / C_d
 * (exact; implemented as b / max_d (L / v_{k_d}) C_d with L the lcm of the v's in
 * use). Applies from the next ppipe_enumerate; invalidates the last results.
 * Envelope: T_eff * L / min v < 2^31 (else PPIPE_ERANGE at ppipe_enumerate).
 * Errors: PPIPE_EINVAL. */
int ppipe_set_vgpu(ppipe_ctx *ctx, const uint8_t *vgpu);

/* SLO sweep from one enumeration (Fig. 12a).
 * The frontier at a lower latency target is a prefix of every segment of the
 * frontier at a higher one (invariant I3: a point's dominators all have smaller or
 * equal E, so they stay feasible), so this derives the frontier for new per-model
 * SLOs slo_us[n_models] and margin_permille from the last ppipe_pareto result
 * without re-enumerating: per segment, the points with E <= T'_m =
 * floor(slo'_m * (1000 - margin') / 1000). Requires T'_m <= T_m of the last
 * ppipe_enumerate for every model (else PPIPE_EINVAL: raise the base SLO and
 * re-enumerate instead). The last ppipe_pareto result stays valid and can be swept
 * again. out: n_points, n_segments, points / seg_offsets (host, if copy_to_host;
 * the page-locked buffer is shared with ppipe_pareto's, so its previous host copy
 * is overwritten), d_points / d_seg_offsets (device, valid until the next
 * ppipe_frontier_at / ppipe_enumerate / ppipe_free); n_candidates is that of the
 * base enumeration; n_feasible, n_survivors and the _local counts are 0 (not
 * recomputed). Device work only (no collective), also under world > 1 where the
 * base result is replicated. Errors: PPIPE_ESTATE (no prior ppipe_pareto),
 * PPIPE_EINVAL, PPIPE_ECUDA. */
int ppipe_frontier_at(ppipe_ctx *ctx, const uint32_t *slo_us, uint32_t margin_permille, int copy_to_host,
                      ppipe_frontier *out);

/* Greedy equal-runtime pre-partitioning into n_blocks blocks (PAPER.md:1005-1010,
 * §5.2): per model, starting at layer 0, a block takes
 * consecutive layers while that brings its runtime t_l = lat[ref_class][l][ref_batch]
 * at least as close to total/N (ties take the layer; compared exactly as
 * |N*acc - total|), leaving one layer for every remaining block; the last block takes
 * the rest. Standalone device call (no context): models as for ppipe_load_profiles
 * (validated the same way), n_blocks in 1..min(n_layers), ref_class < n_classes,
 * ref_batch < n_batches (an index into the batch list). Host outputs, caller-owned:
 *   bounds      [n_models][n_blocks + 1]  block q = layers [bounds[q], bounds[q+1])
 *   block_lat   [n_models][n_classes][n_blocks][n_batches]  sums of member layers
 *   block_bytes [n_models][n_blocks]  act_bytes of each block's last layer
 * The outputs are block-level profiles ready for ppipe_load_profiles. device: CUDA
 * ordinal, -1 = current. Blocks until done. Errors: PPIPE_EINVAL, PPIPE_ERANGE,
 * PPIPE_ECUDA (message via ppipe_last_error(NULL)). */
int ppipe_prepartition(uint32_t n_models, const ppipe_model *models, uint32_t n_classes, uint32_t n_batches,
                       uint32_t n_blocks, uint32_t ref_class, uint32_t ref_batch, int32_t device, uint32_t *bounds,
                       uint32_t *block_lat, uint64_t *block_bytes);

/* Free everything the context owns. NULL-safe. */
void ppipe_free(ppipe_ctx *ctx);

/* Last error message: for ctx == NULL, the calling thread's last failed load. */
const char *ppipe_last_error(const ppipe_ctx *ctx);

/* ---- helpers (not part of the four-call path) ---- */

/* Write a fresh 128-byte ncclUniqueId into out (call on rank 0, broadcast it). */
int ppipe_nccl_unique_id(void *out128);

/* The CUDA stream (cudaStream_t) all of ctx's work is enqueued on. */
void *ppipe_stream(ppipe_ctx *ctx);

/* Device time (ms) of the last ppipe_enumerate's launches, measured with CUDA
 * events on ctx's stream: [0] pack, [1] score (dominant kernel), [2] frontier
 * (sort + scan), [3] merge (all-gather + final pass). Valid after ppipe_pareto. */
int ppipe_phase_ms(ppipe_ctx *ctx, float out_ms[4]);

/* Number of kernel launches the last enumerate + pareto issued (for bench accounting). */
uint64_t ppipe_launch_count(ppipe_ctx *ctx);

/* Host-only: this rank's first-cut row range per model under the row partition
 * (see ppipe_dist). rows[2*m] = lo, rows[2*m+1] = hi (half-open; row 0 = the K=1
 * candidates, row r >= 1 = candidates whose first cut c_1 = r). Returns
 * PPIPE_OK. Usable without a GPU. */
int ppipe_partition_rows(uint32_t n_models, const uint32_t *n_layers, uint32_t n_classes, uint32_t n_batches,
                         uint32_t max_partitions, int32_t rank, int32_t world, uint32_t *rows);

#ifdef __cplusplus
}
#endif
#endif /* PPIPE_H */
