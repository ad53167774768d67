// ppipe_abi.cpp -- C-ABI shim of libppipe_b200.so (include/ppipe.h).
//
// Host side of the hot path: input validation with named errors (SURVEY.md
// §8(b)), the first-cut-row partition across ranks (§8(e)), device memory and
// stream ownership, kernel orchestration (pack -> score -> frontier), and the
// NCCL frontier merge (all-gather of counts and local frontiers, then one final
// frontier pass). No arithmetic of the method runs here except closed-form
// bookkeeping (segment bases, row weights); every candidate is scored on the GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "ppipe_internal.h"

#define PPIPE_API extern "C" __attribute__((visibility("default")))

using namespace ppipe;

namespace {

thread_local std::string g_tls_error;

// ---- NCCL, loaded at run time (the process's already-loaded libnccl.so.2 if any) ----
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

bool load_nccl(std::string* err) {
  if (g_nccl.tried) {
    if (!g_nccl.ok && err) *err = "NCCL library could not be loaded";
    return g_nccl.ok;
  }
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    if (err) *err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
    return false;
  }
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllGather && g_nccl.CommDestroy;
  if (!g_nccl.ok && err) *err = "libnccl.so.2 lacks a required symbol";
  return g_nccl.ok;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;  // capacity in elements
  cudaError_t reserve(size_t want) {
    if (want <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(want, 1) * sizeof(T));
    if (e == cudaSuccess) n = std::max<size_t>(want, 1);
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// Page-locked host buffer (grow-only): D2H results land here at full link speed.
template <typename T>
struct HostBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaError_t reserve(size_t want) {
    if (want <= n && p) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    const size_t cap = std::max<size_t>(want + want / 4, 1);
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), cap * sizeof(T), cudaHostAllocDefault);
    if (e == cudaSuccess) n = cap;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
};

// Row weights of the partition (candidates per first-cut row, §8(e)).
// row 0: K = 1 (C * B); row r in [1, M-1]: K = 2 (C^2 B) + K = 3 with c_1 = r (C^3 B (M-1-r)).
inline unsigned __int128 row_weight(uint32_t M, uint32_t r, uint64_t C, uint64_t B, uint32_t kmax) {
  if (r == 0) return (unsigned __int128)C * B;
  unsigned __int128 w = 0;
  if (kmax >= 2 && M >= 2) w += (unsigned __int128)C * C * B;
  if (kmax >= 3 && M >= 3 && r <= M - 2) w += (unsigned __int128)C * C * C * B * (M - 1 - r);
  return w;
}

inline unsigned __int128 model_weight(uint32_t M, uint64_t C, uint64_t B, uint32_t kmax) {
  unsigned __int128 w = (unsigned __int128)C * B;
  if (kmax >= 2 && M >= 2) w += (unsigned __int128)C * C * B * (M - 1);
  if (kmax >= 3 && M >= 3) w += (unsigned __int128)C * C * C * B * ((uint64_t)(M - 1) * (M - 2) / 2);
  return w;
}

// Contiguous equal-weight split of the (model, row) sequence. A row whose
// starting prefix weight s satisfies q*W <= s*world < (q+1)*W goes to rank q.
void partition_rows(const std::vector<uint32_t>& Ms, uint64_t C, uint64_t B, uint32_t kmax, int rank, int world,
                    std::vector<uint32_t>& rows) {
  const size_t n = Ms.size();
  rows.assign(2 * n, 0);
  unsigned __int128 W = 0;
  for (uint32_t M : Ms) W += model_weight(M, C, B, kmax);
  if (world <= 1) {
    for (size_t m = 0; m < n; ++m) {
      rows[2 * m] = 0;
      rows[2 * m + 1] = Ms[m];
    }
    return;
  }
  auto owner = [&](unsigned __int128 s) -> int {
    unsigned __int128 q = s * (unsigned __int128)world / W;
    return (int)std::min<unsigned __int128>(q, (unsigned __int128)(world - 1));
  };
  unsigned __int128 s = 0;
  for (size_t m = 0; m < n; ++m) {
    const uint32_t M = Ms[m];
    const unsigned __int128 wm = model_weight(M, C, B, kmax);
    int64_t lo = -1, hi = -1;
    if (owner(s) == rank && owner(s + wm - 1) == rank) {
      lo = 0;
      hi = M;  // whole model
    } else if (owner(s) <= rank && owner(s + wm - 1) >= rank) {
      unsigned __int128 t = s;
      for (uint32_t r = 0; r < M; ++r) {
        const int o = owner(t);
        if (o == rank) {
          if (lo < 0) lo = r;
          hi = r + 1;
        }
        t += row_weight(M, r, C, B, kmax);
      }
    }
    if (lo >= 0) {
      rows[2 * m] = (uint32_t)lo;
      rows[2 * m + 1] = (uint32_t)hi;
    }
    s += wm;
  }
}

}  // namespace

struct ppipe_ctx {
  std::string err;
  int rank = 0, world = 1, device = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  uint32_t C = 0, B = 0, n_models = 0, V = 0;
  std::vector<uint32_t> Ms;        // all models
  std::vector<uint32_t> h_batches;
  std::vector<uint32_t> rows;      // [2*n_models] this rank's row ranges
  std::vector<int> local;          // local model ids (work order)
  std::vector<uint64_t> h_segbase; // [n_models + 1] first global segment of each model (last enumerate)
  DevBuf<uint64_t> d_segtmp;       // merge: segment id per final point
  DevBuf<ppipe_point> d_merged;    // merge: re-reduced frontier of the straddling models
  std::vector<DevModel> h_models;  // per local model
  uint32_t max_M = 0;
  // device inputs
  DevBuf<uint32_t> d_lat;
  DevBuf<uint64_t> d_s;
  DevBuf<int32_t> d_P, d_Y;
  DevBuf<DevModel> d_models;
  DevBuf<uint16_t> d_batches;
  DevBuf<uint32_t> d_bwv;
  DevBuf<uint8_t> d_pairv;
  DevBuf<uint64_t> d_segbase;
  // outputs
  DevBuf<unsigned long long> d_counters;
  DevBuf<uint4> d_hot;
  DevBuf<uint64_t> d_hot_tab;
  DevBuf<uint32_t> d_hot_order;  // pass-2 order of the hot units (heaviest first)
  DevBuf<uint32_t> d_hot_w;      // pass-1 feasible count per hot unit
  uint64_t hot_cap = 0;
  DevBuf<ppipe_point> d_surv, d_local, d_gather, d_union, d_final;
  DevBuf<uint64_t> d_segoff_local, d_segoff_final, d_cnt_send, d_cnt_recv;
  FrontierScratch scratch;
  HostBuf<ppipe_point> h_points;  // pinned: last copy_to_host result (valid until the next ppipe_pareto)
  HostBuf<uint64_t> h_segoff;
  bool profiles_ok = true;  // false after a failed ppipe_update_profiles
  unsigned long long* h_counters = nullptr;  // pinned [5]
  // enumerate state
  bool enumerated = false;
  uint32_t wpack = 0x11111111u;  // per-class virtual-GPU weights (ppipe_set_vgpu), 4 bits each
  int w_bits = 0;
  uint32_t w_max = 1;
  // last ppipe_pareto result (base of ppipe_frontier_at)
  bool have_result = false;
  const ppipe_point* res_pts = nullptr;
  const uint64_t* res_off = nullptr;
  uint64_t res_n = 0, res_ncand = 0, res_nfeas = 0, res_nsurv = 0;
  bool res_local = false;
  DevBuf<ppipe_point> d_trunc;
  DevBuf<uint64_t> d_trunc_off;
  DevBuf<uint32_t> d_Tnew;
  ppipe_enum_params last_params{};
  std::vector<uint32_t> last_slo;
  uint64_t n_seg_total = 0;
  uint64_t surv_cap = 1ull << 22;
  cudaEvent_t ev[8] = {};
  // ppipe_update_profiles_async: host descriptors whose copy the next enumerate
  // issues in chunks on cstream, overlapped with scoring earlier chunks
#ifndef PPIPE_MAX_CHUNKS
#define PPIPE_MAX_CHUNKS 8  // chunk events of the async upload (at most 8 chunks)
#endif
  static constexpr int kMaxChunks = PPIPE_MAX_CHUNKS;
  bool pending_upload = false, check_err = false;
  std::vector<ppipe_model> pending;
  cudaStream_t cstream = nullptr;
  cudaStream_t stream2 = nullptr;  // second compute stream: consecutive chunks' score3a overlap (no tail gaps)
  cudaEvent_t sev[2] = {};         // fork / join between stream and stream2
  cudaEvent_t cev[kMaxChunks + 1] = {};
  DevBuf<unsigned long long> d_err;
  // F2 (ppipe_pareto_f2)
  DevBuf<int32_t> d_G, d_F, d_E23, d_pbsd, d_minA;
  DevBuf<unsigned long long> d_gfold;  // cross-batch fold of the K = 3 segments (Problem::gfold)
  DevBuf<uint16_t> d_inv;  // F2 inverse stage tables PF, PFs, SF, SFs
  DevBuf<ppipe_point> d_f2surv, d_f2tmp;
  uint64_t f2_cap = 1ull << 20;
  float phase_ms[4] = {0, 0, 0, 0};
  uint64_t launches = 0;
  int launches_i = 0;
};

namespace {

int fail(ppipe_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  else g_tls_error = buf;
  return code;
}

#define CU(ctx, call)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail((ctx), e_ == cudaErrorMemoryAllocation ? PPIPE_ENOMEM : PPIPE_ECUDA,       \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);      \
  } while (0)

#define NC_(ctx, call)                                                                       \
  do {                                                                                       \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      return fail((ctx), PPIPE_ENCCL, "%s: %s", #call,                                       \
                  g_nccl.GetErrorString ? g_nccl.GetErrorString(r_) : "nccl error");         \
  } while (0)

void free_ctx(ppipe_ctx* c) {
  if (!c) return;
  if (c->device >= 0) cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  c->d_lat.release();
  c->d_s.release();
  c->d_P.release();
  c->d_Y.release();
  c->d_models.release();
  c->d_batches.release();
  c->d_bwv.release();
  c->d_pairv.release();
  c->d_segbase.release();
  c->d_counters.release();
  c->d_hot.release();
  c->d_hot_tab.release();
  c->d_hot_order.release();
  c->d_hot_w.release();
  c->d_surv.release();
  c->d_local.release();
  c->d_gather.release();
  c->d_union.release();
  c->d_final.release();
  c->d_segoff_local.release();
  c->d_segoff_final.release();
  c->d_cnt_send.release();
  c->d_cnt_recv.release();
  c->d_segtmp.release();
  c->d_merged.release();
  c->d_trunc.release();
  c->d_trunc_off.release();
  c->d_Tnew.release();
  c->h_points.release();
  c->h_segoff.release();
  if (c->scratch.buf) cudaFree(c->scratch.buf);
  if (c->h_counters) cudaFreeHost(c->h_counters);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->cstream) cudaStreamDestroy(c->cstream);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  for (auto& e : c->sev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->cev)
    if (e) cudaEventDestroy(e);
  c->d_err.release();
  c->d_G.release();
  c->d_F.release();
  c->d_E23.release();
  c->d_pbsd.release();
  c->d_minA.release();
  c->d_gfold.release();
  c->d_inv.release();
  c->d_f2surv.release();
  c->d_f2tmp.release();
  delete c;
}

}  // namespace

// Per-model checks of the exact-int32 envelope (threaded over models; the
// first failing model in index order is reported, so the message is deterministic).
static int validate_models(uint32_t n_models, const ppipe_model* models, uint32_t C, uint32_t B, const uint32_t* batches,
                    std::string* err) {
  const uint64_t bmax = batches[B - 1];
  std::vector<int> code(n_models, PPIPE_OK);
  std::vector<std::string> msg(n_models);
  auto check = [&](uint32_t m) {
    const ppipe_model& md = models[m];
    char buf[256];
    if (md.n_layers < 1 || md.n_layers > (uint32_t)kMaxLayers) {
      snprintf(buf, sizeof buf, "model %u: n_layers %u must be 1..%d", m, md.n_layers, kMaxLayers);
      code[m] = PPIPE_EINVAL;
      msg[m] = buf;
      return;
    }
    if (!md.lat_us || !md.act_bytes) {
      snprintf(buf, sizeof buf, "model %u: NULL profile pointer", m);
      code[m] = PPIPE_EINVAL;
      msg[m] = buf;
      return;
    }
    const uint32_t M = md.n_layers;
    std::vector<uint64_t> tot((size_t)C * B, 0);
    for (uint32_t k = 0; k < C; ++k)
      for (uint32_t l = 0; l < M; ++l) {
        const uint32_t* row = md.lat_us + ((size_t)k * M + l) * B;
        uint64_t* t = tot.data() + (size_t)k * B;
        for (uint32_t bi = 0; bi < B; ++bi) t[bi] += row[bi];
      }
    for (uint32_t k = 0; k < C; ++k)
      for (uint32_t bi = 0; bi < B; ++bi)
        if (tot[(size_t)k * B + bi] >= (uint64_t)kRangeLimit) {
          snprintf(buf, sizeof buf, "model %u class %u batch %u: whole-model latency %llu us >= 2^28 (int32 envelope)",
                   m, k, batches[bi], (unsigned long long)tot[(size_t)k * B + bi]);
          code[m] = PPIPE_ERANGE;
          msg[m] = buf;
          return;
        }
    const uint64_t smax = (uint64_t)INT64_MAX / (8 * bmax);
    for (uint32_t l = 0; l < M; ++l)
      if (md.act_bytes[l] > smax) {
        snprintf(buf, sizeof buf, "model %u layer %u: act_bytes %llu too large (8*S*b >= 2^63)", m, l,
                 (unsigned long long)md.act_bytes[l]);
        code[m] = PPIPE_ERANGE;
        msg[m] = buf;
        return;
      }
  };
  const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
  if (n_models < 4 || nt == 1) {
    for (uint32_t m = 0; m < n_models; ++m) check(m);
  } else {
    std::atomic<uint32_t> next{0};
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
      th.emplace_back([&] {
        for (uint32_t m; (m = next.fetch_add(1)) < n_models;) check(m);
      });
    for (auto& t : th) t.join();
  }
  for (uint32_t m = 0; m < n_models; ++m)
    if (code[m] != PPIPE_OK) {
      *err = msg[m];
      return code[m];
    }
  return PPIPE_OK;
}

// ===========================================================================
// ABI
// ===========================================================================

PPIPE_API const char* ppipe_last_error(const ppipe_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  return g_tls_error.c_str();
}

PPIPE_API int ppipe_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, PPIPE_EINVAL, "ppipe_nccl_unique_id: NULL output");
  std::string err;
  if (!load_nccl(&err)) return fail(nullptr, PPIPE_ENCCL, "%s", err.c_str());
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, PPIPE_ENCCL, "ncclGetUniqueId failed");
  std::memcpy(out128, &id, sizeof id);
  return PPIPE_OK;
}

PPIPE_API int ppipe_prepartition(uint32_t n_models, const ppipe_model* models, uint32_t n_classes, uint32_t n_batches,
                                 uint32_t n_blocks, uint32_t ref_class, uint32_t ref_batch, int32_t device,
                                 uint32_t* bounds, uint32_t* block_lat, uint64_t* block_bytes) {
  if (n_models == 0) return PPIPE_OK;
  if (!models || !bounds || !block_lat || !block_bytes)
    return fail(nullptr, PPIPE_EINVAL, "ppipe_prepartition: NULL argument");
  if (n_classes < 1 || n_classes > 8 || n_batches < 1)
    return fail(nullptr, PPIPE_EINVAL, "ppipe_prepartition: n_classes %u / n_batches %u invalid", n_classes,
                n_batches);
  if (ref_class >= n_classes || ref_batch >= n_batches)
    return fail(nullptr, PPIPE_EINVAL, "ppipe_prepartition: reference class %u / batch index %u out of range",
                ref_class, ref_batch);
  {
    std::vector<uint32_t> ones(n_batches, 1);  // block bytes are layer bytes: check S alone
    std::string verr;
    const int vrc = validate_models(n_models, models, n_classes, n_batches, ones.data(), &verr);
    if (vrc != PPIPE_OK) return fail(nullptr, vrc, "%s", verr.c_str());
  }
  for (uint32_t m = 0; m < n_models; ++m)
    if (n_blocks < 1 || n_blocks > models[m].n_layers)
      return fail(nullptr, PPIPE_EINVAL, "model %u: n_blocks %u must be 1..%u (its layer count)", m, n_blocks,
                  models[m].n_layers);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, PPIPE_ECUDA, "no CUDA device: this library has no CPU fallback");
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess)
    return fail(nullptr, PPIPE_ECUDA, "cudaSetDevice(%d) failed", device);
  const uint64_t C = n_classes, B = n_batches, N = n_blocks;
  std::vector<uint64_t> lat_off(n_models), s_off(n_models);
  std::vector<uint32_t> Ms(n_models);
  uint64_t nl = 0, ns = 0;
  for (uint32_t m = 0; m < n_models; ++m) {
    lat_off[m] = nl;
    s_off[m] = ns;
    Ms[m] = models[m].n_layers;
    nl += C * Ms[m] * B;
    ns += Ms[m];
  }
  struct Local {
    DevBuf<uint32_t> lat, M, bounds, blat;
    DevBuf<uint64_t> S, lo, so, bS;
    DevBuf<int64_t> prefix;
    cudaStream_t s = nullptr;
    ~Local() {
      lat.release(); M.release(); bounds.release(); blat.release();
      S.release(); lo.release(); so.release(); bS.release(); prefix.release();
      if (s) cudaStreamDestroy(s);
    }
  } d;
#define CUP(x)                                                                                   \
  do {                                                                                           \
    const cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(nullptr, PPIPE_ECUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)
  CUP(cudaStreamCreateWithFlags(&d.s, cudaStreamNonBlocking));
  CUP(d.lat.reserve(nl));
  CUP(d.S.reserve(ns));
  CUP(d.lo.reserve(n_models));
  CUP(d.so.reserve(n_models));
  CUP(d.M.reserve(n_models));
  CUP(d.prefix.reserve(ns + n_models));
  CUP(d.bounds.reserve((size_t)n_models * (N + 1)));
  CUP(d.blat.reserve((size_t)n_models * C * N * B));
  CUP(d.bS.reserve((size_t)n_models * N));
  for (uint32_t m = 0; m < n_models; ++m) {
    CUP(cudaMemcpyAsync(d.lat.p + lat_off[m], models[m].lat_us, 4 * C * Ms[m] * B, cudaMemcpyHostToDevice, d.s));
    CUP(cudaMemcpyAsync(d.S.p + s_off[m], models[m].act_bytes, 8 * (size_t)Ms[m], cudaMemcpyHostToDevice, d.s));
  }
  CUP(cudaMemcpyAsync(d.lo.p, lat_off.data(), 8 * (size_t)n_models, cudaMemcpyHostToDevice, d.s));
  CUP(cudaMemcpyAsync(d.so.p, s_off.data(), 8 * (size_t)n_models, cudaMemcpyHostToDevice, d.s));
  CUP(cudaMemcpyAsync(d.M.p, Ms.data(), 4 * (size_t)n_models, cudaMemcpyHostToDevice, d.s));
  PrepartProblem pp{d.lat.p, d.S.p, d.lo.p, d.so.p, d.M.p, d.prefix.p, d.bounds.p, d.blat.p, d.bS.p,
                    (int)n_models, (int)C, (int)B, (int)N, (int)ref_class, (int)ref_batch};
  CUP(launch_prepartition(pp, d.s));
  CUP(cudaMemcpyAsync(bounds, d.bounds.p, 4 * (size_t)n_models * (N + 1), cudaMemcpyDeviceToHost, d.s));
  CUP(cudaMemcpyAsync(block_lat, d.blat.p, 4 * (size_t)n_models * C * N * B, cudaMemcpyDeviceToHost, d.s));
  CUP(cudaMemcpyAsync(block_bytes, d.bS.p, 8 * (size_t)n_models * N, cudaMemcpyDeviceToHost, d.s));
  CUP(cudaStreamSynchronize(d.s));
#undef CUP
  return PPIPE_OK;
}

PPIPE_API int ppipe_partition_rows(uint32_t n_models, const uint32_t* n_layers, uint32_t n_classes,
                                   uint32_t n_batches, uint32_t max_partitions, int32_t rank, int32_t world,
                                   uint32_t* rows) {
  if (!n_layers || !rows || n_models == 0 || world < 1 || rank < 0 || rank >= world || n_classes == 0 ||
      n_batches == 0 || max_partitions < 1 || max_partitions > 3)
    return fail(nullptr, PPIPE_EINVAL, "ppipe_partition_rows: invalid arguments");
  std::vector<uint32_t> Ms(n_layers, n_layers + n_models), r;
  partition_rows(Ms, n_classes, n_batches, max_partitions, rank, world, r);
  std::memcpy(rows, r.data(), r.size() * sizeof(uint32_t));
  return PPIPE_OK;
}

PPIPE_API void* ppipe_stream(ppipe_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

PPIPE_API uint64_t ppipe_launch_count(ppipe_ctx* ctx) { return ctx ? ctx->launches : 0; }

PPIPE_API int ppipe_phase_ms(ppipe_ctx* ctx, float out_ms[4]) {
  if (!ctx || !out_ms) return PPIPE_EINVAL;
  std::memcpy(out_ms, ctx->phase_ms, sizeof ctx->phase_ms);
  return PPIPE_OK;
}

PPIPE_API void ppipe_free(ppipe_ctx* ctx) { free_ctx(ctx); }

PPIPE_API int ppipe_load_profiles(ppipe_ctx** out, uint32_t n_models, const ppipe_model* models, uint32_t n_classes,
                                  uint32_t n_batches, const uint32_t* batches, const uint32_t* bw_bits_per_us,
                                  const ppipe_dist* dist) {
  if (!out) return fail(nullptr, PPIPE_EINVAL, "ppipe_load_profiles: out is NULL");
  *out = nullptr;
  if (n_models == 0 || !models) return fail(nullptr, PPIPE_EINVAL, "ppipe_load_profiles: no models");
  if (n_classes < 1 || n_classes > (uint32_t)kMaxClasses)
    return fail(nullptr, PPIPE_EINVAL, "n_classes %u: must be 1..%d", n_classes, kMaxClasses);
  if (n_batches < 1 || n_batches > 65535 || !batches)
    return fail(nullptr, PPIPE_EINVAL, "n_batches %u: must be 1..65535 with a batch list", n_batches);
  for (uint32_t i = 0; i < n_batches; ++i) {
    if (batches[i] < 1 || batches[i] > 65535)
      return fail(nullptr, PPIPE_EINVAL, "batch %u value %u: must be 1..65535", i, batches[i]);
    if (i && batches[i] <= batches[i - 1])
      return fail(nullptr, PPIPE_EINVAL, "batch %u value %u: batches must be strictly increasing", i, batches[i]);
  }
  if (!bw_bits_per_us) return fail(nullptr, PPIPE_EINVAL, "bandwidth matrix is NULL");
  for (uint32_t i = 0; i < n_classes * n_classes; ++i)
    if (bw_bits_per_us[i] == 0)
      return fail(nullptr, PPIPE_EINVAL, "bandwidth class %u -> class %u: must be >= 1 bits/us", i / n_classes,
                  i % n_classes);
  {
    std::string verr;
    const int vrc = validate_models(n_models, models, n_classes, n_batches, batches, &verr);
    if (vrc != PPIPE_OK) return fail(nullptr, vrc, "%s", verr.c_str());
  }
  int rank = 0, world = 1, device = -1;
  const void* nccl_id = nullptr;
  if (dist) {
    rank = dist->rank;
    world = dist->world;
    device = dist->device;
    nccl_id = dist->nccl_id;
    if (world < 1 || rank < 0 || rank >= world)
      return fail(nullptr, PPIPE_EINVAL, "dist: rank %d / world %d invalid", rank, world);
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, PPIPE_ECUDA, "no CUDA device: this library has no CPU fallback");
  if (device < 0) cudaGetDevice(&device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
    return fail(nullptr, PPIPE_ECUDA, "cudaGetDeviceProperties(%d) failed", device);
  if (prop.major != 10 || prop.minor != 0)
    return fail(nullptr, PPIPE_ECUDA, "device %d is sm_%d%d; this build targets sm_100a (B200) only", device,
                prop.major, prop.minor);

  ppipe_ctx* c = new ppipe_ctx();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->C = n_classes;
  c->B = n_batches;
  c->n_models = n_models;
  c->h_batches.assign(batches, batches + n_batches);
  if (const char* cap = getenv("PPIPE_SURVIVOR_CAP")) {  // initial survivor capacity (tests of the regrow path)
    const long long v = atoll(cap);
    if (v > 0) c->surv_cap = (uint64_t)v;
  }
  if (const char* cap = getenv("PPIPE_HOT_CAP")) {  // initial hot-unit capacity (tests of the regrow path)
    const long long v = atoll(cap);
    if (v > 0) c->hot_cap = (uint64_t)v;
  }
  auto bail = [&](int code) {
    g_tls_error = c->err;
    free_ctx(c);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) {
    fail(c, PPIPE_ECUDA, "cudaSetDevice(%d) failed", device);
    return bail(PPIPE_ECUDA);
  }
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    fail(c, PPIPE_ECUDA, "cudaStreamCreate failed");
    return bail(PPIPE_ECUDA);
  }
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) {
      fail(c, PPIPE_ECUDA, "cudaEventCreate failed");
      return bail(PPIPE_ECUDA);
    }
  if (cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking) != cudaSuccess) {
    fail(c, PPIPE_ECUDA, "cudaStreamCreate failed");
    return bail(PPIPE_ECUDA);
  }
  for (auto& e : c->sev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      fail(c, PPIPE_ECUDA, "cudaEventCreate failed");
      return bail(PPIPE_ECUDA);
    }
  if (cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking) != cudaSuccess) {
    fail(c, PPIPE_ECUDA, "cudaStreamCreate failed");
    return bail(PPIPE_ECUDA);
  }
  for (auto& e : c->cev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      fail(c, PPIPE_ECUDA, "cudaEventCreate failed");
      return bail(PPIPE_ECUDA);
    }
  if (cudaMallocHost(&c->h_counters, 16 * sizeof(unsigned long long)) != cudaSuccess) {
    fail(c, PPIPE_ENOMEM, "cudaMallocHost failed");
    return bail(PPIPE_ENOMEM);
  }
  if (world > 1 && nccl_id) {
    std::string err;
    if (!load_nccl(&err)) {
      fail(c, PPIPE_ENCCL, "%s", err.c_str());
      return bail(PPIPE_ENCCL);
    }
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    ncclResult_t r = g_nccl.CommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
      fail(c, PPIPE_ENCCL, "ncclCommInitRank(world=%d, rank=%d): %s", world, rank,
           g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "error");
      return bail(PPIPE_ENCCL);
    }
  }
  // partition (weights with Kmax = 3; valid for any Kmax)
  c->Ms.resize(n_models);
  for (uint32_t m = 0; m < n_models; ++m) c->Ms[m] = models[m].n_layers;
  partition_rows(c->Ms, n_classes, n_batches, 3, rank, world, c->rows);
  for (uint32_t m = 0; m < n_models; ++m)
    if (c->rows[2 * m + 1] > c->rows[2 * m]) c->local.push_back((int)m);
  // heavy models first (K = 3 work ~ M^2) for a short tail
  std::stable_sort(c->local.begin(), c->local.end(), [&](int a, int b) { return c->Ms[a] > c->Ms[b]; });
  // distinct bandwidth values and the class-pair map
  std::vector<uint32_t> bwv(bw_bits_per_us, bw_bits_per_us + n_classes * n_classes);
  std::sort(bwv.begin(), bwv.end());
  bwv.erase(std::unique(bwv.begin(), bwv.end()), bwv.end());
  std::vector<uint8_t> pairv(n_classes * n_classes);
  for (uint32_t i = 0; i < n_classes * n_classes; ++i)
    pairv[i] = (uint8_t)(std::lower_bound(bwv.begin(), bwv.end(), bw_bits_per_us[i]) - bwv.begin());
  c->V = (uint32_t)bwv.size();
  // device layout
  uint64_t lat_n = 0, s_n = 0, p_n = 0, y_n = 0;
  for (int m : c->local) {
    DevModel d{};
    d.M = c->Ms[m];
    d.Mp = (d.M + 1 + 3) / 4 * 4;
    d.lat_off = lat_n;
    d.s_off = s_n;
    d.p_off = p_n;
    d.y_off = y_n;
    d.model = (uint32_t)m;
    d.row_lo = c->rows[2 * m];
    d.row_hi = c->rows[2 * m + 1];
    lat_n += (uint64_t)n_classes * d.M * n_batches;
    s_n += d.M;
    p_n += (uint64_t)n_classes * n_batches * d.Mp;
    y_n += (uint64_t)c->V * n_batches * d.Mp;
    c->max_M = std::max(c->max_M, d.M);
    c->h_models.push_back(d);
  }
  int rc;
#define CUL(call)                                                                                          \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess) {                                                                               \
      rc = fail(c, e_ == cudaErrorMemoryAllocation ? PPIPE_ENOMEM : PPIPE_ECUDA, "%s: %s", #call,          \
                cudaGetErrorString(e_));                                                                   \
      return bail(rc);                                                                                     \
    }                                                                                                      \
  } while (0)
  CUL(c->d_lat.reserve(lat_n));
  CUL(c->d_s.reserve(s_n));
  CUL(c->d_P.reserve(p_n));
  CUL(c->d_Y.reserve(y_n));
  CUL(c->d_models.reserve(c->h_models.size()));
  CUL(c->d_batches.reserve(n_batches));
  CUL(c->d_bwv.reserve(c->V));
  CUL(c->d_pairv.reserve(pairv.size()));
  CUL(c->d_segbase.reserve(n_models));
  CUL(c->d_counters.reserve(16));
  // host -> device: the profiles this rank needs
  for (size_t i = 0; i < c->local.size(); ++i) {
    const int m = c->local[i];
    const DevModel& d = c->h_models[i];
    CUL(cudaMemcpyAsync(c->d_lat.p + d.lat_off, models[m].lat_us, sizeof(uint32_t) * n_classes * d.M * n_batches,
                        cudaMemcpyHostToDevice, c->stream));
    CUL(cudaMemcpyAsync(c->d_s.p + d.s_off, models[m].act_bytes, sizeof(uint64_t) * d.M, cudaMemcpyHostToDevice,
                        c->stream));
  }
  std::vector<uint16_t> b16(batches, batches + n_batches);
  CUL(cudaMemcpyAsync(c->d_batches.p, b16.data(), 2 * n_batches, cudaMemcpyHostToDevice, c->stream));
  CUL(cudaMemcpyAsync(c->d_bwv.p, bwv.data(), 4 * bwv.size(), cudaMemcpyHostToDevice, c->stream));
  CUL(cudaMemcpyAsync(c->d_pairv.p, pairv.data(), pairv.size(), cudaMemcpyHostToDevice, c->stream));
  CUL(cudaStreamSynchronize(c->stream));
#undef CUL
  *out = c;
  return PPIPE_OK;
}

static int report_validation(ppipe_ctx* c, unsigned long long key, const ppipe_model* models);

PPIPE_API int ppipe_update_profiles(ppipe_ctx* c, uint32_t n_models, const ppipe_model* models) {
  if (!c) return fail(nullptr, PPIPE_EINVAL, "ppipe_update_profiles: NULL ctx");
  if (n_models != c->n_models || !models)
    return fail(c, PPIPE_EINVAL, "ppipe_update_profiles: %u models, context has %u", n_models, c->n_models);
  for (uint32_t m = 0; m < n_models; ++m)
    if (models[m].n_layers != c->Ms[m])
      return fail(c, PPIPE_EINVAL, "model %u: n_layers %u differs from the loaded %u", m, models[m].n_layers,
                  c->Ms[m]);
  // Copy, then validate on the device (the values are there anyway): one pass over
  // the profiles at HBM speed instead of a host pass over the caller's memory. A
  // failed validation leaves the context without usable profiles until the next
  // successful update. Ranks with NCCL agree on the first failing model.
  c->profiles_ok = false;
  c->enumerated = false;
  c->have_result = false;
  c->res_local = false;
  c->pending_upload = false;  // a synchronous update supersedes a pending asynchronous one
  CU(c, cudaSetDevice(c->device));
  for (size_t i = 0; i < c->local.size(); ++i) {
    const int m = c->local[i];
    const DevModel& d = c->h_models[i];
    CU(c, cudaMemcpyAsync(c->d_lat.p + d.lat_off, models[m].lat_us, sizeof(uint32_t) * c->C * d.M * c->B,
                          cudaMemcpyHostToDevice, c->stream));
    CU(c, cudaMemcpyAsync(c->d_s.p + d.s_off, models[m].act_bytes, sizeof(uint64_t) * d.M, cudaMemcpyHostToDevice,
                          c->stream));
  }
  CU(c, c->d_models.reserve(std::max<size_t>(c->h_models.size(), 1)));
  CU(c, cudaMemcpyAsync(c->d_models.p, c->h_models.data(), sizeof(DevModel) * c->h_models.size(),
                        cudaMemcpyHostToDevice, c->stream));
  CU(c, c->d_cnt_send.reserve(4));
  const unsigned long long none = ~0ull;
  CU(c, cudaMemcpyAsync(c->d_cnt_send.p, &none, 8, cudaMemcpyHostToDevice, c->stream));
  const uint64_t bmax = c->h_batches[c->B - 1];
  CU(c, launch_validate(c->d_models.p, (int)c->local.size(), c->d_lat.p, c->d_s.p, (int)c->C, (int)c->B,
                        (uint64_t)INT64_MAX / (8 * bmax), reinterpret_cast<unsigned long long*>(c->d_cnt_send.p),
                        c->stream));
  unsigned long long key = none;
  if (c->world > 1 && c->comm) {
    CU(c, c->d_cnt_recv.reserve((size_t)c->world));
    NC_(c, g_nccl.AllGather(c->d_cnt_send.p, c->d_cnt_recv.p, 1, ncclUint64, c->comm, c->stream));
    std::vector<unsigned long long> keys(c->world);
    CU(c, cudaMemcpyAsync(keys.data(), c->d_cnt_recv.p, 8 * keys.size(), cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    for (auto k : keys) key = std::min(key, k);
  } else {
    CU(c, cudaMemcpyAsync(&key, c->d_cnt_send.p, 8, cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
  }
  if (key != none) return report_validation(c, key, models);  // same wording as ppipe_load_profiles

  c->profiles_ok = true;
  c->enumerated = false;
  return PPIPE_OK;
}

PPIPE_API int ppipe_update_profiles_async(ppipe_ctx* c, uint32_t n_models, const ppipe_model* models) {
  if (!c) return fail(nullptr, PPIPE_EINVAL, "ppipe_update_profiles_async: NULL ctx");
  if (n_models != c->n_models || !models)
    return fail(c, PPIPE_EINVAL, "ppipe_update_profiles_async: %u models, context has %u", n_models, c->n_models);
  for (uint32_t m = 0; m < n_models; ++m) {
    if (models[m].n_layers != c->Ms[m])
      return fail(c, PPIPE_EINVAL, "model %u: n_layers %u differs from the loaded %u", m, models[m].n_layers,
                  c->Ms[m]);
    if (!models[m].lat_us || !models[m].act_bytes) return fail(c, PPIPE_EINVAL, "model %u: NULL profile pointer", m);
  }
  c->pending.assign(models, models + n_models);
  c->pending_upload = true;
  c->profiles_ok = true;  // values are checked on the device; errors surface in ppipe_pareto
  c->enumerated = false;
  c->have_result = false;
  c->res_local = false;
  return PPIPE_OK;
}

// First failing (model, kind, index) of a device validation key -> the host check's message.
static int report_validation(ppipe_ctx* c, unsigned long long key, const ppipe_model* models) {
  const uint32_t m = (uint32_t)(key >> 40), idx = (uint32_t)(key & ((1ull << 39) - 1));
  if (key & (1ull << 39))
    return fail(c, PPIPE_ERANGE, "model %u layer %u: act_bytes %llu too large (8*S*b >= 2^63)", m, idx,
                (unsigned long long)models[m].act_bytes[idx]);
  const uint32_t k = idx / c->B, bi = idx % c->B, M = models[m].n_layers;
  uint64_t tot = 0;
  for (uint32_t l = 0; l < M; ++l) tot += models[m].lat_us[((size_t)k * M + l) * c->B + bi];
  return fail(c, PPIPE_ERANGE, "model %u class %u batch %u: whole-model latency %llu us >= 2^28 (int32 envelope)", m,
              k, c->h_batches[bi], (unsigned long long)tot);
}

// Segment bases, per-model SLOs and the kernel parameter block for c->last_params
// (shared by the (E, theta) path and F2).
static int setup_problem(ppipe_ctx* c, Problem* out) {
  const ppipe_enum_params* p = &c->last_params;
  // global segment bases (all models; same on every rank)
  std::vector<uint64_t> segbase(c->n_models);
  uint64_t acc = 0;
  for (uint32_t m = 0; m < c->n_models; ++m) {
    segbase[m] = acc;
    uint64_t pw = 1;
    for (uint32_t K = 1; K <= p->max_partitions && K <= c->Ms[m]; ++K) {
      pw *= c->C;
      acc += pw;
    }
  }
  c->n_seg_total = acc;
  c->h_segbase = segbase;
  c->h_segbase.push_back(acc);
  for (size_t i = 0; i < c->local.size(); ++i) c->h_models[i].slo_us = c->last_slo[c->local[i]];
  CU(c, cudaMemcpyAsync(c->d_segbase.p, segbase.data(), 8 * segbase.size(), cudaMemcpyHostToDevice, c->stream));
  CU(c, cudaMemcpyAsync(c->d_models.p, c->h_models.data(), sizeof(DevModel) * c->h_models.size(),
                        cudaMemcpyHostToDevice, c->stream));
  Problem pb{};
  pb.C = (int)c->C;
  pb.B = (int)c->B;
  pb.V = (int)c->V;
  pb.Kmax = (int)p->max_partitions;
  pb.margin = (int)p->margin_permille;
  pb.batches = c->d_batches.p;
  pb.bw_v = c->d_bwv.p;
  pb.pair_v = c->d_pairv.p;
  pb.wpack = c->wpack;
  pb.w_bits = c->w_bits;
  pb.models = c->d_models.p;
  pb.n_local = (int)c->local.size();
  pb.raw_lat = c->d_lat.p;
  pb.raw_s = c->d_s.p;
  pb.P = c->d_P.p;
  pb.Y = c->d_Y.p;
  pb.seg_base = c->d_segbase.p;
  pb.max_M = c->max_M;
  pb.neg_one = -1;
  {
    const char* dbg = getenv("PPIPE_DEBUG_FLAGS");
    pb.debug_flags = dbg ? atoi(dbg) : 0;
  }
  pb.model_base = 0;
  pb.n_chunk = pb.n_local;
  // per-tile minimum of A for the K = 3 early tile skip (ppipe_kernels.cu tile_mina_kernel)
  pb.max_tiles = (int)((c->max_M + 32 * kJ1 - 1) / (32 * kJ1)) + 1;
  const size_t mina_n = (size_t)std::max<size_t>(c->local.size(), 1) * c->C * c->B * pb.max_tiles;
  CU(c, c->d_minA.reserve(mina_n));
  pb.minA = c->d_minA.p;
  *out = pb;
  return PPIPE_OK;
}

// kernels launch_pack issues (pack_p, pack_y, and tile_mina for K = 3)
static int pack_launches(const Problem& pb) { return pb.n_chunk ? (pb.Kmax >= 3 && pb.minA ? 3 : 2) : 0; }

static int run_enumerate(ppipe_ctx* c) {
  CU(c, cudaSetDevice(c->device));
  Problem pb{};
  int rc = setup_problem(c, &pb);
  if (rc != PPIPE_OK) return rc;
  CU(c, c->d_surv.reserve(c->surv_cap));
  if (c->hot_cap == 0) {
    const uint64_t units = (uint64_t)c->local.size() * c->C * c->C * c->B;
    c->hot_cap = std::max<uint64_t>(1, std::min<uint64_t>(units, std::max<uint64_t>(4096, units / 8)));
  }
  const size_t tab_words = hot_unit_table_bytes(pb) / 8;
  CU(c, c->d_hot.reserve(c->hot_cap));
  CU(c, c->d_hot_tab.reserve(c->hot_cap * tab_words));
  CU(c, c->d_hot_order.reserve(c->hot_cap));
  CU(c, c->d_hot_w.reserve(c->hot_cap));
  if (pb.Kmax >= 3 && !getenv("PPIPE_NO_GFOLD")) {  // (the env switch is for measurements only)
    const size_t ng = gfold_elems(pb);
    CU(c, c->d_gfold.reserve(ng));
    CU(c, cudaMemsetAsync(c->d_gfold.p, 0, sizeof(unsigned long long) * ng, c->stream));
    pb.gfold = c->d_gfold.p;
  }
  ScoreOut so{c->d_surv.p, c->d_counters.p, (unsigned long long)c->d_surv.n, c->d_hot.p, c->d_hot_tab.p,
              (unsigned long long)c->hot_cap, getenv("PPIPE_NO_HOT_ORDER") ? nullptr : c->d_hot_order.p,
              c->d_hot_w.p};
  c->launches_i = 0;
  pb.model_base = 0;
  pb.n_chunk = pb.n_local;
  if (c->pending_upload && pb.n_local == 0) {
    // nothing of it lives on this rank; still take part in ppipe_pareto's error all-gather
    // (every rank issues the same collectives)
    c->pending_upload = false;
    CU(c, c->d_err.reserve(1));
    CU(c, cudaMemsetAsync(c->d_err.p, 0xff, 8, c->stream));
    c->check_err = true;
  }
  if (c->pending_upload) {
    // Chunked pipeline: chunk i is uploaded on the copy stream and, as soon as it lands,
    // packed (and validated, pb.err_key) and scored (score3a) on one of two compute streams
    // while chunk i + 1 uploads; score3b / score12 follow once. The first chunk is small
    // (the upload nobody overlaps) and so are the last ones (local models are heavy-first, so
    // the last bytes carry the least work). Launches for a chunk are issued right after its
    // copies, so the GPU starts scoring while the host still issues later chunks.
    CU(c, c->d_err.reserve(1));
    const unsigned long long none = ~0ull;
    CU(c, cudaMemcpyAsync(c->d_err.p, &none, 8, cudaMemcpyHostToDevice, c->stream));
    CU(c, cudaEventRecord(c->ev[0], c->stream));
    CU(c, cudaEventRecord(c->cev[ppipe_ctx::kMaxChunks], c->stream));  // earlier readers of the buffers
    CU(c, cudaStreamWaitEvent(c->cstream, c->cev[ppipe_ctx::kMaxChunks], 0));
    CU(c, cudaMemsetAsync(c->d_counters.p, 0, 16 * sizeof(unsigned long long), c->stream));
    CU(c, cudaEventRecord(c->sev[0], c->stream));  // fork: stream2 after the resets
    CU(c, cudaStreamWaitEvent(c->stream2, c->sev[0], 0));
    // chunk boundaries at cumulative byte fractions
    std::vector<uint64_t> cum(pb.n_local + 1, 0);
    for (int i = 0; i < pb.n_local; ++i)
      cum[i + 1] = cum[i] + sizeof(uint32_t) * (uint64_t)c->C * c->h_models[i].M * c->B + 8ull * c->h_models[i].M;
    // cumulative byte fractions (measured, config 5 e2e: 1/16, 1/4, 1/2, 1 -> 75.6 ms; these
    // 7 -> 72.5 ms: the copy engine finishes at ~22 ms, so the last chunks must be small
    // enough for their scoring to start before it ends)
    std::vector<double> frac = {0.05, 0.15, 0.3, 0.45, 0.6, 0.8, 1.0};
    if (const char* f = getenv("PPIPE_CHUNK_FRACS")) {  // measurements: "0.05,0.25,0.5" (then 1)
      frac.clear();
      for (const char* q = f; *q;) {
        char* end = nullptr;
        const double v = strtod(q, &end);
        if (end == q) break;
        if (v > 0 && v < 1 && (frac.empty() || v > frac.back())) frac.push_back(v);
        q = *end == ',' ? end + 1 : end;
      }
      frac.push_back(1.0);
      if ((int)frac.size() > ppipe_ctx::kMaxChunks) frac.erase(frac.begin() + (ppipe_ctx::kMaxChunks - 1), frac.end() - 1);
    }
    const int nfrac = (int)frac.size();
    std::vector<int> lo(1, 0);
    for (int k = 0; k < nfrac && lo.back() < pb.n_local; ++k) {
      int e = k == nfrac - 1 ? pb.n_local : (int)(std::lower_bound(cum.begin(), cum.end(), (uint64_t)(frac[k] * cum.back())) - cum.begin());
      e = std::max(e, lo.back() + 1);
      e = std::min(e, pb.n_local);
      lo.push_back(e);
    }
    const int nch = (int)lo.size() - 1;
    const uint64_t bmax = c->h_batches[c->B - 1];
    pb.err_key = c->d_err.p;
    pb.smax = (uint64_t)INT64_MAX / (8 * bmax);
    // PPIPE_DEBUG_FLAGS & 256: per-chunk upload / compute completion times on stderr
    const char* dbgs = getenv("PPIPE_DEBUG_FLAGS");
    const bool dbg_chunks = dbgs && (atoi(dbgs) & 256);
    static cudaEvent_t dev_up[ppipe_ctx::kMaxChunks], dev_done[ppipe_ctx::kMaxChunks];
    static bool dev_init = false;
    if (dbg_chunks && !dev_init) {
      for (int i = 0; i < ppipe_ctx::kMaxChunks; ++i) cudaEventCreate(&dev_up[i]), cudaEventCreate(&dev_done[i]);
      dev_init = true;
    }
    // Copies of consecutive local models whose host arrays are also adjacent are merged
    // (each copy costs a few microseconds of setup: 1,000 separate 785 KB copies reach
    // 43 GB/s, one copy 55 GB/s). Local models are ordered heavy-first, so for config 5
    // this merges little; the upload is not on the critical path there.
    struct Run {
      char* dst;
      const char* src;
      size_t n;
    };
    std::vector<Run> runs_lat, runs_s;
    auto add = [](std::vector<Run>& v, void* dst, const void* src, size_t n) {
      if (!v.empty() && v.back().dst + v.back().n == (char*)dst && v.back().src + v.back().n == (const char*)src)
        v.back().n += n;
      else
        v.push_back({(char*)dst, (const char*)src, n});
    };
    for (int ch = 0; ch < nch; ++ch) {
      runs_lat.clear();
      runs_s.clear();
      for (int i = lo[ch]; i < lo[ch + 1]; ++i) {
        const int m = c->local[i];
        const DevModel& d = c->h_models[i];
        add(runs_lat, c->d_lat.p + d.lat_off, c->pending[m].lat_us, sizeof(uint32_t) * c->C * d.M * c->B);
        add(runs_s, c->d_s.p + d.s_off, c->pending[m].act_bytes, sizeof(uint64_t) * d.M);
      }
      for (const auto* v : {&runs_s, &runs_lat})
        for (const Run& r : *v) CU(c, cudaMemcpyAsync(r.dst, r.src, r.n, cudaMemcpyHostToDevice, c->cstream));
      CU(c, cudaEventRecord(c->cev[ch], c->cstream));
      // chunks alternate between the two compute streams (independent models; every shared
      // output is appended through atomics), so one chunk's score3a tail overlaps the next
      const cudaStream_t cs = (ch & 1) ? c->stream2 : c->stream;
      CU(c, cudaStreamWaitEvent(cs, c->cev[ch], 0));
      pb.model_base = lo[ch];
      pb.n_chunk = lo[ch + 1] - lo[ch];
      // (validated inside the pack launch: pb.err_key)
      CU(c, launch_pack(pb, cs));
      CU(c, launch_score_part(pb, so, cs, &c->launches_i, 1));
      if (dbg_chunks) {
        cudaEventRecord(dev_up[ch], c->cstream);
        cudaEventRecord(dev_done[ch], cs);
      }
      c->launches_i += pack_launches(pb);
    }
    CU(c, cudaEventRecord(c->sev[1], c->stream2));  // join
    CU(c, cudaStreamWaitEvent(c->stream, c->sev[1], 0));
    CU(c, cudaEventRecord(c->ev[1], c->stream));  // phase 0 = upload + pack + score3a, interleaved
    if (dbg_chunks) {
      cudaEventSynchronize(c->ev[1]);
      for (int ch = 0; ch < nch; ++ch) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, c->ev[0], dev_up[ch]);
        cudaEventElapsedTime(&b, c->ev[0], dev_done[ch]);
        fprintf(stderr, "ppipe chunk %d (models %d..%d): uploaded at %.2f ms, scored at %.2f ms\n", ch, lo[ch],
                lo[ch + 1] - 1, a, b);
      }
    }
    pb.err_key = nullptr;
    pb.model_base = 0;
    pb.n_chunk = pb.n_local;
    CU(c, launch_score_part(pb, so, c->stream, &c->launches_i, 2));
    CU(c, cudaEventRecord(c->ev[2], c->stream));
    c->pending_upload = false;
    c->check_err = true;
    return PPIPE_OK;
  }
  CU(c, cudaEventRecord(c->ev[0], c->stream));
  CU(c, launch_pack(pb, c->stream));
  c->launches_i += pack_launches(pb);
  CU(c, cudaEventRecord(c->ev[1], c->stream));
  CU(c, cudaMemsetAsync(c->d_counters.p, 0, 16 * sizeof(unsigned long long), c->stream));
  CU(c, launch_score(pb, so, c->stream, &c->launches_i));
  CU(c, cudaEventRecord(c->ev[2], c->stream));
  return PPIPE_OK;
}

static int check_params(ppipe_ctx* ctx, const ppipe_enum_params* p, const char* who) {
  if (!p || !p->slo_us) return fail(ctx, PPIPE_EINVAL, "%s: NULL params or slo_us", who);
  if (p->max_partitions < 1 || p->max_partitions > 3)
    return fail(ctx, PPIPE_EINVAL, "max_partitions %u: must be 1..3", p->max_partitions);
  if (p->margin_permille >= 1000)
    return fail(ctx, PPIPE_EINVAL, "margin_permille %u: must be < 1000", p->margin_permille);
  if (!ctx->profiles_ok)
    return fail(ctx, PPIPE_ESTATE, "%s: the last ppipe_update_profiles failed; profiles are unusable", who);
  for (uint32_t m = 0; m < ctx->n_models; ++m) {
    const uint64_t T = (uint64_t)p->slo_us[m] * (1000 - p->margin_permille) / 1000;
    if (T >= (uint64_t)kRangeLimit)
      return fail(ctx, PPIPE_ERANGE, "model %u: T_eff %llu us >= 2^28 (int32 envelope)", m,
                  (unsigned long long)T);
    if (T * ctx->w_max >= (1ull << 31))
      return fail(ctx, PPIPE_ERANGE, "model %u: T_eff %llu us x virtual-GPU weight %u >= 2^31 (int32 envelope)", m,
                  (unsigned long long)T, ctx->w_max);
  }
  return PPIPE_OK;
}

PPIPE_API int ppipe_enumerate(ppipe_ctx* ctx, const ppipe_enum_params* p) {
  if (!ctx) return fail(nullptr, PPIPE_EINVAL, "ppipe_enumerate: NULL ctx");
  int rc0 = check_params(ctx, p, "ppipe_enumerate");
  if (rc0 != PPIPE_OK) return rc0;
  ctx->have_result = false;
  ctx->res_local = false;
  ctx->last_params = *p;
  ctx->last_slo.assign(p->slo_us, p->slo_us + ctx->n_models);
  ctx->last_params.slo_us = ctx->last_slo.data();
  ctx->enumerated = false;
  int rc = run_enumerate(ctx);
  if (rc == PPIPE_OK) ctx->enumerated = true;
  return rc;
}

// ---- frontier merge ----
// Per rank: [n_points, n_cand, n_feas, n_surv, first model + 1, last model + 1, points of
// the first model, points of the last model] of its local frontier (0 models: 0, 0).
constexpr int kMergeCnt = 8;

static int local_counters(ppipe_ctx* c, uint64_t n_local_pts, uint64_t n_cand, uint64_t n_feas, uint64_t n_surv,
                          uint64_t out[kMergeCnt]) {
  int mf = -1, ml = -1;
  for (int m : c->local) {
    mf = mf < 0 ? m : std::min(mf, m);
    ml = std::max(ml, m);
  }
  uint64_t nfirst = 0, nlast = 0;
  if (mf >= 0) {
    uint64_t b[4];
    const uint64_t at[4] = {c->h_segbase[mf], c->h_segbase[mf + 1], c->h_segbase[ml], c->h_segbase[ml + 1]};
    for (int i = 0; i < 4; ++i)
      CU(c, cudaMemcpyAsync(&b[i], c->d_segoff_local.p + at[i], 8, cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    nfirst = b[1] - b[0];
    nlast = b[3] - b[2];
  }
  const uint64_t hs[kMergeCnt] = {n_local_pts, n_cand, n_feas, n_surv, (uint64_t)(mf + 1), (uint64_t)(ml + 1),
                                  nfirst, nlast};
  std::memcpy(out, hs, sizeof hs);
  return PPIPE_OK;
}

// Every model lies on one rank except the <= world - 1 models at range boundaries, and
// each rank's local frontier is in canonical order, so the global frontier is the
// rank-ordered concatenation of the local ones with only the straddling models' points
// re-reduced (decomposability: F(A u B) = F(F(A) u F(B))). Input: every rank's counters
// (cnts, kMergeCnt per rank) and its local frontier at d_gather + r * maxc. Output:
// d_final / d_segoff_final of c, *n_pts; *n_cand / *n_feas summed over the ranks.
static int merge_assemble(ppipe_ctx* c, const std::vector<uint64_t>& cnts, uint64_t maxc, int* nl, uint64_t* n_cand,
                          uint64_t* n_feas, uint64_t* n_pts) {
  uint64_t tot = 0;
  *n_cand = *n_feas = 0;
  for (int r = 0; r < c->world; ++r) {
    tot += cnts[kMergeCnt * r];
    *n_cand += cnts[kMergeCnt * r + 1];
    *n_feas += cnts[kMergeCnt * r + 2];
  }
  // pieces in rank order: (model or -1 for a run of whole models, source, count)
  struct Piece {
    long long model;
    uint64_t src, n;
  };
  std::vector<Piece> pieces;
  for (int r = 0; r < c->world; ++r) {
    const uint64_t* q = &cnts[kMergeCnt * (size_t)r];
    if (q[4] == 0) continue;  // no rows on rank r
    const long long f = (long long)q[4] - 1, l = (long long)q[5] - 1;
    const uint64_t base = (uint64_t)r * maxc, n = q[0];
    if (f == l) {
      pieces.push_back({f, base, n});
    } else {
      pieces.push_back({f, base, q[6]});
      pieces.push_back({-1, base + q[6], n - q[6] - q[7]});
      pieces.push_back({l, base + n - q[7], q[7]});
    }
  }
  // a model with pieces from two or more ranks straddles: re-reduce its points
  std::vector<char> dirty(pieces.size(), 0);
  std::vector<long long> straddle;
  for (size_t i = 0; i < pieces.size(); ++i)
    for (size_t k = i + 1; k < pieces.size() && pieces[k].model == pieces[i].model && pieces[i].model >= 0; ++k) {
      dirty[i] = dirty[k] = 1;
      if (straddle.empty() || straddle.back() != pieces[i].model) straddle.push_back(pieces[i].model);
    }
  uint64_t n_dirty = 0;
  for (size_t i = 0; i < pieces.size(); ++i)
    if (dirty[i]) n_dirty += pieces[i].n;
  CU(c, c->d_union.reserve(std::max<uint64_t>(n_dirty, 1)));
  uint64_t off = 0;
  for (size_t i = 0; i < pieces.size(); ++i)
    if (dirty[i] && pieces[i].n) {
      CU(c, cudaMemcpyAsync(c->d_union.p + off, c->d_gather.p + pieces[i].src, sizeof(ppipe_point) * pieces[i].n,
                            cudaMemcpyDeviceToDevice, c->stream));
      off += pieces[i].n;
    }
  CU(c, c->d_final.reserve(std::max<uint64_t>(tot, 1)));
  CU(c, c->d_segoff_final.reserve(c->n_seg_total + 1));
  CU(c, c->d_merged.reserve(std::max<uint64_t>(n_dirty, 1)));
  uint64_t n_merged = 0;
  std::vector<uint64_t> mcount(straddle.size(), 0);
  const char* dbgs_ = getenv("PPIPE_DEBUG_FLAGS");
  const bool mdbg = dbgs_ && (atoi(dbgs_) & 32);
  cudaEvent_t aev[4] = {};
  if (mdbg) {
    for (auto& x : aev) cudaEventCreate(&x);
    cudaEventRecord(aev[0], c->stream);
  }
  if (n_dirty) {
    CU(c, frontier_pass(c->d_union.p, n_dirty, c->d_segbase.p, (int)c->C, c->n_seg_total, c->d_merged.p,
                        c->d_segoff_final.p, &n_merged, &c->scratch, c->stream, nl, c->wpack));
    std::vector<uint64_t> b(2 * straddle.size());
    for (size_t i = 0; i < straddle.size(); ++i) {
      CU(c, cudaMemcpyAsync(&b[2 * i], c->d_segoff_final.p + c->h_segbase[straddle[i]], 8, cudaMemcpyDeviceToHost,
                            c->stream));
      CU(c, cudaMemcpyAsync(&b[2 * i + 1], c->d_segoff_final.p + c->h_segbase[straddle[i] + 1], 8,
                            cudaMemcpyDeviceToHost, c->stream));
    }
    CU(c, cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < straddle.size(); ++i) mcount[i] = b[2 * i + 1] - b[2 * i];
  }
  if (mdbg) cudaEventRecord(aev[1], c->stream);
  // assemble in order: clean pieces from the gathered frontiers, each straddling
  // model's merged block in place of its first piece
  uint64_t w = 0, moff = 0;
  size_t si = 0;
  for (size_t i = 0; i < pieces.size(); ++i) {
    const ppipe_point* src = c->d_gather.p + pieces[i].src;
    uint64_t n = pieces[i].n;
    if (dirty[i]) {
      if (i > 0 && dirty[i - 1] && pieces[i - 1].model == pieces[i].model) continue;
      src = c->d_merged.p + moff;
      n = mcount[si];
      moff += n;
      ++si;
    }
    if (n) CU(c, cudaMemcpyAsync(c->d_final.p + w, src, sizeof(ppipe_point) * n, cudaMemcpyDeviceToDevice, c->stream));
    w += n;
  }
  *n_pts = w;
  if (mdbg) cudaEventRecord(aev[2], c->stream);
  CU(c, c->d_segtmp.reserve(std::max<uint64_t>(w, 1)));
  CU(c, segment_offsets(c->d_final.p, w, c->d_segbase.p, (int)c->C, c->n_seg_total, c->d_segoff_final.p,
                        c->d_segtmp.p, c->stream, nl));
  if (mdbg) {
    cudaEventRecord(aev[3], c->stream);
    cudaEventSynchronize(aev[3]);
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, aev[0], aev[1]);
    cudaEventElapsedTime(&b, aev[1], aev[2]);
    cudaEventElapsedTime(&d, aev[2], aev[3]);
    fprintf(stderr, "ppipe assemble rank %d: straddlers (%llu records) %.3f ms, concat %.3f ms, offsets %.3f ms\n",
            c->rank, (unsigned long long)n_dirty, a, b, d);
    for (auto& x : aev) cudaEventDestroy(x);
  }
  return PPIPE_OK;
}

PPIPE_API int ppipe_pareto(ppipe_ctx* c, int copy_to_host, ppipe_frontier* out) {
  if (!c) return fail(nullptr, PPIPE_EINVAL, "ppipe_pareto: NULL ctx");
  if (!out) return fail(c, PPIPE_EINVAL, "ppipe_pareto: NULL output");
  if (!c->enumerated) return fail(c, PPIPE_ESTATE, "ppipe_pareto called before ppipe_enumerate");
  CU(c, cudaSetDevice(c->device));
  if (c->check_err) {  // values uploaded by ppipe_update_profiles_async were validated on the device
    c->check_err = false;
    unsigned long long key = ~0ull;
    if (c->world > 1 && c->comm) {  // every rank fails alike
      CU(c, c->d_cnt_recv.reserve((size_t)c->world));
      NC_(c, g_nccl.AllGather(c->d_err.p, c->d_cnt_recv.p, 1, ncclUint64, c->comm, c->stream));
      std::vector<unsigned long long> keys(c->world);
      CU(c, cudaMemcpyAsync(keys.data(), c->d_cnt_recv.p, 8 * keys.size(), cudaMemcpyDeviceToHost, c->stream));
      CU(c, cudaStreamSynchronize(c->stream));
      for (auto k : keys) key = std::min(key, k);
    } else {
      CU(c, cudaMemcpyAsync(&key, c->d_err.p, 8, cudaMemcpyDeviceToHost, c->stream));
      CU(c, cudaStreamSynchronize(c->stream));
    }
    if (key != ~0ull) {
      c->profiles_ok = false;
      c->enumerated = false;
      return report_validation(c, key, c->pending.data());
    }
  }
  // survivors; grow and re-run on overflow (deterministic, so the result is unchanged)
  for (;;) {
    CU(c, cudaMemcpyAsync(c->h_counters, c->d_counters.p, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    const bool surv_ok = c->h_counters[0] <= c->d_surv.n;
    const bool hot_ok = c->h_counters[3] <= c->hot_cap;
    if (surv_ok && hot_ok) break;
    if (!surv_ok) c->surv_cap = c->h_counters[0] + c->h_counters[0] / 4 + 1024;
    if (!hot_ok) c->hot_cap = c->h_counters[3] + c->h_counters[3] / 4 + 64;
    int rc = run_enumerate(c);
    if (rc != PPIPE_OK) return rc;
  }
  const uint64_t n_surv = c->h_counters[0];
  if (const char* dbg = getenv("PPIPE_DEBUG_FLAGS"))
    if (atoi(dbg) & 8)
      fprintf(stderr, "ppipe debug: hot units %llu, pass-2 tiles %llu, visits %llu, slot-hits %llu, emit-calls %llu, "
              "survivors %llu, feasible %llu\n", c->h_counters[3], c->h_counters[7], c->h_counters[5],
              c->h_counters[6], c->h_counters[8], c->h_counters[0], c->h_counters[1]);
  uint64_t n_feas = c->h_counters[1], n_cand = c->h_counters[2];
  int nl = c->launches_i;
  // local frontier
  CU(c, c->d_local.reserve(std::max<uint64_t>(n_surv, 1)));
  CU(c, c->d_segoff_local.reserve(c->n_seg_total + 1));
  uint64_t n_local_pts = 0;
  CU(c, frontier_pass(c->d_surv.p, n_surv, c->d_segbase.p, (int)c->C, c->n_seg_total, c->d_local.p,
                      c->d_segoff_local.p, &n_local_pts, &c->scratch, c->stream, &nl, c->wpack));
  CU(c, cudaEventRecord(c->ev[3], c->stream));
  const ppipe_point* d_pts = c->d_local.p;
  const uint64_t* d_off = c->d_segoff_local.p;
  uint64_t n_pts = n_local_pts;
  if (c->world > 1 && c->comm) {
    // The only multi-GPU-specific step: all-gather every rank's counters and its padded
    // local frontier over NCCL into d_gather; merge_assemble (shared with the one-GPU
    // ppipe_merge_shards) does the rest.
    uint64_t hs[kMergeCnt];
    int rc = local_counters(c, n_local_pts, n_cand, n_feas, n_surv, hs);
    if (rc != PPIPE_OK) return rc;
    CU(c, c->d_cnt_send.reserve(kMergeCnt));
    CU(c, c->d_cnt_recv.reserve(kMergeCnt * (size_t)c->world));
    CU(c, cudaMemcpyAsync(c->d_cnt_send.p, hs, sizeof hs, cudaMemcpyHostToDevice, c->stream));
    NC_(c, g_nccl.AllGather(c->d_cnt_send.p, c->d_cnt_recv.p, kMergeCnt, ncclUint64, c->comm, c->stream));
    std::vector<uint64_t> cnts(kMergeCnt * (size_t)c->world);
    CU(c, cudaMemcpyAsync(cnts.data(), c->d_cnt_recv.p, 8 * cnts.size(), cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    uint64_t maxc = 1;
    for (int r = 0; r < c->world; ++r) maxc = std::max(maxc, cnts[kMergeCnt * r]);
    // padded all-gather of local frontiers (32-byte records as bytes)
    if (c->d_local.n < maxc) {
      DevBuf<ppipe_point> tmp;
      CU(c, tmp.reserve(maxc));
      CU(c, cudaMemcpyAsync(tmp.p, c->d_local.p, sizeof(ppipe_point) * n_local_pts, cudaMemcpyDeviceToDevice,
                            c->stream));
      CU(c, cudaStreamSynchronize(c->stream));
      c->d_local.release();
      c->d_local = tmp;
    }
    CU(c, c->d_gather.reserve(maxc * c->world));
    NC_(c, g_nccl.AllGather(c->d_local.p, c->d_gather.p, maxc * sizeof(ppipe_point), ncclUint8, c->comm,
                            c->stream));
    nl += 2;  // the two all-gathers
    const char* dbgs = getenv("PPIPE_DEBUG_FLAGS");
    const bool dbg = dbgs && (atoi(dbgs) & 32);
    cudaEvent_t mev[2] = {};
    if (dbg) {
      for (auto& x : mev) cudaEventCreate(&x);
      cudaEventRecord(mev[0], c->stream);
    }
    rc = merge_assemble(c, cnts, maxc, &nl, &n_cand, &n_feas, &n_pts);
    if (rc != PPIPE_OK) return rc;
    if (dbg) {
      cudaEventRecord(mev[1], c->stream);
      cudaEventSynchronize(mev[1]);
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, c->ev[3], mev[0]);
      cudaEventElapsedTime(&b, mev[0], mev[1]);
      fprintf(stderr, "ppipe merge rank %d: counters + all-gathers %.3f ms, assemble %.3f ms (maxc %llu)\n", c->rank,
              a, b, (unsigned long long)maxc);
      for (auto& x : mev) cudaEventDestroy(x);
    }
    d_pts = c->d_final.p;
    d_off = c->d_segoff_final.p;
  }
  CU(c, cudaEventRecord(c->ev[4], c->stream));
  CU(c, cudaEventSynchronize(c->ev[4]));
  cudaEventElapsedTime(&c->phase_ms[0], c->ev[0], c->ev[1]);
  cudaEventElapsedTime(&c->phase_ms[1], c->ev[1], c->ev[2]);
  cudaEventElapsedTime(&c->phase_ms[2], c->ev[2], c->ev[3]);
  cudaEventElapsedTime(&c->phase_ms[3], c->ev[3], c->ev[4]);
  c->launches = (uint64_t)nl;
  std::memset(out, 0, sizeof *out);
  out->n_candidates = n_cand;
  out->n_feasible = n_feas;
  out->n_points = n_pts;
  out->n_segments = c->n_seg_total;
  out->d_points = d_pts;
  out->d_seg_offsets = d_off;
  out->n_survivors = n_surv;
  out->n_candidates_local = c->h_counters[2];
  out->n_feasible_local = c->h_counters[1];
  c->have_result = true;
  c->res_pts = d_pts;
  c->res_off = d_off;
  c->res_n = n_pts;
  c->res_ncand = n_cand;
  c->res_nfeas = n_feas;
  c->res_nsurv = n_surv;
  c->res_local = !(c->world > 1 && c->comm);  // a shard's local frontier (ppipe_merge_shards input)
  if (copy_to_host) {
    CU(c, c->h_points.reserve(n_pts));
    CU(c, c->h_segoff.reserve(c->n_seg_total + 1));
    if (n_pts)
      CU(c, cudaMemcpyAsync(c->h_points.p, d_pts, sizeof(ppipe_point) * n_pts, cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaMemcpyAsync(c->h_segoff.p, d_off, 8 * (c->n_seg_total + 1), cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    out->points = c->h_points.p;
    out->seg_offsets = c->h_segoff.p;
  }
  return PPIPE_OK;
}

// F2: the MILP-lossless frontier (include/ppipe.h; ppipe_f2.cu). Every model is
// scored whole by the rank that holds its row 0 (its K = 1 row), so each rank's
// frontier is final for its models and the global one is the rank-ordered
// concatenation.
static_assert(sizeof(ppipe_point_pb) == sizeof(ppipe_point) && offsetof(ppipe_point_pb, K) == offsetof(ppipe_point, K) &&
                  offsetof(ppipe_point_pb, cls) == offsetof(ppipe_point, cls),
              "per-stage-batch records share the point buffers and the segment-offset kernels");

// Models owned by this rank for the whole-model paths (F2, per-stage batch): the rank
// holding a model's row 0 (its K = 1 row) scores all of it.
static int owned_models(ppipe_ctx* c, std::vector<int>* own, const char* who) {
  own->clear();
  for (size_t i = 0; i < c->local.size(); ++i)
    if (c->h_models[i].row_lo == 0 && c->h_models[i].row_hi > 0) own->push_back((int)i);
  (void)who;
  return PPIPE_OK;
}

// Candidate count of the owned models: sum_K C(M-1, K-1) * C^K * B^(K if per_stage else 1).
static uint64_t owned_candidates(ppipe_ctx* c, const std::vector<int>& own, int Kmax, bool per_stage) {
  uint64_t n = 0;
  for (int i : own) {
    const uint32_t M = c->h_models[i].M;
    uint64_t pw = 1, bw = 1, comb = 1;
    for (uint32_t K = 1; K <= (uint32_t)Kmax && K <= M; ++K) {
      pw *= c->C;
      bw = per_stage ? bw * c->B : c->B;
      n += comb * pw * bw;
      comb = comb * (M - K) / K;
    }
  }
  return n;
}

// Whole-model paths under NCCL: every rank's points (32-byte records in canonical
// order, owned models only) are final, so the global result is their rank-ordered
// concatenation (counts all-gather + one padded all-gather), then the CSR.
static int concat_owned(ppipe_ctx* c, uint64_t* n_pts, uint64_t n_cand, uint64_t n_feas_local, uint64_t* n_cand_all,
                        uint64_t* n_feas_all, const ppipe_point** d_pts, const uint64_t** d_off, int* nl) {
  *d_pts = c->d_local.p;
  *d_off = c->d_segoff_local.p;
  *n_cand_all = n_cand;
  *n_feas_all = n_feas_local;
  if (!(c->world > 1 && c->comm)) return PPIPE_OK;
  constexpr int kCnt = 3;
  CU(c, c->d_cnt_send.reserve(kCnt));
  CU(c, c->d_cnt_recv.reserve(kCnt * (size_t)c->world));
  uint64_t hs[kCnt] = {*n_pts, n_cand, n_feas_local};
  CU(c, cudaMemcpyAsync(c->d_cnt_send.p, hs, sizeof hs, cudaMemcpyHostToDevice, c->stream));
  NC_(c, g_nccl.AllGather(c->d_cnt_send.p, c->d_cnt_recv.p, kCnt, ncclUint64, c->comm, c->stream));
  std::vector<uint64_t> cnts(kCnt * (size_t)c->world);
  CU(c, cudaMemcpyAsync(cnts.data(), c->d_cnt_recv.p, 8 * cnts.size(), cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  uint64_t maxc = 1, tot = 0;
  *n_cand_all = *n_feas_all = 0;
  for (int r = 0; r < c->world; ++r) {
    maxc = std::max(maxc, cnts[kCnt * r]);
    tot += cnts[kCnt * r];
    *n_cand_all += cnts[kCnt * r + 1];
    *n_feas_all += cnts[kCnt * r + 2];
  }
  if (c->d_local.n < maxc) {
    DevBuf<ppipe_point> tmp;
    CU(c, tmp.reserve(maxc));
    if (*n_pts)
      CU(c, cudaMemcpyAsync(tmp.p, c->d_local.p, sizeof(ppipe_point) * *n_pts, cudaMemcpyDeviceToDevice, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    c->d_local.release();
    c->d_local = tmp;
  }
  CU(c, c->d_gather.reserve(maxc * c->world));
  NC_(c, g_nccl.AllGather(c->d_local.p, c->d_gather.p, maxc * sizeof(ppipe_point), ncclUint8, c->comm, c->stream));
  CU(c, c->d_final.reserve(std::max<uint64_t>(tot, 1)));
  uint64_t w = 0;
  for (int r = 0; r < c->world; ++r) {
    const uint64_t n = cnts[kCnt * r];
    if (n)
      CU(c, cudaMemcpyAsync(c->d_final.p + w, c->d_gather.p + (uint64_t)r * maxc, sizeof(ppipe_point) * n,
                            cudaMemcpyDeviceToDevice, c->stream));
    w += n;
  }
  *n_pts = w;
  CU(c, c->d_segoff_final.reserve(c->n_seg_total + 1));
  CU(c, c->d_segtmp.reserve(std::max<uint64_t>(w, 1)));
  CU(c, segment_offsets(c->d_final.p, w, c->d_segbase.p, (int)c->C, c->n_seg_total, c->d_segoff_final.p,
                        c->d_segtmp.p, c->stream, nl));
  *nl += 2;
  *d_pts = c->d_final.p;
  *d_off = c->d_segoff_final.p;
  return PPIPE_OK;
}

// Phase times, launch count and the optional host copy (into the page-locked buffers)
// of a whole-model path's result.
static int publish_owned(ppipe_ctx* c, int nl, const ppipe_point* d_pts, const uint64_t* d_off, uint64_t n_pts,
                         int copy_to_host, const ppipe_point** h_pts, const uint64_t** h_off) {
  CU(c, cudaEventRecord(c->ev[4], c->stream));
  CU(c, cudaEventSynchronize(c->ev[4]));
  cudaEventElapsedTime(&c->phase_ms[0], c->ev[0], c->ev[1]);
  cudaEventElapsedTime(&c->phase_ms[1], c->ev[1], c->ev[2]);
  cudaEventElapsedTime(&c->phase_ms[2], c->ev[2], c->ev[3]);
  cudaEventElapsedTime(&c->phase_ms[3], c->ev[3], c->ev[4]);
  c->launches = (uint64_t)nl;
  *h_pts = nullptr;
  *h_off = nullptr;
  if (copy_to_host) {
    CU(c, c->h_points.reserve(n_pts));
    CU(c, c->h_segoff.reserve(c->n_seg_total + 1));
    if (n_pts)
      CU(c, cudaMemcpyAsync(c->h_points.p, d_pts, sizeof(ppipe_point) * n_pts, cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaMemcpyAsync(c->h_segoff.p, d_off, 8 * (c->n_seg_total + 1), cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    *h_pts = c->h_points.p;
    *h_off = c->h_segoff.p;
  }
  return PPIPE_OK;
}

PPIPE_API int ppipe_merge_shards(ppipe_ctx* const* shards, int n_shards, int copy_to_host, ppipe_frontier* out) {
  if (!shards || n_shards < 1 || !out) return fail(nullptr, PPIPE_EINVAL, "ppipe_merge_shards: NULL argument");
  ppipe_ctx* c = shards[0];
  if (!c) return fail(nullptr, PPIPE_EINVAL, "ppipe_merge_shards: shard 0 is NULL");
  for (int r = 0; r < n_shards; ++r) {
    const ppipe_ctx* x = shards[r];
    if (!x) return fail(c, PPIPE_EINVAL, "ppipe_merge_shards: shard %d is NULL", r);
    if (x->world != n_shards || x->rank != r || x->comm)
      return fail(c, PPIPE_EINVAL, "ppipe_merge_shards: shard %d is rank %d of %d%s; expected rank %d of %d in shard mode",
                  r, x->rank, x->world, x->comm ? " with NCCL" : "", r, n_shards);
    if (x->device != c->device || x->n_models != c->n_models || x->C != c->C || x->B != c->B || x->Ms != c->Ms)
      return fail(c, PPIPE_EINVAL, "ppipe_merge_shards: shard %d was loaded with another device or workload shape", r);
    if (!x->have_result || !x->res_local)
      return fail(c, PPIPE_ESTATE, "ppipe_merge_shards: shard %d has no local ppipe_pareto result", r);
    if (x->last_params.max_partitions != c->last_params.max_partitions ||
        x->last_params.margin_permille != c->last_params.margin_permille || x->last_slo != c->last_slo ||
        x->wpack != c->wpack)
      return fail(c, PPIPE_EINVAL, "ppipe_merge_shards: shard %d was enumerated with other parameters", r);
  }
  CU(c, cudaSetDevice(c->device));
  int nl = 0;
  CU(c, cudaEventRecord(c->ev[3], c->stream));
  // the same inputs the NCCL path all-gathers: every shard's counters and its local
  // frontier, padded to the largest, at d_gather + r * maxc
  std::vector<uint64_t> cnts(kMergeCnt * (size_t)n_shards);
  uint64_t maxc = 1;
  for (int r = 0; r < n_shards; ++r) {
    ppipe_ctx* x = shards[r];
    int rc = local_counters(x, x->res_n, x->res_ncand, x->res_nfeas, x->res_nsurv, &cnts[kMergeCnt * (size_t)r]);
    if (rc != PPIPE_OK) return fail(c, rc, "shard %d: %s", r, x->err.c_str());
    maxc = std::max(maxc, x->res_n);
  }
  CU(c, c->d_gather.reserve(maxc * n_shards));
  for (int r = 0; r < n_shards; ++r)
    if (shards[r]->res_n)
      CU(c, cudaMemcpyAsync(c->d_gather.p + (size_t)r * maxc, shards[r]->res_pts, sizeof(ppipe_point) * shards[r]->res_n,
                            cudaMemcpyDeviceToDevice, c->stream));
  uint64_t n_cand = 0, n_feas = 0, n_pts = 0;
  int rc = merge_assemble(c, cnts, maxc, &nl, &n_cand, &n_feas, &n_pts);
  if (rc != PPIPE_OK) return rc;
  CU(c, cudaEventRecord(c->ev[4], c->stream));
  CU(c, cudaEventSynchronize(c->ev[4]));
  cudaEventElapsedTime(&c->phase_ms[3], c->ev[3], c->ev[4]);
  c->launches = (uint64_t)nl;
  std::memset(out, 0, sizeof *out);
  out->n_candidates = n_cand;
  out->n_feasible = n_feas;
  out->n_points = n_pts;
  out->n_segments = c->n_seg_total;
  out->d_points = c->d_final.p;
  out->d_seg_offsets = c->d_segoff_final.p;
  out->n_survivors = c->res_nsurv;
  out->n_candidates_local = c->res_ncand;
  out->n_feasible_local = c->res_nfeas;
  c->have_result = true;
  c->res_local = false;  // now the merged frontier
  c->res_pts = c->d_final.p;
  c->res_off = c->d_segoff_final.p;
  c->res_n = n_pts;
  c->res_ncand = n_cand;
  c->res_nfeas = n_feas;
  if (copy_to_host) {
    CU(c, c->h_points.reserve(n_pts));
    CU(c, c->h_segoff.reserve(c->n_seg_total + 1));
    if (n_pts)
      CU(c, cudaMemcpyAsync(c->h_points.p, c->d_final.p, sizeof(ppipe_point) * n_pts, cudaMemcpyDeviceToHost,
                            c->stream));
    CU(c, cudaMemcpyAsync(c->h_segoff.p, c->d_segoff_final.p, 8 * (c->n_seg_total + 1), cudaMemcpyDeviceToHost,
                          c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    out->points = c->h_points.p;
    out->seg_offsets = c->h_segoff.p;
  }
  return PPIPE_OK;
}

// Shared prologue of the whole-model paths: parameter checks, owned models, problem setup.
static int whole_model_setup(ppipe_ctx* c, const ppipe_enum_params* p, const char* who, std::vector<int>* own,
                             Problem* pb) {
  int rc = check_params(c, p, who);
  if (rc != PPIPE_OK) return rc;
  if (c->pending_upload)
    return fail(c, PPIPE_ESTATE, "%s: profiles from ppipe_update_profiles_async are uploaded by ppipe_enumerate only; "
                                 "use ppipe_update_profiles", who);
  owned_models(c, own, who);
  CU(c, cudaSetDevice(c->device));
  c->have_result = false;
  c->res_local = false;
  c->enumerated = false;
  c->last_params = *p;
  c->last_slo.assign(p->slo_us, p->slo_us + c->n_models);
  c->last_params.slo_us = c->last_slo.data();
  return setup_problem(c, pb);
}

PPIPE_API int ppipe_pareto_f2(ppipe_ctx* c, const ppipe_enum_params* p, int copy_to_host, ppipe_frontier* out) {
  if (!c) return fail(nullptr, PPIPE_EINVAL, "ppipe_pareto_f2: NULL ctx");
  if (!out) return fail(c, PPIPE_EINVAL, "ppipe_pareto_f2: NULL output");
  std::vector<int> own;
  if (p)
    for (size_t i = 0; i < c->local.size(); ++i)
      if (c->h_models[i].row_lo == 0 && c->h_models[i].M > kF2MaxLayers)
        return fail(c, PPIPE_ERANGE, "model %d: %u layers; F2 supports at most %u", c->local[i], c->h_models[i].M,
                    kF2MaxLayers);
  Problem pb{};
  int rc = whole_model_setup(c, p, "ppipe_pareto_f2", &own, &pb);
  if (rc != PPIPE_OK) return rc;
  if (c->n_seg_total >= (1ull << 28)) return fail(c, PPIPE_ERANGE, "F2: %llu segments >= 2^28",
                                                  (unsigned long long)c->n_seg_total);
  const int Kmax = (int)p->max_partitions;
  // G: all C^3 segments of the largest model, capped at PPIPE_F2_G_BYTES (default 8 GiB), at least one segment
  size_t g_need = 0, f_need = 1;
  for (int i : own) {
    const uint32_t M = c->h_models[i].M;
    g_need = std::max(g_need, f2_g3_elems_per_segment((int)c->B, M) * c->C * c->C * c->C);
    f_need = std::max<size_t>(f_need, (size_t)c->C * c->C * c->B * M);
  }
  const uint64_t n_cand = owned_candidates(c, own, Kmax, false);
  size_t g_budget = 8ull << 30;
  if (const char* gb = getenv("PPIPE_F2_G_BYTES")) g_budget = (size_t)strtoull(gb, nullptr, 10);
  size_t g_cap = std::min(g_need, g_budget / sizeof(int32_t));
  for (int i : own) g_cap = std::max(g_cap, f2_g3_elems_per_segment((int)c->B, c->h_models[i].M));
  if (Kmax >= 3) CU(c, c->d_G.reserve(std::max<size_t>(g_cap, 1)));
  if (Kmax >= 2) CU(c, c->d_F.reserve(f_need));
  if (Kmax >= 3) CU(c, c->d_E23.reserve(2 * f_need));
  const size_t inv_n = f_need / c->C * ((c->B + 3) & ~3u);  // C * B * 4 ceil(B / 4) * max M
  if (Kmax >= 2) CU(c, c->d_inv.reserve(4 * inv_n));
  const int q3_grid = f2_q3_grid(c->device);
  int nl = 0;
  for (int attempt = 0;; ++attempt) {
    CU(c, c->d_f2surv.reserve(c->f2_cap));
    F2Out fo{c->d_f2surv.p, c->d_counters.p, (unsigned long long)c->d_f2surv.n, c->d_G.p, c->d_G.n, c->d_F.p,
             c->d_inv.p, c->d_inv.p + inv_n, c->d_inv.p + 2 * inv_n, c->d_inv.p + 3 * inv_n, c->d_E23.p,
             q3_grid};
    nl = 0;
    CU(c, cudaEventRecord(c->ev[0], c->stream));
    CU(c, launch_pack(pb, c->stream));
    nl += pack_launches(pb);
    CU(c, cudaEventRecord(c->ev[1], c->stream));
    CU(c, cudaMemsetAsync(c->d_counters.p, 0, 16 * sizeof(unsigned long long), c->stream));
    for (int i : own) CU(c, launch_f2_model(pb, i, c->h_models[i].M, Kmax, fo, c->stream, &nl));
    CU(c, cudaEventRecord(c->ev[2], c->stream));
    CU(c, cudaMemcpyAsync(c->h_counters, c->d_counters.p, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    if (c->h_counters[0] <= c->d_f2surv.n) break;
    c->f2_cap = c->h_counters[0] + c->h_counters[0] / 4 + 1024;  // deterministic: re-run with room
  }
  const uint64_t n_surv = c->h_counters[0], n_feas_local = c->h_counters[1];
  CU(c, c->d_f2tmp.reserve(std::max<uint64_t>(n_surv, 1)));
  CU(c, c->d_local.reserve(std::max<uint64_t>(n_surv, 1)));
  CU(c, c->d_segoff_local.reserve(c->n_seg_total + 1));
  CU(c, c->d_segtmp.reserve(std::max<uint64_t>(n_surv, 2)));  // f2_finalize keeps two cursors there
  uint64_t n_pts = 0;
  CU(c, f2_finalize(c->d_f2surv.p, n_surv, c->d_segbase.p, (int)c->C, c->n_seg_total, c->d_local.p, c->d_f2tmp.p,
                    c->d_segoff_local.p, c->d_segtmp.p, &n_pts, &c->scratch, c->stream, &nl));
  CU(c, cudaEventRecord(c->ev[3], c->stream));
  const ppipe_point* d_pts = nullptr;
  const uint64_t* d_off = nullptr;
  uint64_t n_cand_all = 0, n_feas_all = 0;
  if ((rc = concat_owned(c, &n_pts, n_cand, n_feas_local, &n_cand_all, &n_feas_all, &d_pts, &d_off, &nl)) != PPIPE_OK)
    return rc;
  std::memset(out, 0, sizeof *out);
  if ((rc = publish_owned(c, nl, d_pts, d_off, n_pts, copy_to_host, &out->points, &out->seg_offsets)) != PPIPE_OK)
    return rc;
  out->n_candidates = n_cand_all;
  out->n_feasible = n_feas_all;
  out->n_points = n_pts;
  out->n_segments = c->n_seg_total;
  out->d_points = d_pts;
  out->d_seg_offsets = d_off;
  out->n_survivors = n_surv;
  out->n_candidates_local = n_cand;
  out->n_feasible_local = n_feas_local;
  return PPIPE_OK;
}

PPIPE_API int ppipe_pareto_pb(ppipe_ctx* c, const ppipe_enum_params* p, int copy_to_host, ppipe_frontier_pb* out) {
  if (!c) return fail(nullptr, PPIPE_EINVAL, "ppipe_pareto_pb: NULL ctx");
  if (!out) return fail(c, PPIPE_EINVAL, "ppipe_pareto_pb: NULL output");
  if (c->B > 255) return fail(c, PPIPE_ERANGE, "ppipe_pareto_pb: %u batch sizes; at most 255", c->B);
  std::vector<int> own;
  Problem pb{};
  int rc = whole_model_setup(c, p, "ppipe_pareto_pb", &own, &pb);
  if (rc != PPIPE_OK) return rc;
  const int Kmax = (int)p->max_partitions;
  const uint64_t n_cand = owned_candidates(c, own, Kmax, true);
  // suffix-minimum rows for the K = 3 unit bound, when they fit in 2 GiB
  uint32_t maxM = 0;
  for (int i : own) maxM = std::max(maxM, c->h_models[i].M);
  const size_t sd_n = (size_t)c->C * c->C * c->B * c->B * maxM;
  int32_t* sd = nullptr;
  if (Kmax >= 3 && sd_n > 0 && sd_n * sizeof(int32_t) <= (2ull << 30)) {
    CU(c, c->d_pbsd.reserve(sd_n));
    sd = c->d_pbsd.p;
  }
  int nl = 0;
  for (;;) {
    CU(c, c->d_f2surv.reserve(c->f2_cap));
    PbOut po{reinterpret_cast<ppipe_point_pb*>(c->d_f2surv.p), c->d_counters.p, (unsigned long long)c->d_f2surv.n, sd};
    nl = 0;
    CU(c, cudaEventRecord(c->ev[0], c->stream));
    CU(c, launch_pack(pb, c->stream));
    nl += pack_launches(pb);
    CU(c, cudaEventRecord(c->ev[1], c->stream));
    CU(c, cudaMemsetAsync(c->d_counters.p, 0, 16 * sizeof(unsigned long long), c->stream));
    for (int i : own) CU(c, launch_pb_model(pb, i, c->h_models[i].M, Kmax, po, c->stream, &nl));
    CU(c, cudaEventRecord(c->ev[2], c->stream));
    CU(c, cudaMemcpyAsync(c->h_counters, c->d_counters.p, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    if (c->h_counters[0] <= c->d_f2surv.n) break;
    c->f2_cap = c->h_counters[0] + c->h_counters[0] / 4 + 1024;  // deterministic: re-run with room
  }
  const uint64_t n_surv = c->h_counters[0], n_feas_local = c->h_counters[1];
  CU(c, c->d_local.reserve(std::max<uint64_t>(n_surv, 1)));
  CU(c, c->d_segoff_local.reserve(c->n_seg_total + 1));
  uint64_t n_pts = 0;
  CU(c, pb_frontier_pass(reinterpret_cast<const ppipe_point_pb*>(c->d_f2surv.p), n_surv, c->d_segbase.p, (int)c->C,
                         c->n_seg_total, c->d_batches.p, (int)c->B, reinterpret_cast<ppipe_point_pb*>(c->d_local.p),
                         c->d_segoff_local.p, &n_pts, &c->scratch, c->stream, &nl));
  CU(c, cudaEventRecord(c->ev[3], c->stream));
  const ppipe_point* d_pts = nullptr;
  const uint64_t* d_off = nullptr;
  uint64_t n_cand_all = 0, n_feas_all = 0;
  if ((rc = concat_owned(c, &n_pts, n_cand, n_feas_local, &n_cand_all, &n_feas_all, &d_pts, &d_off, &nl)) != PPIPE_OK)
    return rc;
  std::memset(out, 0, sizeof *out);
  const ppipe_point* h_pts = nullptr;
  if ((rc = publish_owned(c, nl, d_pts, d_off, n_pts, copy_to_host, &h_pts, &out->seg_offsets)) != PPIPE_OK)
    return rc;
  out->points = reinterpret_cast<const ppipe_point_pb*>(h_pts);
  out->n_candidates = n_cand_all;
  out->n_feasible = n_feas_all;
  out->n_points = n_pts;
  out->n_segments = c->n_seg_total;
  out->d_points = reinterpret_cast<const ppipe_point_pb*>(d_pts);
  out->d_seg_offsets = d_off;
  out->n_survivors = n_surv;
  return PPIPE_OK;
}

PPIPE_API int ppipe_set_vgpu(ppipe_ctx* c, const uint8_t* vgpu) {
  if (!c) return fail(nullptr, PPIPE_EINVAL, "ppipe_set_vgpu: NULL ctx");
  uint32_t v[8] = {1, 1, 1, 1, 1, 1, 1, 1};
  if (vgpu)
    for (uint32_t k = 0; k < c->C; ++k) {
      if (vgpu[k] < 1 || vgpu[k] > 4)
        return fail(c, PPIPE_EINVAL, "class %u: vgpu %u must be 1..4 (1/v of a GPU per instance)", k, vgpu[k]);
      v[k] = vgpu[k];
    }
  uint32_t L = 1;  // lcm of the v's in use: weights L / v are integers <= 12
  for (uint32_t k = 0; k < c->C; ++k) L = L * v[k] / std::gcd(L, v[k]);
  uint32_t pack = 0, wmax = 1;
  for (uint32_t k = 0; k < 8; ++k) {
    const uint32_t w = k < c->C ? L / v[k] : 1;
    pack |= w << (4 * k);
    wmax = std::max(wmax, w);
  }
  int bits = 0;
  while ((1u << bits) < wmax) ++bits;
  c->wpack = pack;
  c->w_max = wmax;
  c->w_bits = bits;
  c->enumerated = false;
  c->have_result = false;
  c->res_local = false;
  return PPIPE_OK;
}

PPIPE_API int ppipe_frontier_at(ppipe_ctx* c, const uint32_t* slo_us, uint32_t margin_permille, int copy_to_host,
                                ppipe_frontier* out) {
  if (!c) return fail(nullptr, PPIPE_EINVAL, "ppipe_frontier_at: NULL ctx");
  if (!out || !slo_us) return fail(c, PPIPE_EINVAL, "ppipe_frontier_at: NULL slo_us or output");
  if (!c->have_result) return fail(c, PPIPE_ESTATE, "ppipe_frontier_at called before ppipe_pareto");
  if (margin_permille >= 1000) return fail(c, PPIPE_EINVAL, "margin_permille %u: must be < 1000", margin_permille);
  std::vector<uint32_t> Tn(c->n_models);
  for (uint32_t m = 0; m < c->n_models; ++m) {
    const uint64_t T0 = (uint64_t)c->last_slo[m] * (1000 - c->last_params.margin_permille) / 1000;
    const uint64_t T1 = (uint64_t)slo_us[m] * (1000 - margin_permille) / 1000;
    if (T1 > T0)
      return fail(c, PPIPE_EINVAL,
                  "model %u: T_eff %llu us exceeds the enumerated %llu us (a sweep can only lower the target)", m,
                  (unsigned long long)T1, (unsigned long long)T0);
    Tn[m] = (uint32_t)T1;
  }
  CU(c, cudaSetDevice(c->device));
  CU(c, c->d_Tnew.reserve(std::max<size_t>(c->n_models, 1)));
  CU(c, c->d_trunc.reserve(std::max<uint64_t>(c->res_n, 1)));
  CU(c, c->d_trunc_off.reserve(c->n_seg_total + 1));
  CU(c, cudaMemcpyAsync(c->d_Tnew.p, Tn.data(), 4 * Tn.size(), cudaMemcpyHostToDevice, c->stream));
  uint64_t n_pts = 0;
  int nl = 0;
  CU(c, truncate_frontier(c->res_pts, c->res_off, c->res_n, c->n_seg_total, c->d_Tnew.p, c->d_trunc.p,
                          c->d_trunc_off.p, &n_pts, &c->scratch, c->stream, &nl));
  std::memset(out, 0, sizeof *out);
  out->n_candidates = c->res_ncand;
  out->n_points = n_pts;
  out->n_segments = c->n_seg_total;
  out->d_points = c->d_trunc.p;
  out->d_seg_offsets = c->d_trunc_off.p;
  if (copy_to_host) {
    CU(c, c->h_points.reserve(n_pts));
    CU(c, c->h_segoff.reserve(c->n_seg_total + 1));
    if (n_pts)
      CU(c, cudaMemcpyAsync(c->h_points.p, c->d_trunc.p, sizeof(ppipe_point) * n_pts, cudaMemcpyDeviceToHost,
                            c->stream));
    CU(c, cudaMemcpyAsync(c->h_segoff.p, c->d_trunc_off.p, 8 * (c->n_seg_total + 1), cudaMemcpyDeviceToHost,
                          c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    out->points = c->h_points.p;
    out->seg_offsets = c->h_segoff.p;
  }
  return PPIPE_OK;
}
