/*
 * ppipe_oracle.c -- plain, slow, obviously-correct CPU oracle for the PPipe
 * plan-enumeration hot path (arXiv 2507.18748).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library. It
 * shares no code, header, table or constant with the CUDA path
 * (paper_2507_18748_b200/); it reads the same plain input arrays.
 *
 * What it computes (DESIGN.md §2 "The path"):
 *
 *   for m in models                                 per-model independence, PAPER.md:2299-2302 (A.1)
 *     T = floor(slo_us[m] * (1000 - margin) / 1000)  SLO margin, PAPER.md:1386-1394 (§5.4), 1690-1693 (§7.1)
 *     for K in 1..min(Kmax, M)                       <=3 partitions, PAPER.md:562-571 (§3 "Encoding")
 *       for cuts 0 = c_0 < c_1 < .. < c_{K-1} < c_K = M  (lexicographic)
 *                                                  well-formed partitions, eqs. 1.1-1.5
 *         for class tuple (k_1..k_K) in classes^K  (lexicographic, repeats allowed; 14 for C=2)
 *           for b in batches                        unified batch, eq. 3.3, PAPER.md:2369-2370 (A.2)
 *             C_d = sum_{l=c_{d-1}}^{c_d - 1} lat[k_d][l][b]      eq. 1.9 / C_{ldbij}
 *             Y_d = ceil(8 * S[c_d - 1] * b / bw[k_d][k_{d+1}])  d = 1..K-1; Y_{bj}, eq. 1.11
 *                   (no transfer before partition 1 or after partition K: readings A2/A3)
 *             E   = sum_d C_d + sum_d Y_d                          eq. 1.12
 *             feasible iff E <= T                                  eq. 1.12 "<= T" (reading A6)
 *             theta = b / max_d C_d  (exact rational; C = 0 => +inf) X_{ldbij} = b / C, x_l = min_d x_ld,
 *                     (with virtual GPUs: min_d v_{k_d} b / C_d, see oracle_set_vgpu)
 *                                                                  PAPER.md:2245, 2281, 2284 (reading A11)
 *   per segment (m, K, k_1..k_K): sort feasible candidates by
 *       (E asc, theta desc, b asc, (c_1, c_2) lexicographic asc)
 *     and keep p iff theta_p > best theta so far (strict)  -- the (E min, theta max) Pareto
 *     frontier with the canonical tie-break of reading A1/A17.
 *
 * Hoisting (allowed by SURVEY.md §8(c)): C_d over a fixed (range, class, b) and
 * Y_d over a fixed (cut, class pair, b) are computed once by the definitions
 * above (direct summation over the layer range, ceil-division) and reused
 * across the loops that do not change them. No prefix-difference table is used.
 *
 * Parallelism: pthreads over first-cut rows of one model; results are sorted
 * per segment afterwards, so they do not depend on the thread count.
 *
 * Parity: every function here is pinned by tests/test_oracle_pins.py (hand-worked
 * fixtures P0a/P0b, printed numbers P1-P4, closed forms P5/P6/P9, the textbook
 * min-max partition P7, and the literal O(n^2) Pareto definition P8);
 * oracle_prepartition (end of file) by tests/test_prepartition_pins.py (the
 * SPEC.md examples, closed forms for N = 1, N = M and uniform layers, and the
 * half-layer balance bound that the greedy stopping rule implies); the F2
 * reduction (oracle_set_frontier(2), below) by tests/test_f2_pins.py (an
 * independent Fraction-based literal definition on random tiny inputs, a
 * hand-worked fixture, the K = 1 closed form, the single-batch all-kept case and
 * the MILP-losslessness property); oracle_run_pb (per-stage batch sizes, end of
 * file) by tests/test_pb_pins.py (the unified oracle at one batch size, a Fraction
 * literal definition, closed-form counts, a hand-worked mixed-batch plan and the
 * superset property over the unified frontier).
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* Output record: 32 bytes, same field layout as the library's documented
 * point record. Declared here independently on purpose. */
typedef struct {
  uint32_t model;
  uint16_t cut[2];
  uint8_t K;
  uint8_t cls[3];
  uint16_t batch;
  uint16_t reserved;
  uint32_t e2e_us;
  uint32_t stage_us[3];
} oracle_point;

typedef struct {
  uint32_t n_layers;
  const uint32_t *lat_us;    /* [C][M][B] */
  const uint64_t *act_bytes; /* [M] */
} oracle_model;

typedef struct {
  int64_t E;
  int64_t st[3]; /* C_1..C_K */
  int32_t c1, c2;
  int32_t b;
} cand;

typedef struct {
  cand *v;
  size_t n, cap;
} cvec;

static void cvec_push(cvec *a, const cand *c) {
  if (a->n == a->cap) {
    size_t nc = a->cap ? a->cap * 2 : 64;
    cand *nv = (cand *)realloc(a->v, nc * sizeof(cand));
    if (!nv) {
      fprintf(stderr, "oracle: out of memory\n");
      abort();
    }
    a->v = nv;
    a->cap = nc;
  }
  a->v[a->n++] = *c;
}

/*
 * Virtual GPUs (§5.1; App. A.2 L_{kvbi}):
 * class k may be a "pseudo-class" running on 1/v_k of a physical GPU (MPS), so
 * v_k instances share one GPU and a stage's per-physical-GPU throughput is
 * v_k * b / C_d. The plan's throughput is its bottleneck, the minimum over stages
 * (x_l = min_d x_ld): theta = min_d v_{k_d} * b / C_d. With every
 * v = 1 (the default) this is b / max_d C_d. theta is kept as the exact fraction
 * (num, den) = (v_d* b, C_d*) of the minimising stage d* (den = 0 is +inf).
 */
static uint8_t g_vgpu[256]; /* per class; 0 = unset = 1 */

void oracle_set_vgpu(const uint8_t *v, uint32_t n_classes) {
  memset(g_vgpu, 0, sizeof g_vgpu);
  if (v)
    for (uint32_t k = 0; k < n_classes && k < 256; k++) g_vgpu[k] = v[k];
}

static int64_t vgpu_of(int k) { return g_vgpu[k] ? g_vgpu[k] : 1; }

/* theta_p > theta_q for fractions num/den (den = 0 is +inf; two +inf tie) */
static int theta_gt(int64_t np_, int64_t dp, int64_t nq, int64_t dq) { return np_ * dq > nq * dp; }

static void theta_of(const cand *c, int K, const int *cls, int64_t *num, int64_t *den) {
  *num = vgpu_of(cls[0]) * c->b;
  *den = c->st[0];
  for (int d = 1; d < K; d++) {
    const int64_t n2 = vgpu_of(cls[d]) * c->b, d2 = c->st[d];
    if (theta_gt(*num, *den, n2, d2)) { /* stage d is slower: it is the bottleneck so far */
      *num = n2;
      *den = d2;
    }
  }
}

static int g_sort_K; /* qsort has no context argument; sorting is single-threaded */
static int g_sort_cls[3];
static int cand_cmp(const void *pa, const void *pb) {
  const cand *p = (const cand *)pa, *q = (const cand *)pb;
  if (p->E != q->E) return p->E < q->E ? -1 : 1;
  int64_t np_, dp, nq, dq;
  theta_of(p, g_sort_K, g_sort_cls, &np_, &dp);
  theta_of(q, g_sort_K, g_sort_cls, &nq, &dq);
  if (theta_gt(np_, dp, nq, dq)) return -1; /* theta descending */
  if (theta_gt(nq, dq, np_, dp)) return 1;
  if (p->b != q->b) return p->b < q->b ? -1 : 1;
  if (p->c1 != q->c1) return p->c1 < q->c1 ? -1 : 1;
  if (p->c2 != q->c2) return p->c2 < q->c2 ? -1 : 1;
  return 0;
}

/*
 * F2, the MILP-lossless frontier (DESIGN.md §3 readings
 * F2-1..F2-4). PPipe's MILP gives a chosen pipeline g_d GPUs in stage d and its
 * throughput is x_l = min_d g_d * X_d with X_d = b / C_d the per-GPU throughput of
 * stage d (eqs. 1.10, 1.13); E only has to meet the SLO
 * (eq. 1.12). So per segment the objective is the per-stage vector
 * x = (X_1, .., X_K) (with virtual GPUs X_d = v_{k_d} b / C_d),
 * and a feasible candidate q makes p redundant iff x_q >= x_p in every stage and
 * either x_q != x_p (strict Pareto dominance) or x_q == x_p and q comes first in
 * (E, b, c_1, c_2) ascending (E is the tie-break only). Kept points are listed in
 * (b, c_1, c_2) ascending order. Below is that definition as written: every pair.
 */
static int g_frontier = 1; /* 1 = (E, theta) staircase (A1), 2 = F2 */

void oracle_set_frontier(int kind) { g_frontier = kind == 2 ? 2 : 1; }

/* q makes p redundant under F2 (see above). X_q,d >= X_p,d  <=>  v b_q C_p,d >= v b_p C_q,d
 * (C = 0 reads as +inf: two +inf are equal). */
static int f2_beats(const cand *q, const cand *p, int K, const int *cls) {
  int all_eq = 1;
  for (int d = 0; d < K; d++) {
    const int64_t v = vgpu_of(cls[d]);
    const int64_t lhs = v * q->b * p->st[d], rhs = v * p->b * q->st[d];
    if (lhs < rhs) return 0;
    if (lhs != rhs) all_eq = 0;
  }
  if (!all_eq) return 1;
  if (q->E != p->E) return q->E < p->E;
  if (q->b != p->b) return q->b < p->b;
  if (q->c1 != p->c1) return q->c1 < p->c1;
  return q->c2 < p->c2; /* p itself: not redundant */
}

static int f2_out_cmp(const void *pa, const void *pb) {
  const cand *p = (const cand *)pa, *q = (const cand *)pb;
  if (p->b != q->b) return p->b < q->b ? -1 : 1;
  if (p->c1 != q->c1) return p->c1 < q->c1 ? -1 : 1;
  if (p->c2 != q->c2) return p->c2 < q->c2 ? -1 : 1;
  return 0;
}

typedef struct {
  const cand *v;
  size_t n;
  int K;
  const int *cls;
  uint8_t *keep;
  int t, nt;
} f2_job;

static void *f2_worker(void *arg) {
  f2_job *j = (f2_job *)arg;
  for (size_t i = (size_t)j->t; i < j->n; i += (size_t)j->nt) {
    int redundant = 0;
    for (size_t q = 0; q < j->n && !redundant; q++) redundant = f2_beats(&j->v[q], &j->v[i], j->K, j->cls);
    j->keep[i] = (uint8_t)!redundant;
  }
  return NULL;
}

/* F2 reduction of one segment's feasible candidates, in place: returns the kept count,
 * kept points first, in (b, c_1, c_2) order. */
static size_t f2_reduce(cand *v, size_t n, int K, const int *cls, int nthreads) {
  if (!n) return 0;
  uint8_t *keep = (uint8_t *)calloc(n, 1);
  int nt = nthreads;
  if ((size_t)nt > n) nt = (int)n;
  f2_job *jobs = (f2_job *)calloc((size_t)nt, sizeof(f2_job));
  pthread_t *th = (pthread_t *)calloc((size_t)nt, sizeof(pthread_t));
  for (int t = 0; t < nt; t++) {
    jobs[t] = (f2_job){v, n, K, cls, keep, t, nt};
    pthread_create(&th[t], NULL, f2_worker, &jobs[t]);
  }
  for (int t = 0; t < nt; t++) pthread_join(th[t], NULL);
  size_t k = 0;
  for (size_t i = 0; i < n; i++)
    if (keep[i]) v[k++] = v[i];
  qsort(v, k, sizeof(cand), f2_out_cmp);
  free(keep);
  free(jobs);
  free(th);
  return k;
}

/* ---- problem description shared by the worker threads ---- */
typedef struct {
  const oracle_model *md;
  uint32_t C, B, M;
  const uint32_t *batches;
  const uint32_t *bw; /* [C][C] */
  int64_t T;
  int Kmax;
  int only_K;               /* 0 = all */
  const uint8_t *only_cls;  /* NULL = all tuples */
  int32_t row_lo, row_hi;   /* row sample [row_lo, row_hi): row 0 = K=1, row r>=1 = first cut r; row_hi <= 0 = all */
  uint32_t nseg[4];         /* C^K */
  /* hoisted direct quantities */
  int64_t *pre;  /* pre[c][k][b]  = sum_{l<c} lat[k][l][b]   for c=0..M, by direct summation */
  int64_t *suf;  /* suf[c][k][b]  = sum_{l>=c} lat[k][l][b]  for c=0..M, by direct summation */
  int64_t *Y;    /* Y[c][k][k'][b] = ceil(8*S[c-1]*b / bw[k][k']) for c=1..M-1 */
  int next_row;
  pthread_mutex_t mu;
  uint64_t n_cand, n_feas;
} problem;

typedef struct {
  problem *pb;
  cvec *segs[4]; /* per K, C^K vectors */
  uint64_t n_cand, n_feas;
} worker;

static inline uint32_t LAT(const problem *pb, uint32_t k, uint32_t l, uint32_t bi) {
  return pb->md->lat_us[((size_t)k * pb->M + l) * pb->B + bi];
}

/* C_d by direct summation over layers [i, j) on class k at batch index bi. */
static int64_t direct_sum(const problem *pb, uint32_t k, uint32_t i, uint32_t j, uint32_t bi) {
  int64_t s = 0;
  for (uint32_t l = i; l < j; l++) s += LAT(pb, k, l, bi);
  return s;
}

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static int tuple_allowed(const problem *pb, int K, const uint32_t *k) {
  if (pb->only_K && pb->only_K != K) return 0;
  if (!pb->only_cls) return 1;
  for (int d = 0; d < K; d++)
    if (pb->only_cls[d] != k[d]) return 0;
  return 1;
}

static void emit(worker *w, int K, const uint32_t *k, const cand *c) {
  uint32_t idx = 0;
  for (int d = 0; d < K; d++) idx = idx * w->pb->C + k[d];
  cvec_push(&w->segs[K][idx], c);
}

/* One row of the enumeration: K=1 (row = -1), or K>=2 with first cut c1 = row. */
static void do_row(worker *w, int K, int32_t c1) {
  problem *pb = w->pb;
  const uint32_t C = pb->C, B = pb->B, M = pb->M;
  const uint64_t *S = pb->md->act_bytes;
  uint32_t k[3];
  cand c;
  if (K == 1) {
    for (k[0] = 0; k[0] < C; k[0]++) {
      if (!tuple_allowed(pb, 1, k)) continue;
      for (uint32_t bi = 0; bi < B; bi++) {
        memset(&c, 0, sizeof c);
        c.st[0] = pb->pre[((size_t)M * C + k[0]) * B + bi]; /* whole model on class k */
        c.E = c.st[0];
        c.b = (int32_t)pb->batches[bi];
        w->n_cand++;
        if (c.E > pb->T) continue;
        w->n_feas++;
        emit(w, 1, k, &c);
      }
    }
    return;
  }
  if (K == 2) {
    for (k[0] = 0; k[0] < C; k[0]++)
      for (k[1] = 0; k[1] < C; k[1]++) {
        if (!tuple_allowed(pb, 2, k)) continue;
        for (uint32_t bi = 0; bi < B; bi++) {
          memset(&c, 0, sizeof c);
          c.st[0] = pb->pre[((size_t)c1 * C + k[0]) * B + bi];
          c.st[1] = pb->suf[((size_t)c1 * C + k[1]) * B + bi];
          int64_t y = pb->Y[(((size_t)c1 * C + k[0]) * C + k[1]) * B + bi];
          c.E = c.st[0] + c.st[1] + y;
          c.c1 = c1;
          c.b = (int32_t)pb->batches[bi];
          w->n_cand++;
          if (c.E > pb->T) continue;
          w->n_feas++;
          emit(w, 2, k, &c);
        }
      }
    return;
  }
  /* K == 3: C_2 over [c1, c2) by direct summation for each c2 (hoisted over the tuple loop). */
  int64_t *mid = (int64_t *)malloc(sizeof(int64_t) * C * B);
  for (int32_t c2 = c1 + 1; c2 <= (int32_t)M - 1; c2++) {
    for (uint32_t kk = 0; kk < C; kk++)
      for (uint32_t bi = 0; bi < B; bi++) mid[kk * B + bi] = direct_sum(pb, kk, (uint32_t)c1, (uint32_t)c2, bi);
    for (k[0] = 0; k[0] < C; k[0]++)
      for (k[1] = 0; k[1] < C; k[1]++)
        for (k[2] = 0; k[2] < C; k[2]++) {
          if (!tuple_allowed(pb, 3, k)) continue;
          for (uint32_t bi = 0; bi < B; bi++) {
            c.st[0] = pb->pre[((size_t)c1 * C + k[0]) * B + bi];
            c.st[1] = mid[k[1] * B + bi];
            c.st[2] = pb->suf[((size_t)c2 * C + k[2]) * B + bi];
            int64_t y1 = pb->Y[(((size_t)c1 * C + k[0]) * C + k[1]) * B + bi];
            int64_t y2 = pb->Y[(((size_t)c2 * C + k[1]) * C + k[2]) * B + bi];
            c.E = c.st[0] + c.st[1] + c.st[2] + y1 + y2;
            c.c1 = c1;
            c.c2 = c2;
            c.b = (int32_t)pb->batches[bi];
            w->n_cand++;
            if (c.E > pb->T) continue;
            w->n_feas++;
            emit(w, 3, k, &c);
          }
        }
  }
  (void)S;
  free(mid);
}

static void *worker_main(void *arg) {
  worker *w = (worker *)arg;
  problem *pb = w->pb;
  const int32_t M = (int32_t)pb->M;
  for (;;) {
    pthread_mutex_lock(&pb->mu);
    int32_t r = pb->next_row++;
    pthread_mutex_unlock(&pb->mu);
    /* row 0: K=1 (no cuts). row r in 1..M-1: K=2 and K=3 with first cut c_1 = r. */
    if (r >= M) break;
    int in_sample = pb->row_hi <= 0 || (r >= pb->row_lo && r < pb->row_hi);
    if (!in_sample) continue;
    if (r == 0) {
      do_row(w, 1, -1);
      continue;
    }
    if (pb->Kmax >= 2) do_row(w, 2, r);                /* c_1 in [1, M-1] */
    if (pb->Kmax >= 3 && r <= M - 2) do_row(w, 3, r);  /* c_1 < c_2 <= M-1 */
  }
  return NULL;
}

/* ---- public oracle API (ctypes) ---- */

typedef struct {
  oracle_point *pts;
  uint64_t n_pts;
  uint64_t *seg_off; /* CSR over all segments in canonical order */
  uint64_t n_seg;
  uint64_t n_cand, n_feas;
} oracle_result;

static int g_threads = 0;

void oracle_set_threads(int n) { g_threads = n; }

void oracle_result_free(oracle_result *r) {
  if (!r) return;
  free(r->pts);
  free(r->seg_off);
  free(r);
}

/*
 * Enumerate models [model_lo, model_hi), all K <= Kmax (or only_K), all tuples
 * (or only_cls). row_lo/row_hi restrict the enumeration to rows [row_lo, row_hi)
 * where row 0 holds the K=1 candidates and row r >= 1 the candidates with first
 * cut c_1 = r (sampling and rank shards; row_hi <= 0 disables). Returns 0 on success.
 */
int oracle_run(uint32_t n_models, const oracle_model *models, uint32_t n_classes, uint32_t n_batches,
               const uint32_t *batches, const uint32_t *bw, uint32_t kmax, const uint32_t *slo_us,
               uint32_t margin_permille, uint32_t model_lo, uint32_t model_hi, int only_K,
               const uint8_t *only_cls, int32_t row_lo, int32_t row_hi, oracle_result **out) {
  if (!out || n_classes == 0 || n_batches == 0 || kmax < 1 || kmax > 3 || margin_permille >= 1000) return -1;
  if (model_hi > n_models || model_lo > model_hi) return -1;
  oracle_result *res = (oracle_result *)calloc(1, sizeof *res);
  size_t cap_pts = 0;
  const uint32_t C = n_classes, B = n_batches;
  /* total segments in canonical order */
  uint64_t total_seg = 0;
  for (uint32_t m = model_lo; m < model_hi; m++) {
    uint32_t M = models[m].n_layers;
    uint64_t p = 1;
    for (uint32_t K = 1; K <= kmax && K <= M; K++) {
      p *= C;
      total_seg += p;
    }
  }
  res->seg_off = (uint64_t *)calloc(total_seg + 1, sizeof(uint64_t));
  res->n_seg = total_seg;
  uint64_t seg_cursor = 0;

  int nthreads = g_threads > 0 ? g_threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads < 1) nthreads = 1;

  for (uint32_t m = model_lo; m < model_hi; m++) {
    problem pb;
    memset(&pb, 0, sizeof pb);
    pb.md = &models[m];
    pb.C = C;
    pb.B = B;
    pb.M = models[m].n_layers;
    pb.batches = batches;
    pb.bw = bw;
    pb.T = (int64_t)slo_us[m] * (int64_t)(1000 - margin_permille) / 1000; /* floor */
    pb.Kmax = (int)kmax;
    pb.only_K = only_K;
    pb.only_cls = only_cls;
    pb.row_lo = row_lo;
    pb.row_hi = row_hi;
    const uint32_t M = pb.M;
    pthread_mutex_init(&pb.mu, NULL);
    /* hoisted direct sums: pre[c] over [0, c), suf[c] over [c, M) */
    pb.pre = (int64_t *)malloc(sizeof(int64_t) * (M + 1) * C * B);
    pb.suf = (int64_t *)malloc(sizeof(int64_t) * (M + 1) * C * B);
    for (uint32_t c = 0; c <= M; c++)
      for (uint32_t k = 0; k < C; k++)
        for (uint32_t bi = 0; bi < B; bi++) {
          pb.pre[((size_t)c * C + k) * B + bi] = direct_sum(&pb, k, 0, c, bi);
          pb.suf[((size_t)c * C + k) * B + bi] = direct_sum(&pb, k, c, M, bi);
        }
    pb.Y = (int64_t *)calloc((size_t)(M + 1) * C * C * B, sizeof(int64_t));
    for (uint32_t c = 1; c + 1 <= M; c++)
      for (uint32_t k = 0; k < C; k++)
        for (uint32_t k2 = 0; k2 < C; k2++)
          for (uint32_t bi = 0; bi < B; bi++)
            pb.Y[(((size_t)c * C + k) * C + k2) * B + bi] =
                ceil_div(8 * (int64_t)models[m].act_bytes[c - 1] * (int64_t)batches[bi], (int64_t)bw[k * C + k2]);
    for (uint32_t K = 1; K <= 3; K++) {
      uint32_t p = 1;
      for (uint32_t d = 0; d < K; d++) p *= C;
      pb.nseg[K] = p;
    }
    worker *ws = (worker *)calloc((size_t)nthreads, sizeof(worker));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; t++) {
      ws[t].pb = &pb;
      for (int K = 1; K <= 3; K++) ws[t].segs[K] = (cvec *)calloc(pb.nseg[K], sizeof(cvec));
      pthread_create(&th[t], NULL, worker_main, &ws[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; t++) {
      res->n_cand += ws[t].n_cand;
      res->n_feas += ws[t].n_feas;
    }
    /* per segment, canonical order: K asc, tuple lexicographic asc */
    for (uint32_t K = 1; K <= kmax && K <= M; K++) {
      for (uint32_t s = 0; s < pb.nseg[K]; s++) {
        cvec all = {0};
        for (int t = 0; t < nthreads; t++)
          for (size_t i = 0; i < ws[t].segs[K][s].n; i++) cvec_push(&all, &ws[t].segs[K][s].v[i]);
        g_sort_K = (int)K;
        {
          uint32_t t = s; /* the segment's class tuple (lexicographic index) */
          for (int d = (int)K - 1; d >= 0; d--) {
            g_sort_cls[d] = (int)(t % C);
            t /= C;
          }
        }
        size_t n_out = all.n;
        if (g_frontier == 2) {
          n_out = f2_reduce(all.v, all.n, (int)K, g_sort_cls, nthreads);
        } else if (all.n) {
          qsort(all.v, all.n, sizeof(cand), cand_cmp);
        }
        int64_t best_n = 0, best_d = 1; /* theta = 0 */
        for (size_t i = 0; i < n_out; i++) {
          const cand *p = &all.v[i];
          if (g_frontier != 2) {
            int64_t tn, td;
            theta_of(p, (int)K, g_sort_cls, &tn, &td);
            if (!theta_gt(tn, td, best_n, best_d)) continue; /* keep iff theta > best (strict) */
            best_n = tn;
            best_d = td;
          }
          if (res->n_pts == cap_pts) {
            cap_pts = cap_pts ? cap_pts * 2 : 1024;
            res->pts = (oracle_point *)realloc(res->pts, cap_pts * sizeof(oracle_point));
          }
          oracle_point *o = &res->pts[res->n_pts++];
          memset(o, 0, sizeof *o);
          o->model = m;
          o->K = (uint8_t)K;
          o->cut[0] = (uint16_t)(K >= 2 ? p->c1 : 0);
          o->cut[1] = (uint16_t)(K >= 3 ? p->c2 : 0);
          uint32_t idx = s;
          for (int d = (int)K - 1; d >= 0; d--) {
            o->cls[d] = (uint8_t)(idx % C);
            idx /= C;
          }
          for (int d = (int)K; d < 3; d++) o->cls[d] = 0xFF;
          o->batch = (uint16_t)p->b;
          o->e2e_us = (uint32_t)p->E;
          for (int d = 0; d < (int)K; d++) o->stage_us[d] = (uint32_t)p->st[d];
        }
        free(all.v);
        res->seg_off[++seg_cursor] = res->n_pts;
      }
    }
    for (int t = 0; t < nthreads; t++) {
      for (int K = 1; K <= 3; K++) {
        for (uint32_t s = 0; s < pb.nseg[K]; s++) free(ws[t].segs[K][s].v);
        free(ws[t].segs[K]);
      }
    }
    free(ws);
    free(th);
    free(pb.pre);
    free(pb.suf);
    free(pb.Y);
    pthread_mutex_destroy(&pb.mu);
  }
  *out = res;
  return 0;
}

/*
 * Greedy equal-runtime pre-partitioning (§5.2).
 *
 *   "we start from the first layer and sequentially group consecutive layers
 *    together until their combined runtime is as close as possible to 1/N of the
 *    runtime of the entire DNN; this process is repeated until we reach the last
 *    layer."
 *
 * Runtime t_l = lat[ref_class][l][ref_b] (a selected GPU type at one batch). A block
 * starts at the first unassigned layer with that layer, then takes the next layer
 * while doing so brings its runtime at least as close to total/N (ties include the
 * layer), and stops early enough to leave one layer for every
 * remaining block; block N takes the rest. "As close as possible" is
 * compared exactly in integers: |N*(acc + t) - total| <= |N*acc - total|.
 * Block latency per (class, batch) = sum over member layers; block output bytes =
 * the last member layer's. lat is [C][M][B]; outputs bounds[N+1],
 * block_lat[C][N][B] (uint64, so sums cannot wrap), block_S[N].
 * Returns 0, or -1 if N < 1, N > M or the reference indices are out of range.
 */
int oracle_prepartition(uint32_t M, uint32_t C, uint32_t B, const uint32_t *lat, const uint64_t *S, uint32_t N,
                        uint32_t ref_class, uint32_t ref_b, uint32_t *bounds, uint64_t *block_lat, uint64_t *block_S) {
  if (N < 1 || N > M || ref_class >= C || ref_b >= B) return -1;
  int64_t total = 0;
  for (uint32_t l = 0; l < M; ++l) total += lat[((size_t)ref_class * M + l) * B + ref_b];
  uint32_t i = 0;
  bounds[0] = 0;
  for (uint32_t blk = 0; blk + 1 < N; ++blk) {
    const uint32_t remaining = N - blk - 1; /* blocks still to come after this one */
    int64_t acc = lat[((size_t)ref_class * M + i) * B + ref_b];
    uint32_t j = i + 1;
    while (j < M - remaining) {
      const int64_t t = lat[((size_t)ref_class * M + j) * B + ref_b];
      int64_t with = (int64_t)N * (acc + t) - total, without = (int64_t)N * acc - total;
      if (with < 0) with = -with;
      if (without < 0) without = -without;
      if (with <= without) {
        acc += t;
        ++j;
      } else {
        break;
      }
    }
    bounds[blk + 1] = j;
    i = j;
  }
  bounds[N] = M;
  for (uint32_t k = 0; k < C; ++k)
    for (uint32_t q = 0; q < N; ++q)
      for (uint32_t b = 0; b < B; ++b) {
        uint64_t sum = 0;
        for (uint32_t l = bounds[q]; l < bounds[q + 1]; ++l) sum += lat[((size_t)k * M + l) * B + b];
        block_lat[((size_t)k * N + q) * B + b] = sum;
      }
  for (uint32_t q = 0; q < N; ++q) block_S[q] = S[bounds[q + 1] - 1];
  return 0;
}

/*
 * Per-stage batch sizes (DESIGN.md §3 readings PB-1..PB-4).
 *
 * The basic MILP of App. A.1 lets every partition pick its own batch size: eq. 1.1
 * sums p_{ldbij} over (b, i, j) per partition d, so partition d runs
 * at b_d. Per candidate (cuts, classes, b_1..b_K):
 *   C_d = sum_{l in [c_{d-1}, c_d)} lat[k_d][l][b_d]                  eq. 1.9 (C_{ldbij} at b_d)
 *   Y_d = ceil(8 * S[c_d - 1] * b_d / bw[k_d][k_{d+1}])  for d < K    eq. 1.11: n_ld = Y_{bj} of
 *         partition d's own (b, j), i.e. the sender's batch
 *   E   = sum_d C_d + sum_d Y_d <= T                                  eq. 1.12
 *   theta = min_d b_d / C_d  (x_l = min_d x_ld, X = b / C, one GPU per stage)
 * and per segment (m, K, k_1..k_K) the (E min, theta max) staircase with ties on
 * identical (E, theta) broken by the smallest (b_1, .., b_K) (lexicographic), then the
 * smallest (c_1, c_2). With one batch size this is oracle_run's frontier.
 * Records carry batch INDICES (bidx[d] into the batch list; 0xFF when unused).
 * Pinned by tests/test_pb_pins.py.
 */
typedef struct {
  uint32_t model;
  uint16_t cut[2];
  uint8_t K;
  uint8_t cls[3];
  uint8_t bidx[3];
  uint8_t reserved;
  uint32_t e2e_us;
  uint32_t stage_us[3];
} oracle_point_pb;

typedef struct {
  int64_t E;
  int64_t st[3];
  int32_t c1, c2;
  int32_t bi[3];
} cand_pb;

typedef struct {
  cand_pb *v;
  size_t n, cap;
} cvec_pb;

static void cvec_pb_push(cvec_pb *a, const cand_pb *c) {
  if (a->n == a->cap) {
    size_t nc = a->cap ? a->cap * 2 : 64;
    cand_pb *nv = (cand_pb *)realloc(a->v, nc * sizeof(cand_pb));
    if (!nv) {
      fprintf(stderr, "oracle: out of memory\n");
      abort();
    }
    a->v = nv;
    a->cap = nc;
  }
  a->v[a->n++] = *c;
}

static const uint32_t *g_pb_batches; /* qsort context (sorting is single-threaded) */
static int g_pb_K;

/* theta = min_d b_d / C_d as the fraction (num, den) of the minimising stage (den 0 = +inf) */
static void theta_pb(const cand_pb *c, int K, int64_t *num, int64_t *den) {
  *num = g_pb_batches[c->bi[0]];
  *den = c->st[0];
  for (int d = 1; d < K; d++) {
    const int64_t n2 = g_pb_batches[c->bi[d]], d2 = c->st[d];
    if (theta_gt(*num, *den, n2, d2)) {
      *num = n2;
      *den = d2;
    }
  }
}

static int cand_pb_cmp(const void *pa, const void *pb_) {
  const cand_pb *p = (const cand_pb *)pa, *q = (const cand_pb *)pb_;
  if (p->E != q->E) return p->E < q->E ? -1 : 1;
  int64_t np_, dp, nq, dq;
  theta_pb(p, g_pb_K, &np_, &dp);
  theta_pb(q, g_pb_K, &nq, &dq);
  if (theta_gt(np_, dp, nq, dq)) return -1;
  if (theta_gt(nq, dq, np_, dp)) return 1;
  for (int d = 0; d < g_pb_K; d++)
    if (p->bi[d] != q->bi[d]) return p->bi[d] < q->bi[d] ? -1 : 1;
  if (p->c1 != q->c1) return p->c1 < q->c1 ? -1 : 1;
  if (p->c2 != q->c2) return p->c2 < q->c2 ? -1 : 1;
  return 0;
}

typedef struct {
  problem *pb;
  cvec_pb *segs[4];
  uint64_t n_cand, n_feas;
} worker_pb;

static void emit_pb(worker_pb *w, int K, const uint32_t *k, const cand_pb *c) {
  uint32_t idx = 0;
  for (int d = 0; d < K; d++) idx = idx * w->pb->C + k[d];
  cvec_pb_push(&w->segs[K][idx], c);
}

/* One row: K=1 (c1 = -1) or first cut c1 for K=2 / K=3; every class and batch per stage. */
static void do_row_pb(worker_pb *w, int K, int32_t c1) {
  problem *pb = w->pb;
  const uint32_t C = pb->C, B = pb->B, M = pb->M;
  uint32_t k[3];
  cand_pb c;
  memset(&c, 0, sizeof c);
  if (K == 1) {
    for (k[0] = 0; k[0] < C; k[0]++)
      for (uint32_t b1 = 0; b1 < B; b1++) {
        memset(&c, 0, sizeof c);
        c.st[0] = pb->pre[((size_t)M * C + k[0]) * B + b1];
        c.E = c.st[0];
        c.bi[0] = (int32_t)b1;
        w->n_cand++;
        if (c.E > pb->T) continue;
        w->n_feas++;
        emit_pb(w, 1, k, &c);
      }
    return;
  }
  if (K == 2) {
    for (k[0] = 0; k[0] < C; k[0]++)
      for (k[1] = 0; k[1] < C; k[1]++)
        for (uint32_t b1 = 0; b1 < B; b1++)
          for (uint32_t b2 = 0; b2 < B; b2++) {
            memset(&c, 0, sizeof c);
            c.st[0] = pb->pre[((size_t)c1 * C + k[0]) * B + b1];
            c.st[1] = pb->suf[((size_t)c1 * C + k[1]) * B + b2];
            c.E = c.st[0] + c.st[1] + pb->Y[(((size_t)c1 * C + k[0]) * C + k[1]) * B + b1]; /* sender's batch */
            c.c1 = c1;
            c.bi[0] = (int32_t)b1;
            c.bi[1] = (int32_t)b2;
            w->n_cand++;
            if (c.E > pb->T) continue;
            w->n_feas++;
            emit_pb(w, 2, k, &c);
          }
    return;
  }
  int64_t *mid = (int64_t *)malloc(sizeof(int64_t) * C * B);
  for (int32_t c2 = c1 + 1; c2 <= (int32_t)M - 1; c2++) {
    for (uint32_t kk = 0; kk < C; kk++)
      for (uint32_t bi = 0; bi < B; bi++) mid[kk * B + bi] = direct_sum(pb, kk, (uint32_t)c1, (uint32_t)c2, bi);
    for (k[0] = 0; k[0] < C; k[0]++)
      for (k[1] = 0; k[1] < C; k[1]++)
        for (k[2] = 0; k[2] < C; k[2]++)
          for (uint32_t b1 = 0; b1 < B; b1++)
            for (uint32_t b2 = 0; b2 < B; b2++)
              for (uint32_t b3 = 0; b3 < B; b3++) {
                c.st[0] = pb->pre[((size_t)c1 * C + k[0]) * B + b1];
                c.st[1] = mid[k[1] * B + b2];
                c.st[2] = pb->suf[((size_t)c2 * C + k[2]) * B + b3];
                c.E = c.st[0] + c.st[1] + c.st[2] + pb->Y[(((size_t)c1 * C + k[0]) * C + k[1]) * B + b1] +
                      pb->Y[(((size_t)c2 * C + k[1]) * C + k[2]) * B + b2];
                c.c1 = c1;
                c.c2 = c2;
                c.bi[0] = (int32_t)b1;
                c.bi[1] = (int32_t)b2;
                c.bi[2] = (int32_t)b3;
                w->n_cand++;
                if (c.E > pb->T) continue;
                w->n_feas++;
                emit_pb(w, 3, k, &c);
              }
  }
  free(mid);
}

static void *worker_pb_main(void *arg) {
  worker_pb *w = (worker_pb *)arg;
  problem *pb = w->pb;
  const int32_t M = (int32_t)pb->M;
  for (;;) {
    pthread_mutex_lock(&pb->mu);
    int32_t r = pb->next_row++;
    pthread_mutex_unlock(&pb->mu);
    if (r >= M) break;
    if (r == 0) {
      do_row_pb(w, 1, -1);
      continue;
    }
    if (pb->Kmax >= 2) do_row_pb(w, 2, r);
    if (pb->Kmax >= 3 && r <= M - 2) do_row_pb(w, 3, r);
  }
  return NULL;
}

typedef struct {
  oracle_point_pb *pts;
  uint64_t n_pts;
  uint64_t *seg_off;
  uint64_t n_seg;
  uint64_t n_cand, n_feas;
} oracle_result_pb;

void oracle_result_pb_free(oracle_result_pb *r) {
  if (!r) return;
  free(r->pts);
  free(r->seg_off);
  free(r);
}

/* Models [model_lo, model_hi), every K <= kmax; batches <= 255 entries. Returns 0 on success. */
int oracle_run_pb(uint32_t n_models, const oracle_model *models, uint32_t n_classes, uint32_t n_batches,
                  const uint32_t *batches, const uint32_t *bw, uint32_t kmax, const uint32_t *slo_us,
                  uint32_t margin_permille, uint32_t model_lo, uint32_t model_hi, oracle_result_pb **out) {
  if (!out || n_classes == 0 || n_batches == 0 || n_batches > 255 || kmax < 1 || kmax > 3 || margin_permille >= 1000)
    return -1;
  if (model_hi > n_models || model_lo > model_hi) return -1;
  oracle_result_pb *res = (oracle_result_pb *)calloc(1, sizeof *res);
  size_t cap_pts = 0;
  const uint32_t C = n_classes, B = n_batches;
  uint64_t total_seg = 0;
  for (uint32_t m = model_lo; m < model_hi; m++) {
    uint64_t p = 1;
    for (uint32_t K = 1; K <= kmax && K <= models[m].n_layers; K++) {
      p *= C;
      total_seg += p;
    }
  }
  res->seg_off = (uint64_t *)calloc(total_seg + 1, sizeof(uint64_t));
  res->n_seg = total_seg;
  uint64_t seg_cursor = 0;
  int nthreads = g_threads > 0 ? g_threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads < 1) nthreads = 1;
  g_pb_batches = batches;
  for (uint32_t m = model_lo; m < model_hi; m++) {
    problem pb;
    memset(&pb, 0, sizeof pb);
    pb.md = &models[m];
    pb.C = C;
    pb.B = B;
    pb.M = models[m].n_layers;
    pb.batches = batches;
    pb.bw = bw;
    pb.T = (int64_t)slo_us[m] * (int64_t)(1000 - margin_permille) / 1000;
    pb.Kmax = (int)kmax;
    const uint32_t M = pb.M;
    pthread_mutex_init(&pb.mu, NULL);
    pb.pre = (int64_t *)malloc(sizeof(int64_t) * (M + 1) * C * B);
    pb.suf = (int64_t *)malloc(sizeof(int64_t) * (M + 1) * C * B);
    for (uint32_t c = 0; c <= M; c++)
      for (uint32_t k = 0; k < C; k++)
        for (uint32_t bi = 0; bi < B; bi++) {
          pb.pre[((size_t)c * C + k) * B + bi] = direct_sum(&pb, k, 0, c, bi);
          pb.suf[((size_t)c * C + k) * B + bi] = direct_sum(&pb, k, c, M, bi);
        }
    pb.Y = (int64_t *)calloc((size_t)(M + 1) * C * C * B, sizeof(int64_t));
    for (uint32_t c = 1; c + 1 <= M; c++)
      for (uint32_t k = 0; k < C; k++)
        for (uint32_t k2 = 0; k2 < C; k2++)
          for (uint32_t bi = 0; bi < B; bi++)
            pb.Y[(((size_t)c * C + k) * C + k2) * B + bi] =
                ceil_div(8 * (int64_t)models[m].act_bytes[c - 1] * (int64_t)batches[bi], (int64_t)bw[k * C + k2]);
    for (uint32_t K = 1; K <= 3; K++) {
      uint32_t p = 1;
      for (uint32_t d = 0; d < K; d++) p *= C;
      pb.nseg[K] = p;
    }
    worker_pb *ws = (worker_pb *)calloc((size_t)nthreads, sizeof(worker_pb));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; t++) {
      ws[t].pb = &pb;
      for (int K = 1; K <= 3; K++) ws[t].segs[K] = (cvec_pb *)calloc(pb.nseg[K], sizeof(cvec_pb));
      pthread_create(&th[t], NULL, worker_pb_main, &ws[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; t++) {
      res->n_cand += ws[t].n_cand;
      res->n_feas += ws[t].n_feas;
    }
    for (uint32_t K = 1; K <= kmax && K <= M; K++) {
      for (uint32_t s = 0; s < pb.nseg[K]; s++) {
        cvec_pb all = {0};
        for (int t = 0; t < nthreads; t++)
          for (size_t i = 0; i < ws[t].segs[K][s].n; i++) cvec_pb_push(&all, &ws[t].segs[K][s].v[i]);
        g_pb_K = (int)K;
        if (all.n) qsort(all.v, all.n, sizeof(cand_pb), cand_pb_cmp);
        int64_t best_n = 0, best_d = 1;
        for (size_t i = 0; i < all.n; i++) {
          const cand_pb *p = &all.v[i];
          int64_t tn, td;
          theta_pb(p, (int)K, &tn, &td);
          if (!theta_gt(tn, td, best_n, best_d)) continue;
          best_n = tn;
          best_d = td;
          if (res->n_pts == cap_pts) {
            cap_pts = cap_pts ? cap_pts * 2 : 1024;
            res->pts = (oracle_point_pb *)realloc(res->pts, cap_pts * sizeof(oracle_point_pb));
          }
          oracle_point_pb *o = &res->pts[res->n_pts++];
          memset(o, 0, sizeof *o);
          o->model = m;
          o->K = (uint8_t)K;
          o->cut[0] = (uint16_t)(K >= 2 ? p->c1 : 0);
          o->cut[1] = (uint16_t)(K >= 3 ? p->c2 : 0);
          uint32_t idx = s;
          for (int d = (int)K - 1; d >= 0; d--) {
            o->cls[d] = (uint8_t)(idx % C);
            idx /= C;
          }
          for (int d = 0; d < 3; d++) {
            if (d >= (int)K) o->cls[d] = 0xFF;
            o->bidx[d] = d < (int)K ? (uint8_t)p->bi[d] : (uint8_t)0xFF;
          }
          o->e2e_us = (uint32_t)p->E;
          for (int d = 0; d < (int)K; d++) o->stage_us[d] = (uint32_t)p->st[d];
        }
        free(all.v);
        res->seg_off[++seg_cursor] = res->n_pts;
      }
    }
    for (int t = 0; t < nthreads; t++) {
      for (int K = 1; K <= 3; K++) {
        for (uint32_t s = 0; s < pb.nseg[K]; s++) free(ws[t].segs[K][s].v);
        free(ws[t].segs[K]);
      }
    }
    free(ws);
    free(th);
    free(pb.pre);
    free(pb.suf);
    free(pb.Y);
    pthread_mutex_destroy(&pb.mu);
  }
  *out = res;
  return 0;
}
