#define _POSIX_C_SOURCE 200809L
/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle. Never linked into, called by, or
 * shipped with the product path (paper_2504_08784_b200/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and only
 * as the checker / CPU baseline.
 *
 * A plain-C restatement of the SLOs-Serve multi-SLO DP planner as implemented by
 * the reference (proj/src/{perf_model,batch_planner,dp_scheduler}.cpp). It is a
 * sequential, line-by-line restatement of the reference ALGORITHM (not of its
 * code structure): std::map/std::vector containers become hash tables and flat
 * arrays, and the two ordering-sensitive pieces of libstdc++ the reference relies
 * on are restated explicitly:
 *   - std::stable_sort (libstdc++ 13 __stable_sort_adaptive: 7-element insertion
 *     chunks, buffered merge loop, forward/backward adaptive merge), because the
 *     chain comparator's eps-tie is not a strict weak ordering
 *     (dp_scheduler.cpp:393-397, 121-124);
 *   - std::map iteration order of per-slot owner bins (ascending owner,
 *     batch_planner.cpp:258, 306).
 * Pinning: tests/test_oracle_pinning.py checks this library against
 * oracle/_ref/libslos_ref.so (the reference compiled from its own sources) and
 * against the committed golden fixtures in tests/golden/ (written by
 * oracle/make_golden.py from the reference), bit-exact on every output field.
 *
 * Built with -O2 -ffp-contract=off (oracle/Makefile) so fp64 rounds like the
 * reference objects. Errors thrown deep inside (infeasible-budget from time2bs,
 * internal-inconsistency) unwind with longjmp; temporaries are leaked on that
 * path (test-only code).
 */
#include <math.h>
#include <setjmp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "slos_planner.h"

#define K_TIME_EPS 1e-9  /* common.hpp:29 */
#define K_VALUE_EPS 1e-9 /* dp_scheduler.cpp:47 */

static int time_le(double a, double b) { return a <= b + K_TIME_EPS; } /* common.hpp:31 */
static int time_lt(double a, double b) { return a < b - K_TIME_EPS; }  /* common.hpp:32 */
/* std::max / std::min semantics (return the first argument on ties / NaN). */
static double dmax(double a, double b) { return (a < b) ? b : a; }
static double dmin(double a, double b) { return (b < a) ? b : a; }
static int64_t imax(int64_t a, int64_t b) { return (a < b) ? b : a; }
static int64_t imin(int64_t a, int64_t b) { return (b < a) ? b : a; }

/* ---------------------------------------------------------------- errors --- */

static __thread char g_err[256];
static __thread jmp_buf* g_jmp;
static __thread int g_jmp_code;

static void fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s: %s", slos_status_slug(code), msg);
  g_jmp_code = code;
  if (g_jmp) longjmp(*g_jmp, 1);
  abort();
}

const char* slos_status_slug(int s) {
  switch (s) {
    case SLOS_OK: return "ok";
    case SLOS_ERR_INVALID_PARAMETERS: return "invalid-parameters";
    case SLOS_ERR_INTERNAL_INCONSISTENCY: return "internal-inconsistency";
    case SLOS_ERR_INFEASIBLE_BUDGET: return "infeasible-budget";
    case SLOS_ERR_CUDA: return "cuda-error";
    case SLOS_ERR_CAPACITY: return "capacity";
    case SLOS_ERR_NO_DEVICE: return "no-device";
    case SLOS_ERR_ALLOC: return "alloc";
    case SLOS_ERR_RANGE: return "range";
    default: return "error";
  }
}
const char* slos_last_error(void) { return g_err; }
const char* slos_backend(void) { return "oracle-c"; }

/* --------------------------------------------------------- small vectors --- */

#define VEC(T) struct { T* v; int64_t n, cap; }
#define VPUSH(vec, x)                                                              \
  do {                                                                             \
    if ((vec).n == (vec).cap) {                                                    \
      (vec).cap = (vec).cap ? 2 * (vec).cap : 16;                                  \
      (vec).v = realloc((vec).v, (size_t)(vec).cap * sizeof(*(vec).v));            \
      if (!(vec).v) abort();                                                       \
    }                                                                              \
    (vec).v[(vec).n++] = (x);                                                      \
  } while (0)
typedef struct { int* v; int64_t n, cap; } ivec_t;
#define VFREE(vec) do { free((vec).v); (vec).v = NULL; (vec).n = (vec).cap = 0; } while (0)

/* ------------------------------------------------ libstdc++ stable_sort --- */
/* Restatement of libstdc++-13 std::stable_sort (bits/stl_algo.h:5023-5052 and
 * helpers) for an element size `sz` and a `less(a, b)` predicate. */

typedef int (*less_fn)(const void* a, const void* b, const void* ctx);

#define ELT(base, i) ((char*)(base) + (size_t)(i) * sz)

static void ss_insertion(char* first, int64_t n, size_t sz, less_fn lt, const void* ctx,
                         char* tmp) {
  if (n <= 0) return;
  for (int64_t i = 1; i < n; ++i) {
    if (lt(ELT(first, i), first, ctx)) {
      memcpy(tmp, ELT(first, i), sz);
      memmove(ELT(first, 1), first, (size_t)i * sz);
      memcpy(first, tmp, sz);
    } else { /* __unguarded_linear_insert */
      memcpy(tmp, ELT(first, i), sz);
      int64_t last = i, next = i - 1;
      while (lt(tmp, ELT(first, next), ctx)) {
        memcpy(ELT(first, last), ELT(first, next), sz);
        last = next;
        --next;
      }
      memcpy(ELT(first, last), tmp, sz);
    }
  }
}

/* __move_merge: returns elements written */
static char* ss_move_merge(char* f1, char* l1, char* f2, char* l2, char* out, size_t sz,
                           less_fn lt, const void* ctx) {
  while (f1 != l1 && f2 != l2) {
    if (lt(f2, f1, ctx)) { memcpy(out, f2, sz); f2 += sz; }
    else { memcpy(out, f1, sz); f1 += sz; }
    out += sz;
  }
  memmove(out, f1, (size_t)(l1 - f1)); out += (l1 - f1);
  memmove(out, f2, (size_t)(l2 - f2)); out += (l2 - f2);
  return out;
}

static void ss_merge_loop(char* first, char* last, char* result, int64_t step, size_t sz,
                          less_fn lt, const void* ctx) {
  const int64_t two = 2 * step;
  while ((last - first) / (int64_t)sz >= two) {
    result = ss_move_merge(first, ELT(first, step), ELT(first, step), ELT(first, two), result,
                           sz, lt, ctx);
    first = ELT(first, two);
  }
  int64_t rest = (last - first) / (int64_t)sz;
  if (rest < step) step = rest;
  ss_move_merge(first, ELT(first, step), ELT(first, step), last, result, sz, lt, ctx);
}

static void ss_merge_sort_with_buffer(char* first, int64_t len, char* buf, size_t sz, less_fn lt,
                                      const void* ctx, char* tmp) {
  int64_t step = 7; /* _S_chunk_size */
  { /* __chunk_insertion_sort */
    char* f = first;
    int64_t left = len;
    while (left >= step) { ss_insertion(f, step, sz, lt, ctx, tmp); f = ELT(f, step); left -= step; }
    ss_insertion(f, left, sz, lt, ctx, tmp);
  }
  while (step < len) {
    ss_merge_loop(first, ELT(first, len), buf, step, sz, lt, ctx);
    step *= 2;
    ss_merge_loop(buf, ELT(buf, len), first, step, sz, lt, ctx);
    step *= 2;
  }
}

static void stable_sort_ls(void* base, int64_t n, size_t sz, less_fn lt, const void* ctx) {
  if (n <= 0) return;
  char* first = (char*)base;
  int64_t half = (n + 1) / 2;
  char* buf = malloc((size_t)half * sz + sz);
  char* tmp = malloc(sz);
  char* middle = ELT(first, half);
  char* last = ELT(first, n);
  ss_merge_sort_with_buffer(first, half, buf, sz, lt, ctx, tmp);
  ss_merge_sort_with_buffer(middle, n - half, buf, sz, lt, ctx, tmp);
  int64_t len1 = half, len2 = n - half;
  if (len1 <= len2) { /* __move_merge_adaptive */
    memcpy(buf, first, (size_t)len1 * sz);
    char *f1 = buf, *l1 = ELT(buf, len1), *f2 = middle, *out = first;
    while (f1 != l1 && f2 != last) {
      if (lt(f2, f1, ctx)) { memcpy(out, f2, sz); f2 += sz; }
      else { memcpy(out, f1, sz); f1 += sz; }
      out += sz;
    }
    if (f1 != l1) memcpy(out, f1, (size_t)(l1 - f1));
  } else { /* __move_merge_adaptive_backward(first, middle, buf, buf_end, last) */
    memcpy(buf, middle, (size_t)len2 * sz);
    char *f1 = first, *l1 = middle, *f2 = buf, *l2 = ELT(buf, len2), *res = last;
    if (f1 == l1) { memmove(res - (l2 - f2), f2, (size_t)(l2 - f2)); goto done; }
    if (f2 == l2) goto done;
    l1 -= sz; l2 -= sz;
    for (;;) {
      if (lt(l2, l1, ctx)) {
        res -= sz; memcpy(res, l1, sz);
        if (f1 == l1) { l2 += sz; memmove(res - (l2 - f2), f2, (size_t)(l2 - f2)); goto done; }
        l1 -= sz;
      } else {
        res -= sz; memcpy(res, l2, sz);
        if (f2 == l2) goto done;
        l2 -= sz;
      }
    }
  }
done:
  free(buf);
  free(tmp);
}

/* -------------------------------------------------------------- planner --- */

struct slos_planner {
  slos_perf_term* terms;
  int n_terms;
  double tpot[SLOS_MAX_TIERS * 4]; /* num_tiers may exceed 8 (rejected by run()) */
  double slow[SLOS_MAX_TIERS * 4];
  int L;
  int tpot_window;
  slos_planner_config cfg;
};

void slos_planner_config_default(slos_planner_config* c) {
  c->max_chunk_tokens = 2048;
  c->max_batch_tokens = 16384;
  c->speculative = 0;
  c->spec_max_len = 8;
  c->spec_alpha = 0.8;
  c->plan_margin = 0.0;
}

#define TRY_BEGIN                       \
  jmp_buf jb__;                         \
  jmp_buf* prev__ = g_jmp;              \
  g_jmp = &jb__;                        \
  if (setjmp(jb__)) {                   \
    g_jmp = prev__;                     \
    return_code__ = g_jmp_code;         \
    goto catch__;                       \
  }
#define TRY_END g_jmp = prev__;

int slos_planner_create(const slos_perf_term* terms, int32_t n_terms, const double* tpot,
                        const double* slow, int32_t n_tiers, int32_t tpot_window,
                        const slos_planner_config* cfg, slos_planner** out) {
  *out = NULL;
  /* PerfModel::PerfModel perf_model.cpp:98-104 */
  if (n_terms < 1) { fail_soft: snprintf(g_err, sizeof g_err, "invalid-parameters"); return SLOS_ERR_INVALID_PARAMETERS; }
  for (int i = 0; i < n_terms; ++i)
    if (terms[i].k1 < 0 || terms[i].k2 < 0 || terms[i].b < 0) goto fail_soft;
  /* SloConfig::validate workload.cpp:18-30 */
  if (n_tiers < 1 || n_tiers > SLOS_MAX_TIERS * 4) goto fail_soft;
  for (int i = 0; i < n_tiers; ++i) {
    if (tpot[i] <= 0) goto fail_soft;
    if (i > 0 && tpot[i] < tpot[i - 1]) goto fail_soft;
    if (slow[i] < 1.0) goto fail_soft;
  }
  if (tpot_window < 1) goto fail_soft;
  slos_planner_config c;
  if (cfg) c = *cfg; else slos_planner_config_default(&c);
  /* BatchPlanner::BatchPlanner batch_planner.cpp:117-123 */
  if (c.max_chunk_tokens < 1 || c.max_batch_tokens < 1) goto fail_soft;
  if (c.max_chunk_tokens > INT32_MAX || c.max_batch_tokens > INT32_MAX) goto fail_soft; /* 32-bit slos_entry */
  if (c.speculative && c.spec_max_len > SLOS_ENTRY_MAX_SPEC) goto fail_soft;             /* 7-bit spec_len */
  if (c.plan_margin < 0) goto fail_soft;
  slos_planner* p = calloc(1, sizeof *p);
  p->terms = malloc(sizeof(slos_perf_term) * (size_t)n_terms);
  memcpy(p->terms, terms, sizeof(slos_perf_term) * (size_t)n_terms);
  p->n_terms = n_terms;
  for (int i = 0; i < n_tiers; ++i) { p->tpot[i] = tpot[i]; p->slow[i] = slow[i]; }
  p->L = n_tiers;
  p->tpot_window = tpot_window;
  p->cfg = c;
  *out = p;
  return SLOS_OK;
}

void slos_planner_destroy(slos_planner* p) {
  if (!p) return;
  free(p->terms);
  free(p);
}

/* PerfModel::predict perf_model.cpp:106-114 */
static double predict(const slos_planner* p, int64_t n, int64_t s) {
  if (n < 0 || s < 0) fail(SLOS_ERR_INVALID_PARAMETERS, "predict needs nonnegative num_tokens and spec_step");
  double best = 0.0;
  for (int i = 0; i < p->n_terms; ++i) {
    const slos_perf_term* t = &p->terms[i];
    double v = t->k1 * (double)n + t->k2 * (double)s + t->b; /* term_value :92-94 */
    best = dmax(best, v);
  }
  return best;
}

/* PerfModel::time2bs perf_model.cpp:116-130 */
static int64_t time2bs(const slos_planner* p, double budget, int64_t spec, int64_t max_tokens) {
  if (max_tokens < 1) fail(SLOS_ERR_INVALID_PARAMETERS, "max_tokens must be positive");
  if (!time_le(predict(p, 1, spec), budget))
    fail(SLOS_ERR_INFEASIBLE_BUDGET, "budget below single-token latency");
  int64_t lo = 1, hi = max_tokens;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (time_le(predict(p, mid, spec), budget)) lo = mid; else hi = mid - 1;
  }
  return lo;
}

/* BatchPlanner::plan_predict / min_slot_s / plan_time2bs / quantize_gap
 * batch_planner.cpp:125-139 */
static double plan_predict(const slos_planner* p, int64_t n, int64_t s) {
  return predict(p, n, s) * (1.0 + p->cfg.plan_margin);
}
static int64_t plan_time2bs(const slos_planner* p, double budget, int64_t s) {
  return time2bs(p, budget / (1.0 + p->cfg.plan_margin), s, p->cfg.max_batch_tokens);
}
static double quantize_gap(double g) {
  if (g <= 0) return 0.0;
  return floor(g * 1000.0 + 1e-6) / 1000.0;
}

/* expected_accepted batch_planner.cpp:32-37 */
static double expected_accepted(double alpha, int sl) {
  if (sl < 1) fail(SLOS_ERR_INVALID_PARAMETERS, "speculation length must be >= 1");
  if (alpha >= 1.0) return (double)sl;
  if (alpha <= 0.0) return 1.0;
  return (1.0 - pow(alpha, sl)) / (1.0 - alpha);
}

double slos_expected_accepted(double alpha, int32_t sl) {
  if (sl < 1) return NAN;
  if (alpha >= 1.0) return (double)sl;
  if (alpha <= 0.0) return 1.0;
  return (1.0 - pow(alpha, sl)) / (1.0 - alpha);
}

/* min_len_covering batch_planner.cpp:42-47 */
static int min_len_covering(double tpot, double target, double alpha, int max_len) {
  for (int sl = 1; sl <= max_len; ++sl)
    if (tpot * expected_accepted(alpha, sl) >= target - K_TIME_EPS) return sl;
  return 0;
}

typedef struct {
  int lengths[SLOS_MAX_TIERS * 4];
  double batch_time_s;
  int64_t batch_capacity;
  int64_t decode_tokens;
  double prefill_throughput;
} spec_plan_t;

static int lens_less(const int* a, const int* b, int n) { /* std::vector<int> operator< */
  for (int i = 0; i < n; ++i) {
    if (a[i] < b[i]) return 1;
    if (b[i] < a[i]) return 0;
  }
  return 0;
}

/* solve_spec_lengths batch_planner.cpp:51-115. Returns 1 with *out, else 0. */
static int solve_spec(const slos_planner* p, const int64_t* counts, int n_counts, double alpha,
                      int max_len, spec_plan_t* out) {
  const int L = p->L;
  if (n_counts != L) fail(SLOS_ERR_INVALID_PARAMETERS, "census width does not match tier count");
  if (alpha <= 0.0 || alpha > 1.0) fail(SLOS_ERR_INVALID_PARAMETERS, "alpha must be in (0, 1]");
  if (max_len < 1) fail(SLOS_ERR_INVALID_PARAMETERS, "spec_max_len must be >= 1");
  int present[SLOS_MAX_TIERS * 4], np = 0;
  for (int l = 0; l < L; ++l) if (counts[l] > 0) present[np++] = l;
  if (np == 0) return 0;
  const double margin = 1.0 + p->cfg.plan_margin;
  int have = 0;
  spec_plan_t best;
  memset(&best, 0, sizeof best);
  for (int bi = 0; bi < np; ++bi) {
    const int bind = present[bi];
    for (int sl_bind = 1; sl_bind <= max_len; ++sl_bind) {
      const double t_batch = p->tpot[bind] * expected_accepted(alpha, sl_bind);
      int lens[SLOS_MAX_TIERS * 4];
      for (int l = 0; l < L; ++l) lens[l] = 0;
      lens[bind] = sl_bind;
      int ok = 1;
      for (int k = 0; k < np; ++k) {
        const int l = present[k];
        if (l == bind) continue;
        const int sl = min_len_covering(p->tpot[l], t_batch, alpha, max_len);
        if (sl == 0) { ok = 0; break; }
        lens[l] = sl;
      }
      if (!ok) continue;
      int64_t spec_step = 0, decode = 0;
      for (int k = 0; k < np; ++k) {
        const int l = present[k];
        spec_step = imax(spec_step, lens[l]);
        decode += counts[l] * lens[l];
      }
      if (!time_le(predict(p, 1, spec_step) * margin, t_batch)) continue;
      int64_t cap = 1;
      {
        int64_t lo = 1, hi = p->cfg.max_batch_tokens;
        while (lo < hi) {
          const int64_t mid = lo + (hi - lo + 1) / 2;
          if (time_le(predict(p, mid, spec_step) * margin, t_batch)) lo = mid; else hi = mid - 1;
        }
        cap = lo;
      }
      if (cap < decode) continue;
      const int64_t budget = imin(cap - decode, p->cfg.max_chunk_tokens);
      const double tpt = (double)budget / t_batch;
      if (!have || tpt > best.prefill_throughput + 1e-12 ||
          (fabs(tpt - best.prefill_throughput) <= 1e-12 &&
           (t_batch < best.batch_time_s - K_TIME_EPS ||
            (fabs(t_batch - best.batch_time_s) <= K_TIME_EPS && lens_less(lens, best.lengths, L))))) {
        have = 1;
        memcpy(best.lengths, lens, sizeof lens);
        best.batch_time_s = t_batch;
        best.batch_capacity = cap;
        best.decode_tokens = decode;
        best.prefill_throughput = tpt;
      }
    }
  }
  if (have) *out = best;
  return have;
}

/* ------------------------------------------------------------ gap tiling --- */

typedef struct {
  int tier;
  int owner;
  double phase;
  int64_t backlog;
  int64_t remaining;
} member_t; /* DecodeMember batch_planner.hpp:19-25 */

typedef struct {
  int64_t counts[SLOS_MAX_TIERS * 4];
  int n_counts;
  member_t* exact;
  int64_t n_exact;
} census_t; /* DecodeCensus batch_planner.hpp:27-34 */

typedef struct { int64_t owner, tok; } owner_tok_t;

typedef struct {
  double start_s, end_s;
  int64_t capacity, spec_step;
  int64_t first_owner, n_owner; /* into gapplan.owners */
  int64_t per_tier[SLOS_MAX_TIERS * 4];
  int64_t decode_tokens, prefill_budget;
} pbatch_t; /* PlannedBatch batch_planner.hpp:38-49 */

typedef struct {
  VEC(pbatch_t) b;
  VEC(owner_tok_t) own;
  int64_t prefill_budget;
  int n_spec;
  int spec_lengths[SLOS_MAX_TIERS * 4];
} gapplan_t; /* GapPlan batch_planner.hpp:51-55 */

static void gp_free(gapplan_t* g) { VFREE(g->b); VFREE(g->own); }
static void gp_reset(gapplan_t* g) { g->b.n = 0; g->own.n = 0; g->prefill_budget = 0; g->n_spec = 0; }

static int census_empty(const census_t* c) { /* batch_planner.cpp:11-16 */
  if (c->n_exact) return 0;
  for (int l = 0; l < c->n_counts; ++l) if (c->counts[l] > 0) return 0;
  return 1;
}

static void merged_counts(const census_t* c, int L, int64_t* out) { /* :24-30 */
  for (int l = 0; l < L; ++l) out[l] = 0;
  for (int l = 0; l < c->n_counts && l < L; ++l) out[l] = c->counts[l];
  for (int64_t i = 0; i < c->n_exact; ++i) out[c->exact[i].tier] += 1;
}

typedef struct {
  double time;
  int owner;
  int tier;
  int late;
  int64_t ins; /* insertion index: the stable-sort tie-break */
} due_t;

static int due_cmp(const void* a, const void* b) { /* batch_planner.cpp:224-227, stable */
  const due_t* x = a;
  const due_t* y = b;
  if (x->late != y->late) return x->late ? -1 : 1;
  if (x->time < y->time) return -1;
  if (y->time < x->time) return 1;
  return (x->ins < y->ins) ? -1 : (x->ins > y->ins);
}

typedef struct { int64_t slot, owner, ins; } bin_t;
static int bin_cmp(const void* a, const void* b) {
  const bin_t* x = a;
  const bin_t* y = b;
  if (x->slot != y->slot) return x->slot < y->slot ? -1 : 1;
  if (x->owner != y->owner) return x->owner < y->owner ? -1 : 1;
  return (x->ins < y->ins) ? -1 : (x->ins > y->ins);
}

typedef struct {
  int64_t dues, slots; /* reference work counters D and S */
} work_t;

/* BatchPlanner::tile_gap_ar batch_planner.cpp:152-313. Returns 1 = plan, 0 = nullopt. */
static int tile_gap_ar(const slos_planner* p, double gap_s, const census_t* c,
                       double due_horizon_s, gapplan_t* plan, work_t* w) {
  gp_reset(plan);
  const int L = p->L;
  const double horizon = dmax(gap_s, due_horizon_s);
  if (gap_s <= K_TIME_EPS) { /* :156-164 */
    int any_due = 0;
    for (int64_t i = 0; i < c->n_exact; ++i) {
      const member_t* m = &c->exact[i];
      if (m->remaining <= 0) continue;
      if (m->backlog > 0) any_due = 1;
      if (horizon > K_TIME_EPS && time_le(m->phase, horizon)) any_due = 1;
    }
    return any_due ? 0 : 1;
  }
  const double min_slot = plan_predict(p, 1, 0);

  int tiers_present[SLOS_MAX_TIERS * 4], n_present = 0; /* :167-175 */
  for (int l = 0; l < L; ++l) {
    const int canonical = l < c->n_counts && c->counts[l] > 0;
    int exact = 0;
    for (int64_t i = 0; i < c->n_exact; ++i)
      if (c->exact[i].tier == l && c->exact[i].remaining > 0) exact = 1;
    if (canonical || exact) tiers_present[n_present++] = l;
  }

  if (n_present == 0) goto prefill_only;

  VEC(due_t) dues = {0};
  for (int64_t i = 0; i < c->n_exact; ++i) { /* :199-213 */
    const member_t* m = &c->exact[i];
    int64_t issued = 0;
    for (int64_t b = 0; b < m->backlog && issued < m->remaining; ++b, ++issued) {
      due_t d = {0.0, m->owner, m->tier, 1, dues.n};
      VPUSH(dues, d);
    }
    const double tpot = p->tpot[m->tier];
    const double phase = dmax(m->phase, 0.0);
    for (double d = phase; time_le(d, horizon) && issued < m->remaining; d += tpot, ++issued) {
      if (d <= K_TIME_EPS) {
        due_t x = {0.0, m->owner, m->tier, 1, dues.n};
        VPUSH(dues, x);
      } else {
        due_t x = {d, m->owner, m->tier, 0, dues.n};
        VPUSH(dues, x);
      }
    }
  }
  for (int l = 0; l < c->n_counts; ++l) { /* :214-220 */
    const double tpot = p->tpot[l];
    for (double d = tpot; time_le(d, gap_s); d += tpot)
      for (int64_t k = 0; k < c->counts[l]; ++k) {
        due_t x = {d, -1, l, 0, dues.n};
        VPUSH(dues, x);
      }
  }
  if (w) w->dues += dues.n;
  if (dues.n == 0) { VFREE(dues); goto prefill_only; } /* :223 */
  qsort(dues.v, (size_t)dues.n, sizeof(due_t), due_cmp);

  double t0 = INFINITY; /* :229-231 */
  for (int k = 0; k < n_present; ++k) t0 = dmin(t0, p->tpot[tiers_present[k]]);
  if (min_slot > t0 + K_TIME_EPS) { VFREE(dues); return 0; }

  double t0_first = t0; /* :234-239 */
  for (int64_t i = 0; i < c->n_exact; ++i) {
    const member_t* m = &c->exact[i];
    if (m->remaining <= 0) continue;
    if (m->phase > K_TIME_EPS && m->phase < t0_first - K_TIME_EPS) t0_first = dmax(m->phase, min_slot);
  }
  VEC(double) ends = {0};
  for (double e = t0_first; time_le(e, gap_s); e += t0) VPUSH(ends, e); /* :240-246 */
  if (ends.n == 0) {
    if (time_le(min_slot, gap_s)) VPUSH(ends, gap_s);
  } else if (gap_s - ends.v[ends.n - 1] >= min_slot - K_TIME_EPS) {
    VPUSH(ends, gap_s);
  }
  const int64_t S = ends.n;
  if (w) w->slots += S;
  if (S == 0) { VFREE(dues); VFREE(ends); return 0; }

  int64_t* cap = malloc(sizeof(int64_t) * (size_t)S);
  int64_t* free_cap = malloc(sizeof(int64_t) * (size_t)S);
  for (int64_t s = 0; s < S; ++s) { /* :250-255 */
    const double dur = ends.v[s] - (s == 0 ? 0.0 : ends.v[s - 1]);
    cap[s] = imin(plan_time2bs(p, dur, 0), p->cfg.max_batch_tokens);
    free_cap[s] = cap[s];
  }
  int64_t* per_tier = calloc((size_t)S * (size_t)L, sizeof(int64_t));
  VEC(bin_t) bins = {0};
  int ok = 1;
  for (int64_t k = 0; k < dues.n; ++k) { /* :261-298 */
    const due_t* d = &dues.v[k];
    int64_t placed = -1;
    if (d->late) {
      for (int64_t s = 0; s < S; ++s) if (free_cap[s] > 0) { placed = s; break; }
    } else {
      int64_t jit = -1, lo = 0, hi = S - 1;
      while (lo <= hi) {
        const int64_t mid = (lo + hi) / 2;
        if (time_le(ends.v[mid], d->time)) { jit = mid; lo = mid + 1; } else { hi = mid - 1; }
      }
      for (int64_t s = jit; s >= 0; --s) if (free_cap[s] > 0) { placed = s; break; }
    }
    if (placed < 0) { ok = 0; break; }
    --free_cap[placed];
    if (d->owner >= 0) { bin_t bn = {placed, d->owner, k}; VPUSH(bins, bn); }
    else per_tier[placed * L + d->tier] += 1;
  }
  if (ok) {
    /* std::map<int,int64_t> per slot: ascending owner (:258, :306) */
    qsort(bins.v, (size_t)bins.n, sizeof(bin_t), bin_cmp);
    int64_t bi = 0;
    for (int64_t s = 0; s < S; ++s) { /* :300-311 */
      pbatch_t b;
      memset(&b, 0, sizeof b);
      b.start_s = s == 0 ? 0.0 : ends.v[s - 1];
      b.end_s = ends.v[s];
      b.capacity = cap[s];
      for (int l = 0; l < L; ++l) b.per_tier[l] = per_tier[s * L + l];
      b.first_owner = plan->own.n;
      while (bi < bins.n && bins.v[bi].slot == s) {
        owner_tok_t ot = {bins.v[bi].owner, 0};
        while (bi < bins.n && bins.v[bi].slot == s && bins.v[bi].owner == ot.owner) { ot.tok++; bi++; }
        VPUSH(plan->own, ot);
      }
      b.n_owner = plan->own.n - b.first_owner;
      b.decode_tokens = cap[s] - free_cap[s];
      b.prefill_budget = imin(free_cap[s], p->cfg.max_chunk_tokens);
      plan->prefill_budget += b.prefill_budget;
      VPUSH(plan->b, b);
    }
  }
  free(cap); free(free_cap); free(per_tier);
  VFREE(bins); VFREE(dues); VFREE(ends);
  return ok;

prefill_only: { /* :177-195 */
    double t = 0.0;
    while (gap_s - t >= min_slot - K_TIME_EPS) {
      int64_t size = plan_time2bs(p, gap_s - t, 0);
      size = imin(size, p->cfg.max_chunk_tokens);
      const double dur = plan_predict(p, size, 0);
      pbatch_t b;
      memset(&b, 0, sizeof b);
      b.start_s = t;
      b.end_s = t + dur;
      b.capacity = size;
      b.first_owner = plan->own.n;
      b.prefill_budget = size;
      VPUSH(plan->b, b);
      plan->prefill_budget += size;
      t += dur;
    }
    return 1;
  }
}

/* BatchPlanner::tile_gap batch_planner.cpp:315-406 */
static int tile_gap(const slos_planner* p, double gap_s, const census_t* c, double due_horizon_s,
                    gapplan_t* out, work_t* w) {
  const int L = p->L;
  int ar_ok = tile_gap_ar(p, gap_s, c, due_horizon_s, out, w);
  if (!p->cfg.speculative || census_empty(c)) return ar_ok;

  int spec_serviceable = 1; /* :320-334 */
  for (int64_t i = 0; i < c->n_exact; ++i) if (c->exact[i].backlog > 0) spec_serviceable = 0;
  if (due_horizon_s > gap_s + K_TIME_EPS) {
    for (int64_t i = 0; i < c->n_exact; ++i) {
      const member_t* m = &c->exact[i];
      if (m->remaining <= 0) continue;
      const double tpot = p->tpot[m->tier];
      int64_t issued = imin(m->backlog, m->remaining);
      for (double d = dmax(m->phase, 0.0); time_le(d, due_horizon_s) && issued < m->remaining;
           d += tpot, ++issued)
        if (!time_le(d, gap_s)) spec_serviceable = 0;
    }
  }
  spec_plan_t sp;
  int have_sp = 0;
  if (spec_serviceable) {
    int64_t mc[SLOS_MAX_TIERS * 4];
    merged_counts(c, L, mc);
    have_sp = solve_spec(p, mc, L, p->cfg.spec_alpha, p->cfg.spec_max_len, &sp);
  }
  if (have_sp) { /* :340-347 */
    for (int64_t i = 0; i < c->n_exact; ++i) {
      if (c->exact[i].remaining > 0 && c->exact[i].phase < sp.batch_time_s - K_TIME_EPS) {
        have_sp = 0;
        break;
      }
    }
  }
  if (!have_sp) return ar_ok;

  const int full = (int)floor(gap_s / sp.batch_time_s + K_TIME_EPS); /* :350 */
  if (full == 0) return ar_ok;

  gapplan_t plan;
  memset(&plan, 0, sizeof plan);
  plan.n_spec = L;
  memcpy(plan.spec_lengths, sp.lengths, sizeof(int) * (size_t)L);
  int64_t* left = malloc(sizeof(int64_t) * (size_t)(c->n_exact + 1));
  for (int64_t i = 0; i < c->n_exact; ++i) left[i] = c->exact[i].remaining;
  for (int k = 0; k < full; ++k) { /* :357-387 */
    pbatch_t b;
    memset(&b, 0, sizeof b);
    b.start_s = k * sp.batch_time_s;
    b.end_s = (k + 1) * sp.batch_time_s;
    b.capacity = sp.batch_capacity;
    b.spec_step = 0;
    int64_t decode = 0;
    for (int l = 0; l < c->n_counts; ++l) {
      const int64_t n = c->counts[l] * sp.lengths[l];
      b.per_tier[l] = n;
      decode += n;
    }
    b.first_owner = plan.own.n;
    for (int64_t i = 0; i < c->n_exact; ++i) {
      const int tier = c->exact[i].tier;
      const int64_t n = imin(left[i], sp.lengths[tier]);
      if (n <= 0) continue;
      owner_tok_t ot = {c->exact[i].owner, n};
      VPUSH(plan.own, ot);
      left[i] -= n;
      decode += n;
      b.spec_step = imax(b.spec_step, sp.lengths[tier]);
    }
    b.n_owner = plan.own.n - b.first_owner;
    for (int l = 0; l < L; ++l)
      if (b.per_tier[l] > 0) b.spec_step = imax(b.spec_step, sp.lengths[l]);
    b.decode_tokens = decode;
    b.prefill_budget = imax(0, imin(sp.batch_capacity - decode, p->cfg.max_chunk_tokens));
    plan.prefill_budget += b.prefill_budget;
    VPUSH(plan.b, b);
  }
  free(left);

  const double used = full * sp.batch_time_s; /* :390-402 */
  if (gap_s - used > K_TIME_EPS) {
    census_t rest;
    memset(&rest, 0, sizeof rest);
    rest.n_counts = L;
    merged_counts(c, L, rest.counts);
    gapplan_t tail;
    memset(&tail, 0, sizeof tail);
    int tok = tile_gap_ar(p, gap_s - used, &rest, 0.0, &tail, w);
    if (!tok) { gp_free(&tail); gp_free(&plan); return ar_ok; }
    for (int64_t k = 0; k < tail.b.n; ++k) {
      pbatch_t b = tail.b.v[k];
      b.start_s += used;
      b.end_s += used;
      plan.prefill_budget += b.prefill_budget;
      b.first_owner = plan.own.n; /* canonical-only tail: no owners */
      b.n_owner = 0;
      VPUSH(plan.b, b);
    }
    gp_free(&tail);
  }
  if (ar_ok && out->prefill_budget >= plan.prefill_budget) { gp_free(&plan); return 1; } /* :404 */
  gp_free(out);
  *out = plan;
  return 1;
}

/* ---------------------------------------------------- hash table helpers --- */

typedef struct {
  uint64_t k0, k1, k2; /* key words */
  int64_t val;
  int32_t used;
  int32_t has;
} hent_t;

typedef struct {
  hent_t* t;
  int64_t cap, n;
} htab_t;

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
static uint64_t hkey(uint64_t a, uint64_t b, uint64_t c) {
  return mix64(a * 0x9E3779B97F4A7C15ULL ^ mix64(b + 0x632BE59BD9B4E019ULL) ^ mix64(c ^ 0x85EBCA77C2B2AE63ULL));
}
static hent_t* hfind(htab_t* h, uint64_t a, uint64_t b, uint64_t c, int insert) {
  if (insert && 2 * (h->n + 1) > h->cap) {
    int64_t ncap = h->cap ? 2 * h->cap : 1024;
    hent_t* nt = calloc((size_t)ncap, sizeof(hent_t));
    for (int64_t i = 0; i < h->cap; ++i)
      if (h->t[i].used) {
        uint64_t q = hkey(h->t[i].k0, h->t[i].k1, h->t[i].k2) & (uint64_t)(ncap - 1);
        while (nt[q].used) q = (q + 1) & (uint64_t)(ncap - 1);
        nt[q] = h->t[i];
      }
    free(h->t);
    h->t = nt;
    h->cap = ncap;
  }
  if (!h->cap) return NULL;
  uint64_t q = hkey(a, b, c) & (uint64_t)(h->cap - 1);
  while (h->t[q].used) {
    if (h->t[q].k0 == a && h->t[q].k1 == b && h->t[q].k2 == c) return &h->t[q];
    q = (q + 1) & (uint64_t)(h->cap - 1);
  }
  if (!insert) return NULL;
  h->t[q].used = 1;
  h->t[q].k0 = a; h->t[q].k1 = b; h->t[q].k2 = c;
  h->n++;
  return &h->t[q];
}

/* ------------------------------------------------------------- scheduler --- */

typedef struct {
  int forced;
  const char* id;
  int32_t ref; /* running index (>=0) or SLOS_PENDING_REF(pending index) */
  double deadline;
  int64_t prefill;
  int tier;
  int64_t memory;
  double value;
} chain_t; /* ChainItem dp_scheduler.cpp:17-25 */

static int chain_less(const void* a, const void* b, const void* ctx) { /* :393-397 */
  (void)ctx;
  const chain_t* x = a;
  const chain_t* y = b;
  if (fabs(x->deadline - y->deadline) > K_TIME_EPS) return x->deadline < y->deadline;
  if (x->forced != y->forced) return x->forced;
  return strcmp(x->id, y->id) < 0;
}

/* pack_add / pack_get dp_scheduler.cpp:28-35 */
static uint64_t pack_add(uint64_t c, int tier) { return c + ((uint64_t)1 << (8 * tier)); }
static int64_t pack_get(uint64_t c, int tier) { return (int64_t)((c >> (8 * tier)) & 0xff); }

typedef struct {
  int item;
  uint64_t counts;
  int64_t mem, pb;
  double value;
  int n_admitted;
  int parent;
  int alive; /* still in its Pareto bucket */
} state_t; /* DpState dp_scheduler.cpp:37-45 */

/* members_at dp_scheduler.cpp:55-91 */
static int64_t members_at(const slos_planner* p, const slos_input* in, double at, double pull,
                          member_t* out) {
  int64_t n = 0;
  for (int32_t i = 0; i < in->n_running; ++i) {
    const slos_running* r = &in->running[i];
    if (r->prefill_remaining > 0 || r->decode_remaining <= 0) continue;
    if (r->decode_tier < 0 || r->decode_tier >= p->L) fail(SLOS_ERR_INVALID_PARAMETERS, "vector::at");
    const double tpot = p->tpot[r->decode_tier];
    int64_t remaining = r->decode_remaining;
    int64_t backlog = imin(r->backlog, remaining);
    double next = r->next_due_s;
    if (at > in->now + K_TIME_EPS) {
      int64_t served = backlog;
      backlog = 0;
      if (time_le(next, at + pull)) {
        int64_t k = (int64_t)floor((at + pull - next) / tpot + K_TIME_EPS) + 1;
        served += k;
        next += (double)k * tpot;
      }
      remaining -= imin(served, remaining);
      if (remaining <= 0) continue;
    } else {
      while (backlog < remaining && time_lt(next - at, pull)) {
        backlog += 1;
        next += tpot;
      }
    }
    member_t m;
    m.tier = r->decode_tier;
    m.phase = dmax(next - at, 0.0);
    m.backlog = backlog;
    m.remaining = remaining;
    m.owner = i;
    out[n++] = m;
  }
  return n;
}

typedef struct {
  int32_t req;
  int32_t spec_len;
  int64_t prefill, decode;
} pentry_t;

typedef struct {
  double start_s, end_s;
  int64_t capacity, spec_step, budget_left;
  int64_t first_entry, n_entries;
} obatch_t;

typedef struct {
  VEC(obatch_t) b;
  VEC(pentry_t) e;
  double exact_until_s;
} splan_t;

static void sp_free(splan_t* s) { VFREE(s->b); VFREE(s->e); }

typedef struct {
  size_t idx;
  double ddl;
  int64_t left;
  const char* id;
} pre_t;
static int pre_less(const void* a, const void* b, const void* ctx) { /* :121-124 */
  (void)ctx;
  const pre_t* x = a;
  const pre_t* y = b;
  if (fabs(x->ddl - y->ddl) > K_TIME_EPS) return x->ddl < y->ddl;
  return strcmp(x->id, y->id) < 0;
}

/* edf_fallback dp_scheduler.cpp:96-188 */
static void edf_fallback(const slos_planner* p, const slos_input* in, splan_t* plan) {
  typedef struct { size_t idx; double tpot, next; int64_t backlog, left; } dec_t;
  pre_t* pre = malloc(sizeof(pre_t) * (size_t)(in->n_running + 1));
  dec_t* dec = malloc(sizeof(dec_t) * (size_t)(in->n_running + 1));
  int64_t npre = 0, ndec = 0;
  for (int32_t i = 0; i < in->n_running; ++i) {
    const slos_running* r = &in->running[i];
    if (r->prefill_remaining > 0) {
      pre_t x = {(size_t)i, r->prefill_deadline, r->prefill_remaining, r->id};
      pre[npre++] = x;
    } else if (r->decode_remaining > 0) {
      if (r->decode_tier < 0 || r->decode_tier >= p->L) fail(SLOS_ERR_INVALID_PARAMETERS, "vector::at");
      dec_t x = {(size_t)i, p->tpot[r->decode_tier], r->next_due_s, imin(r->backlog, r->decode_remaining),
                 r->decode_remaining};
      dec[ndec++] = x;
    }
  }
  stable_sort_ls(pre, npre, sizeof(pre_t), pre_less, NULL);
  double t0 = 0.0;
  for (int64_t k = 0; k < ndec; ++k) t0 = (t0 == 0.0) ? dec[k].tpot : dmin(t0, dec[k].tpot);

  double t = in->now;
  const int64_t chunk_cap = p->cfg.max_chunk_tokens;
  for (int guard = 0; guard < 100000; ++guard) {
    int prefills = 0, decodes = 0;
    for (int64_t k = 0; k < npre; ++k) if (pre[k].left > 0) { prefills = 1; break; }
    for (int64_t k = 0; k < ndec; ++k) if (dec[k].left > 0) { decodes = 1; break; }
    if (!prefills && !decodes) break;
    obatch_t b;
    memset(&b, 0, sizeof b);
    b.start_s = t;
    b.first_entry = plan->e.n;
    int64_t dtok = 0;
    if (decodes) {
      const double slot_end = t + t0;
      for (int64_t k = 0; k < ndec; ++k) {
        dec_t* d = &dec[k];
        if (d->left <= 0) continue;
        int64_t due = imin(d->backlog, d->left);
        d->backlog -= due;
        while (d->left - due > 0 && time_le(d->next, slot_end)) { ++due; d->next += d->tpot; }
        if (due > 0) {
          d->left -= due;
          pentry_t e = {(int32_t)d->idx, 0, 0, due};
          VPUSH(plan->e, e);
          dtok += due;
        }
      }
      const int64_t cap = plan_time2bs(p, t0, 0);
      const int64_t freec = imax(0, imin(cap - dtok, chunk_cap));
      int64_t spent = 0;
      for (int64_t k = 0; k < npre; ++k) {
        if (freec - spent <= 0) break;
        if (pre[k].left <= 0) continue;
        const int64_t s = imin(pre[k].left, freec - spent);
        pre[k].left -= s;
        spent += s;
        pentry_t e = {(int32_t)pre[k].idx, 0, s, 0};
        VPUSH(plan->e, e);
      }
      const int64_t total = dtok + spent;
      const double dur = dmax(t0, total > 0 ? plan_predict(p, total, 0) : 0.0);
      b.end_s = t + dur;
      b.capacity = imax(cap, total);
      b.budget_left = imax(0, freec - spent);
    } else {
      int64_t spent = 0;
      for (int64_t k = 0; k < npre; ++k) {
        if (chunk_cap - spent <= 0) break;
        if (pre[k].left <= 0) continue;
        const int64_t s = imin(pre[k].left, chunk_cap - spent);
        pre[k].left -= s;
        spent += s;
        pentry_t e = {(int32_t)pre[k].idx, 0, s, 0};
        VPUSH(plan->e, e);
      }
      b.end_s = t + plan_predict(p, spent, 0);
      b.capacity = spent;
    }
    t = b.end_s;
    b.n_entries = plan->e.n - b.first_entry;
    VPUSH(plan->b, b);
  }
  plan->exact_until_s = t;
  free(pre);
  free(dec);
}

typedef struct {
  const chain_t* item;
  int64_t prefill_left;
  int64_t decode_assigned;
} bmember_t;

/* chain_member lambda dp_scheduler.cpp:238-252 */
static member_t chain_member(const slos_planner* p, const slos_input* in, const bmember_t* mem,
                             int64_t mi, double a, double span, double pull) {
  const bmember_t* m = &mem[mi];
  const double tpot = p->tpot[m->item->tier];
  member_t e;
  memset(&e, 0, sizeof e);
  e.tier = m->item->tier;
  e.remaining = (int64_t)ceil(span / tpot) + 2;
  double next = m->item->deadline + (double)(m->decode_assigned + 1) * tpot;
  while (e.backlog < e.remaining && time_lt(next - a, pull)) {
    e.backlog += 1;
    next += tpot;
  }
  e.phase = next - a;
  e.owner = (int)(in->n_running + mi);
  return e;
}

/* build_plan dp_scheduler.cpp:196-354 */
static void build_plan(const slos_planner* p, const slos_input* in, const chain_t* chain,
                       const int* sel, int nsel, int* tail_infeasible, splan_t* plan) {
  const int L = p->L;
  const double pull = plan_predict(p, 1, 0);
  *tail_infeasible = 0;
  const int64_t R = in->n_running;
  bmember_t* mem = malloc(sizeof(bmember_t) * (size_t)(nsel + 1));
  for (int k = 0; k < nsel; ++k) { mem[k].item = &chain[sel[k]]; mem[k].prefill_left = chain[sel[k]].prefill; mem[k].decode_assigned = 0; }
  double* bounds = malloc(sizeof(double) * (size_t)(nsel + 2));
  int nb = 0;
  bounds[nb++] = in->now;
  for (int k = 0; k < nsel; ++k)
    if (mem[k].item->deadline > bounds[nb - 1] + K_TIME_EPS) bounds[nb++] = mem[k].item->deadline;

  member_t* ex = malloc(sizeof(member_t) * (size_t)(R + nsel + 1));
  int64_t edf = 0;
  int fill_late = 0;
  gapplan_t gp;
  memset(&gp, 0, sizeof gp);

#define ENTRY_REF(owner) ((owner) < R ? (int32_t)(owner) : mem[(owner)-R].item->ref)
#define ENTRY_TIER(owner) ((owner) < R ? in->running[(owner)].decode_tier : mem[(owner)-R].item->tier)
#define FILL_PREFILL(B, BUDGET)                                                              \
  do {                                                                                       \
    int64_t budget_ = (BUDGET);                                                              \
    while (budget_ > 0) {                                                                    \
      while (edf < nsel && mem[edf].prefill_left == 0) ++edf;                                \
      if (edf == nsel) break;                                                                \
      bmember_t* m_ = &mem[edf];                                                             \
      int64_t spend_ = imin(budget_, m_->prefill_left);                                      \
      m_->prefill_left -= spend_;                                                            \
      budget_ -= spend_;                                                                     \
      if (m_->prefill_left == 0 && (B).end_s > m_->item->deadline + K_TIME_EPS) fill_late = 1; \
      pentry_t e_ = {m_->item->ref, 0, spend_, 0};                                           \
      VPUSH(plan->e, e_);                                                                    \
    }                                                                                        \
    (B).budget_left = budget_;                                                               \
  } while (0)

  for (int k = 0; k + 1 < nb; ++k) { /* :262-293 */
    const double a = bounds[k];
    const double raw = bounds[k + 1] - a;
    const double len = quantize_gap(raw);
    census_t cen;
    memset(&cen, 0, sizeof cen);
    cen.n_counts = L;
    cen.exact = ex;
    cen.n_exact = members_at(p, in, a, pull, ex);
    for (int mi = 0; mi < nsel; ++mi)
      if (mem[mi].item->deadline <= a + K_TIME_EPS)
        ex[cen.n_exact++] = chain_member(p, in, mem, mi, a, raw + pull, pull);
    if (!tile_gap(p, len, &cen, raw + pull, &gp, NULL)) {
      *tail_infeasible = 1;
      goto out;
    }
    for (int64_t bi = 0; bi < gp.b.n; ++bi) {
      const pbatch_t* pb = &gp.b.v[bi];
      obatch_t o;
      memset(&o, 0, sizeof o);
      o.start_s = a + pb->start_s;
      o.end_s = a + pb->end_s;
      o.capacity = pb->capacity;
      o.spec_step = pb->spec_step;
      o.first_entry = plan->e.n;
      const int spec_batch = pb->spec_step > 0 && gp.n_spec > 0;
      for (int64_t q = 0; q < pb->n_owner; ++q) {
        const int64_t owner = gp.own.v[pb->first_owner + q].owner;
        const int64_t tok = gp.own.v[pb->first_owner + q].tok;
        const int sl = spec_batch ? gp.spec_lengths[ENTRY_TIER(owner)] : 0;
        if (owner >= R) mem[owner - R].decode_assigned += tok;
        pentry_t e = {ENTRY_REF(owner), sl, 0, tok};
        VPUSH(plan->e, e);
      }
      FILL_PREFILL(o, pb->prefill_budget);
      o.n_entries = plan->e.n - o.first_entry;
      VPUSH(plan->b, o);
    }
  }
  {
    int shortfall = fill_late; /* :294-300 */
    for (int k = 0; k < nsel; ++k) if (mem[k].prefill_left > 0) shortfall = 1;
    if (shortfall) { *tail_infeasible = 1; goto out; }
  }
  { /* decode tail :302-349 */
    const double t_last = bounds[nb - 1];
    census_t tail;
    memset(&tail, 0, sizeof tail);
    tail.n_counts = L;
    tail.exact = ex;
    tail.n_exact = members_at(p, in, t_last, pull, ex);
    double tail_len = 0.0, max_tpot = 0.0;
    for (int l = 0; l < L; ++l) max_tpot = dmax(max_tpot, p->tpot[l]);
    for (int64_t i = 0; i < tail.n_exact; ++i) {
      const double tpot = p->tpot[ex[i].tier];
      tail_len = dmax(tail_len, ex[i].phase + (double)ex[i].remaining * tpot);
    }
    if (nsel > 0 || in->tail_horizon_s > K_TIME_EPS) {
      double capv = dmax(2.0 * max_tpot, in->tail_horizon_s);
      for (int64_t i = 0; i < tail.n_exact; ++i) {
        if (ex[i].remaining <= 0) continue;
        capv = dmax(capv, ex[i].phase + p->tpot[ex[i].tier]);
      }
      tail_len = dmin(tail_len, capv);
    }
    for (int mi = 0; mi < nsel; ++mi) ex[tail.n_exact++] = chain_member(p, in, mem, mi, t_last, tail_len, pull);
    const double tlen = quantize_gap(tail_len);
    if (tlen > K_TIME_EPS && tail.n_exact > 0) {
      if (!tile_gap(p, tlen, &tail, tail_len, &gp, NULL)) {
        *tail_infeasible = 1;
      } else {
        for (int64_t bi = 0; bi < gp.b.n; ++bi) {
          const pbatch_t* pb = &gp.b.v[bi];
          obatch_t o;
          memset(&o, 0, sizeof o);
          o.start_s = t_last + pb->start_s;
          o.end_s = t_last + pb->end_s;
          o.capacity = pb->capacity;
          o.spec_step = pb->spec_step;
          o.first_entry = plan->e.n;
          const int spec_batch = pb->spec_step > 0 && gp.n_spec > 0;
          for (int64_t q = 0; q < pb->n_owner; ++q) {
            const int64_t owner = gp.own.v[pb->first_owner + q].owner;
            const int64_t tok = gp.own.v[pb->first_owner + q].tok;
            const int sl = spec_batch ? gp.spec_lengths[ENTRY_TIER(owner)] : 0;
            pentry_t e = {ENTRY_REF(owner), sl, 0, tok};
            VPUSH(plan->e, e);
          }
          FILL_PREFILL(o, pb->prefill_budget);
          o.n_entries = plan->e.n - o.first_entry;
          VPUSH(plan->b, o);
        }
      }
    }
  }
  plan->exact_until_s = plan->b.n == 0 ? in->now : plan->b.v[plan->b.n - 1].end_s;
out:
#undef ENTRY_REF
#undef ENTRY_TIER
#undef FILL_PREFILL
  gp_free(&gp);
  free(mem);
  free(bounds);
  free(ex);
}

/* --------------------------------------------------------- result output --- */

static void emit_result(const slos_input* in, int infeasible, double value, const int32_t* adm,
                        int nadm, const int32_t* dec, int ndec, const splan_t* plan,
                        const slos_counters* ctr, slos_result* out) {
  (void)in;
  for (int64_t k = 0; k < plan->e.n; ++k) { /* the 8-byte slos_entry (include/slos_planner.h) */
    const int bad = plan->e.v[k].prefill > INT32_MAX || plan->e.v[k].decode > INT32_MAX ||
                    plan->e.v[k].prefill < INT32_MIN || plan->e.v[k].decode < INT32_MIN ||
                    plan->e.v[k].spec_len < 0 || plan->e.v[k].spec_len > SLOS_ENTRY_MAX_SPEC;
    const int both = plan->e.v[k].prefill != 0 && (plan->e.v[k].decode != 0 || plan->e.v[k].spec_len != 0);
    if (bad || both) {
      memset(out, 0, sizeof *out);
      out->status = bad ? SLOS_ERR_INVALID_PARAMETERS : SLOS_ERR_INTERNAL_INCONSISTENCY;
      return;
    }
  }
  size_t bytes = sizeof(obatch_t) + sizeof(slos_batch) * (size_t)plan->b.n +
                 sizeof(slos_entry) * (size_t)plan->e.n + sizeof(int32_t) * (size_t)(nadm + ndec) + 64;
  char* mem = calloc(1, bytes);
  slos_batch* b = (slos_batch*)mem;
  slos_entry* e = (slos_entry*)(b + plan->b.n);
  int32_t* ids = (int32_t*)(e + plan->e.n);
  for (int64_t k = 0; k < plan->b.n; ++k) {
    b[k].start_s = plan->b.v[k].start_s;
    b[k].end_s = plan->b.v[k].end_s;
    b[k].capacity_tokens = plan->b.v[k].capacity;
    b[k].spec_step = plan->b.v[k].spec_step;
    b[k].prefill_budget_left = plan->b.v[k].budget_left;
    b[k].first_entry = plan->b.v[k].first_entry;
    b[k].n_entries = plan->b.v[k].n_entries;
  }
  for (int64_t k = 0; k < plan->e.n; ++k) {
    e[k] = (plan->e.v[k].decode != 0 || plan->e.v[k].spec_len != 0)
               ? slos_entry_decode(plan->e.v[k].req, (int32_t)plan->e.v[k].decode, plan->e.v[k].spec_len)
               : slos_entry_prefill(plan->e.v[k].req, (int32_t)plan->e.v[k].prefill);
  }
  for (int k = 0; k < nadm; ++k) ids[k] = adm[k];
  for (int k = 0; k < ndec; ++k) ids[nadm + k] = dec[k];
  out->status = SLOS_OK;
  out->running_set_infeasible = infeasible;
  out->admitted_value = value;
  out->n_admitted = nadm;
  out->n_declined = ndec;
  out->n_deferred = 0;
  out->admitted = ids;
  out->declined = ids + nadm;
  out->deferred = ids + nadm + ndec;
  out->n_batches = plan->b.n;
  out->batches = b;
  out->n_entries = plan->e.n;
  out->entries = e;
  out->exact_until_s = plan->exact_until_s;
  if (ctr) out->counters = *ctr;
  out->owner_ = mem;
}

/* SloScheduler::run dp_scheduler.cpp:364-558 */
static void run(const slos_planner* p, const slos_input* in, int unit_value, slos_result* out) {
  const int L = p->L;
  if (L > 8) fail(SLOS_ERR_INVALID_PARAMETERS, "at most 8 SLO tiers supported");
  if (in->n_running >= SLOS_ENTRY_MAX_REQS || in->n_pending >= SLOS_ENTRY_MAX_REQS) /* 24-bit entry refs */
    fail(SLOS_ERR_INVALID_PARAMETERS, "too many requests for the plan entry format");
  const int64_t cap_chain = (int64_t)in->n_running + in->n_pending;
  chain_t* chain = malloc(sizeof(chain_t) * (size_t)(cap_chain + 1));
  int N = 0;
  for (int32_t i = 0; i < in->n_running; ++i) { /* :370-379 */
    const slos_running* r = &in->running[i];
    if (r->prefill_remaining <= 0) continue;
    chain_t it;
    memset(&it, 0, sizeof it);
    it.forced = 1;
    it.id = r->id;
    it.ref = i;
    it.deadline = r->prefill_deadline;
    it.prefill = r->prefill_remaining;
    it.tier = r->decode_tier;
    chain[N++] = it;
  }
  for (int32_t i = 0; i < in->n_pending; ++i) { /* :380-389 */
    const slos_pending* q = &in->pending[i];
    chain_t it;
    memset(&it, 0, sizeof it);
    it.id = q->id;
    it.ref = SLOS_PENDING_REF(i);
    it.deadline = q->prefill_deadline;
    it.prefill = q->prefill_tokens;
    it.tier = q->decode_tier;
    it.memory = q->memory_units;
    it.value = unit_value ? 1.0 : q->value;
    chain[N++] = it;
  }
  if (N > 250) fail(SLOS_ERR_INVALID_PARAMETERS, "admission chain too large");
  for (int i = 0; i < N; ++i)
    if (chain[i].tier < 0 || chain[i].tier >= L) fail(SLOS_ERR_INVALID_PARAMETERS, "bad SLO tier");
  stable_sort_ls(chain, N, sizeof(chain_t), chain_less, NULL);

  int last_forced = -1; /* :399-408 */
  int* floor_at = malloc(sizeof(int) * (size_t)(N + 1));
  for (int i = 0; i < N; ++i) { floor_at[i] = last_forced; if (chain[i].forced) last_forced = i; }
  int64_t* suffix = calloc((size_t)N + 1, sizeof(int64_t));
  for (int i = N - 1; i >= 0; --i) suffix[i] = suffix[i + 1] + chain[i].prefill;
  const int64_t mem_budget = in->memory_total - in->memory_standard_resident;

  const double pull = plan_predict(p, 1, 0); /* :413-436 */
  int have_running_decode = 0;
  for (int32_t i = 0; i < in->n_running; ++i)
    if (in->running[i].prefill_remaining <= 0 && in->running[i].decode_remaining > 0) have_running_decode = 1;
  htab_t memo = {0};
  member_t* ex = malloc(sizeof(member_t) * (size_t)(in->n_running + 1));
  gapplan_t gp;
  memset(&gp, 0, sizeof gp);
  slos_counters ctr;
  memset(&ctr, 0, sizeof ctr);
  work_t work = {0, 0};

  VEC(state_t) arena = {0};
  { state_t s0 = {-1, 0, 0, 0, 0.0, 0, -1, 1}; VPUSH(arena, s0); }
  htab_t buckets = {0}; /* (item, counts) -> index into bucket lists */
  VEC(ivec_t) blist = {0};
  VEC(ivec_t) states_at = {0};
  for (int i = 0; i <= N; ++i) { ivec_t e = {0}; VPUSH(states_at, e); }
  VPUSH(states_at.v[0], 0);
  {
    hent_t* h = hfind(&buckets, (uint64_t)(int64_t)-1, 0, 0, 1);
    h->has = 1;
    h->val = blist.n;
    ivec_t e = {0};
    VPUSH(e, 0);
    VPUSH(blist, e);
  }

  for (int i = 0; i < N; ++i) { /* :467-502 */
    const chain_t* it = &chain[i];
    for (int j = floor_at[i]; j < i; ++j) {
      const int64_t nsrc = states_at.v[j + 1].n; /* snapshot: inserts go to states_at[i+1] */
      for (int64_t si = 0; si < nsrc; ++si) {
        const int sidx = states_at.v[j + 1].v[si];
        const state_t s = arena.v[sidx];
        if (!s.alive) continue; /* :475-478 */
        ctr.transitions++;
        const double t_j = (j < 0) ? in->now : chain[j].deadline;
        /* gap_budget :418-436 */
        const double diff = it->deadline - t_j;
        const double raw = dmax(0.0, diff);
        const double len = quantize_gap(raw);
        int has;
        int64_t dpb = 0;
        uint64_t k0, k1;
        if (!have_running_decode) { /* BatchPlanner::prefill_budget :408-422 (pure memo) */
          const double gap = quantize_gap(len);
          k0 = 0xFFFFFFFFFFFFFFFFULL;
          k1 = (uint64_t)llround(gap * 1000.0);
        } else {
          k0 = (uint64_t)llround(t_j * 1e6);
          k1 = (uint64_t)llround(raw * 1e6);
        }
        hent_t* h = hfind(&memo, k0, k1, s.counts, 0);
        if (h) {
          has = h->has;
          dpb = h->val;
        } else {
          ctr.gap_evals++;
          census_t cen;
          memset(&cen, 0, sizeof cen);
          cen.n_counts = L;
          for (int l = 0; l < L; ++l) cen.counts[l] = pack_get(s.counts, l);
          int okg;
          if (!have_running_decode) {
            const double gap = quantize_gap(len);
            okg = tile_gap(p, gap, &cen, 0.0, &gp, &work);
          } else {
            cen.exact = ex;
            cen.n_exact = members_at(p, in, t_j, pull, ex);
            okg = tile_gap(p, len, &cen, raw + pull, &gp, &work);
          }
          has = okg;
          dpb = okg ? gp.prefill_budget : 0;
          h = hfind(&memo, k0, k1, s.counts, 1);
          h->has = has;
          h->val = dpb;
        }
        if (!has) continue;
        const int64_t avail = s.pb + dpb;
        if (avail < it->prefill) continue;
        state_t ns;
        ns.item = i;
        ns.counts = pack_add(s.counts, it->tier);
        if (pack_get(ns.counts, it->tier) > 250) fail(SLOS_ERR_INTERNAL_INCONSISTENCY, "tier count overflow");
        if (it->forced) {
          ns.mem = s.mem;
        } else {
          ns.mem = s.mem + it->memory;
          if (ns.mem > mem_budget) continue;
        }
        ns.pb = imin(avail - it->prefill, suffix[i + 1]);
        ns.value = s.value + (it->forced ? 0.0 : it->value);
        ns.n_admitted = s.n_admitted + (it->forced ? 0 : 1);
        ns.parent = sidx;
        ns.alive = 1;
        /* try_insert :445-465 */
        hent_t* bh = hfind(&buckets, (uint64_t)(int64_t)ns.item, ns.counts, 0, 1);
        if (!bh->has) {
          bh->has = 1;
          bh->val = blist.n;
          ivec_t e = {0};
          VPUSH(blist, e);
        }
        int64_t bidx = bh->val;
        int reject = 0;
        for (int64_t q = 0; q < blist.v[bidx].n; ++q) {
          const state_t* e = &arena.v[blist.v[bidx].v[q]];
          if (e->value >= ns.value - K_VALUE_EPS && e->mem <= ns.mem && e->pb >= ns.pb) {
            const int equal = fabs(e->value - ns.value) <= K_VALUE_EPS && e->mem == ns.mem && e->pb == ns.pb;
            if (!equal || e->n_admitted >= ns.n_admitted) { reject = 1; break; }
          }
        }
        if (reject) continue;
        int64_t wq = 0;
        for (int64_t q = 0; q < blist.v[bidx].n; ++q) {
          const int idx = blist.v[bidx].v[q];
          state_t* e = &arena.v[idx];
          if (ns.value >= e->value - K_VALUE_EPS && ns.mem <= e->mem && ns.pb >= e->pb) {
            e->alive = 0;
          } else {
            blist.v[bidx].v[wq++] = idx;
          }
        }
        blist.v[bidx].n = wq;
        const int id = (int)arena.n;
        VPUSH(arena, ns);
        VPUSH(blist.v[bidx], id);
        VPUSH(states_at.v[i + 1], id);
      }
    }
  }
  ctr.dues = work.dues;
  ctr.slots = work.slots;
  ctr.states = arena.n - 1;

  int best = -1; /* :504-522 */
  for (int item = (last_forced > -1 ? last_forced : -1); item < N; ++item) {
    if (item == -1 && last_forced != -1) continue;
    for (int64_t q = 0; q < states_at.v[item + 1].n; ++q) {
      const int idx = states_at.v[item + 1].v[q];
      if (!arena.v[idx].alive) continue;
      int better = 0;
      if (best < 0) better = 1;
      else {
        const state_t* x = &arena.v[idx];
        const state_t* y = &arena.v[best];
        if (fabs(x->value - y->value) > K_VALUE_EPS) better = x->value > y->value;
        else if (x->n_admitted != y->n_admitted) better = x->n_admitted > y->n_admitted;
        else if (x->mem != y->mem) better = x->mem < y->mem;
        else if (x->pb != y->pb) better = x->pb > y->pb;
        else better = idx < best;
      }
      if (better) best = idx;
    }
  }

  splan_t plan;
  memset(&plan, 0, sizeof plan);
  int32_t* adm = malloc(sizeof(int32_t) * (size_t)(N + in->n_pending + 1));
  int32_t* dec = malloc(sizeof(int32_t) * (size_t)(N + in->n_pending + 1));
  int nadm = 0, ndec = 0;
  double value = 0.0;
  int infeasible = 0;
  if (best < 0) { /* :525-530 */
    infeasible = 1;
    for (int32_t q = 0; q < in->n_pending; ++q) dec[ndec++] = q;
    edf_fallback(p, in, &plan);
  } else {
    int* sel = malloc(sizeof(int) * (size_t)(N + 1)); /* :532-544 */
    int nsel = 0;
    for (int s = best; s > 0; s = arena.v[s].parent) sel[nsel++] = arena.v[s].item;
    for (int a = 0, b = nsel - 1; a < b; ++a, --b) { int t = sel[a]; sel[a] = sel[b]; sel[b] = t; }
    char* in_chain = calloc((size_t)N + 1, 1);
    for (int k = 0; k < nsel; ++k) in_chain[sel[k]] = 1;
    for (int k = 0; k < nsel; ++k)
      if (!chain[sel[k]].forced) { adm[nadm++] = -chain[sel[k]].ref - 1; value += chain[sel[k]].value; }
    for (int q = 0; q < N; ++q)
      if (!chain[q].forced && !in_chain[q]) dec[ndec++] = -chain[q].ref - 1;
    int tail_infeasible = 0;
    build_plan(p, in, chain, sel, nsel, &tail_infeasible, &plan);
    if (tail_infeasible) { /* :546-556 */
      sp_free(&plan);
      memset(&plan, 0, sizeof plan);
      infeasible = 1;
      nadm = 0;
      ndec = 0;
      value = 0.0;
      for (int32_t q = 0; q < in->n_pending; ++q) dec[ndec++] = q;
      edf_fallback(p, in, &plan);
    }
    free(sel);
    free(in_chain);
  }
  emit_result(in, infeasible, value, adm, nadm, dec, ndec, &plan, &ctr, out);

  sp_free(&plan);
  free(adm); free(dec);
  for (int64_t q = 0; q < blist.n; ++q) VFREE(blist.v[q]);
  VFREE(blist);
  for (int64_t q = 0; q < states_at.n; ++q) VFREE(states_at.v[q]);
  VFREE(states_at);
  VFREE(arena);
  free(buckets.t);
  free(memo.t);
  gp_free(&gp);
  free(ex);
  free(chain);
  free(floor_at);
  free(suffix);
}

/* ------------------------------------------------------------ C-ABI entry --- */

int slos_plan(slos_planner* p, const slos_input* in, int32_t unit_value, slos_result* out) {
  memset(out, 0, sizeof *out);
  int return_code__ = SLOS_OK;
  TRY_BEGIN
  run(p, in, unit_value, out);
  TRY_END
  return SLOS_OK;
catch__:
  memset(out, 0, sizeof *out);
  out->status = return_code__;
  return return_code__;
}

int slos_plan_batch(slos_planner* const* planners, int32_t n, const slos_input* inputs,
                    int32_t unit_value, slos_result* outs, void* stream) {
  (void)stream;
  for (int32_t k = 0; k < n; ++k) slos_plan(planners[k], &inputs[k], unit_value, &outs[k]);
  return SLOS_OK;
}

void slos_result_free(slos_result* r) {
  if (!r) return;
  free(r->owner_);
  memset(r, 0, sizeof *r);
}

static void export_gap(const slos_planner* p, int ok, const gapplan_t* g, slos_gap_result* out) {
  memset(out, 0, sizeof *out);
  out->status = SLOS_OK;
  if (!ok) return;
  out->feasible = 1;
  out->prefill_budget = g->prefill_budget;
  out->n_spec_lengths = g->n_spec;
  for (int l = 0; l < g->n_spec && l < SLOS_MAX_TIERS; ++l) out->spec_lengths[l] = g->spec_lengths[l];
  char* mem = calloc(1, sizeof(slos_gap_batch) * (size_t)g->b.n + sizeof(int64_t) * 2 * (size_t)g->own.n + 64);
  slos_gap_batch* bs = (slos_gap_batch*)mem;
  int64_t* own = (int64_t*)(bs + g->b.n);
  for (int64_t k = 0; k < g->b.n; ++k) {
    const pbatch_t* b = &g->b.v[k];
    bs[k].start_s = b->start_s;
    bs[k].end_s = b->end_s;
    bs[k].capacity_tokens = b->capacity;
    bs[k].spec_step = b->spec_step;
    bs[k].decode_tokens = b->decode_tokens;
    bs[k].prefill_budget = b->prefill_budget;
    for (int l = 0; l < p->L && l < SLOS_MAX_TIERS; ++l) bs[k].decode_per_tier[l] = b->per_tier[l];
    bs[k].first_owner = b->first_owner;
    bs[k].n_owners = b->n_owner;
  }
  for (int64_t k = 0; k < g->own.n; ++k) { own[2 * k] = g->own.v[k].owner; own[2 * k + 1] = g->own.v[k].tok; }
  out->n_batches = g->b.n;
  out->batches = bs;
  out->n_owner_pairs = g->own.n;
  out->owner_tokens = own;
  out->owner_ = mem;
}

int slos_tile_gap_batch(slos_planner* p, int32_t n, const slos_gap_query* q, slos_gap_result* outs) {
  for (int32_t k = 0; k < n; ++k) {
    gapplan_t g;
    memset(&g, 0, sizeof g);
    member_t* ex = malloc(sizeof(member_t) * (size_t)(q[k].n_exact + 1));
    census_t c;
    memset(&c, 0, sizeof c);
    c.n_counts = p->L;
    for (int l = 0; l < p->L && l < SLOS_MAX_TIERS; ++l) c.counts[l] = q[k].counts_per_tier[l];
    int return_code__ = SLOS_OK;
    int ok = 0;
    TRY_BEGIN
    if (q[k].mode != SLOS_GAP_PREFILL_BUDGET) {
      for (int32_t i = 0; i < q[k].n_exact; ++i) {
        ex[i].tier = q[k].exact[i].tier;
        ex[i].owner = q[k].exact[i].owner;
        ex[i].phase = q[k].exact[i].phase_s;
        ex[i].backlog = q[k].exact[i].backlog;
        ex[i].remaining = q[k].exact[i].remaining;
      }
      c.exact = ex;
      c.n_exact = q[k].n_exact;
      if (q[k].mode == SLOS_GAP_TILE_AR) ok = tile_gap_ar(p, q[k].gap_s, &c, q[k].due_horizon_s, &g, NULL);
      else ok = tile_gap(p, q[k].gap_s, &c, q[k].due_horizon_s, &g, NULL);
      export_gap(p, ok, &g, &outs[k]);
    } else {
      const double gap = quantize_gap(q[k].gap_s); /* prefill_budget :408-422 */
      ok = tile_gap(p, gap, &c, 0.0, &g, NULL);
      memset(&outs[k], 0, sizeof outs[k]);
      outs[k].feasible = ok;
      outs[k].prefill_budget = ok ? g.prefill_budget : 0;
    }
    TRY_END
    gp_free(&g);
    free(ex);
    continue;
  catch__: /* g was modified after setjmp: leak it rather than read it */
    memset(&outs[k], 0, sizeof outs[k]);
    outs[k].status = return_code__;
    free(ex);
  }
  return SLOS_OK;
}

void slos_gap_result_free(slos_gap_result* r) {
  if (!r) return;
  free(r->owner_);
  memset(r, 0, sizeof *r);
}

int slos_time2bs_batch(slos_planner* p, int32_t n, const double* budget, const int64_t* spec,
                       int64_t max_tokens, int64_t* out, int32_t* status) {
  for (int32_t k = 0; k < n; ++k) {
    int return_code__ = SLOS_OK;
    out[k] = 0;
    TRY_BEGIN
    out[k] = time2bs(p, budget[k], spec ? spec[k] : 0, max_tokens);
    TRY_END
    status[k] = SLOS_OK;
    continue;
  catch__:
    status[k] = return_code__;
  }
  return SLOS_OK;
}

int slos_predict_batch(slos_planner* p, int32_t n, const int64_t* tokens, const int64_t* spec,
                       double* out) {
  int return_code__ = SLOS_OK;
  TRY_BEGIN
  for (int32_t k = 0; k < n; ++k) out[k] = predict(p, tokens[k], spec ? spec[k] : 0);
  TRY_END
  return SLOS_OK;
catch__:
  return return_code__;
}

int slos_solve_spec_lengths(slos_planner* p, const int64_t* counts, int32_t n_tiers, double alpha,
                            int32_t max_len, slos_spec_plan* out) {
  memset(out, 0, sizeof *out);
  int return_code__ = SLOS_OK;
  TRY_BEGIN
  spec_plan_t sp;
  if (solve_spec(p, counts, n_tiers, alpha, max_len, &sp)) {
    out->feasible = 1;
    for (int l = 0; l < p->L && l < SLOS_MAX_TIERS; ++l) out->lengths[l] = sp.lengths[l];
    out->batch_time_s = sp.batch_time_s;
    out->batch_capacity = sp.batch_capacity;
    out->decode_tokens = sp.decode_tokens;
    out->prefill_throughput = sp.prefill_throughput;
  }
  TRY_END
  return SLOS_OK;
catch__:
  return return_code__;
}


/* device-resident workspace API: synchronous CPU version (test infrastructure) */
struct slos_workspace {
  slos_planner* const* planners;
  const slos_input* inputs;
  int32_t n;
  int32_t unit_value;
  slos_result* res; /* results of the last solve, owned until download */
  double solve_ms;
};
static void ws_clear(slos_workspace* b) {
  if (b->res) {
    for (int32_t k = 0; k < b->n; ++k) slos_result_free(&b->res[k]);
    free(b->res);
    b->res = NULL;
  }
}
int slos_workspace_create(slos_workspace** out) {
  *out = calloc(1, sizeof(slos_workspace));
  return *out ? SLOS_OK : SLOS_ERR_ALLOC;
}
void slos_workspace_destroy(slos_workspace* b) {
  if (!b) return;
  ws_clear(b);
  free(b);
}
int slos_workspace_upload(slos_workspace* b, slos_planner* const* planners, int32_t n, const slos_input* inputs,
                          int32_t unit_value, slos_result* outs, void* stream) {
  (void)stream;
  ws_clear(b);
  for (int32_t k = 0; k < n; ++k) memset(&outs[k], 0, sizeof outs[k]);
  b->planners = planners;
  b->inputs = inputs;
  b->n = n;
  b->unit_value = unit_value;
  return SLOS_OK;
}
int slos_workspace_solve(slos_workspace* b, void* stream) {
  struct timespec t0, t1;
  ws_clear(b);
  b->res = calloc((size_t)(b->n > 0 ? b->n : 1), sizeof(slos_result));
  clock_gettime(CLOCK_MONOTONIC, &t0);
  int r = slos_plan_batch(b->planners, b->n, b->inputs, b->unit_value, b->res, stream);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  b->solve_ms = (double)(t1.tv_sec - t0.tv_sec) * 1e3 + (double)(t1.tv_nsec - t0.tv_nsec) * 1e-6;
  return r;
}
int slos_workspace_download(slos_workspace* b, slos_result* outs, void* stream) {
  (void)stream;
  if (!b->res) return SLOS_ERR_INVALID_PARAMETERS;
  memcpy(outs, b->res, sizeof(slos_result) * (size_t)b->n);
  free(b->res);
  b->res = NULL;
  return SLOS_OK;
}
int slos_workspace_records(slos_workspace* b, slos_record* out, void* stream) {
  (void)stream;
  if (!b->res) return SLOS_ERR_INVALID_PARAMETERS;
  for (int32_t k = 0; k < b->n; ++k) {
    const slos_result* r = &b->res[k];
    slos_record x;
    memset(&x, 0, sizeof x);
    x.status = r->status;
    x.running_set_infeasible = r->running_set_infeasible;
    x.n_admitted = r->n_admitted;
    x.n_declined = r->n_declined;
    x.admitted_value = r->admitted_value;
    x.n_batches = r->n_batches;
    x.n_entries = r->n_entries;
    x.exact_until_s = r->exact_until_s;
    x.counters = r->counters;
    out[k] = x;
  }
  return SLOS_OK;
}
int slos_workspace_launches(slos_workspace* b, int64_t* n) {
  (void)b;
  *n = 0; /* no device kernels in the CPU checker */
  return SLOS_OK;
}

int slos_workspace_stage_ms(slos_workspace* b, float* ms, int32_t n) {
  (void)b;
  for (int k = 0; k < n; ++k) ms[k] = 0.0f;
  return SLOS_OK;
}

int slos_workspace_kernel_ms(slos_workspace* b, float* ms2) {
  ms2[0] = (float)b->solve_ms;
  ms2[1] = 0.0f;
  return SLOS_OK;
}
/* ---- plan broker: the CPU checker plans immediately (no batching) ---- */
struct slos_broker {
  int32_t unit_value;
  int64_t plans;
};
int slos_broker_create(int32_t unit_value, slos_broker** out) {
  *out = (slos_broker*)calloc(1, sizeof(slos_broker));
  if (!*out) return SLOS_ERR_ALLOC;
  (*out)->unit_value = unit_value;
  return SLOS_OK;
}
void slos_broker_destroy(slos_broker* b) { free(b); }
void slos_broker_join(slos_broker* b) { (void)b; }
void slos_broker_leave(slos_broker* b) { (void)b; }
int slos_broker_plan(slos_broker* b, slos_planner* p, const slos_input* in, slos_result* out) {
  __atomic_fetch_add(&b->plans, 1, __ATOMIC_RELAXED);
  return slos_plan(p, in, b->unit_value, out);
}
void slos_broker_stats(slos_broker* b, int64_t* flushes, int64_t* plans) {
  *plans = __atomic_load_n(&b->plans, __ATOMIC_RELAXED);
  *flushes = *plans;
}

void slos_last_transfer_bytes(int64_t* h2d, int64_t* d2h) {
  *h2d = 0;
  *d2h = 0;
}
