/*
 * slos_planner.h -- C-ABI boundary of the multi-SLO DP token-allocation planner.
 *
 * This is the drop-in boundary for the SLOs-Serve planner hot path
 * (`slosim::SloScheduler::schedule`, reference proj/src/dp_scheduler.cpp:360-558).
 * Three libraries export exactly this ABI:
 *   - libslos_b200.so      the product: sm_100a CUDA kernels + C++ host shim
 *                          (paper_2504_08784_b200/csrc/)
 *   - liboracle_slos.so    test-only CPU restatement in plain C (oracle/)
 *   - oracle/_ref/libslos_ref.so  test-only adapter over the reference sources
 * so that the parity tests can drive all three through one binding.
 *
 * Conventions (mirroring the reference):
 *   - Plain pointers and sizes only; no C++ or torch types.
 *   - Inputs are caller-owned and read-only for the duration of a call.
 *   - Request ids cross the ABI as NUL-terminated strings on input (the chain
 *     sort tie-breaks on them, dp_scheduler.cpp:393-397) and as indices into
 *     running[] / pending[] on output.
 *   - Results are library-allocated; release them with slos_result_free().
 *   - Reference exceptions (slosim::Error, common.hpp:12-25) become status codes;
 *     slos_status_slug() returns the reference's code slug and
 *     slos_last_error() a thread-local message.
 *   - `running_set_infeasible` is a RESULT, not an error (dp_scheduler.cpp:524-556).
 */
#ifndef SLOS_PLANNER_H
#define SLOS_PLANNER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLOS_ABI_VERSION 1
#define SLOS_MAX_TIERS 8 /* dp_scheduler.cpp:367 */
#define SLOS_MAX_CHAIN 250 /* dp_scheduler.cpp:390 */

/* Status codes. 1..3 carry the reference's error slugs. */
enum {
  SLOS_OK = 0,
  SLOS_ERR_INVALID_PARAMETERS = 1,     /* "invalid-parameters" */
  SLOS_ERR_INTERNAL_INCONSISTENCY = 2, /* "internal-inconsistency" */
  SLOS_ERR_INFEASIBLE_BUDGET = 3,      /* "infeasible-budget" (perf_model.cpp:120) */
  SLOS_ERR_CUDA = 10,                  /* CUDA runtime failure */
  SLOS_ERR_CAPACITY = 11,              /* device arena too small even after regrowth */
  SLOS_ERR_NO_DEVICE = 12,             /* no sm_100 device: the product never falls back to CPU */
  SLOS_ERR_ALLOC = 13,                 /* host allocation failure */
  SLOS_ERR_RANGE = 14                  /* a value exceeds the device wire format */
};

/* ---- planner construction: PerfModel + SloConfig + PlannerConfig ---------- */

/* One max-of-affine latency term (perf_model.hpp:21-25). */
typedef struct slos_perf_term {
  double k1; /* seconds per batched token */
  double k2; /* seconds per speculation step */
  double b;  /* fixed per-batch overhead */
} slos_perf_term;

/* PlannerConfig (batch_planner.hpp:57-66). */
typedef struct slos_planner_config {
  int64_t max_chunk_tokens; /* default 2048 */
  int64_t max_batch_tokens; /* default 16384 (PerfModel::kDefaultMaxTokens) */
  int32_t speculative;      /* default 0 */
  int32_t spec_max_len;     /* default 8 */
  double spec_alpha;        /* default 0.8 */
  double plan_margin;       /* default 0.0 */
} slos_planner_config;

void slos_planner_config_default(slos_planner_config* cfg);

typedef struct slos_planner slos_planner;

/* Replaces `BatchPlanner(const PerfModel&, const SloConfig&, PlannerConfig)`
 * (batch_planner.hpp:89) + `SloScheduler(const BatchPlanner&)` (dp_scheduler.hpp:94).
 * Unlike the reference (which holds `const PerfModel&`, batch_planner.hpp:130)
 * the handle OWNS copies of every argument. Validation follows
 * PerfModel::PerfModel (perf_model.cpp:98-104), SloConfig::validate
 * (workload.cpp:18-30) and BatchPlanner::BatchPlanner (batch_planner.cpp:117-123).
 * A handle is externally synchronised, like the reference planner. */
int slos_planner_create(const slos_perf_term* terms, int32_t n_terms,
                        const double* tpot_tiers_s, const double* ttft_slowdowns,
                        int32_t n_tiers, int32_t tpot_window,
                        const slos_planner_config* cfg, slos_planner** out);
void slos_planner_destroy(slos_planner* planner);

/* ---- ScheduleInput (dp_scheduler.hpp:15-47) ------------------------------- */

typedef struct slos_running { /* RunningRequest dp_scheduler.hpp:28-36 */
  const char* id;
  int64_t prefill_remaining;
  double prefill_deadline;
  int32_t decode_tier;
  int32_t reserved0;
  double next_due_s;
  int64_t backlog;
  int64_t decode_remaining;
} slos_running;

typedef struct slos_pending { /* PendingRequest dp_scheduler.hpp:16-23 */
  const char* id;
  double prefill_deadline;
  int64_t prefill_tokens;
  int32_t decode_tier;
  int32_t reserved0;
  int64_t memory_units;
  double value;
} slos_pending;

typedef struct slos_input { /* ScheduleInput dp_scheduler.hpp:38-47 */
  double now;
  const slos_running* running;
  int32_t n_running;
  int32_t n_pending;
  const slos_pending* pending;
  int64_t memory_total;
  int64_t memory_standard_resident;
  double tail_horizon_s;
} slos_input;

/* ---- ScheduleResult (dp_scheduler.hpp:49-79) ------------------------------ */

/* Entry request reference: req >= 0 is running[req]; req < 0 is pending[-req-1]. */
#define SLOS_PENDING_REF(p) (-(int32_t)(p)-1)

/* PlanEntry dp_scheduler.hpp:49-54, 8 bytes on the wire (plans are the bulk of the
 * device->host traffic). Every entry the planner emits is EITHER a prefill chunk
 * (decode_tokens = spec_len = 0) OR a decode allocation (prefill_tokens = 0):
 * dp_scheduler.cpp:150,163,178,229,288,343. So one 32-bit token count and a kind
 * bit carry it:
 *   ref bits  0-23  request reference (SLOS_PENDING_REF convention, 24-bit signed)
 *   ref bits 24-30  spec_len of a decode entry (0 = autoregressive)
 *   ref bit  31     1 = decode entry, 0 = prefill entry
 *   tokens          prefill_tokens (prefill entry) or decode_tokens (decode entry)
 * The limits that keep this lossless are enforced, never truncated: slos_plan*
 * rejects n_running or n_pending >= SLOS_ENTRY_MAX_REQS, slos_planner_create
 * rejects max_batch_tokens / max_chunk_tokens above INT32_MAX and speculative
 * spec_max_len above SLOS_ENTRY_MAX_SPEC, and a plan whose count would still not
 * fit (only possible with absurd decode backlogs in the EDF fallback) fails with
 * SLOS_ERR_INVALID_PARAMETERS. Read entries through the accessors below; the
 * adapter widens the counts back to the reference's int64. */
typedef struct slos_entry {
  uint32_t ref;
  int32_t tokens;
} slos_entry;

#define SLOS_ENTRY_MAX_REQS (1 << 23)
#define SLOS_ENTRY_MAX_SPEC 127

#if defined(__CUDACC__)
#define SLOS_ENTRY_FN static inline __host__ __device__
#else
#define SLOS_ENTRY_FN static inline
#endif
SLOS_ENTRY_FN int32_t slos_entry_req(const slos_entry* e) { return ((int32_t)(e->ref << 8)) >> 8; }
SLOS_ENTRY_FN int32_t slos_entry_is_decode(const slos_entry* e) { return (int32_t)(e->ref >> 31); }
SLOS_ENTRY_FN int32_t slos_entry_spec_len(const slos_entry* e) { return (int32_t)((e->ref >> 24) & 0x7Fu); }
SLOS_ENTRY_FN int64_t slos_entry_prefill_tokens(const slos_entry* e) {
  return slos_entry_is_decode(e) ? 0 : (int64_t)e->tokens;
}
SLOS_ENTRY_FN int64_t slos_entry_decode_tokens(const slos_entry* e) {
  return slos_entry_is_decode(e) ? (int64_t)e->tokens : 0;
}
SLOS_ENTRY_FN slos_entry slos_entry_prefill(int32_t req, int32_t tokens) {
  slos_entry e;
  e.ref = (uint32_t)req & 0xFFFFFFu;
  e.tokens = tokens;
  return e;
}
SLOS_ENTRY_FN slos_entry slos_entry_decode(int32_t req, int32_t tokens, int32_t spec_len) {
  slos_entry e;
  e.ref = ((uint32_t)req & 0xFFFFFFu) | ((uint32_t)spec_len & 0x7Fu) << 24 | 0x80000000u;
  e.tokens = tokens;
  return e;
}

typedef struct slos_batch { /* PlanBatch dp_scheduler.hpp:56-63 */
  double start_s;
  double end_s;
  int64_t capacity_tokens;
  int64_t spec_step;
  int64_t prefill_budget_left;
  int64_t first_entry; /* index into slos_result.entries */
  int64_t n_entries;
} slos_batch;

/* Work counters, defined by the REFERENCE traversal (SURVEY.md §8 preamble):
 * transitions = DP transitions with a surviving source (dp_scheduler.cpp:479),
 * gap_evals   = unique gap evaluations (memo misses, dp_scheduler.cpp:427 /
 *               batch_planner.cpp:414),
 * dues        = dues materialised inside those evaluations (batch_planner.cpp:198-220),
 * slots       = slots built inside those evaluations (batch_planner.cpp:247),
 * states      = DP states created (arena size - 1).  Counted for the admission
 * DP only (build_plan / fallback excluded). */
typedef struct slos_counters {
  int64_t transitions;
  int64_t gap_evals;
  int64_t dues;
  int64_t slots;
  int64_t states;
} slos_counters;

typedef struct slos_result {
  int32_t status; /* SLOS_OK or an error code; on error the rest is empty */
  int32_t running_set_infeasible;
  double admitted_value;
  int32_t n_admitted;
  int32_t n_declined;
  int32_t n_deferred; /* always 0 for this scheduler */
  int32_t reserved0;
  const int32_t* admitted; /* pending indices, chain (pDDL) order */
  const int32_t* declined; /* pending indices; chain order, or input order on fallback */
  const int32_t* deferred;
  int64_t n_batches;
  const slos_batch* batches;
  int64_t n_entries;
  const slos_entry* entries;
  double exact_until_s;
  slos_counters counters;
  void* owner_; /* library bookkeeping; do not touch */
} slos_result;

/* `SloScheduler::schedule` (unit_value = 0, dp_scheduler.cpp:360) and
 * `SloScheduler::schedule_throughput` (unit_value = 1, dp_scheduler.cpp:362). */
int slos_plan(slos_planner* planner, const slos_input* input, int32_t unit_value,
              slos_result* out);

/* Batched plan(): n independent instances (one per replica / routing candidate /
 * scheduling window / sweep point). planners[k] serves inputs[k]; handles may
 * repeat. `stream` is a cudaStream_t (NULL = the library's stream); the call is
 * synchronous on return. Each outs[k] must be released with slos_result_free().
 * Returns SLOS_OK when the batch ran; per-instance errors land in outs[k].status. */
int slos_plan_batch(slos_planner* const* planners, int32_t n, const slos_input* inputs,
                    int32_t unit_value, slos_result* outs, void* stream);

void slos_result_free(slos_result* result);

/* Device-resident batches: the three stages of slos_plan_batch exposed so a
 * caller (and bench.py) can keep instances resident in HBM and re-solve them.
 *   upload   -- host preparation + one H2D copy (instances become resident);
 *               invalid instances get their status in outs[k] immediately
 *   solve    -- enqueue the kernel pipeline on `stream` (asynchronous)
 *   download -- synchronise, regrow the rare overflowed instance, compact and
 *               copy the results back (one D2H); fills outs[k]
 * `inputs` must stay valid until download returns. The CPU checkers implement
 * the same calls synchronously. */
typedef struct slos_workspace slos_workspace;
int slos_workspace_create(slos_workspace** out);
void slos_workspace_destroy(slos_workspace* ws);
int slos_workspace_upload(slos_workspace* batch, slos_planner* const* planners, int32_t n,
                      const slos_input* inputs, int32_t unit_value, slos_result* outs,
                      void* stream);
int slos_workspace_solve(slos_workspace* batch, void* stream);
int slos_workspace_download(slos_workspace* batch, slos_result* outs, void* stream);

/* Fixed-size per-instance result record (what a multi-GPU sweep all-gathers). */
typedef struct slos_record {
  int32_t status;
  int32_t running_set_infeasible;
  int32_t n_admitted;
  int32_t n_declined;
  double admitted_value;
  int64_t n_batches;
  int64_t n_entries;
  double exact_until_s;
  slos_counters counters;
} slos_record;

/* Write the n records of the last solve to `out` (n slos_record), in input order,
 * asynchronously on `stream`. `out` is DEVICE memory for the product (a device-to-
 * device copy that feeds an NCCL gather without a host round trip) and host
 * memory for the CPU checkers. */
int slos_workspace_records(slos_workspace* ws, slos_record* out, void* stream);

/* Device time (ms) of the last solve's kernels: [0] admission DP, [1] plan
 * reconstruction. CPU checkers report wall time of the whole solve in [0]. */
int slos_workspace_kernel_ms(slos_workspace* ws, float* ms2);

/* Device time (ms) of the last solve's stages, n <= 3 entries: [0] anchor caches
 * and pair groups (anchor_kernel, group_kernel), [1] admission DP until its last
 * part ends (dp_kernel; solve parts are pipelined, so earlier parts'
 * reconstruction overlaps it), [2] the remaining plan reconstruction
 * (build_kernel*). CPU checkers write zeros. */
int slos_workspace_stage_ms(slos_workspace* ws, float* ms, int32_t n);

/* Number of kernels the last solve launched (anchor / group / DP per solve part and
 * one per non-empty reconstruction queue; the records and compaction kernels are
 * separate calls). CPU checkers write 0. */
int slos_workspace_launches(slos_workspace* ws, int64_t* n);

/* Bytes moved host->device and device->host by the calling thread's last
 * slos_plan_batch / slos_workspace_* sequence. */
void slos_last_transfer_bytes(int64_t* h2d, int64_t* d2h);

/* ---- the plan broker: concurrent schedule() calls -> one batched launch --------
 * The reference calls `Scheduler::schedule` synchronously, one replica at a time
 * (sim_executor.cpp:344); many replicas / simulations / sweep points running in
 * their own threads each block in schedule(). The broker turns those concurrent
 * calls into ONE slos_plan_batch (SURVEY.md §8 b: "a broker aggregates concurrent
 * schedule() calls into one launch").
 * Protocol: a client thread is ACTIVE while it computes and may still call
 * slos_broker_plan. slos_broker_join() marks the calling client active,
 * slos_broker_leave() marks it inactive (it will not plan until it joins again).
 * slos_broker_plan() queues one plan and blocks the (still registered) client;
 * as soon as no registered client is active, the thread that made it so runs
 * every queued plan as one batch and wakes their callers, which are active again.
 * Results are exactly those of slos_plan (plans are independent). The CPU
 * checkers implement slos_broker_plan as an immediate slos_plan. */
typedef struct slos_broker slos_broker;
int slos_broker_create(int32_t unit_value, slos_broker** out);
void slos_broker_destroy(slos_broker* broker);
void slos_broker_join(slos_broker* broker);
void slos_broker_leave(slos_broker* broker);
int slos_broker_plan(slos_broker* broker, slos_planner* planner, const slos_input* input,
                     slos_result* out);
/* flushes = batched launches so far, plans = plans served */
void slos_broker_stats(slos_broker* broker, int64_t* flushes, int64_t* plans);

/* ---- batch planner primitives (batch_planner.hpp:68-134, perf_model.hpp:25-61) */

typedef struct slos_decode_member { /* DecodeMember batch_planner.hpp:19-25 */
  int32_t tier;
  int32_t owner;
  double phase_s;
  int64_t backlog;
  int64_t remaining;
} slos_decode_member;

enum { SLOS_GAP_TILE_AR = 0, SLOS_GAP_TILE = 1, SLOS_GAP_PREFILL_BUDGET = 2 };

typedef struct slos_gap_query {
  int32_t mode;     /* SLOS_GAP_* : tile_gap_ar / tile_gap / prefill_budget */
  int32_t n_exact;
  double gap_s;
  double due_horizon_s;
  int64_t counts_per_tier[SLOS_MAX_TIERS]; /* canonical members; n_tiers used */
  const slos_decode_member* exact;         /* ignored for SLOS_GAP_PREFILL_BUDGET */
} slos_gap_query;

typedef struct slos_gap_batch { /* PlannedBatch batch_planner.hpp:38-49 */
  double start_s;
  double end_s;
  int64_t capacity_tokens;
  int64_t spec_step;
  int64_t decode_tokens;
  int64_t prefill_budget;
  int64_t decode_per_tier[SLOS_MAX_TIERS];
  int64_t first_owner; /* index into slos_gap_result.owner_tokens (pairs) */
  int64_t n_owners;
} slos_gap_batch;

typedef struct slos_gap_result { /* std::optional<GapPlan> batch_planner.hpp:51-55 */
  int32_t status;
  int32_t feasible; /* 0 = nullopt */
  int64_t prefill_budget;
  int32_t n_spec_lengths; /* 0 for autoregressive plans */
  int32_t spec_lengths[SLOS_MAX_TIERS];
  int64_t n_batches;
  const slos_gap_batch* batches;
  int64_t n_owner_pairs;
  const int64_t* owner_tokens; /* (owner, tokens) pairs, 2*n_owner_pairs values */
  void* owner_;
} slos_gap_result;

/* Evaluate n gap queries. For SLOS_GAP_PREFILL_BUDGET only feasible and
 * prefill_budget are filled (batch_planner.cpp:408-422). */
int slos_tile_gap_batch(slos_planner* planner, int32_t n, const slos_gap_query* queries,
                        slos_gap_result* outs);
void slos_gap_result_free(slos_gap_result* r);

/* PerfModel::time2bs(budget, spec_step, max_tokens) (perf_model.cpp:116-130) over n
 * budgets; status[k] = SLOS_ERR_INFEASIBLE_BUDGET reproduces the reference throw. */
int slos_time2bs_batch(slos_planner* planner, int32_t n, const double* budget_s,
                       const int64_t* spec_step, int64_t max_tokens, int64_t* out,
                       int32_t* status);

/* PerfModel::predict (perf_model.cpp:106-114). */
int slos_predict_batch(slos_planner* planner, int32_t n, const int64_t* num_tokens,
                       const int64_t* spec_step, double* out);

/* solve_spec_lengths (batch_planner.cpp:51-115) with the planner's alpha/max_len. */
typedef struct slos_spec_plan {
  int32_t feasible;
  int32_t lengths[SLOS_MAX_TIERS];
  double batch_time_s;
  int64_t batch_capacity;
  int64_t decode_tokens;
  double prefill_throughput;
} slos_spec_plan;
int slos_solve_spec_lengths(slos_planner* planner, const int64_t* decoders_per_tier,
                            int32_t n_tiers, double alpha, int32_t max_len,
                            slos_spec_plan* out);

/* expected_accepted (batch_planner.cpp:32-37). */
double slos_expected_accepted(double alpha, int32_t sl);

/* ---- diagnostics ----------------------------------------------------------- */

const char* slos_status_slug(int status);
const char* slos_last_error(void);
/* "b200-cuda", "oracle-c" or "reference-cpp". */
const char* slos_backend(void);

#ifdef __cplusplus
}
#endif

#endif /* SLOS_PLANNER_H */
