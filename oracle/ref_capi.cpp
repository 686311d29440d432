// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// C-ABI adapter (include/slos_planner.h) over the UNMODIFIED reference planner.
// Built by oracle/Makefile together with the reference's own sources, read in
// place from /root/reference/proj/src, into oracle/_ref/libslos_ref.so. It is the
// parity anchor for the C restatement (oracle/slos_oracle.c) and the
// `cpu_baseline.kind = "reference"` arm of bench.py.
//
// Each entry point forwards to the reference function it is named after:
//   slos_plan            -> SloScheduler::schedule / schedule_throughput  dp_scheduler.cpp:360-362
//   slos_tile_gap_batch  -> BatchPlanner::tile_gap_ar / tile_gap / prefill_budget
//                           batch_planner.cpp:152, 315, 408
//   slos_time2bs_batch   -> PerfModel::time2bs  perf_model.cpp:116
//   slos_predict_batch   -> PerfModel::predict  perf_model.cpp:106
//   slos_solve_spec_lengths -> solve_spec_lengths batch_planner.cpp:51
//   slos_expected_accepted  -> expected_accepted  batch_planner.cpp:32

#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <memory>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "slos_plan_json.h"
#include "slos_planner.h"
#include "slosim/batch_planner.hpp"
#include "slosim/common.hpp"
#include "slosim/dp_scheduler.hpp"
#include "slosim/perf_model.hpp"
#include "slosim/workload.hpp"

using namespace slosim;

#ifdef SLOS_REF_INSTR
// oracle/instrument_ref.py: the reference sources patched with work counters
namespace slos_instr { extern thread_local long long T, G, D, S, snap[5]; extern thread_local int on; }
#endif

struct slos_planner {
  PerfModel model;
  SloConfig slo;
  PlannerConfig cfg;
  std::unique_ptr<BatchPlanner> planner;
  std::unique_ptr<SloScheduler> sched;
};

namespace {

thread_local std::string g_last_error;

int status_of(const Error& e) {
  if (e.code() == "invalid-parameters") return SLOS_ERR_INVALID_PARAMETERS;
  if (e.code() == "internal-inconsistency") return SLOS_ERR_INTERNAL_INCONSISTENCY;
  if (e.code() == "infeasible-budget") return SLOS_ERR_INFEASIBLE_BUDGET;
  return SLOS_ERR_INVALID_PARAMETERS;
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    g_last_error = e.what();
    return status_of(e);
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SLOS_ERR_INVALID_PARAMETERS;
  }
}

ScheduleInput to_input(const slos_input* in) {
  ScheduleInput s;
  s.now = in->now;
  s.memory_total = in->memory_total;
  s.memory_standard_resident = in->memory_standard_resident;
  s.tail_horizon_s = in->tail_horizon_s;
  s.running.reserve(in->n_running);
  for (int i = 0; i < in->n_running; ++i) {
    const slos_running& r = in->running[i];
    RunningRequest rr;
    rr.id = r.id;
    rr.prefill_remaining = r.prefill_remaining;
    rr.prefill_deadline = r.prefill_deadline;
    rr.decode_tier = r.decode_tier;
    rr.next_due_s = r.next_due_s;
    rr.backlog = r.backlog;
    rr.decode_remaining = r.decode_remaining;
    s.running.push_back(std::move(rr));
  }
  s.pending.reserve(in->n_pending);
  for (int i = 0; i < in->n_pending; ++i) {
    const slos_pending& p = in->pending[i];
    PendingRequest pp;
    pp.id = p.id;
    pp.prefill_deadline = p.prefill_deadline;
    pp.prefill_tokens = p.prefill_tokens;
    pp.decode_tier = p.decode_tier;
    pp.memory_units = p.memory_units;
    pp.value = p.value;
    s.pending.push_back(std::move(pp));
  }
  return s;
}

// One malloc per result; every array points into it.
void fill_result(const slos_input* in, const ScheduleResult& res, slos_result* out) {
  std::unordered_map<std::string, int32_t> ref;
  for (int i = 0; i < in->n_running; ++i) ref.emplace(in->running[i].id, i);
  for (int i = 0; i < in->n_pending; ++i) ref.emplace(in->pending[i].id, SLOS_PENDING_REF(i));
  size_t n_entries = 0;
  for (const auto& b : res.plan.batches) {
    n_entries += b.entries.size();
    for (const PlanEntry& pe : b.entries) {  // the 8-byte slos_entry (include/slos_planner.h)
      if (pe.prefill_tokens > INT32_MAX || pe.decode_tokens > INT32_MAX || pe.prefill_tokens < INT32_MIN ||
          pe.decode_tokens < INT32_MIN)
        fail("invalid-parameters", "a plan token count exceeds the 32-bit entry range");
      if (pe.spec_len < 0 || pe.spec_len > SLOS_ENTRY_MAX_SPEC)
        fail("invalid-parameters", "a plan spec_len exceeds the entry range");
      if (pe.prefill_tokens != 0 && (pe.decode_tokens != 0 || pe.spec_len != 0))
        fail("internal-inconsistency", "a plan entry carries both prefill and decode tokens");
    }
  }
  const size_t n_adm = res.admitted.size(), n_dec = res.declined.size(),
               n_def = res.deferred.size(), n_b = res.plan.batches.size();
  size_t bytes = sizeof(slos_batch) * n_b + sizeof(slos_entry) * n_entries +
                 sizeof(int32_t) * (n_adm + n_dec + n_def) + 64;
  char* mem = static_cast<char*>(std::calloc(1, bytes));
  slos_batch* batches = reinterpret_cast<slos_batch*>(mem);
  slos_entry* entries = reinterpret_cast<slos_entry*>(batches + n_b);
  int32_t* ids = reinterpret_cast<int32_t*>(entries + n_entries);
  auto pidx = [&](const std::string& id) { return -ref.at(id) - 1; };
  for (size_t k = 0; k < n_adm; ++k) ids[k] = pidx(res.admitted[k]);
  for (size_t k = 0; k < n_dec; ++k) ids[n_adm + k] = pidx(res.declined[k]);
  for (size_t k = 0; k < n_def; ++k) ids[n_adm + n_dec + k] = pidx(res.deferred[k]);
  size_t e = 0;
  for (size_t k = 0; k < n_b; ++k) {
    const PlanBatch& b = res.plan.batches[k];
    batches[k].start_s = b.start_s;
    batches[k].end_s = b.end_s;
    batches[k].capacity_tokens = b.capacity_tokens;
    batches[k].spec_step = b.spec_step;
    batches[k].prefill_budget_left = b.prefill_budget_left;
    batches[k].first_entry = (int64_t)e;
    batches[k].n_entries = (int64_t)b.entries.size();
    for (const PlanEntry& pe : b.entries) {
      const int32_t rq = ref.at(pe.id);
      entries[e] = (pe.decode_tokens != 0 || pe.spec_len != 0)
                       ? slos_entry_decode(rq, (int32_t)pe.decode_tokens, pe.spec_len)
                       : slos_entry_prefill(rq, (int32_t)pe.prefill_tokens);
      ++e;
    }
  }
  out->status = SLOS_OK;
  out->running_set_infeasible = res.running_set_infeasible ? 1 : 0;
  out->admitted_value = res.admitted_value;
  out->n_admitted = (int32_t)n_adm;
  out->n_declined = (int32_t)n_dec;
  out->n_deferred = (int32_t)n_def;
  out->admitted = ids;
  out->declined = ids + n_adm;
  out->deferred = ids + n_adm + n_dec;
  out->n_batches = (int64_t)n_b;
  out->batches = batches;
  out->n_entries = (int64_t)n_entries;
  out->entries = entries;
  out->exact_until_s = res.plan.exact_until_s;
  std::memset(&out->counters, 0, sizeof(out->counters));
  out->owner_ = mem;
}

DecodeCensus to_census(const slos_gap_query& q, int num_tiers) {
  DecodeCensus c;
  c.counts_per_tier.assign(q.counts_per_tier, q.counts_per_tier + num_tiers);
  if (q.mode != SLOS_GAP_PREFILL_BUDGET) {
    for (int i = 0; i < q.n_exact; ++i) {
      DecodeMember m;
      m.tier = q.exact[i].tier;
      m.owner = q.exact[i].owner;
      m.phase_s = q.exact[i].phase_s;
      m.backlog = q.exact[i].backlog;
      m.remaining = q.exact[i].remaining;
      c.exact.push_back(m);
    }
  }
  return c;
}

void fill_gap(const std::optional<GapPlan>& gp, int num_tiers, slos_gap_result* out) {
  std::memset(out, 0, sizeof(*out));
  out->status = SLOS_OK;
  if (!gp) return;
  out->feasible = 1;
  out->prefill_budget = gp->prefill_budget;
  out->n_spec_lengths = (int32_t)gp->spec_lengths.size();
  for (size_t l = 0; l < gp->spec_lengths.size() && l < SLOS_MAX_TIERS; ++l)
    out->spec_lengths[l] = gp->spec_lengths[l];
  size_t pairs = 0;
  for (const auto& b : gp->batches) pairs += b.decode_by_owner.size();
  const size_t n_b = gp->batches.size();
  char* mem = static_cast<char*>(
      std::calloc(1, sizeof(slos_gap_batch) * n_b + sizeof(int64_t) * 2 * pairs + 64));
  slos_gap_batch* bs = reinterpret_cast<slos_gap_batch*>(mem);
  int64_t* own = reinterpret_cast<int64_t*>(bs + n_b);
  size_t p = 0;
  for (size_t k = 0; k < n_b; ++k) {
    const PlannedBatch& b = gp->batches[k];
    bs[k].start_s = b.start_s;
    bs[k].end_s = b.end_s;
    bs[k].capacity_tokens = b.capacity_tokens;
    bs[k].spec_step = b.spec_step;
    bs[k].decode_tokens = b.decode_tokens;
    bs[k].prefill_budget = b.prefill_budget;
    for (size_t l = 0; l < b.decode_per_tier.size() && l < (size_t)num_tiers; ++l)
      bs[k].decode_per_tier[l] = b.decode_per_tier[l];
    bs[k].first_owner = (int64_t)p;
    bs[k].n_owners = (int64_t)b.decode_by_owner.size();
    for (const auto& [o, t] : b.decode_by_owner) {
      own[2 * p] = o;
      own[2 * p + 1] = t;
      ++p;
    }
  }
  out->n_batches = (int64_t)n_b;
  out->batches = bs;
  out->n_owner_pairs = (int64_t)pairs;
  out->owner_tokens = own;
  out->owner_ = mem;
}

}  // namespace

extern "C" {

void slos_planner_config_default(slos_planner_config* cfg) {
  PlannerConfig d;
  cfg->max_chunk_tokens = d.max_chunk_tokens;
  cfg->max_batch_tokens = d.max_batch_tokens;
  cfg->speculative = d.speculative ? 1 : 0;
  cfg->spec_max_len = d.spec_max_len;
  cfg->spec_alpha = d.spec_alpha;
  cfg->plan_margin = d.plan_margin;
}

int slos_planner_create(const slos_perf_term* terms, int32_t n_terms, const double* tpot,
                        const double* slow, int32_t n_tiers, int32_t tpot_window,
                        const slos_planner_config* cfg, slos_planner** out) {
  *out = nullptr;
  return guarded([&] {
    auto p = std::make_unique<slos_planner>();
    std::vector<PerfTerm> t;
    for (int i = 0; i < n_terms; ++i) t.push_back({terms[i].k1, terms[i].k2, terms[i].b});
    p->model = PerfModel(t);
    p->slo.tpot_tiers_s.assign(tpot, tpot + n_tiers);
    p->slo.ttft_slowdowns.assign(slow, slow + n_tiers);
    p->slo.tpot_window = tpot_window;
    slos_planner_config c;
    if (cfg) c = *cfg; else slos_planner_config_default(&c);
    p->cfg.max_chunk_tokens = c.max_chunk_tokens;
    p->cfg.max_batch_tokens = c.max_batch_tokens;
    p->cfg.speculative = c.speculative != 0;
    p->cfg.spec_alpha = c.spec_alpha;
    p->cfg.spec_max_len = c.spec_max_len;
    p->cfg.plan_margin = c.plan_margin;
    p->planner = std::make_unique<BatchPlanner>(p->model, p->slo, p->cfg);
    p->sched = std::make_unique<SloScheduler>(*p->planner);
    if (c.max_chunk_tokens > INT32_MAX || c.max_batch_tokens > INT32_MAX)  // 32-bit slos_entry
      fail("invalid-parameters", "batch and chunk caps must fit the 32-bit plan entries");
    if (c.speculative && c.spec_max_len > SLOS_ENTRY_MAX_SPEC)  // 7-bit entry spec_len
      fail("invalid-parameters", "spec_max_len must fit the plan entry format");
    *out = p.release();
    return SLOS_OK;
  });
}

void slos_planner_destroy(slos_planner* p) { delete p; }

int slos_plan(slos_planner* p, const slos_input* in, int32_t unit_value, slos_result* out) {
  std::memset(out, 0, sizeof(*out));
  int st = guarded([&] {
    if (in->n_running >= SLOS_ENTRY_MAX_REQS || in->n_pending >= SLOS_ENTRY_MAX_REQS)  // 24-bit entry refs
      fail("invalid-parameters", "too many requests for the plan entry format");
    ScheduleInput s = to_input(in);
#ifdef SLOS_REF_INSTR
    // a fresh BatchPlanner per plan (cold prefill_budget memo, acceptance_main.cpp:606),
    // so the memo-miss counter G is a per-plan quantity
    BatchPlanner fresh(p->model, p->slo, p->cfg);
    SloScheduler sched(fresh);
    ScheduleResult r = unit_value ? sched.schedule_throughput(s) : sched.schedule(s);
    fill_result(in, r, out);
    out->counters.transitions = slos_instr::snap[0];
    out->counters.gap_evals = slos_instr::snap[1];
    out->counters.dues = slos_instr::snap[2];
    out->counters.slots = slos_instr::snap[3];
    out->counters.states = slos_instr::snap[4];
#else
    ScheduleResult r = unit_value ? p->sched->schedule_throughput(s) : p->sched->schedule(s);
    fill_result(in, r, out);
#endif
    return SLOS_OK;
  });
  out->status = st;
  return st;
}

// Single-thread latency as the reference's own criterion measures it
// (acceptance_main.cpp:606-609): a FRESH BatchPlanner + SloScheduler per instance
// (cold memo), and only schedule() inside the clock.
int slos_ref_schedule_timed(slos_planner* p, const slos_input* in, int32_t unit_value, slos_result* out,
                            double* seconds) {
  std::memset(out, 0, sizeof(*out));
  *seconds = 0.0;
  int st = guarded([&] {
    ScheduleInput s = to_input(in);
    BatchPlanner planner(p->model, p->slo, p->cfg);
    SloScheduler sched(planner);
    timespec a, b;
    clock_gettime(CLOCK_MONOTONIC, &a);
    ScheduleResult r = unit_value ? sched.schedule_throughput(s) : sched.schedule(s);
    clock_gettime(CLOCK_MONOTONIC, &b);
    *seconds = (double)(b.tv_sec - a.tv_sec) + 1e-9 * (double)(b.tv_nsec - a.tv_nsec);
    fill_result(in, r, out);
    return SLOS_OK;
  });
  out->status = st;
  return st;
}

// Reference CPU batch: a std::thread pool over all host cores, one planner per
// instance handle. Handles shared between instances are
// serialised by giving each worker its own private copy of the planner.
int slos_plan_batch(slos_planner* const* planners, int32_t n, const slos_input* inputs,
                    int32_t unit_value, slos_result* outs, void* /*stream*/) {
  const char* env = std::getenv("SLOS_REF_THREADS");
  int workers = env ? std::atoi(env) : (int)std::thread::hardware_concurrency();
  if (workers < 1) workers = 1;
  std::vector<std::thread> pool;
  std::atomic<int> next{0};
  for (int w = 0; w < workers; ++w) {
    pool.emplace_back([&] {
      std::unordered_map<const slos_planner*, std::unique_ptr<slos_planner>> own;
      for (int k = next.fetch_add(1); k < n; k = next.fetch_add(1)) {
        const slos_planner* src = planners[k];
        auto& mine = own[src];
        if (!mine) {
          mine = std::make_unique<slos_planner>();
          mine->model = src->model;
          mine->slo = src->slo;
          mine->cfg = src->cfg;
          mine->planner = std::make_unique<BatchPlanner>(mine->model, mine->slo, mine->cfg);
          mine->sched = std::make_unique<SloScheduler>(*mine->planner);
        }
        slos_plan(mine.get(), &inputs[k], unit_value, &outs[k]);
      }
    });
  }
  for (auto& t : pool) t.join();
  return SLOS_OK;
}

void slos_result_free(slos_result* r) {
  if (r && r->owner_) std::free(r->owner_);
  if (r) std::memset(r, 0, sizeof(*r));
}

int slos_tile_gap_batch(slos_planner* p, int32_t n, const slos_gap_query* q,
                        slos_gap_result* outs) {
  const int L = p->slo.num_tiers();
  for (int k = 0; k < n; ++k) {
    int st = guarded([&] {
      DecodeCensus c = to_census(q[k], L);
      if (q[k].mode == SLOS_GAP_TILE_AR) {
        fill_gap(p->planner->tile_gap_ar(q[k].gap_s, c, q[k].due_horizon_s), L, &outs[k]);
      } else if (q[k].mode == SLOS_GAP_TILE) {
        fill_gap(p->planner->tile_gap(q[k].gap_s, c, q[k].due_horizon_s), L, &outs[k]);
      } else {
        auto b = p->planner->prefill_budget(q[k].gap_s, c.counts_per_tier);
        std::memset(&outs[k], 0, sizeof(outs[k]));
        outs[k].feasible = b.has_value();
        outs[k].prefill_budget = b ? *b : 0;
      }
      return SLOS_OK;
    });
    if (st != SLOS_OK) {
      std::memset(&outs[k], 0, sizeof(outs[k]));
      outs[k].status = st;
    }
  }
  return SLOS_OK;
}

void slos_gap_result_free(slos_gap_result* r) {
  if (r && r->owner_) std::free(r->owner_);
  if (r) std::memset(r, 0, sizeof(*r));
}

int slos_time2bs_batch(slos_planner* p, int32_t n, const double* budget, const int64_t* spec,
                       int64_t max_tokens, int64_t* out, int32_t* status) {
  for (int k = 0; k < n; ++k) {
    out[k] = 0;
    status[k] = guarded([&] {
      out[k] = p->model.time2bs(budget[k], spec ? spec[k] : 0, max_tokens);
      return SLOS_OK;
    });
  }
  return SLOS_OK;
}

int slos_predict_batch(slos_planner* p, int32_t n, const int64_t* tokens, const int64_t* spec,
                       double* out) {
  return guarded([&] {
    for (int k = 0; k < n; ++k) out[k] = p->model.predict(tokens[k], spec ? spec[k] : 0);
    return SLOS_OK;
  });
}

int slos_solve_spec_lengths(slos_planner* p, const int64_t* counts, int32_t n_tiers, double alpha,
                            int32_t max_len, slos_spec_plan* out) {
  std::memset(out, 0, sizeof(*out));
  return guarded([&] {
    std::vector<int64_t> c(counts, counts + n_tiers);
    auto sp = solve_spec_lengths(c, alpha, max_len, p->model, p->slo, p->cfg);
    if (sp) {
      out->feasible = 1;
      for (size_t l = 0; l < sp->lengths.size() && l < SLOS_MAX_TIERS; ++l)
        out->lengths[l] = sp->lengths[l];
      out->batch_time_s = sp->batch_time_s;
      out->batch_capacity = sp->batch_capacity;
      out->decode_tokens = sp->decode_tokens;
      out->prefill_throughput = sp->prefill_throughput;
    }
    return SLOS_OK;
  });
}

double slos_expected_accepted(double alpha, int32_t sl) { return expected_accepted(alpha, sl); }


/* device-resident workspace API: synchronous CPU version (test infrastructure) */
struct slos_workspace {
  slos_planner* const* planners;
  const slos_input* inputs;
  int32_t n;
  int32_t unit_value;
  slos_result* res; /* results of the last solve, owned until download */
  double solve_ms;
};
static void ws_clear_cpu(slos_workspace* b) {
  if (b->res) {
    for (int32_t k = 0; k < b->n; ++k) slos_result_free(&b->res[k]);
    free(b->res);
    b->res = NULL;
  }
}
int slos_workspace_create(slos_workspace** out) {
  *out = static_cast<slos_workspace*>(std::calloc(1, sizeof(slos_workspace)));
  return *out ? SLOS_OK : SLOS_ERR_ALLOC;
}
void slos_workspace_destroy(slos_workspace* b) {
  if (!b) return;
  ws_clear_cpu(b);
  free(b);
}
int slos_workspace_upload(slos_workspace* b, slos_planner* const* planners, int32_t n, const slos_input* inputs,
                          int32_t unit_value, slos_result* outs, void* stream) {
  (void)stream;
  ws_clear_cpu(b);
  for (int32_t k = 0; k < n; ++k) memset(&outs[k], 0, sizeof outs[k]);
  b->planners = planners;
  b->inputs = inputs;
  b->n = n;
  b->unit_value = unit_value;
  return SLOS_OK;
}
int slos_workspace_solve(slos_workspace* b, void* stream) {
  timespec t0, t1;
  ws_clear_cpu(b);
  b->res = static_cast<slos_result*>(std::calloc((size_t)(b->n > 0 ? b->n : 1), sizeof(slos_result)));
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
  *n = 0;  // no device kernels in the CPU reference
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
// ---- plan broker: the CPU reference plans immediately (no batching) ----
struct slos_broker {
  int32_t unit_value = 0;
  std::atomic<int64_t> plans{0};
};
int slos_broker_create(int32_t unit_value, slos_broker** out) {
  *out = new slos_broker();
  (*out)->unit_value = unit_value;
  return SLOS_OK;
}
void slos_broker_destroy(slos_broker* b) { delete b; }
void slos_broker_join(slos_broker* b) { (void)b; }
void slos_broker_leave(slos_broker* b) { (void)b; }
int slos_broker_plan(slos_broker* b, slos_planner* p, const slos_input* in, slos_result* out) {
  b->plans.fetch_add(1);
  return slos_plan(p, in, b->unit_value, out);
}
void slos_broker_stats(slos_broker* b, int64_t* flushes, int64_t* plans) {
  *plans = b->plans.load();
  *flushes = *plans;
}

void slos_last_transfer_bytes(int64_t* h2d, int64_t* d2h) {
  *h2d = 0;
  *d2h = 0;
}


const char* slos_status_slug(int s) {
  switch (s) {
    case SLOS_OK: return "ok";
    case SLOS_ERR_INVALID_PARAMETERS: return "invalid-parameters";
    case SLOS_ERR_INTERNAL_INCONSISTENCY: return "internal-inconsistency";
    case SLOS_ERR_INFEASIBLE_BUDGET: return "infeasible-budget";
    default: return "error";
  }
}

const char* slos_last_error(void) { return g_last_error.c_str(); }
const char* slos_backend(void) { return "reference-cpp"; }

}  // extern "C"

// plan_to_json parity (include/slos_plan_json.h): the slos_result is turned back into
// the reference's ScheduleResult and serialised by the reference's own plan_to_json
// (dp_scheduler.cpp:560-589).
extern "C" int slos_plan_to_json(const slos_input* in, const slos_result* r, double now_s, char* buf, int64_t cap,
                                 int64_t* len) {
  if (len) *len = 0;
  if (!in || !r) return SLOS_ERR_INVALID_PARAMETERS;
  std::string text;
  const int st = guarded([&] {
    auto pid = [&](int32_t k) -> std::string {
      if (k < 0 || k >= in->n_pending) fail("invalid-parameters", "pending index out of range");
      return in->pending[k].id ? in->pending[k].id : "";
    };
    ScheduleResult res;
    for (int k = 0; k < r->n_admitted; ++k) res.admitted.push_back(pid(r->admitted[k]));
    for (int k = 0; k < r->n_declined; ++k) res.declined.push_back(pid(r->declined[k]));
    for (int k = 0; k < r->n_deferred; ++k) res.deferred.push_back(pid(r->deferred[k]));
    res.admitted_value = r->admitted_value;
    res.running_set_infeasible = r->running_set_infeasible != 0;
    res.plan.exact_until_s = r->exact_until_s;
    for (int64_t b = 0; b < r->n_batches; ++b) {
      const slos_batch& cb = r->batches[b];
      PlanBatch pb;
      pb.start_s = cb.start_s;
      pb.end_s = cb.end_s;
      pb.capacity_tokens = cb.capacity_tokens;
      pb.spec_step = cb.spec_step;
      pb.prefill_budget_left = cb.prefill_budget_left;
      if (cb.first_entry < 0 || cb.n_entries < 0 || cb.first_entry + cb.n_entries > r->n_entries)
        fail("invalid-parameters", "batch entry range out of range");
      for (int64_t e = cb.first_entry; e < cb.first_entry + cb.n_entries; ++e) {
        const slos_entry* ce = &r->entries[e];
        const int32_t ref = slos_entry_req(ce);
        PlanEntry pe;
        if (ref >= 0 && ref < in->n_running) pe.id = in->running[ref].id ? in->running[ref].id : "";
        else if (ref < 0 && -ref - 1 < in->n_pending) pe.id = pid(-ref - 1);
        else fail("invalid-parameters", "entry reference out of range");
        pe.prefill_tokens = slos_entry_prefill_tokens(ce);
        pe.decode_tokens = slos_entry_decode_tokens(ce);
        pe.spec_len = slos_entry_spec_len(ce);
        pb.entries.push_back(std::move(pe));
      }
      res.plan.batches.push_back(std::move(pb));
    }
    try {
      text = plan_to_json(res, now_s);
    } catch (const std::exception& e) {  // nlohmann: ill-formed UTF-8 in an id
      fail("invalid-parameters", e.what());
    }
    return SLOS_OK;
  });
  if (st != SLOS_OK) return st;
  if (len) *len = (int64_t)text.size();
  if (buf && cap > 0) {
    const size_t m = (size_t)cap > text.size() ? text.size() : (size_t)cap;
    std::memcpy(buf, text.data(), m);
    if ((size_t)cap > text.size()) buf[text.size()] = '\0';
  }
  return SLOS_OK;
}
