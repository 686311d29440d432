// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// The drop-in proof, end to end: the reference's own discrete-event simulator
// (ReplicaSim / ClusterSim, sim_executor.cpp + tiers_router.cpp) and capacity
// sweep (simulate_scenario / capacity_search, metrics.cpp:214-313), compiled
// UNMODIFIED from /root/reference, with the planner behind the reference's
// `Scheduler` interface (dp_scheduler.hpp:81-86) swapped at the factory.
//
// oracle/Makefile links this file with the reference objects into
// oracle/_ref/libslos_refsim.so using `-Wl,--wrap=<make_scheduler>`: ReplicaSim's
// call to make_scheduler (sim_executor.cpp:59) lands in __wrap_make_scheduler
// below, which returns
//   * the reference SloScheduler (backend unset) -- optionally a recording
//     subclass that captures every ScheduleInput (the C5 sweep corpus), or
//   * GpuSloScheduler: the adapter of INTEGRATION.md, forwarding schedule() to
//     any library that exports include/slos_planner.h (the product
//     libslos_b200.so on the GPU box), loaded with dlopen.
// Comparing the RequestRecords of both runs checks the planner in the loop of
// the reference's routing (ClusterSim::on_decline, tiers_router.cpp:80-108) and
// sweep driver -- SURVEY.md §8 rows a13 and a14.

#include <dlfcn.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "slos_planner.h"
#include "slosim/baselines.hpp"
#include "slosim/common.hpp"
#include "slosim/dp_scheduler.hpp"
#include "slosim/metrics.hpp"
#include "slosim/perf_model.hpp"
#include "slosim/sim_executor.hpp"
#include "slosim/tiers_router.hpp"
#include "slosim/workload.hpp"

using namespace slosim;

namespace {

// ---- the backend: a dlopen'd library exporting include/slos_planner.h ----
struct Backend {
  void* dl = nullptr;
  int (*create)(const slos_perf_term*, int32_t, const double*, const double*, int32_t, int32_t,
                const slos_planner_config*, slos_planner**) = nullptr;
  void (*destroy)(slos_planner*) = nullptr;
  int (*plan)(slos_planner*, const slos_input*, int32_t, slos_result*) = nullptr;
  void (*free_result)(slos_result*) = nullptr;
  const char* (*slug)(int) = nullptr;
  const char* (*last_error)(void) = nullptr;
};

std::mutex g_mu;
Backend g_backend;          // dl == nullptr: the reference SloScheduler
bool g_record = false;
std::vector<ScheduleInput> g_recorded;
int64_t g_plans = 0;

// INTEGRATION.md's adapter, verbatim in behaviour: ScheduleInput -> slos_input,
// slos_plan, slos_result -> ScheduleResult (ids mapped back from indices).
class GpuSloScheduler : public Scheduler {
 public:
  GpuSloScheduler(const BatchPlanner& p, const Backend& be) : be_(be) {
    std::vector<slos_perf_term> t;
    for (const PerfTerm& x : p.model().terms()) t.push_back({x.k1, x.k2, x.b});
    const PlannerConfig& c = p.config();
    slos_planner_config cfg{c.max_chunk_tokens, c.max_batch_tokens, c.speculative ? 1 : 0,
                            c.spec_max_len, c.spec_alpha, c.plan_margin};
    const SloConfig& s = p.slo();
    check(be_.create(t.data(), (int)t.size(), s.tpot_tiers_s.data(), s.ttft_slowdowns.data(),
                     s.num_tiers(), s.tpot_window, &cfg, &h_));
  }
  ~GpuSloScheduler() override {
    if (h_) be_.destroy(h_);
  }
  std::string name() const override { return "slos"; }

  ScheduleResult schedule(const ScheduleInput& in) override {
    {
      std::lock_guard<std::mutex> g(g_mu);
      ++g_plans;
    }
    std::vector<slos_running> run;
    run.reserve(in.running.size());
    for (const RunningRequest& r : in.running)
      run.push_back({r.id.c_str(), r.prefill_remaining, r.prefill_deadline, r.decode_tier, 0, r.next_due_s,
                     r.backlog, r.decode_remaining});
    std::vector<slos_pending> pen;
    pen.reserve(in.pending.size());
    for (const PendingRequest& q : in.pending)
      pen.push_back({q.id.c_str(), q.prefill_deadline, q.prefill_tokens, q.decode_tier, 0, q.memory_units,
                     q.value});
    slos_input ci{in.now, run.data(), (int32_t)run.size(), (int32_t)pen.size(), pen.data(), in.memory_total,
                  in.memory_standard_resident, in.tail_horizon_s};
    slos_result r;
    check(be_.plan(h_, &ci, /*unit_value=*/0, &r));
    auto id = [&](int32_t ref) -> const std::string& {
      return ref >= 0 ? in.running[ref].id : in.pending[-ref - 1].id;
    };
    ScheduleResult out;
    for (int k = 0; k < r.n_admitted; ++k) out.admitted.push_back(in.pending[r.admitted[k]].id);
    for (int k = 0; k < r.n_declined; ++k) out.declined.push_back(in.pending[r.declined[k]].id);
    out.admitted_value = r.admitted_value;
    out.running_set_infeasible = r.running_set_infeasible != 0;
    out.plan.exact_until_s = r.exact_until_s;
    for (int64_t b = 0; b < r.n_batches; ++b) {
      const slos_batch& cb = r.batches[b];
      PlanBatch pb;
      pb.start_s = cb.start_s;
      pb.end_s = cb.end_s;
      pb.capacity_tokens = cb.capacity_tokens;
      pb.spec_step = cb.spec_step;
      pb.prefill_budget_left = cb.prefill_budget_left;
      for (int64_t e = cb.first_entry; e < cb.first_entry + cb.n_entries; ++e) {
        PlanEntry pe;
        pe.id = id(slos_entry_req(&r.entries[e]));
        pe.prefill_tokens = slos_entry_prefill_tokens(&r.entries[e]);
        pe.decode_tokens = slos_entry_decode_tokens(&r.entries[e]);
        pe.spec_len = slos_entry_spec_len(&r.entries[e]);
        pb.entries.push_back(std::move(pe));
      }
      out.plan.batches.push_back(std::move(pb));
    }
    be_.free_result(&r);
    return out;
  }

 private:
  void check(int st) const {
    if (st != SLOS_OK) fail(be_.slug(st), be_.last_error());  // the reference's slugs
  }
  const Backend& be_;
  slos_planner* h_ = nullptr;
};

// The reference planner, counting calls and optionally recording every input.
class RecordingScheduler : public SloScheduler {
 public:
  explicit RecordingScheduler(const BatchPlanner& p) : SloScheduler(p) {}
  ScheduleResult schedule(const ScheduleInput& in) override {
    {
      std::lock_guard<std::mutex> g(g_mu);
      ++g_plans;
      if (g_record) g_recorded.push_back(in);
    }
    return SloScheduler::schedule(in);
  }
};

// ---- deterministic digest of the simulation's records (FNV-1a over fields) ----
struct Fnv {
  uint64_t h = 1469598103934665603ULL;
  void bytes(const void* p, size_t n) {
    const unsigned char* c = (const unsigned char*)p;
    for (size_t k = 0; k < n; ++k) { h ^= c[k]; h *= 1099511628211ULL; }
  }
  template <typename T>
  void put(const T& v) { bytes(&v, sizeof v); }
  void str(const std::string& s) { put((uint64_t)s.size()); bytes(s.data(), s.size()); }
};

uint64_t digest(const std::vector<RequestRecord>& recs) {
  Fnv f;
  for (const RequestRecord& r : recs) {
    f.str(r.id);
    f.put(r.value); f.put((int)r.best_effort); f.put((int)r.dropped); f.put((int)r.completed);
    f.put(r.arrival_s); f.put(r.completion_s); f.put(r.first_token_s);
    f.put(r.hops); f.put(r.preemptions); f.put(r.tokens_out); f.put(r.total_tokens);
    for (const StageRecord& s : r.stages) {
      f.put((int)s.kind); f.put(s.tier); f.put(s.tokens); f.put(s.available_s); f.put(s.deadline_s);
      f.put(s.line_start_s); f.put(s.completed_s); f.put((int)s.on_time);
      f.put(s.windows_total); f.put(s.windows_violated);
      for (double x : s.tpot_samples) f.put(x);
    }
  }
  return f.h;
}

thread_local std::string g_err;

template <typename F>
int guarded(F&& fn) {
  try {
    return fn();
  } catch (const Error& e) {
    g_err = e.what();
    return e.code() == "infeasible-budget" ? SLOS_ERR_INFEASIBLE_BUDGET
           : e.code() == "internal-inconsistency" ? SLOS_ERR_INTERNAL_INCONSISTENCY
                                                  : SLOS_ERR_INVALID_PARAMETERS;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SLOS_ERR_INVALID_PARAMETERS;
  }
}

}  // namespace

// ---- the factory hook (ReplicaSim -> make_scheduler, sim_executor.cpp:59) ----
// --wrap=SYM sends sim_executor.o's undefined reference to SYM to __wrap_SYM and
// __real_SYM to the reference definition (baselines.cpp:175); SYM is the mangled
// slosim::make_scheduler(const std::string&, const BatchPlanner&).
#define SLOS_MK_SYM _ZN6slosim14make_schedulerERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEERKNS_12BatchPlannerE
extern "C" std::unique_ptr<Scheduler> __real__ZN6slosim14make_schedulerERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEERKNS_12BatchPlannerE(
    const std::string& name, const BatchPlanner& planner);

extern "C" std::unique_ptr<Scheduler> __wrap__ZN6slosim14make_schedulerERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEERKNS_12BatchPlannerE(
    const std::string& name, const BatchPlanner& planner) {
  if (name == "slos") {
    if (g_backend.dl) return std::make_unique<GpuSloScheduler>(planner, g_backend);
    return std::make_unique<RecordingScheduler>(planner);
  }
  return __real__ZN6slosim14make_schedulerERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEERKNS_12BatchPlannerE(
      name, planner);
}

extern "C" {

// Simulation knobs (ExecConfig sim_executor.hpp:24-41, ClusterConfig tiers_router.hpp:14-21).
typedef struct slos_sim_config {
  int32_t speculative;
  int32_t spec_max_len;
  double spec_alpha;
  double noise;
  int64_t memory_units;
  int64_t max_chunk_tokens;
  int64_t max_batch_tokens;
  int32_t replicas;
  int32_t routing_limit;
  int32_t backup_best_effort;  // 0: "decline", 1: "best_effort_on_origin"
  int32_t reserved0;
  double net_delay_s;
} slos_sim_config;

typedef struct slos_sim_summary {
  int64_t requests, standard, attained, best_effort, dropped, total_hops, plans, tokens_out;
  double attainment, overall_attainment;
  uint64_t digest;
} slos_sim_summary;

const char* slos_sim_last_error(void) { return g_err.c_str(); }

// Route the "slos" scheduler to `lib_path` (a library exporting slos_planner.h);
// NULL or "" restores the reference SloScheduler.
int slos_sim_set_backend(const char* lib_path) {
  std::lock_guard<std::mutex> g(g_mu);
  if (g_backend.dl) dlclose(g_backend.dl);
  g_backend = Backend{};
  if (!lib_path || !*lib_path) return SLOS_OK;
  void* dl = dlopen(lib_path, RTLD_NOW | RTLD_LOCAL);
  if (!dl) { g_err = dlerror(); return SLOS_ERR_INVALID_PARAMETERS; }
  Backend b;
  b.dl = dl;
  b.create = (decltype(b.create))dlsym(dl, "slos_planner_create");
  b.destroy = (decltype(b.destroy))dlsym(dl, "slos_planner_destroy");
  b.plan = (decltype(b.plan))dlsym(dl, "slos_plan");
  b.free_result = (decltype(b.free_result))dlsym(dl, "slos_result_free");
  b.slug = (decltype(b.slug))dlsym(dl, "slos_status_slug");
  b.last_error = (decltype(b.last_error))dlsym(dl, "slos_last_error");
  if (!b.create || !b.destroy || !b.plan || !b.free_result || !b.slug || !b.last_error) {
    dlclose(dl);
    g_err = "backend library lacks the slos_planner.h entry points";
    return SLOS_ERR_INVALID_PARAMETERS;
  }
  g_backend = b;
  return SLOS_OK;
}

void slos_sim_set_recording(int32_t on) {
  std::lock_guard<std::mutex> g(g_mu);
  g_record = on != 0;
  g_recorded.clear();
}

int64_t slos_sim_recorded_count(void) { return (int64_t)g_recorded.size(); }

// Append the recorded inputs to `path` (binary, little endian; parsed by
// paper_2504_08784_b200/workload.py load_corpus): per instance
//   f64 now, f64 tail_horizon_s, i64 memory_total, i64 memory_standard_resident,
//   i32 n_running, i32 n_pending,
//   n_running x {i64 prefill_remaining, f64 prefill_deadline, i32 decode_tier, i32 pad,
//                f64 next_due_s, i64 backlog, i64 decode_remaining}
//   n_pending x {f64 prefill_deadline, i64 prefill_tokens, i32 decode_tier, i32 pad,
//                i64 memory_units, f64 value}
//   then every id (running first, then pending) as u16 length + bytes.
int slos_sim_recorded_write(const char* path) {
  FILE* f = std::fopen(path, "ab");
  if (!f) { g_err = "cannot open corpus file"; return SLOS_ERR_INVALID_PARAMETERS; }
  auto w = [&](const void* p, size_t n) { std::fwrite(p, 1, n, f); };
  const int32_t pad = 0;
  for (const ScheduleInput& in : g_recorded) {
    const int32_t nr = (int32_t)in.running.size(), np = (int32_t)in.pending.size();
    w(&in.now, 8); w(&in.tail_horizon_s, 8); w(&in.memory_total, 8); w(&in.memory_standard_resident, 8);
    w(&nr, 4); w(&np, 4);
    for (const RunningRequest& r : in.running) {
      const int32_t t = r.decode_tier;
      w(&r.prefill_remaining, 8); w(&r.prefill_deadline, 8); w(&t, 4); w(&pad, 4);
      w(&r.next_due_s, 8); w(&r.backlog, 8); w(&r.decode_remaining, 8);
    }
    for (const PendingRequest& q : in.pending) {
      const int32_t t = q.decode_tier;
      w(&q.prefill_deadline, 8); w(&q.prefill_tokens, 8); w(&t, 4); w(&pad, 4);
      w(&q.memory_units, 8); w(&q.value, 8);
    }
    auto ws = [&](const std::string& s) {
      const uint16_t n = (uint16_t)s.size();
      w(&n, 2);
      w(s.data(), s.size());
    };
    for (const RunningRequest& r : in.running) ws(r.id);
    for (const PendingRequest& q : in.pending) ws(q.id);
  }
  std::fclose(f);
  return SLOS_OK;
}

static ExecConfig exec_of(const slos_sim_config* c) {
  ExecConfig e;
  e.scheduler = "slos";
  e.speculative = c->speculative != 0;
  e.spec_max_len = c->spec_max_len;
  e.spec_alpha = c->spec_alpha;
  e.noise = c->noise;
  e.memory_units = c->memory_units;
  e.max_chunk_tokens = c->max_chunk_tokens;
  e.max_batch_tokens = c->max_batch_tokens;
  return e;
}

static ClusterConfig cluster_of(const slos_sim_config* c) {
  ClusterConfig k;
  k.replicas = c->replicas;
  k.routing_limit = c->routing_limit;
  k.backup = c->backup_best_effort ? "best_effort_on_origin" : "decline";
  k.net_delay_s = c->net_delay_s;
  return k;
}

// simulate_scenario(scale_scenario(scenario, scale), ...) (metrics.cpp:214-232)
// with the configured scheduler backend; fills a summary and the record digest.
static PerfModel model_of(const slos_perf_term* terms, int32_t n) {
  std::vector<PerfTerm> t;
  for (int k = 0; k < n; ++k) t.push_back({terms[k].k1, terms[k].k2, terms[k].b});
  return PerfModel(std::move(t));
}

int slos_sim_scenario(const char* scenario_path, const slos_perf_term* terms, int32_t n_terms,
                      const slos_sim_config* cfg, uint64_t seed, double horizon_s, double scale,
                      slos_sim_summary* out) {
  return guarded([&] {
    const ScenarioConfig sc = scale_scenario(load_scenario_file(scenario_path), scale);
    const PerfModel model = model_of(terms, n_terms);
    {
      std::lock_guard<std::mutex> g(g_mu);
      g_plans = 0;
    }
    const std::vector<RequestRecord> recs =
        simulate_scenario(sc, model, exec_of(cfg), cluster_of(cfg), seed, horizon_s);
    const SummaryStats st = summarize(recs);
    std::memset(out, 0, sizeof *out);
    out->requests = st.total_requests;
    out->standard = st.standard_requests;
    out->attained = st.standard_attained;
    out->best_effort = st.best_effort_requests;
    out->dropped = st.dropped_requests;
    for (const RequestRecord& r : recs) out->total_hops += r.hops;
    out->plans = g_plans;
    out->tokens_out = st.tokens_out;
    out->attainment = st.attainment;
    out->overall_attainment = st.overall_attainment;
    out->digest = digest(recs);
    return SLOS_OK;
  });
}

// capacity_search (metrics.cpp:234-313) with the configured scheduler backend.
int slos_sim_capacity(const char* scenario_path, const slos_perf_term* terms, int32_t n_terms,
                      const slos_sim_config* cfg,
                      double target, double lo_scale, double hi_scale, double rel_tol, int32_t seeds,
                      uint64_t base_seed, double horizon_s, double* scale_out, double* per_gpu_rate_out,
                      double* attainment_out, int32_t* evaluations_out) {
  return guarded([&] {
    const ScenarioConfig sc = load_scenario_file(scenario_path);
    const PerfModel model = model_of(terms, n_terms);
    CapacityOptions o;
    o.target_attainment = target;
    o.lo_scale = lo_scale;
    o.hi_scale = hi_scale;
    o.rel_tolerance = rel_tol;
    o.seeds_per_rate = seeds;
    o.base_seed = base_seed;
    o.horizon_s = horizon_s;
    const CapacityResult r = capacity_search(sc, model, exec_of(cfg), cluster_of(cfg), o);
    *scale_out = r.scale;
    *per_gpu_rate_out = r.per_gpu_rate;
    *attainment_out = r.attainment_at;
    *evaluations_out = r.evaluations;
    return SLOS_OK;
  });
}

}  // extern "C"
