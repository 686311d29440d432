// Batched routing rounds and lockstep simulation lanes (include/slos_lockstep.h).
//
// Reference-side integration layer: the reference's ReplicaSim (sim_executor.cpp)
// is reused unmodified as the caller of the planner; what is new is how the
// cluster's replicas and many simulations are advanced so their schedule() calls
// can be served in batches by the plan broker of a library exporting
// include/slos_planner.h.
//
// Equivalence with the reference's sequential ClusterSim::run (tiers_router.cpp:
// 110-174). The reference loop repeatedly takes the earliest of (a) the transfer
// heap's top (ties: transfers first, then heap order (t, seq)) and (b) the replica
// with the smallest next_time() (ties: lowest index), and runs ONE iteration:
// advance that replica (its schedule() calls happen inside), or deliver that
// transfer (advance_to + inject). Replicas interact only through transfers, and a
// transfer created while a replica is at time t (on_decline, :80-108) is due at
// t + net_delay_s, while every iteration happens at a time >= the earliest pending
// event T. Hence all iterations before W = T + net_delay_s are independent of the
// transfers created in them, and a replica's own sequence of iterations before W
// is determined by its state and the transfers already queued for it: transfer x
// precedes the replica's own event at t_own iff t_x <= t_own (the reference's
// `ev_t <= rep_t`). Each replica therefore runs its window on its own thread with
// exactly the reference's sequence of calls; the transfers the window creates are
// then numbered (seq) in the reference's global iteration order -- key (time,
// transfer-before-replica, heap seq | replica index, per-replica order) -- and
// pushed. Lanes (independent simulations) share nothing but the broker.
//
// Built by integration/Makefile with the reference's simulator sources compiled
// in place and `-Wl,--wrap` on slosim::make_scheduler (sim_executor.cpp:59), so a
// replica's "slos" scheduler is a BrokerScheduler over the backend library (or,
// without a backend, the reference SloScheduler itself).

#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "slos_lockstep.h"
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

constexpr double kInf = std::numeric_limits<double>::infinity();

// ---- backend: a dlopen'd library exporting include/slos_planner.h ----------
struct Backend {
  void* dl = nullptr;
  int (*create)(const slos_perf_term*, int32_t, const double*, const double*, int32_t, int32_t,
                const slos_planner_config*, slos_planner**) = nullptr;
  void (*destroy)(slos_planner*) = nullptr;
  void (*free_result)(slos_result*) = nullptr;
  const char* (*slug)(int) = nullptr;
  const char* (*last_error)(void) = nullptr;
  int (*broker_create)(int32_t, slos_broker**) = nullptr;
  void (*broker_destroy)(slos_broker*) = nullptr;
  void (*join)(slos_broker*) = nullptr;
  void (*leave)(slos_broker*) = nullptr;
  int (*plan)(slos_broker*, slos_planner*, const slos_input*, slos_result*) = nullptr;
  void (*stats)(slos_broker*, int64_t*, int64_t*) = nullptr;
};

std::mutex g_mu;
Backend g_be;
slos_broker* g_broker = nullptr;
std::atomic<int64_t> g_plans{0};
std::atomic<int64_t> g_windows{0};
thread_local std::string g_err;
// the lane whose replicas are being constructed on this thread (per-lane plan count)
thread_local std::atomic<int64_t>* tl_lane_plans = nullptr;

void broker_join() {
  if (g_broker) g_be.join(g_broker);
}
void broker_leave() {
  if (g_broker) g_be.leave(g_broker);
}

// Planner handles, one per distinct (model, SLO, config): the plans of one broker
// flush run inside one slos_plan_batch call, and the product's handles are read-only.
std::mutex g_hmu;
std::map<std::string, slos_planner*> g_handles;

slos_planner* handle_for(const BatchPlanner& p) {
  std::vector<slos_perf_term> t;
  for (const PerfTerm& x : p.model().terms()) t.push_back({x.k1, x.k2, x.b});
  const PlannerConfig& c = p.config();
  slos_planner_config cfg{c.max_chunk_tokens, c.max_batch_tokens, c.speculative ? 1 : 0, c.spec_max_len,
                          c.spec_alpha, c.plan_margin};
  const SloConfig& s = p.slo();
  std::string key;
  auto put = [&](const void* q, size_t n) { key.append((const char*)q, n); };
  put(t.data(), t.size() * sizeof(slos_perf_term));
  put(&cfg, sizeof cfg);
  put(s.tpot_tiers_s.data(), s.tpot_tiers_s.size() * sizeof(double));
  put(s.ttft_slowdowns.data(), s.ttft_slowdowns.size() * sizeof(double));
  put(&s.tpot_window, sizeof s.tpot_window);
  std::lock_guard<std::mutex> g(g_hmu);
  auto it = g_handles.find(key);
  if (it != g_handles.end()) return it->second;
  slos_planner* h = nullptr;
  const int st = g_be.create(t.data(), (int)t.size(), s.tpot_tiers_s.data(), s.ttft_slowdowns.data(),
                             s.num_tiers(), s.tpot_window, &cfg, &h);
  if (st != SLOS_OK) fail(g_be.slug(st), g_be.last_error());
  g_handles.emplace(key, h);
  return h;
}

// The INTEGRATION.md adapter with slos_plan replaced by the broker: the calling
// replica thread blocks until its plan's batch has run.
class BrokerScheduler : public Scheduler {
 public:
  explicit BrokerScheduler(const BatchPlanner& p) : h_(handle_for(p)), lane_plans_(tl_lane_plans) {}
  std::string name() const override { return "slos"; }

  ScheduleResult schedule(const ScheduleInput& in) override {
    g_plans.fetch_add(1, std::memory_order_relaxed);
    if (lane_plans_) lane_plans_->fetch_add(1, std::memory_order_relaxed);
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
    std::memset(&r, 0, sizeof r);
    const int st = g_be.plan(g_broker, h_, &ci, &r);
    if (st != SLOS_OK) fail(g_be.slug(st), g_be.last_error());
    auto id = [&](int32_t ref) -> const std::string& {
      return ref >= 0 ? in.running[ref].id : in.pending[-ref - 1].id;
    };
    ScheduleResult out;
    out.admitted.reserve((size_t)r.n_admitted);
    for (int k = 0; k < r.n_admitted; ++k) out.admitted.push_back(in.pending[r.admitted[k]].id);
    for (int k = 0; k < r.n_declined; ++k) out.declined.push_back(in.pending[r.declined[k]].id);
    out.admitted_value = r.admitted_value;
    out.running_set_infeasible = r.running_set_infeasible != 0;
    out.plan.exact_until_s = r.exact_until_s;
    out.plan.batches.reserve((size_t)r.n_batches);
    for (int64_t b = 0; b < r.n_batches; ++b) {
      const slos_batch& cb = r.batches[b];
      PlanBatch pb;
      pb.start_s = cb.start_s;
      pb.end_s = cb.end_s;
      pb.capacity_tokens = cb.capacity_tokens;
      pb.spec_step = cb.spec_step;
      pb.prefill_budget_left = cb.prefill_budget_left;
      pb.entries.reserve((size_t)cb.n_entries);
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
    g_be.free_result(&r);
    return out;
  }

 private:
  slos_planner* h_;
  std::atomic<int64_t>* lane_plans_;
};

// The reference planner, counting calls (no backend).
class CountingScheduler : public SloScheduler {
 public:
  explicit CountingScheduler(const BatchPlanner& p) : SloScheduler(p), lane_plans_(tl_lane_plans) {}
  ScheduleResult schedule(const ScheduleInput& in) override {
    g_plans.fetch_add(1, std::memory_order_relaxed);
    if (lane_plans_) lane_plans_->fetch_add(1, std::memory_order_relaxed);
    return SloScheduler::schedule(in);
  }

 private:
  std::atomic<int64_t>* lane_plans_;
};

// ---- deterministic digest of a simulation's records (FNV-1a over fields) ----
struct Fnv {
  uint64_t h = 1469598103934665603ULL;
  void bytes(const void* p, size_t n) {
    const unsigned char* c = (const unsigned char*)p;
    for (size_t k = 0; k < n; ++k) {
      h ^= c[k];
      h *= 1099511628211ULL;
    }
  }
  template <typename T>
  void put(const T& v) {
    bytes(&v, sizeof v);
  }
  void str(const std::string& s) {
    put((uint64_t)s.size());
    bytes(s.data(), s.size());
  }
};

uint64_t digest(const std::vector<RequestRecord>& recs) {
  Fnv f;
  for (const RequestRecord& r : recs) {
    f.str(r.id);
    f.put(r.value);
    f.put((int)r.best_effort);
    f.put((int)r.dropped);
    f.put((int)r.completed);
    f.put(r.arrival_s);
    f.put(r.completion_s);
    f.put(r.first_token_s);
    f.put(r.hops);
    f.put(r.preemptions);
    f.put(r.tokens_out);
    f.put(r.total_tokens);
    for (const StageRecord& s : r.stages) {
      f.put((int)s.kind);
      f.put(s.tier);
      f.put(s.tokens);
      f.put(s.available_s);
      f.put(s.deadline_s);
      f.put(s.line_start_s);
      f.put(s.completed_s);
      f.put((int)s.on_time);
      f.put(s.windows_total);
      f.put(s.windows_violated);
      for (double x : s.tpot_samples) f.put(x);
    }
  }
  return f.h;
}

// ---- per-replica worker threads --------------------------------------------
// One persistent thread per replica of a lane: the lane posts a window task to the
// replicas that have work before W and waits for them.
class Gang {
 public:
  explicit Gang(int n) : n_(n), task_(n), err_(n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~Gang() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // Run fn(i) for every i with want[i] on its thread; returns the first error.
  std::string run(const std::vector<char>& want, const std::function<void(int)>& fn) {
    int k = 0;
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      for (int i = 0; i < n_; ++i) {
        task_[i] = want[i];
        err_[i].clear();
        k += want[i] ? 1 : 0;
      }
      pending_ = k;
      ++gen_;
    }
    // the workers count as active for the broker from the moment they are posted,
    // so no flush can fire between this lane going idle and its workers starting
    for (int j = 0; j < k; ++j) broker_join();
    broker_leave();  // the lane itself waits
    cv_.notify_all();
    {
      std::unique_lock<std::mutex> lk(mu_);
      done_cv_.wait(lk, [&] { return pending_ == 0; });
    }
    broker_join();
    for (int i = 0; i < n_; ++i)
      if (!err_[i].empty()) return err_[i];
    return {};
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    while (true) {
      const std::function<void(int)>* fn = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && task_[i]); });
        if (stop_) return;
        seen = gen_;
        fn = fn_;
      }
      try {
        (*fn)(i);
      } catch (const std::exception& e) {
        err_[i] = e.what();
        if (err_[i].empty()) err_[i] = "error";
      }
      broker_leave();
      {
        std::lock_guard<std::mutex> g(mu_);
        task_[i] = 0;
        if (--pending_ == 0) done_cv_.notify_all();
      }
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::vector<char> task_;
  std::vector<std::string> err_;
  const std::function<void(int)>* fn_ = nullptr;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

// replica_seed (tiers_router.cpp:18-24): spreads replica seeds apart.
uint64_t replica_seed(uint64_t base, int idx) {
  uint64_t x = base + 0x9E3779B97F4A7C15ULL * (uint64_t)(idx + 1);
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  return x;
}

// ---- one lane: ClusterSim (tiers_router.cpp:58-174) in lookahead windows ----
class Lane {
 public:
  Lane(const PerfModel& model, const ScenarioConfig& sc, const ExecConfig& exec, const ClusterConfig& cluster,
       uint64_t seed, double horizon_s)
      : cluster_(cluster) {
    // simulate_scenario (metrics.cpp:223-232)
    trace_ = generate_trace(sc, seed, horizon_s);
    ExecConfig e = exec;
    e.seed = seed;
    cluster_.validate();
    const int n = cluster_.replicas;
    tl_lane_plans = &plans_;
    for (int i = 0; i < n; ++i) {  // ClusterSim::ClusterSim (tiers_router.cpp:58-78)
      ExecConfig rc = e;
      rc.seed = n == 1 ? e.seed : replica_seed(e.seed, i);
      reps_.push_back(std::make_unique<ReplicaSim>(model, sc.slo, rc,
                                                   [this, i](const std::string& id) { return on_decline(i, id); }));
    }
    tl_lane_plans = nullptr;
    key_.resize((size_t)n);
    pushes_.resize((size_t)n);
    drops_.resize((size_t)n);
  }

  std::vector<RequestRecord> run(Gang& gang) {
    // arrivals, round-robin origins (tiers_router.cpp:114-127)
    std::vector<RequestSpec> sorted = trace_;
    std::sort(sorted.begin(), sorted.end(), [](const RequestSpec& a, const RequestSpec& b) {
      if (a.arrival_s != b.arrival_s) return a.arrival_s < b.arrival_s;
      return a.id < b.id;
    });
    const int n = (int)reps_.size();
    int rr = 0;
    for (const RequestSpec& req : sorted) {
      if (routes_.count(req.id)) fail("invalid-parameters", "duplicate request id " + req.id);
      routes_.emplace(req.id, RouteState{req, rr, 0});
      heap_.push({req.arrival_s, seq_++, rr, false, 0, req.id});
      rr = (rr + 1) % n;
    }
    std::vector<double> nt((size_t)n);
    std::vector<char> want((size_t)n);
    std::vector<std::vector<Transfer>> tq((size_t)n);
    const double delay = cluster_.net_delay_s;
    int64_t guard = 0;
    while (true) {
      if (++guard > 200000000LL) fail("internal-inconsistency", "cluster simulation stuck");
      if (heap_.empty()) {
        bool all = true;
        for (auto& rep : reps_)
          if (!rep->drained()) {
            all = false;
            break;
          }
        if (all) break;
      }
      const double ev_t = heap_.empty() ? kInf : heap_.top().t;
      double rep_t = kInf;
      int bi = -1;
      for (int i = 0; i < n; ++i) {
        nt[i] = reps_[i]->next_time();
        if (nt[i] < rep_t) {
          rep_t = nt[i];
          bi = i;
        }
      }
      if (ev_t == kInf && bi < 0) fail("internal-inconsistency", "cluster idle with undrained replicas");
      g_windows.fetch_add(1, std::memory_order_relaxed);
      if (!(delay > 0.0)) {  // no lookahead: exactly one reference iteration
        if (ev_t <= rep_t) {
          Transfer tr = heap_.top();
          heap_.pop();
          ReplicaSim& rep = *reps_[tr.target];
          key_[tr.target] = {tr.t, 0, tr.seq, 0};
          rep.advance_to(tr.t);
          rep.inject(routes_.at(tr.id).spec, tr.t, tr.best_effort, tr.hops);
        } else {
          key_[bi] = {rep_t, 1, bi, 0};
          reps_[bi]->advance_to(rep_t);
        }
        merge();
        continue;
      }
      const double W = std::min(ev_t, rep_t) + delay;
      for (int i = 0; i < n; ++i) tq[i].clear();
      while (!heap_.empty() && heap_.top().t < W) {
        tq[heap_.top().target].push_back(heap_.top());
        heap_.pop();
      }
      int busy = 0, only = -1;
      for (int i = 0; i < n; ++i) {
        want[i] = (!tq[i].empty() || nt[i] < W) ? 1 : 0;
        if (want[i]) {
          ++busy;
          only = i;
        }
      }
      auto task = [&](int i) {
        ReplicaSim& rep = *reps_[i];
        size_t x = 0;
        int64_t k = 0;
        while (true) {
          const double t_own = rep.next_time();
          if (x < tq[i].size() && tq[i][x].t <= t_own) {
            const Transfer& tr = tq[i][x++];
            key_[i] = {tr.t, 0, tr.seq, 0};
            rep.advance_to(tr.t);
            rep.inject(routes_.at(tr.id).spec, tr.t, tr.best_effort, tr.hops);
          } else if (t_own < W) {
            key_[i] = {t_own, 1, i, k++};
            rep.advance_to(t_own);
          } else {
            break;
          }
        }
      };
      if (busy == 1) {
        task(only);  // one replica has work: run it on the lane's own thread
      } else {
        const std::string err = gang.run(want, task);
        if (!err.empty()) fail("internal-inconsistency", err);
      }
      merge();
    }
    std::vector<RequestRecord> out = std::move(dropped_);
    for (auto& rep : reps_) {
      auto part = rep->finalize();
      out.insert(out.end(), std::make_move_iterator(part.begin()), std::make_move_iterator(part.end()));
    }
    std::sort(out.begin(), out.end(), [](const RequestRecord& a, const RequestRecord& b) {
      if (a.arrival_s != b.arrival_s) return a.arrival_s < b.arrival_s;
      return a.id < b.id;
    });
    return out;
  }

  int replicas() const { return (int)reps_.size(); }
  int64_t plans() const { return plans_.load(); }

 private:
  struct Transfer {
    double t = 0.0;
    int64_t seq = 0;
    int target = 0;
    bool best_effort = false;
    int hops = 0;
    std::string id;
    bool operator>(const Transfer& o) const {
      if (t != o.t) return t > o.t;
      return seq > o.seq;
    }
  };
  struct RouteState {
    RequestSpec spec;
    int origin = 0;
    int hops = 0;
  };
  // position of an iteration in the reference loop's order
  struct Key {
    double t = 0.0;
    int kind = 0;     // 0: transfer delivery, 1: replica event
    int64_t a = 0;    // transfer seq | replica index
    int64_t b = 0;    // per-replica order of its own events
    bool operator<(const Key& o) const {
      if (t != o.t) return t < o.t;
      if (kind != o.kind) return kind < o.kind;
      if (a != o.a) return a < o.a;
      return b < o.b;
    }
  };
  struct Push {
    Key key;
    int order;
    Transfer tr;
  };

  // ClusterSim::on_decline (tiers_router.cpp:80-108), on the declining replica's
  // thread: the transfer is queued with the current iteration's key and numbered
  // after the window (merge).
  DeclineAction on_decline(int i, const std::string& id) {
    RouteState& rs = routes_.at(id);
    const int n = (int)reps_.size();
    const int effective_limit = std::min(cluster_.routing_limit, n - 1);
    const double t = reps_[i]->now() + cluster_.net_delay_s;
    auto push = [&](int target, bool be) {
      pushes_[i].push_back({key_[i], (int)pushes_[i].size(), Transfer{t, 0, target, be, rs.hops, id}});
    };
    if (rs.hops < effective_limit) {
      ++rs.hops;
      push((i + 1) % n, false);
      return DeclineAction::kRemove;
    }
    if (cluster_.backup == "best_effort_on_origin") {
      if (i == rs.origin) return DeclineAction::kDemoteBestEffort;
      push(rs.origin, true);
      return DeclineAction::kRemove;
    }
    RequestRecord rec;  // backup "decline": the request leaves the system unserved
    rec.id = id;
    rec.value = rs.spec.value;
    rec.arrival_s = rs.spec.arrival_s;
    rec.total_tokens = rs.spec.total_tokens();
    rec.hops = rs.hops;
    rec.dropped = true;
    drops_[i].push_back(std::move(rec));
    return DeclineAction::kRemove;
  }

  // the window's transfers, numbered in the reference's iteration order
  void merge() {
    std::vector<Push> all;
    for (auto& v : pushes_) {
      for (auto& p : v) all.push_back(std::move(p));
      v.clear();
    }
    std::sort(all.begin(), all.end(), [](const Push& x, const Push& y) {
      if (x.key < y.key) return true;
      if (y.key < x.key) return false;
      return x.order < y.order;
    });
    for (Push& p : all) {
      p.tr.seq = seq_++;
      heap_.push(std::move(p.tr));
    }
    for (auto& v : drops_) {
      for (auto& r : v) dropped_.push_back(std::move(r));
      v.clear();
    }
  }

  ClusterConfig cluster_;
  std::atomic<int64_t> plans_{0};
  std::vector<RequestSpec> trace_;
  std::vector<std::unique_ptr<ReplicaSim>> reps_;
  std::unordered_map<std::string, RouteState> routes_;
  std::priority_queue<Transfer, std::vector<Transfer>, std::greater<Transfer>> heap_;
  int64_t seq_ = 0;
  std::vector<RequestRecord> dropped_;
  std::vector<Key> key_;
  std::vector<std::vector<Push>> pushes_;
  std::vector<std::vector<RequestRecord>> drops_;
};

ExecConfig exec_of(const slos_sim_config* c) {
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

ClusterConfig cluster_of(const slos_sim_config* c) {
  ClusterConfig k;
  k.replicas = c->replicas;
  k.routing_limit = c->routing_limit;
  k.backup = c->backup_best_effort ? "best_effort_on_origin" : "decline";
  k.net_delay_s = c->net_delay_s;
  return k;
}

PerfModel model_of(const slos_perf_term* terms, int32_t n) {
  std::vector<PerfTerm> t;
  for (int k = 0; k < n; ++k) t.push_back({terms[k].k1, terms[k].k2, terms[k].b});
  return PerfModel(std::move(t));
}

// One simulation as a lane on its own thread (lane coordinator + replica gang).
struct LaneJob {
  const PerfModel* model;
  ScenarioConfig sc;
  ExecConfig exec;
  ClusterConfig cluster;
  uint64_t seed;
  double horizon;
  std::vector<RequestRecord> recs;
  int64_t plans = 0;
  std::string err;
};

// Run every job as a concurrent lane; the calling thread only waits.
void run_lanes(std::vector<LaneJob>& jobs) {
  std::vector<std::thread> th;
  th.reserve(jobs.size());
  for (int j = 0; j < (int)jobs.size(); ++j) broker_join();  // lanes are active from the start
  for (LaneJob& J : jobs) {
    th.emplace_back([&J] {
      try {
        Lane lane(*J.model, J.sc, J.exec, J.cluster, J.seed, J.horizon);
        Gang gang(lane.replicas());
        J.recs = lane.run(gang);
        J.plans = lane.plans();
      } catch (const std::exception& e) {
        J.err = e.what();
      }
      broker_leave();
    });
  }
  for (auto& t : th) t.join();
}

template <typename F>
int guarded(F&& fn) {
  try {
    return fn();
  } catch (const Error& e) {
    g_err = e.what();
    return e.code() == "infeasible-budget"        ? SLOS_ERR_INFEASIBLE_BUDGET
           : e.code() == "internal-inconsistency" ? SLOS_ERR_INTERNAL_INCONSISTENCY
                                                  : SLOS_ERR_INVALID_PARAMETERS;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SLOS_ERR_INVALID_PARAMETERS;
  }
}

void fill_summary(const std::vector<RequestRecord>& recs, slos_sim_summary* out) {
  const SummaryStats st = summarize(recs);
  std::memset(out, 0, sizeof *out);
  out->requests = st.total_requests;
  out->standard = st.standard_requests;
  out->attained = st.standard_attained;
  out->best_effort = st.best_effort_requests;
  out->dropped = st.dropped_requests;
  for (const RequestRecord& r : recs) out->total_hops += r.hops;
  out->tokens_out = st.tokens_out;
  out->attainment = st.attainment;
  out->overall_attainment = st.overall_attainment;
  out->digest = digest(recs);
}

struct StatScope {  // plans / flushes / windows / wall of one call
  slos_lockstep_stats* out;
  int64_t p0, f0, w0;
  std::chrono::steady_clock::time_point t0;
  explicit StatScope(slos_lockstep_stats* o) : out(o) {
    p0 = g_plans.load();
    w0 = g_windows.load();
    int64_t pl = 0;
    f0 = 0;
    if (g_broker) g_be.stats(g_broker, &f0, &pl);
    t0 = std::chrono::steady_clock::now();
  }
  ~StatScope() {
    if (!out) return;
    out->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    out->plans = g_plans.load() - p0;
    out->windows = g_windows.load() - w0;
    if (g_broker) {
      int64_t f = 0, pl = 0;
      g_be.stats(g_broker, &f, &pl);
      out->flushes = f - f0;
    } else {
      out->flushes = out->plans;
    }
  }
};

}  // namespace

// ---- the factory hook (ReplicaSim -> make_scheduler, sim_executor.cpp:59) ----
extern "C" std::unique_ptr<Scheduler> __real__ZN6slosim14make_schedulerERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEERKNS_12BatchPlannerE(
    const std::string& name, const BatchPlanner& planner);

extern "C" std::unique_ptr<Scheduler> __wrap__ZN6slosim14make_schedulerERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEERKNS_12BatchPlannerE(
    const std::string& name, const BatchPlanner& planner) {
  if (name == "slos") {
    if (g_be.dl) return std::make_unique<BrokerScheduler>(planner);
    return std::make_unique<CountingScheduler>(planner);
  }
  return __real__ZN6slosim14make_schedulerERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEERKNS_12BatchPlannerE(
      name, planner);
}

extern "C" {

const char* slos_lockstep_last_error(void) { return g_err.c_str(); }

int slos_lockstep_set_backend(const char* lib_path) {
  std::lock_guard<std::mutex> g(g_mu);
  {
    std::lock_guard<std::mutex> h(g_hmu);
    for (auto& kv : g_handles) g_be.destroy(kv.second);
    g_handles.clear();
  }
  if (g_broker) g_be.broker_destroy(g_broker);
  g_broker = nullptr;
  if (g_be.dl) dlclose(g_be.dl);
  g_be = Backend{};
  if (!lib_path || !*lib_path) return SLOS_OK;
  void* dl = dlopen(lib_path, RTLD_NOW | RTLD_LOCAL);
  if (!dl) {
    g_err = dlerror();
    return SLOS_ERR_INVALID_PARAMETERS;
  }
  Backend b;
  b.dl = dl;
  b.create = (decltype(b.create))dlsym(dl, "slos_planner_create");
  b.destroy = (decltype(b.destroy))dlsym(dl, "slos_planner_destroy");
  b.free_result = (decltype(b.free_result))dlsym(dl, "slos_result_free");
  b.slug = (decltype(b.slug))dlsym(dl, "slos_status_slug");
  b.last_error = (decltype(b.last_error))dlsym(dl, "slos_last_error");
  b.broker_create = (decltype(b.broker_create))dlsym(dl, "slos_broker_create");
  b.broker_destroy = (decltype(b.broker_destroy))dlsym(dl, "slos_broker_destroy");
  b.join = (decltype(b.join))dlsym(dl, "slos_broker_join");
  b.leave = (decltype(b.leave))dlsym(dl, "slos_broker_leave");
  b.plan = (decltype(b.plan))dlsym(dl, "slos_broker_plan");
  b.stats = (decltype(b.stats))dlsym(dl, "slos_broker_stats");
  if (!b.create || !b.destroy || !b.free_result || !b.slug || !b.last_error || !b.broker_create ||
      !b.broker_destroy || !b.join || !b.leave || !b.plan || !b.stats) {
    dlclose(dl);
    g_err = "backend library lacks the slos_planner.h entry points (with the plan broker)";
    return SLOS_ERR_INVALID_PARAMETERS;
  }
  slos_broker* br = nullptr;
  if (b.broker_create(0, &br) != SLOS_OK) {
    dlclose(dl);
    g_err = "slos_broker_create failed";
    return SLOS_ERR_INVALID_PARAMETERS;
  }
  g_be = b;
  g_broker = br;
  return SLOS_OK;
}

int slos_lockstep_simulate(int32_t n, const char* const* paths, const slos_perf_term* terms, int32_t n_terms,
                           const slos_sim_config* cfgs, const uint64_t* seeds, const double* horizons,
                           const double* scales, slos_sim_summary* outs, slos_lockstep_stats* stats) {
  std::lock_guard<std::mutex> g(g_mu);
  StatScope scope(stats);
  return guarded([&] {
    const PerfModel model = model_of(terms, n_terms);
    std::vector<LaneJob> jobs((size_t)n);
    for (int k = 0; k < n; ++k) {
      LaneJob& J = jobs[k];
      J.model = &model;
      J.sc = scale_scenario(load_scenario_file(paths[k]), scales[k]);
      J.exec = exec_of(&cfgs[k]);
      J.cluster = cluster_of(&cfgs[k]);
      J.seed = seeds[k];
      J.horizon = horizons[k];
    }
    const int64_t p0 = g_plans.load();
    run_lanes(jobs);
    (void)p0;
    for (int k = 0; k < n; ++k) {
      if (!jobs[k].err.empty()) fail("internal-inconsistency", jobs[k].err);
      fill_summary(jobs[k].recs, &outs[k]);
      outs[k].plans = jobs[k].plans;
    }
    return SLOS_OK;
  });
}

// capacity_search (metrics.cpp:234-313), n searches at once: each search is a
// thread running the bisection; eval_median's seeds are lanes.
int slos_lockstep_capacity(int32_t n, const char* const* paths, const slos_perf_term* terms, int32_t n_terms,
                           const slos_sim_config* cfgs, double target, double lo_scale, double hi_scale,
                           double rel_tol, int32_t seeds_per_rate, uint64_t base_seed, double horizon_s,
                           slos_capacity_result* outs, slos_lockstep_stats* stats) {
  std::lock_guard<std::mutex> g(g_mu);
  StatScope scope(stats);
  return guarded([&] {
    if (lo_scale <= 0 || hi_scale <= lo_scale) fail("invalid-parameters", "need 0 < lo_scale < hi_scale");
    if (target <= 0 || target > 1) fail("invalid-parameters", "target attainment must be in (0, 1]");
    if (rel_tol <= 0) fail("invalid-parameters", "tolerance must be positive");
    if (seeds_per_rate < 1) fail("invalid-parameters", "need at least one seed");
    if (horizon_s <= 0) fail("invalid-parameters", "horizon must be positive");
    const PerfModel model = model_of(terms, n_terms);
    std::vector<std::string> errs((size_t)n);
    std::vector<std::thread> th;
    for (int q = 0; q < n; ++q) {
      th.emplace_back([&, q] {
        try {
          const ScenarioConfig scenario = load_scenario_file(paths[q]);
          const ExecConfig exec = exec_of(&cfgs[q]);
          const ClusterConfig cluster = cluster_of(&cfgs[q]);
          int evals = 0;
          auto eval_median = [&](double scale) -> double {  // metrics.cpp:246-273
            const ScenarioConfig sc = scale_scenario(scenario, scale);
            std::vector<LaneJob> jobs((size_t)seeds_per_rate);
            for (int s = 0; s < seeds_per_rate; ++s) {
              LaneJob& J = jobs[s];
              J.model = &model;
              J.sc = sc;
              J.exec = exec;
              J.cluster = cluster;
              J.seed = base_seed + 1000003ULL * (uint64_t)s;
              J.horizon = horizon_s;
            }
            run_lanes(jobs);
            std::vector<double> atts((size_t)seeds_per_rate, 0.0);
            for (int s = 0; s < seeds_per_rate; ++s) {
              if (!jobs[s].err.empty()) fail("internal-inconsistency", jobs[s].err);
              int64_t attained = 0;
              for (const RequestRecord& r : jobs[s].recs)
                if (!r.best_effort && !r.dropped && r.attained()) ++attained;
              atts[s] = jobs[s].recs.empty() ? 1.0 : (double)attained / (double)jobs[s].recs.size();
            }
            std::sort(atts.begin(), atts.end());
            ++evals;
            return atts[atts.size() / 2];
          };
          double lo = lo_scale, hi = hi_scale;  // metrics.cpp:275-297
          const double att_lo = eval_median(lo);
          if (att_lo < target)
            fail("bounds-not-bracketing",
                 "attainment " + std::to_string(att_lo) + " at lo_scale already misses the target");
          double att_at = att_lo;
          const double att_hi = eval_median(hi);
          if (att_hi >= target) {
            lo = hi;
            att_at = att_hi;
          } else {
            int guard = 0;
            while ((hi - lo) / lo > rel_tol && ++guard <= 64) {
              const double mid = 0.5 * (lo + hi);
              const double a = eval_median(mid);
              if (a >= target) {
                lo = mid;
                att_at = a;
              } else {
                hi = mid;
              }
            }
          }
          const ScenarioConfig sc = scale_scenario(scenario, lo);  // metrics.cpp:299-312
          double total = 0.0;
          for (int s = 0; s < seeds_per_rate; ++s) {
            const uint64_t seed = base_seed + 1000003ULL * (uint64_t)s;
            total += (double)generate_trace(sc, seed, horizon_s).size();
          }
          outs[q].scale = lo;
          outs[q].attainment = att_at;
          outs[q].evaluations = evals;
          outs[q].per_gpu_rate =
              total / ((double)seeds_per_rate * horizon_s) / (double)std::max(1, cluster.replicas);
        } catch (const std::exception& e) {
          errs[q] = e.what();
        }
      });
    }
    for (auto& t : th) t.join();
    for (int q = 0; q < n; ++q)
      if (!errs[q].empty()) fail("internal-inconsistency", errs[q]);
    return SLOS_OK;
  });
}

}  // extern "C"
