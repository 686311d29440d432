// Batched multi-replica routing rounds (include/slos_route.h).
//
// The reference's routing: ClusterSim::on_decline (tiers_router.cpp:80-108) sends a
// declined request to replica (r+1) % R after net_delay_s while its hop count is
// below min(routing_limit, R-1), then applies the backup policy; the target
// replica's next plan sees it as a pending entry (ReplicaSim::inject,
// sim_executor.cpp:111-144) and an admitted request becomes a running prefill whose
// memory joins the resident pool (apply_schedule / snapshot, :265-340). Each replica
// plans alone there. Here every replica offered requests in a round, across every
// cluster, is planned in ONE slos_plan_batch (the sm_100a pipeline), then the
// declines are routed for the next round on the host.
#include <cstring>
#include <string>
#include <vector>

#include "../../include/slos_planner.h"
#include "../../include/slos_route.h"

namespace {

struct Req {
  slos_pending p;  // the caller's entry (id pointer stays caller-owned)
  int origin;      // replica index within its cluster
  int hops;
  int64_t out;     // outcome index
};

struct Replica {
  slos_input snap;
  std::vector<slos_running> running;  // snapshot running set + admitted prefills
  int64_t resident;                   // memory_standard_resident
  std::vector<int32_t> offered;       // request ids offered this round
  std::vector<int32_t> next;          // offered next round
};

}  // namespace

extern "C" int slos_route_rounds(slos_planner* const* planners, int32_t n_clusters, const slos_route_config* cfg,
                                 const slos_input* snapshots, slos_route_outcome* outcomes,
                                 slos_route_stats* stats) {
  if (stats) std::memset(stats, 0, sizeof *stats);
  const int R = cfg->replicas;
  if (R < 1 || n_clusters < 0 || cfg->routing_limit < 0 || !(cfg->net_delay_s >= 0.0))
    return SLOS_ERR_INVALID_PARAMETERS;  // ClusterConfig::validate (tiers_router.cpp:26-33)
  const int eff = cfg->routing_limit < R - 1 ? cfg->routing_limit : R - 1;
  const int NR = n_clusters * R;
  std::vector<Replica> rep((size_t)NR);
  std::vector<Req> reqs;
  int64_t n_out = 0;
  for (int x = 0; x < NR; ++x) {
    Replica& s = rep[x];
    s.snap = snapshots[x];
    s.running.assign(snapshots[x].running, snapshots[x].running + snapshots[x].n_running);
    s.resident = snapshots[x].memory_standard_resident;
    for (int k = 0; k < snapshots[x].n_pending; ++k) {
      reqs.push_back({snapshots[x].pending[k], x % R, 0, n_out});
      outcomes[n_out] = {SLOS_ROUTE_DROPPED, -1, 0, -1};
      s.offered.push_back((int32_t)reqs.size() - 1);
      ++n_out;
    }
  }
  std::vector<int32_t> who;  // replicas planned this round
  std::vector<slos_planner*> ps;
  std::vector<slos_input> ins;
  std::vector<std::vector<slos_pending>> pend((size_t)NR);
  for (int round = 0;; ++round) {
    who.clear();
    ps.clear();
    ins.clear();
    for (int x = 0; x < NR; ++x) {
      Replica& s = rep[x];
      if (s.offered.empty()) continue;
      pend[x].clear();
      for (int32_t q : s.offered) pend[x].push_back(reqs[q].p);
      slos_input in = s.snap;
      in.now = s.snap.now + (double)round * cfg->net_delay_s;
      in.running = s.running.data();
      in.n_running = (int32_t)s.running.size();
      in.pending = pend[x].data();
      in.n_pending = (int32_t)pend[x].size();
      in.memory_standard_resident = s.resident;
      who.push_back(x);
      ps.push_back(planners[x]);
      ins.push_back(in);
    }
    if (who.empty()) break;
    std::vector<slos_result> res(who.size());
    const int st = slos_plan_batch(ps.data(), (int32_t)who.size(), ins.data(), cfg->unit_value, res.data(), nullptr);
    if (st != SLOS_OK) return st;
    int bad = SLOS_OK;
    for (size_t w = 0; w < who.size(); ++w)
      if (res[w].status != SLOS_OK && bad == SLOS_OK) bad = res[w].status;
    if (bad != SLOS_OK) {
      for (auto& r : res) slos_result_free(&r);
      return bad;
    }
    if (stats) {
      stats->rounds += 1;
      stats->plans += (int64_t)who.size();
    }
    for (size_t w = 0; w < who.size(); ++w) {
      const int x = who[w];
      Replica& s = rep[x];
      const slos_result& r = res[w];
      const int c0 = x - x % R;  // first replica of this cluster
      for (int k = 0; k < r.n_admitted; ++k) {  // apply_schedule: admitted -> resident prefill
        Req& q = reqs[s.offered[r.admitted[k]]];
        outcomes[q.out] = {SLOS_ROUTE_ADMITTED, x % R, q.hops, round};
        slos_running run;
        std::memset(&run, 0, sizeof run);
        run.id = q.p.id;
        run.prefill_remaining = q.p.prefill_tokens;
        run.prefill_deadline = q.p.prefill_deadline;
        run.decode_tier = q.p.decode_tier;
        s.running.push_back(run);
        s.resident += q.p.memory_units;
        if (stats) stats->admitted += 1;
      }
      for (int k = 0; k < r.n_declined; ++k) {  // on_decline (tiers_router.cpp:80-108)
        const int32_t qi = s.offered[r.declined[k]];
        Req& q = reqs[qi];
        if (q.hops < eff) {
          ++q.hops;
          rep[c0 + (x % R + 1) % R].next.push_back(qi);
        } else if (cfg->backup_best_effort) {
          outcomes[q.out] = {SLOS_ROUTE_BEST_EFFORT, q.origin, q.hops, round};
          if (stats) stats->best_effort += 1;
        } else {
          outcomes[q.out] = {SLOS_ROUTE_DROPPED, -1, q.hops, round};
          if (stats) stats->dropped += 1;
        }
      }
    }
    for (auto& r : res) slos_result_free(&r);
    for (Replica& s : rep) {
      s.offered.swap(s.next);
      s.next.clear();
    }
  }
  return SLOS_OK;
}
