/*
 * slos_lockstep.h -- batched routing rounds and lockstep simulation lanes.
 *
 * The integration layer on the REFERENCE side of the planner boundary (built by
 * integration/Makefile into integration/_build/libslos_lockstep.so, linked with the
 * reference's own simulator sources compiled unmodified from /root/reference).
 *
 * The reference's ClusterSim (tiers_router.cpp:110-174) advances one replica at a
 * time and calls Scheduler::schedule once per replan (sim_executor.cpp:344), so every
 * plan is a separate synchronous call. This library runs the same simulations with
 *   - conservative-lookahead windows: a declined request reaches the next replica
 *     net_delay_s after the replan that declined it (on_decline, tiers_router.cpp:
 *     80-108), so every replica event earlier than (earliest pending event +
 *     net_delay_s) is independent of every plan made in that window; those replicas
 *     advance concurrently, one host thread each, and the transfers they create are
 *     sequenced afterwards in the reference's own event order;
 *   - lanes: many simulations (sweep points, seeds, scenarios) in flight at once;
 *   - the plan broker (slos_broker_*, include/slos_planner.h) of a library exporting
 *     slos_planner.h: every replan of every replica of every lane that is waiting at
 *     the same moment goes to the GPU in ONE batched launch.
 * Results are identical to the reference's sequential ClusterSim / simulate_scenario
 * / capacity_search (digest over every RequestRecord field), which the tests check.
 */
#ifndef SLOS_LOCKSTEP_H
#define SLOS_LOCKSTEP_H

#include <stdint.h>

#include "slos_planner.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ExecConfig (sim_executor.hpp:24-41) + ClusterConfig (tiers_router.hpp:14-21). */
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
  int32_t backup_best_effort; /* 0: "decline", 1: "best_effort_on_origin" */
  int32_t reserved0;
  double net_delay_s;
} slos_sim_config;

/* summarize() (metrics.cpp:53-92) of one simulation + a digest over every record. */
typedef struct slos_sim_summary {
  int64_t requests, standard, attained, best_effort, dropped, total_hops, plans, tokens_out;
  double attainment, overall_attainment;
  uint64_t digest;
} slos_sim_summary;

/* CapacityResult (metrics.hpp). */
typedef struct slos_capacity_result {
  double scale;
  double per_gpu_rate;
  double attainment;
  int32_t evaluations;
  int32_t reserved0;
} slos_capacity_result;

typedef struct slos_lockstep_stats {
  int64_t plans;    /* schedule() calls served */
  int64_t flushes;  /* batched launches (broker flushes); = plans without a broker */
  int64_t windows;  /* lookahead windows processed over all lanes */
  double wall_s;    /* wall time of the call */
} slos_lockstep_stats;

/* The planner behind every replica's "slos" scheduler: a library exporting
 * include/slos_planner.h (the product libslos_b200.so), served through its plan
 * broker; NULL or "" = the reference SloScheduler itself (lanes and replicas still
 * run concurrently on host threads). */
int slos_lockstep_set_backend(const char* lib_path);

/* n independent simulate_scenario runs (metrics.cpp:223-232) of
 * scale_scenario(load_scenario_file(paths[k]), scales[k]) (:214-221) as concurrent
 * lanes. terms: the PerfModel shared by every lane. */
int slos_lockstep_simulate(int32_t n, const char* const* scenario_paths, const slos_perf_term* terms,
                           int32_t n_terms, const slos_sim_config* cfgs, const uint64_t* seeds,
                           const double* horizons_s, const double* scales, slos_sim_summary* outs,
                           slos_lockstep_stats* stats);

/* n capacity_search bisections (metrics.cpp:234-313) run concurrently; each
 * evaluation's seeds_per_rate simulations are lanes (the reference's OpenMP loop
 * over seeds, metrics.cpp:251). */
int slos_lockstep_capacity(int32_t n, const char* const* scenario_paths, const slos_perf_term* terms,
                           int32_t n_terms, const slos_sim_config* cfgs, double target, double lo_scale,
                           double hi_scale, double rel_tol, int32_t seeds_per_rate, uint64_t base_seed,
                           double horizon_s, slos_capacity_result* outs, slos_lockstep_stats* stats);

const char* slos_lockstep_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SLOS_LOCKSTEP_H */
