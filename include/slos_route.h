/*
 * slos_route.h -- batched multi-replica routing rounds (product, libslos_b200.so).
 *
 * The reference routes a request its replica declines to the next replica of the
 * ring after a network delay, at most min(routing_limit, replicas-1) hops, then
 * applies the backup policy (ClusterSim::on_decline, tiers_router.cpp:80-108);
 * every offer becomes a pending entry of the target's next plan
 * (ReplicaSim::inject / apply_schedule, sim_executor.cpp:111-144, 318-340), and
 * each replica plans alone, synchronously (sim_executor.cpp:344).
 *
 * slos_route_rounds evaluates those routing rounds for MANY clusters at once on
 * frozen replica snapshots (R replicas of G(n_dec, n_new) each):
 * round k (at now + k * net_delay_s) plans, in ONE slos_plan_batch over every
 * cluster, every replica that was offered requests in that round; a request a
 * replica admits joins that replica's running set as a forced running prefill
 * (and its memory joins the resident pool) for the later rounds; a declined one is
 * re-offered to (r+1) % R in round k+1 while hops < min(routing_limit, R-1), then:
 *   backup "best_effort_on_origin": demoted to best effort at its origin,
 *   backup "decline": dropped.
 * Rounds stop when no offer is left (at most min(routing_limit, R-1) + 1 rounds).
 */
#ifndef SLOS_ROUTE_H
#define SLOS_ROUTE_H

#include <stdint.h>

#include "slos_planner.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct slos_route_config { /* ClusterConfig tiers_router.hpp:14-21 */
  int32_t replicas;
  int32_t routing_limit;
  int32_t backup_best_effort; /* 0: "decline", 1: "best_effort_on_origin" */
  int32_t unit_value;         /* 0: schedule(), 1: schedule_throughput() */
  double net_delay_s;
} slos_route_config;

enum { SLOS_ROUTE_ADMITTED = 0, SLOS_ROUTE_BEST_EFFORT = 1, SLOS_ROUTE_DROPPED = 2 };

/* The fate of one arriving request (a pending entry of its origin's snapshot). */
typedef struct slos_route_outcome {
  int32_t fate;     /* SLOS_ROUTE_* */
  int32_t replica;  /* replica that admitted it / its origin (best effort) / -1 (dropped) */
  int32_t hops;     /* re-offers it took (RouteState::hops) */
  int32_t round;    /* planning round of the final decision */
} slos_route_outcome;

typedef struct slos_route_stats {
  int64_t rounds;  /* planning rounds (batched launches) */
  int64_t plans;   /* replica plans over all rounds */
  int64_t admitted, best_effort, dropped;
} slos_route_stats;

/* n_clusters clusters of cfg->replicas replicas each. snapshots[c * R + r] is
 * replica r of cluster c (its running set, memory and now; its pending list are the
 * requests arriving at that replica, which is their origin) and planners[c * R + r]
 * its planner. outcomes: one per pending entry, in snapshot order then pending order.
 * Returns SLOS_OK, or the first error status of a plan (the outcomes are then
 * undefined). */
int slos_route_rounds(slos_planner* const* planners, int32_t n_clusters, const slos_route_config* cfg,
                      const slos_input* snapshots, slos_route_outcome* outcomes, slos_route_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* SLOS_ROUTE_H */
