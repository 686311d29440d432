/* Batched synthetic trace generation.
 *
 * Replaces, for many (scenario, rate scale, seed) points at once, the serial step
 * every capacity-sweep point starts with:
 *   slosim::scale_scenario   proj/src/metrics.cpp:214-221
 *   slosim::generate_trace   proj/src/workload.cpp:159-206
 *     sample_arrivals        proj/src/workload.cpp:125-157 (poisson / bursty)
 *     sample_lognormal       proj/src/workload.cpp:113-123
 *     derive_memory_units    proj/src/workload.cpp:69-73
 *     RequestSpec::validate  proj/src/workload.cpp:51-67
 *     ScenarioConfig::validate proj/src/workload.cpp:86-109, SloConfig::validate :16-29
 * Jobs are independent and run on a host thread pool; each job's requests are
 * identical (every field, every bit) to the reference's generate_trace on the
 * same inputs (tests/test_trace.py checks them against the reference compiled in
 * oracle/_ref). Sampling stays on the host by design: exactness needs libstdc++'s
 * mt19937_64 / normal (polar) / exponential / generate_canonical algorithms and
 * glibc's log/exp, which the device's math library does not reproduce.
 *
 * Request ids are implicit: request k of a job is "<scenario name>-<k, 6 digits,
 * zero padded>" in the reference (workload.cpp:166-169).
 */
#ifndef SLOS_TRACE_H_
#define SLOS_TRACE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SLOS_SHAPE_SINGLE = 0,    /* ScenarioConfig::shape "single" */
  SLOS_SHAPE_REASONING = 1, /* "reasoning" */
  SLOS_SHAPE_TOOL = 2       /* "tool" */
};

enum {
  SLOS_ARRIVAL_POISSON = 0, /* ArrivalConfig::process "poisson" */
  SLOS_ARRIVAL_BURSTY = 1   /* "bursty" */
};

/* status codes beyond slos_planner.h's (common.hpp error slugs) */
enum {
  SLOS_ERR_INVALID_DISTRIBUTION = 20, /* "invalid-distribution-parameters" */
  SLOS_ERR_INVARIANT = 21             /* "invariant-violation" */
};

/* ScenarioConfig (workload.hpp:58-100) with the SloConfig it validates against. */
typedef struct slos_scenario {
  int32_t shape;   /* SLOS_SHAPE_* (any other value: "unknown scenario shape") */
  int32_t process; /* SLOS_ARRIVAL_* (any other value: "unknown arrival process") */
  double rate_per_s, on_multiplier, mean_on_s, mean_off_s;
  double prompt_mean, prompt_std;
  double output_mean, output_std;
  double think_mean, think_std;
  double response_mean, response_std;
  int32_t prefill_tier, decode_tier, think_tier, response_tier;
  double value;
  double tool_pairs_mean, tool_pairs_std;
  double tool_delay_min_s, tool_delay_max_s;
  double memory_overprovision;
  const double* tpot_tiers_s;   /* slo.tpot_tiers_s[n_tiers] */
  const double* ttft_slowdowns; /* slo.ttft_slowdowns[n_tiers] */
  int32_t n_tiers;
  int32_t tpot_window;
} slos_scenario;

/* one trace: scale_scenario(*scenario, rate_scale), then generate_trace(.., seed, duration_s) */
typedef struct slos_trace_job {
  const slos_scenario* scenario;
  double rate_scale;
  uint64_t seed;
  double duration_s;
} slos_trace_job;

typedef struct slos_trace_stage { /* StageSpec (workload.hpp:25-32) */
  int64_t tokens;
  double external_delay_s;
  int32_t kind; /* 0 prefill, 1 decode (StageKind) */
  int32_t slo_tier;
} slos_trace_stage;

typedef struct slos_trace_request { /* RequestSpec (workload.hpp:34-47) */
  double arrival_s;
  double value;
  int64_t memory_units;
  int32_t first_stage; /* index into slos_trace.stages */
  int32_t n_stages;
} slos_trace_request;

typedef struct slos_trace {
  int32_t status;     /* SLOS_OK or the reference's error for this job; on error the rest is empty */
  int32_t n_requests;
  int64_t n_stages;
  slos_trace_request* requests;
  slos_trace_stage* stages;
} slos_trace;

/* Generate n traces; outs[k] belongs to jobs[k] (free each with slos_trace_free).
 * threads <= 0: one per hardware thread. Returns SLOS_OK when the batch ran
 * (per-job errors land in outs[k].status), or an error for bad arguments. */
int slos_trace_batch(const slos_trace_job* jobs, int32_t n, int32_t threads, slos_trace* outs);
void slos_trace_free(slos_trace* t);

#ifdef __cplusplus
}
#endif

#endif /* SLOS_TRACE_H_ */
