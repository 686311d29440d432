// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// Extra exports of oracle/_ref/libslos_ref.so used to generate and pin golden
// fixtures (tests/golden/, written by oracle/make_golden.py):
//   slos_ref_uniforms          std::mt19937_64 + std::uniform_real_distribution<double>(0,1),
//                              the draw sequence of the reference's stress generator
//                              (acceptance_main.cpp:577-605); pins our C generator.
//   slos_ref_oracle_instances  the reference's brute-force instance generator
//                              (tests/oracle.cpp:67-102) serialised as int64 records.
//   slos_ref_trace             slosim::scale_scenario + slosim::generate_trace (the
//                              reference's own code) into include/slos_trace.h's layout,
//                              the checker of the product's batched trace generator.
//   slos_ref_perf_fit          slosim::PerfModel::fit (the reference's own), the checker of
//                              the product's device fit (include/slos_fit.h).
//   slos_ref_oracle_best_value / slos_ref_oracle_subset_feasible
//                              tests/oracle.cpp:8-65 on such a record.

#include <cstdint>
#include <random>
#include <vector>

#include "oracle.hpp"
#include "slos_trace.h"
#include "slos_fit.h"
#include "slosim/perf_model.hpp"
#include "slosim/common.hpp"
#include "slosim/metrics.hpp"
#include "slosim/workload.hpp"
#include <cstdlib>
#include <cstring>

using namespace slosim;

namespace {

constexpr int kRec = 41;  // see encode()

void encode(const oracle::Instance& in, int64_t* r) {
  for (int k = 0; k < kRec; ++k) r[k] = 0;
  r[0] = in.cap;
  r[1] = (int64_t)in.tpots.size();
  for (size_t l = 0; l < in.tpots.size() && l < 2; ++l) r[2 + l] = in.tpots[l];
  r[4] = (int64_t)in.runners.size();
  for (size_t j = 0; j < in.runners.size() && j < 3; ++j) r[5 + j] = in.runners[j].tier;
  r[8] = (int64_t)in.candidates.size();
  for (size_t i = 0; i < in.candidates.size() && i < 6; ++i) {
    const auto& c = in.candidates[i];
    r[9 + 5 * i + 0] = c.deadline;
    r[9 + 5 * i + 1] = c.prefill;
    r[9 + 5 * i + 2] = c.tier;
    r[9 + 5 * i + 3] = c.memory;
    r[9 + 5 * i + 4] = (int64_t)c.value;
  }
  r[39] = in.memory_total;
  r[40] = in.horizon;
}

oracle::Instance decode(const int64_t* r) {
  oracle::Instance in;
  in.cap = (int)r[0];
  for (int l = 0; l < r[1]; ++l) in.tpots.push_back((int)r[2 + l]);
  for (int j = 0; j < r[4]; ++j) in.runners.push_back({(int)r[5 + j]});
  for (int i = 0; i < r[8]; ++i) {
    oracle::Instance::Candidate c;
    c.deadline = (int)r[9 + 5 * i];
    c.prefill = (int)r[9 + 5 * i + 1];
    c.tier = (int)r[9 + 5 * i + 2];
    c.memory = r[9 + 5 * i + 3];
    c.value = (double)r[9 + 5 * i + 4];
    in.candidates.push_back(c);
  }
  in.memory_total = r[39];
  in.horizon = (int)r[40];
  return in;
}

}  // namespace

extern "C" {

int slos_ref_oracle_record_len(void) { return kRec; }

void slos_ref_uniforms(uint64_t seed, int32_t n, double* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (int i = 0; i < n; ++i) out[i] = u(rng);
}

// The reference's stress generator (acceptance_main.cpp:577-605), generalised to
// G(n_dec, n_new, seed, tiers) as SURVEY.md §8 d0 defines it: std::mt19937_64(seed)
// and uniform_real_distribution(0, 1) draws consumed in the harness's order. It
// lets bench.py's reference arm build its inputs from oracle/_ref alone (same
// outputs as the product's generator, paper_2504_08784_b200/csrc/slos_workload.c).
void slos_ref_stress(uint64_t seed, int32_t n_dec, int32_t n_new, int32_t two_tier,
                     const double* tpot_tiers, double now, int32_t* dec_tier, double* dec_next_due,
                     int64_t* dec_remaining, double* new_deadline, int64_t* new_prefill,
                     int32_t* new_tier, int64_t* new_memory, double* new_value) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (int32_t i = 0; i < n_dec; ++i) {
    dec_tier[i] = two_tier ? i % 2 : 0;
    dec_next_due[i] = now + u(rng) * tpot_tiers[dec_tier[i]];
    dec_remaining[i] = 50 + (int64_t)(u(rng) * 200.0);
  }
  for (int32_t i = 0; i < n_new; ++i) {
    new_deadline[i] = now + 0.3 + 0.9 * u(rng);
    new_prefill[i] = 200 + (int64_t)(u(rng) * 700.0);
    new_tier[i] = two_tier ? i % 2 : 0;
    new_memory[i] = 20 + (int64_t)(u(rng) * 60.0);
    new_value[i] = 1.0 + (int64_t)(u(rng) * 8.0);
  }
}

void slos_ref_oracle_instances(uint64_t seed, int32_t count, int64_t* records) {
  std::mt19937_64 rng(seed);
  for (int i = 0; i < count; ++i) encode(oracle::random_instance(rng), records + (size_t)i * kRec);
}

double slos_ref_oracle_best_value(const int64_t* record) {
  return oracle::best_value(decode(record));
}

int32_t slos_ref_oracle_subset_feasible(const int64_t* record, const int32_t* admitted,
                                        int32_t n) {
  std::vector<int> a(admitted, admitted + n);
  return oracle::subset_feasible(decode(record), a) ? 1 : 0;
}

// The reference's trace for one slos_trace_job (include/slos_trace.h layout).
int32_t slos_ref_trace(const slos_trace_job* job, slos_trace* out) {
  std::memset(out, 0, sizeof *out);
  const slos_scenario& s = *job->scenario;
  ScenarioConfig sc;
  sc.name = "ref";
  sc.shape = s.shape == SLOS_SHAPE_SINGLE ? "single"
             : s.shape == SLOS_SHAPE_REASONING ? "reasoning"
             : s.shape == SLOS_SHAPE_TOOL ? "tool" : "unknown";
  sc.arrival.process = s.process == SLOS_ARRIVAL_POISSON ? "poisson" : s.process == SLOS_ARRIVAL_BURSTY ? "bursty" : "other";
  sc.arrival.rate_per_s = s.rate_per_s;
  sc.arrival.on_multiplier = s.on_multiplier;
  sc.arrival.mean_on_s = s.mean_on_s;
  sc.arrival.mean_off_s = s.mean_off_s;
  sc.prompt_tokens = {s.prompt_mean, s.prompt_std};
  sc.output_tokens = {s.output_mean, s.output_std};
  sc.think_tokens = {s.think_mean, s.think_std};
  sc.response_tokens = {s.response_mean, s.response_std};
  sc.prefill_tier = s.prefill_tier;
  sc.decode_tier = s.decode_tier;
  sc.think_tier = s.think_tier;
  sc.response_tier = s.response_tier;
  sc.value = s.value;
  sc.tool_pairs_mean = s.tool_pairs_mean;
  sc.tool_pairs_std = s.tool_pairs_std;
  sc.tool_delay_min_s = s.tool_delay_min_s;
  sc.tool_delay_max_s = s.tool_delay_max_s;
  sc.memory_overprovision = s.memory_overprovision;
  sc.slo.tpot_tiers_s.assign(s.tpot_tiers_s, s.tpot_tiers_s + s.n_tiers);
  sc.slo.ttft_slowdowns.assign(s.ttft_slowdowns, s.ttft_slowdowns + s.n_tiers);
  sc.slo.tpot_window = s.tpot_window;
  std::vector<RequestSpec> reqs;
  try {
    reqs = generate_trace(scale_scenario(sc, job->rate_scale), job->seed, job->duration_s);
  } catch (const Error& e) {
    const std::string c = e.code();
    out->status = c == "invalid-distribution-parameters" ? SLOS_ERR_INVALID_DISTRIBUTION
                  : c == "invariant-violation"           ? SLOS_ERR_INVARIANT
                  : c == "invalid-parameters"            ? 1
                                                         : 2;
    return out->status;
  }
  size_t ns = 0;
  for (const auto& r : reqs) ns += r.stages.size();
  out->stages = (slos_trace_stage*)std::malloc(std::max<size_t>(1, ns * sizeof(slos_trace_stage)));
  out->requests = (slos_trace_request*)std::malloc(std::max<size_t>(1, reqs.size() * sizeof(slos_trace_request)));
  size_t x = 0;
  for (size_t k = 0; k < reqs.size(); ++k) {
    const RequestSpec& r = reqs[k];
    slos_trace_request& q = out->requests[k];
    q.arrival_s = r.arrival_s;
    q.value = r.value;
    q.memory_units = r.memory_units;
    q.first_stage = (int32_t)x;
    q.n_stages = (int32_t)r.stages.size();
    for (const auto& st : r.stages) {
      slos_trace_stage& o = out->stages[x++];
      o.tokens = st.tokens;
      o.external_delay_s = st.external_delay_s;
      o.kind = st.kind == StageKind::kPrefill ? 0 : 1;
      o.slo_tier = st.slo_tier;
    }
  }
  out->n_requests = (int32_t)reqs.size();
  out->n_stages = (int64_t)ns;
  return 0;
}

void slos_ref_trace_free(slos_trace* t) {
  std::free(t->stages);
  std::free(t->requests);
  std::memset(t, 0, sizeof *t);
}

// The reference's PerfModel::fit on one profile set; terms in the model's order.
int32_t slos_ref_perf_fit(const slos_profile_sample* x, int32_t n, int32_t num_terms, int32_t max_iters,
                          slos_perf_term* out) {
  std::vector<ProfileSample> s((size_t)std::max(0, n));
  for (int i = 0; i < n; ++i) s[i] = ProfileSample{x[i].num_tokens, x[i].spec_step, x[i].latency_s};
  try {
    const PerfModel m = PerfModel::fit(s, num_terms, max_iters);
    const auto& t = m.terms();
    for (size_t q = 0; q < t.size(); ++q) out[q] = slos_perf_term{t[q].k1, t[q].k2, t[q].b};
    return (int32_t)t.size() == num_terms ? 0 : 2;
  } catch (const Error& e) {
    const std::string c = e.code();
    return c == "insufficient-samples" ? SLOS_ERR_INSUFFICIENT_SAMPLES
           : c == "degenerate-samples" ? SLOS_ERR_DEGENERATE_SAMPLES
           : c == "invalid-parameters" ? 1
                                       : 2;
  }
}

}  // extern "C"
