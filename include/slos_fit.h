/* PerfModel::fit on the device, batched over profile sets.
 *
 * Replaces slosim::PerfModel::fit (proj/src/perf_model.cpp:132-201, with
 * nonneg_least_squares :19-90 and term_value :92-94): a max-of-affine batch-latency
 * model fitted by iterative regime assignment. Each profile set is one CTA: the
 * regime refits (normal equations, one lane per matrix entry, accumulated in
 * sample order; Gaussian elimination with the reference's pivoting) and the
 * argmax reassignment of every sample (threads over samples) run on the GPU; the
 * host does the argument checks, the reference's initial quantile bands (its own
 * std::sort) and the final term order. Coefficients are bit-identical to the
 * reference's (tests/test_fit_gpu.py).
 */
#ifndef SLOS_FIT_H_
#define SLOS_FIT_H_

#include <stdint.h>

#include "slos_planner.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SLOS_ERR_INSUFFICIENT_SAMPLES = 22, /* "insufficient-samples": fewer than 3 samples per term */
  SLOS_ERR_DEGENERATE_SAMPLES = 23    /* "degenerate-samples": fewer distinct num_tokens than terms */
};

#define SLOS_FIT_MAX_TERMS 32

typedef struct slos_profile_sample { /* ProfileSample (perf_model.hpp:10-14) */
  int64_t num_tokens;
  int64_t spec_step;
  double latency_s;
} slos_profile_sample;

/* Fit n_sets profiles: set k has n_samples[k] samples at sets[k]. terms_out holds
 * num_terms terms per set (set k at terms_out + k * num_terms, ordered by (k1, k2, b)
 * like the reference); status[k] is SLOS_OK or the reference's error for that set.
 * num_terms must be in [1, SLOS_FIT_MAX_TERMS]; max_iters defaults to 100 in the
 * reference (perf_model.hpp:46). Returns SLOS_OK when the batch ran. */
int slos_perf_fit_batch(const slos_profile_sample* const* sets, const int32_t* n_samples, int32_t n_sets,
                        int32_t num_terms, int32_t max_iters, slos_perf_term* terms_out, int32_t* status);

#ifdef __cplusplus
}
#endif

#endif /* SLOS_FIT_H_ */
