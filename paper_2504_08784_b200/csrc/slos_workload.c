/*
 * Synthetic planning-instance generator (host side, benchmark/test input only).
 *
 * Restates the reference's stress-instance generator (acceptance_main.cpp:577-605,
 * generalised as G(n_dec, n_new, seed, tiers) in SURVEY.md §8 d0) so that the GPU
 * box can build the same synthetic instances without the reference tree:
 *   std::mt19937_64(seed) and std::uniform_real_distribution<double>(0, 1), drawn
 *   in the reference's order. The uniform draw is libstdc++'s
 *   generate_canonical<double, 53> on a 64-bit engine: (double)x * 2^-64, clamped
 *   below 1 (bits/random.tcc). Pinned against the reference's own engine by
 *   tests/test_workload.py (oracle/_ref slos_ref_uniforms).
 */
#include <math.h>
#include <stdint.h>

typedef struct {
  uint64_t mt[312];
  int mti;
} mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt64_next(mt64_t* s) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static double u01(mt64_t* s) {
  double r = (double)mt64_next(s) / 18446744073709551616.0;
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}

void slos_wl_uniforms(uint64_t seed, int32_t n, double* out) {
  mt64_t s;
  mt64_seed(&s, seed);
  for (int32_t i = 0; i < n; ++i) out[i] = u01(&s);
}

/* G(n_dec, n_new, seed, two_tier): one stress instance, reference draw order
 * (acceptance_main.cpp:587-605). two_tier != 0 -> tier i%2, else tier 0.
 * now = 100 (acceptance_main.cpp:583). */
void slos_wl_stress(uint64_t seed, int32_t n_dec, int32_t n_new, int32_t two_tier,
                    const double* tpot_tiers, double now,
                    int32_t* dec_tier, double* dec_next_due, int64_t* dec_remaining,
                    double* new_deadline, int64_t* new_prefill, int32_t* new_tier,
                    int64_t* new_memory, double* new_value) {
  mt64_t s;
  mt64_seed(&s, seed);
  for (int32_t i = 0; i < n_dec; ++i) {
    const int tier = two_tier ? i % 2 : 0;
    const double tpot = tpot_tiers[tier];
    dec_tier[i] = tier;
    dec_next_due[i] = now + u01(&s) * tpot;
    dec_remaining[i] = 50 + (int64_t)(u01(&s) * 200.0);
  }
  for (int32_t i = 0; i < n_new; ++i) {
    new_deadline[i] = now + 0.3 + 0.9 * u01(&s);
    new_prefill[i] = 200 + (int64_t)(u01(&s) * 700.0);
    new_tier[i] = two_tier ? i % 2 : 0;
    new_memory[i] = 20 + (int64_t)(u01(&s) * 60.0);
    new_value[i] = 1.0 + (int64_t)(u01(&s) * 8.0);
  }
}
