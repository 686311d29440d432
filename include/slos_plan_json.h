/* slos_plan_json.h -- the reference's canonical result serialisation.
 *
 * Replaces: slosim::plan_to_json (reference proj/include/slosim/dp_scheduler.hpp:108,
 * proj/src/dp_scheduler.cpp:560-589), the string the reference's determinism test
 * compares (proj/tests/test_dp_scheduler.cpp:212-225) and golden diffs are taken on.
 *
 * The output is byte-identical to nlohmann::json::dump() of the reference's object:
 * keys in std::map order, compact separators, int64 counts as integers, doubles in
 * the shortest-digit form nlohmann prints, strings escaped as nlohmann escapes them.
 * Implemented by libslos_b200.so (host code, no device needed) and, for parity, by
 * oracle/_ref/libslos_ref.so (which calls the reference's own plan_to_json).
 */
#ifndef SLOS_PLAN_JSON_H
#define SLOS_PLAN_JSON_H

#include "slos_planner.h"

#ifdef __cplusplus
extern "C" {
#endif

/* plan_to_json(result, now) for the result `r` of planning input `in` (entry and
 * admitted/declined/deferred references resolve to the ids in `in`). Writes at most
 * `cap` bytes to `buf` (NUL-terminated when the text fits), the text length without
 * the NUL to *len (so a call with cap 0 sizes the buffer). Returns SLOS_OK, or
 * SLOS_ERR_INVALID_PARAMETERS when a reference is out of range or an id is not valid
 * UTF-8 (nlohmann's dump throws there). */
int slos_plan_to_json(const slos_input* in, const slos_result* r, double now_s, char* buf, int64_t cap,
                      int64_t* len);

#ifdef __cplusplus
}
#endif

#endif
