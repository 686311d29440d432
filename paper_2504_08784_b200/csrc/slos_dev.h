// Host/device shared layout of the batched planner (product code).
//
// One planning instance = one ScheduleInput (dp_scheduler.hpp:38-47) after the host
// shim has done the host-trivial work the reference does before its DP:
// validation (dp_scheduler.cpp:367-392), the chain stable_sort (:393-397),
// floor_at / suffix_prefill (:399-408), and edf_fallback's prefill order (:121-124).
// Everything else -- the admission DP, gap tiling, speculative search, terminal
// selection, plan reconstruction and the fallback plan -- runs in the sm_100a
// kernels of slos_kernels.cu.
//
// HBM layout is structure-of-arrays per field, instances concatenated; every
// instance carries offsets into those arrays plus offsets/capacities of its
// slice of the device scratch arenas (DP survivors, memo table, candidates,
// plan output). Capacities are host estimates; a kernel that would overflow one
// records SLOS_ERR_CAPACITY with the size it needed and the host re-launches
// that instance with a larger slice.
#pragma once

#include <stdint.h>
#include <cuda_runtime.h>

#include "../../include/slos_planner.h"

namespace slos {

constexpr int kMaxTiers = 8;      // dp_scheduler.cpp:367
constexpr int kMaxParts = 4;      // solve parts pipelined across streams
constexpr int kBuildKinds = 4;    // warp / 128- / 256- / 512-thread CTA reconstruction
constexpr int kQueues = kBuildKinds * kMaxParts;
constexpr int kMaxTerms = 8;      // PerfModel terms carried on device
constexpr int kMaxSpecLen = 64;   // PlannerConfig::spec_max_len carried on device
constexpr double kTimeEps = 1e-9;  // common.hpp:29
constexpr double kValueEps = 1e-9; // dp_scheduler.cpp:47

// Everything a BatchPlanner owns (batch_planner.hpp:129-133), flattened.
struct PlannerDev {
  double k1[kMaxTerms], k2[kMaxTerms], b[kMaxTerms];
  double tpot[kMaxTiers];
  double acc[kMaxSpecLen + 1];  // expected_accepted(alpha, sl), host glibc pow
  double margin1;               // 1.0 + plan_margin
  double spec_alpha;
  int64_t max_chunk;
  int64_t max_batch;
  int32_t n_terms;
  int32_t L;
  int32_t speculative;
  int32_t spec_max_len;
};

// Per-instance header (device copy). Offsets index the SoA arrays / arenas.
struct InstDev {
  double now;
  double tail_horizon;
  int64_t mem_budget;  // memory_total - memory_standard_resident (:408)
  int32_t planner;
  int32_t unit_value;
  int32_t R_total;     // in.running.size()  (chain-member owner base, :250)
  int32_t n_dec;       // running decoders (prefill_remaining<=0 && decode_remaining>0)
  int32_t N;           // chain length
  int32_t n_pre;       // running prefills (edf_fallback order)
  int32_t n_pending;
  int32_t last_forced;
  int32_t have_running_decode;
  int32_t values_integral;  // all chain values integral -> eps ties impossible
  int32_t build_kind;       // plan reconstruction: 0 one warp, 1 a 128-, 2 a 256-, 3 a 512-thread CTA
  int32_t part;             // solve part (dp + build launched per part, pipelined)
  int32_t direct;           // Pareto buckets through a direct count-vector table (dp_kernel)
  int32_t has_shared;       // some DP pair's memo key recurs: dp_kernel clears its memo slice
  int32_t dstride[kMaxTiers];  // its strides: index = sum_l count_l * dstride[l]
  int64_t off_dec;     // into dec_* arrays
  int64_t off_chain;   // into ch_* arrays (N items, suffix has N+1)
  int64_t off_pre;     // into pre_* arrays
  // scratch slices
  int64_t off_surv;  int64_t cap_surv;   // DP survivors storage
  int64_t off_cand;  int64_t cap_cand;   // per-level candidates
  int64_t off_memo;  int64_t cap_memo;   // gap memo (power of two)
  int64_t off_sel;                       // N ints: selected chain indices
  int64_t off_ids;                       // admitted/declined lists (n_pending each)
  int64_t off_batch; int64_t cap_batch;  // plan batches
  int64_t off_entry; int64_t cap_entry;  // plan entries
  int64_t off_work;  int64_t cap_work;   // build/fallback work area (bytes)
  int64_t off_run;                       // running tiers (R_total ints)
  int64_t cap_gb;                        // gap batches per tile_gap call
  int64_t cap_go;                        // owner pairs per tile_gap call
  int64_t off_anchor; int64_t anchor_stride;  // per-anchor caches (bytes), N+1 anchors
  int64_t off_pair;    // into pair_shared: N(N+1)/2 flags, triangular (anchor j+1, item i)
  int64_t off_group;   // into groups (bytes): one GroupHdr + variant arrays per pair
};

// Per-instance result header written by the kernels.
struct OutHdr {
  int32_t status;
  int32_t infeasible;
  int32_t best;          // -1 = no terminal state (fallback)
  int32_t n_sel;
  double value;
  double exact_until;
  int32_t n_admitted;
  int32_t n_declined;
  int64_t n_batches;
  int64_t n_entries;
  int64_t ctr[5];        // transitions, gap_evals, dues, slots, states
  int64_t need_surv, need_cand, need_memo, need_batch, need_entry, need_work;
  int64_t dbg_cycles;  // build_kernel cycles of this instance (phase timing only)
  int64_t dbg_dp_cycles;  // dp_kernel cycles of this instance (phase timing only)
};

// Memo table entry (gap_budget memo, dp_scheduler.cpp:414-435).
struct MemoEnt {
  uint64_t k0, k1, k2;
  int64_t val;
  int32_t state;   // 0 empty, 1 locked, 2 pending(this level), 3 done
  int32_t first;   // first candidate (traversal order) that asked for it
  int32_t has;     // optional<int64_t>::has_value
  int32_t pad;
};

// Device pointers of one batch launch.
struct BatchArgs {
  const PlannerDev* planners;
  const InstDev* inst;
  const int32_t* order;  // launch order of instances (cost-descending)
  int32_t n_inst;
  const int32_t* atask;  // anchor tasks (instance, anchor j) pairs, j = -1 .. N-2
  int32_t n_atask;
  int32_t mixed_spec;    // both speculative and autoregressive planners in the batch
  // decoders
  const int32_t* dec_idx;
  const int32_t* dec_tier;
  const int32_t* dec_bytier;   // per instance: decoder indices grouped by tier (anchor due walk)
  const double* dec_next;
  const int64_t* dec_backlog;
  const int64_t* dec_rem;
  // chain (sorted)
  const double* ch_deadline;
  const int64_t* ch_prefill;
  const int32_t* ch_tier;
  const int64_t* ch_memory;
  const double* ch_value;
  const int32_t* ch_forced;
  const int32_t* ch_ref;
  const int32_t* ch_floor;
  const int64_t* ch_suffix;   // chain arrays use a stride of N+1 per instance
  // edf_fallback prefills (sorted)
  const int32_t* pre_idx;
  const int64_t* pre_left;
  // scratch
  uint64_t* s_counts;
  int64_t* s_mem;
  int64_t* s_pb;
  double* s_value;
  int32_t* s_nadm;
  int32_t* s_parent;
  int32_t* s_arena;
  int32_t* s_level;  // survivor level bookkeeping (N+2 ints per instance in off_surv space)
  // candidates
  int32_t* c_src;
  int32_t* c_j;
  int32_t* c_memo;
  int32_t* c_flag;   // valid / accepted / dead bits
  int32_t* c_bucket;
  int32_t* c_pos;
  int32_t* c_aux;
  uint64_t* c_counts;
  int64_t* c_mem;
  int64_t* c_pb;
  double* c_value;
  int32_t* c_nadm;
  uint64_t* c_bkey;  // bucket hash keys (2*cap_cand)
  int32_t* c_bval;   // bucket hash values
  MemoEnt* memo;
  const int32_t* run_tier;
  int32_t* sel;
  int32_t* ids;
  slos_batch* batches;
  slos_entry* entries;
  unsigned char* work;
  unsigned char* anchors;
  const uint8_t* pair_shared;  // 1: the pair's memo key (a_us, raw_us) recurs in another pair
  unsigned char* groups;       // per-pair gap group records (anchor_kernel -> dp_kernel)
  int32_t* s_sb;               // survivor: dense id of its Pareto bucket within its level
  uint64_t* s_bcnt;            // per level, per surviving bucket: its count vector
  int64_t* k_val;              // per level: fresh-pair key results (budget, or -1 = nullopt)
  double* ctime;               // per instance: canonical due times [Lmax][Sc] (anchor_kernel)
  int32_t* ccnt;               // per instance: canonical due counts [kMaxTiers]
  int32_t* bq;       // build queues: 2 counters per queue, then the queue segments; per
                     // queue, fallback instances from the front, the rest from the back
  int32_t qbase[kQueues];  // queue q = kBuildKinds*part + build_kind: segment offset in bq
  int32_t qn[kQueues];     // and length
  OutHdr* out;
};

// Gap query (slos_tile_gap_batch) device form.
struct GapQueryDev {
  double gap_s;
  double horizon;
  int64_t counts[kMaxTiers];
  int64_t off_exact;   // into gq_* member arrays
  int32_t n_exact;
  int32_t mode;
  int64_t off_out_batch; int64_t cap_batch;
  int64_t off_out_owner; int64_t cap_owner;
  int64_t off_work; int64_t cap_work;
};

struct GapBatchDev {
  double start_s, end_s;
  int64_t capacity, spec_step, decode_tokens, prefill_budget;
  int64_t per_tier[kMaxTiers];
  int64_t first_owner, n_owner;
};

struct GapOutDev {
  int32_t status;
  int32_t feasible;
  int64_t budget;
  int32_t n_spec;
  int32_t spec_lengths[kMaxTiers];
  int64_t n_batches;
  int64_t n_owner_pairs;
  int64_t need_batch, need_owner, need_work;
};

// dp_kernel / anchor_kernel launch parameters (host and device share this layout).
// PerfModel::fit on the device (slos_fit.cuh)
struct FitSet {
  int64_t off;  // first sample in the SoA arrays
  int32_t n;    // samples
  int32_t run;  // 0: skipped (the host already reported an error)
};

struct FitParams {
  const FitSet* sets;
  const int64_t* nt;   // num_tokens
  const int64_t* ss;   // spec_step
  double* lat;         // latency_s (HBM; also the unstaged path's working copy)
  double* nd;          // num_tokens as double (unstaged path)
  double* sd;          // spec_step as double (unstaged path)
  int smem_samples;    // sets with at most this many samples run from shared memory
  int32_t* assign;     // regime per sample (host: initial quantile bands)
  double* e2;          // squared residual per sample (scratch)
  double* out;         // per set: T x (k1, k2, b) of the best iteration
  int32_t* ok;         // per set: 1 when an iteration recorded a best model
  int T;
  int max_iters;
};

struct DpParams {
  BatchArgs a;
  int Sc;              // per-warp slot capacity
  int Lmax;            // max tiers over planners
  int dec_smem_max;    // stage decoders in smem when n_dec <= this
  unsigned char* wscr_global;  // per-CTA-slot warp scratch when not in smem (nullptr = smem)
  size_t wscr_stride;  // bytes per warp in wscr_global
  int wscr_warps;      // warp slots per launch-order position in wscr_global
  unsigned long long* phase_cycles;  // kNumPhases counters, or nullptr
  int Tsm;             // candidates per level kept in shared memory
  size_t overlay_bytes;  // group-variant / candidate-state overlay (bytes)
  size_t anchor_scr_bytes;  // anchor_kernel: due-pass scratch (bytes)
  size_t grec_stride;       // bytes per pair group record
  size_t grec_hdr;          // header bytes before the variant arrays
  size_t grec_stage;        // bytes of a record the DP stages (header + evaluated arrays)
  int blk0;                 // first position in `order` of this launch's part
  int task0;                // first anchor task of this launch (anchor / group kernels)
  int dtab;                 // direct bucket-table entries in shared memory (0: none)
};

// Push an instance onto its plan-reconstruction queue q = kBuildKinds*part + build_kind (the
// counters are bq[2q], bq[2q+1]); fallback instances (a long sequential batch loop)
// are taken first, from the front.
__device__ __forceinline__ void build_queue_push(const BatchArgs& A, int inst, int part, int kind, bool front) {
  const int q = kBuildKinds * part + kind;
  const int base = A.qbase[q];
  const int n = A.qn[q];
  int32_t* c = A.bq + 2 * q;
  if (front) A.bq[base + atomicAdd(&c[0], 1)] = inst;
  else A.bq[base + n - 1 - atomicAdd(&c[1], 1)] = inst;
}

// build_kernel / build_kernel_warp launch parameters.
struct BuildParams {
  BatchArgs a;
  size_t smem_bytes;  // build_kernel: dynamic shared memory per CTA (per-gap working set)
  size_t smem_warp;   // build_kernel_warp: dynamic shared memory per CTA (4 instances)
  size_t smem_big;    // build_kernel_big: dynamic shared memory per CTA (one CTA per SM)
  int part;           // solve part whose queues this launch drains
  unsigned long long* phase_cycles;  // 8 counters or nullptr (SLOS_PHASE_TIMING)
};

// Triangular index of the pair (anchor a = j+1, chain item i), 0 <= a <= i < N:
// row-major by item, so one DP level's pairs (a = floor+1 .. i) are contiguous.
__host__ __device__ __forceinline__ int64_t pair_index(int N, int a, int i) {
  (void)N;
  return (int64_t)i * (i + 1) / 2 + a;
}

}  // namespace slos
