// Warp-level Δpb engine: the leftover prefill budget of one gap for MANY canonical
// count vectors sharing the same exact census (the admission DP's inner primitive,
// dp_scheduler.cpp:418-436 -> BatchPlanner::tile_gap batch_planner.cpp:315-406 ->
// tile_gap_ar :152-313, budget only).
//
// Re-design (not a port): the reference materialises every due, sorts them and
// places them one by one into per-owner std::map bins. For the DP only the budget
// matters, so a gap is reduced to per-slot counts:
//   * exact members (the running decoders at the gap start, members_at) are
//     enumerated ONCE per (chain item i, anchor j, tightest tier) "variant", lanes
//     over members, into a per-slot histogram nx[s] (same repeated-addition due
//     times and the same jit binary search as the reference, so bit-identical);
//   * canonical members contribute c_l * hc_l[s] where hc_l is the per-slot
//     histogram of tier-l canonical dues (independent of the counts);
//   * late dues fill slots first-fit, and latest-fit placement of the jit groups
//     leaves free capacity G(s) - G(s-1) with G(s) = min_{u>=s}(F(u) - D(u))
//     (F = prefix free capacity after late dues, D = prefix due counts); the gap
//     is infeasible iff min_u (F(u) - D(u)) < 0. Warp scans over slots give the
//     budget sum_s min(free_s, max_chunk) in O(S/32) per count vector.
// All fp64 is evaluated in the reference's order (see slos_common.cuh).
#pragma once

#include "slos_common.cuh"

namespace slos {

// Per-warp scratch (shared or global memory), sized by the host-chosen slot cap Sc.
struct WarpScr {
  double* ends;   // Sc
  int64_t* cap;   // Sc
  int32_t* nx;    // Sc   exact non-late dues per slot
  int32_t* hc;    // L*Sc canonical dues per slot per tier
  int64_t* tmp;   // Sc   placement temporaries
  double* ends2;  // Sc   spec-tail canonical variant
  int64_t* cap2;  // Sc
  int32_t* hc2;   // L*Sc
  int64_t* kh;    // Sc+2 spec per-batch exact decode histogram
  int Sc;
  int L;
};

__device__ __forceinline__ size_t warp_scr_bytes(int Sc, int L) {
  return (size_t)Sc * (8 + 8 + 4 + 4 * L + 8 + 8 + 8 + 4 * L) + (size_t)(Sc + 2) * 8 + 64;
}

__device__ __forceinline__ WarpScr warp_scr_carve(unsigned char* base, int Sc, int L) {
  WarpScr w;
  unsigned char* p = base;
  w.ends = (double*)p; p += (size_t)Sc * 8;
  w.cap = (int64_t*)p; p += (size_t)Sc * 8;
  w.tmp = (int64_t*)p; p += (size_t)Sc * 8;
  w.ends2 = (double*)p; p += (size_t)Sc * 8;
  w.cap2 = (int64_t*)p; p += (size_t)Sc * 8;
  w.kh = (int64_t*)p; p += (size_t)(Sc + 2) * 8;
  w.nx = (int32_t*)p; p += (size_t)Sc * 4;
  w.hc = (int32_t*)p; p += (size_t)Sc * 4 * L;
  w.hc2 = (int32_t*)p; p += (size_t)Sc * 4 * L;
  w.Sc = Sc;
  w.L = L;
  return w;
}

// Running decoders of one instance (SoA; shared memory when staged).
struct DecView {
  const double* next;
  const int64_t* backlog;
  const int64_t* rem;
  const int32_t* tier;
  int n;
  const int32_t* bytier = nullptr;  // anchor due walk: member order grouped by tier
};

// One gap (chain item i, anchor j): the exact census is members_at(a).
struct GapGroup {
  double a;        // gap start (t_j)
  double gap;      // tile_gap gap_s (len, or quantize(len) without running decoders)
  double dh;       // due_horizon_s (raw + pull, or 0)
  double horizon;  // max(gap, dh)  (batch_planner.cpp:155)
  double now, pull;
  bool exact;      // census has exact members (have_running_decode)
  // filled by warp_group_setup (group-level facts, independent of counts)
  unsigned exact_mask;        // tiers with an exact member of remaining > 0
  int64_t exact_per_tier[kMaxTiers];  // merged_counts contribution (batch_planner.cpp:28)
  int n_exact;                // valid members
  bool any_due;               // gap<=eps branch (batch_planner.cpp:156-164)
  bool has_backlog;           // spec: any exact backlog > 0 (:321-322)
  double min_phase;           // spec: min phase over members with remaining > 0 (:341-346)
  // prefill-only cache
  int po_state;               // 0 unknown, 1 ok, 2 error
  int64_t po_budget;
};

struct Variant {
  double t0;
  double t0_first;
  int S;            // number of slots (may exceed Sc -> overflow)
  int64_t Lx;       // exact late dues
  int64_t Dx;       // exact dues materialised
  int q[kMaxTiers]; // canonical due times per tier
  int exact_fail;   // an exact non-late due with jit < 0
  unsigned cfail;   // tiers whose canonical dues have jit < 0
  int cap_err;      // plan_time2bs threw on some slot
  int spill;        // spec: an exact due past gap (within due_horizon)
  int valid;
  int inc;          // slot ends strictly increasing -> jit may be walked
  int dues_done;    // exact dues filled from the anchor due pass (no E2 task)
  int packed;       // cnx/hcp valid: L <= 4 and every canonical per-slot count <= 255
};

// A group's shared variant arrays (shared memory).
struct GroupVar {
  double* ends;
  int64_t* cap;
  int32_t* nx;
  int32_t* hc;
  int64_t* cnx;    // cap - nx per slot (group_kernel, when packed)
  uint32_t* hcp;   // canonical dues per slot, 8 bits per tier (tiers 0..3, when packed)
};

struct GroupHdr {
  GapGroup g;
  Variant v;
  int j;
};

__host__ __device__ __forceinline__ size_t group_var_stride(int Sc, int L) {
  return (((size_t)Sc * (8 + 4 + 8 + 4 + 4 * (size_t)L + 8)) + 127) & ~(size_t)127;
}

// Bytes of a group variant a DP level stages into shared memory: the packed
// placement inputs cnx / hcp and the slot capacities (the leading arrays). The
// unpacked nx / hc are read from the HBM record when a group needs them.
__host__ __device__ __forceinline__ size_t group_var_eval_bytes(int Sc, int L) {
  (void)L;
  return (((size_t)Sc * (8 + 4 + 8)) + 15) & ~(size_t)15;
}

// layout: cnx[Sc] (i64), hcp[Sc] (u32), cap[Sc] (i64), nx[Sc] (i32), hc[L][Sc] (i32),
// ends[Sc] (f64)
__device__ __forceinline__ GroupVar group_var_carve(unsigned char* base, int Sc, int L) {
  GroupVar g;
  const size_t S = (size_t)Sc;
  g.cnx = (int64_t*)base;
  g.hcp = (uint32_t*)(base + S * 8);
  g.cap = (int64_t*)(base + ((S * 12 + 7) & ~(size_t)7));
  g.nx = (int32_t*)((unsigned char*)g.cap + S * 8);
  g.hc = (int32_t*)((unsigned char*)g.nx + S * 4);
  g.ends = (double*)(((uintptr_t)((unsigned char*)g.hc + S * 4 * (size_t)L) + 7) & ~(uintptr_t)7);
  return g;
}

// Exact-member dues of one member into a slot histogram (shared by the warp
// variant builder and the block-wide member-chunk tasks). jit is walked forward
// from the previous due (due times increase along a line) when the slot ends
// are strictly increasing, which gives exactly the reference's binary-search
// result; otherwise every due binary-searches like the reference.
__device__ __forceinline__ void member_dues(const PlannerDev& P, const Member& m, const GapGroup& g,
                                            const double* ends, int S, bool fits, bool inc,
                                            int32_t* nx, int64_t& late, int64_t& dues, int& fail,
                                            int& spill) {
  int64_t issued = m.backlog > 0 ? imin(m.backlog, m.rem) : 0;
  late += issued;
  const double tpot = P.tpot[m.tier];
  int jit = -1;
  bool first = true;
  for (double d = dmax(m.phase, 0.0); time_le(d, g.horizon) && issued < m.rem; d += tpot, ++issued) {
    if (!time_le(d, g.gap)) spill = 1;
    if (d <= kTimeEps) {
      ++late;
    } else {
      ++dues;
      if (fits) {
        if (!inc || first) {
          jit = jit_search(ends, S, d);
          first = false;
        } else {
          while (jit + 1 < S && time_le(ends[jit + 1], d)) ++jit;
        }
        if (jit < 0) fail = 1; else atomicAdd(&nx[jit], 1);
      }
    }
  }
  if (m.backlog < 0 && g.dh > g.gap + kTimeEps) {
    // tile_gap's spill scan starts from min(backlog, remaining) (batch_planner.cpp:329):
    // with a negative backlog it runs past the autoregressive loop's last due.
    int64_t is2 = imin(m.backlog, m.rem);
    for (double d = dmax(m.phase, 0.0); time_le(d, g.dh) && is2 < m.rem; d += tpot, ++is2)
      if (!time_le(d, g.gap)) spill = 1;
  }
}


// E2 form of member_dues: the 32 lanes (one member each) walk their lines in
// lockstep, one due per lane per round, so the histogram updates of lanes that
// land in the same slot (the k-th due of every same-tier line usually does)
// aggregate into one shared-memory atomic via __match_any_sync.
__device__ inline void member_dues_warp(const PlannerDev& P, const Member& m, const GapGroup& g,
                                        const double* ends, int S, bool inc, int32_t* nx,
                                        int64_t& late, int64_t& dues, int& fail, int& spill) {
  bool act = m.valid && m.rem > 0;
  int64_t issued = 0;
  double d = 0.0, tpot = 0.0;
  int jit = -1;
  bool first = true;
  if (act) {
    issued = m.backlog > 0 ? imin(m.backlog, m.rem) : 0;
    late += issued;
    tpot = P.tpot[m.tier];
    d = dmax(m.phase, 0.0);
  }
  for (;;) {
    act = act && time_le(d, g.horizon) && issued < m.rem;
    if (!__any_sync(0xffffffffu, act)) break;
    int key = -1;
    if (act) {
      if (!time_le(d, g.gap)) spill = 1;
      if (d <= kTimeEps) {
        ++late;
      } else {
        ++dues;
        if (!inc || first) {
          jit = jit_search(ends, S, d);
          first = false;
        } else {
          while (jit + 1 < S && time_le(ends[jit + 1], d)) ++jit;
        }
        if (jit < 0) fail = 1; else key = jit;
      }
      d += tpot;
      ++issued;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (key >= 0 && lane_id() == __ffs(peers) - 1) atomicAdd(&nx[key], __popc(peers));
  }
  if (m.valid && m.rem > 0 && m.backlog < 0 && g.dh > g.gap + kTimeEps) {
    int64_t is2 = imin(m.backlog, m.rem);  // see member_dues
    for (double e = dmax(m.phase, 0.0); time_le(e, g.dh) && is2 < m.rem; e += tpot, ++is2)
      if (!time_le(e, g.gap)) spill = 1;
  }
}

// Slot capacities cap[s] = min(plan_time2bs(dur_s), max_batch) (batch_planner.cpp:250-255).
// time2bs is monotone in its budget, so when the interior durations (which differ
// only by ulps of the repeated-addition grid) map to the same capacity at their
// min and max, every interior slot shares it: 4 binary searches instead of S.
// Returns 1 if some slot's time2bs throws (infeasible-budget).
__device__ inline int warp_slot_caps(const PlannerDev& P, const double* ends, int S, int64_t* cap) {
  const int lane = lane_id();
  double lo = INFINITY, hi = -INFINITY;
  for (int s = 1 + lane; s < S - 1; s += 32) {
    const double dur = ends[s] - ends[s - 1];
    lo = dmin(lo, dur);
    hi = dmax(hi, dur);
  }
  lo = warp_min(lo);
  for (int o = 16; o; o >>= 1) hi = dmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  int64_t shared_cap = -2;
  if (S > 2) {
    const int64_t a = lane == 0 ? plan_time2bs(P, lo, 0) : 0;
    const int64_t b = lane == 1 ? plan_time2bs(P, hi, 0) : 0;
    const int64_t ca = __shfl_sync(0xffffffffu, a, 0), cb = __shfl_sync(0xffffffffu, b, 1);
    if (ca == cb && ca >= 0) shared_cap = imin(ca, P.max_batch);
  }
  int err = 0;
  for (int s = lane; s < S; s += 32) {
    if (s > 0 && s < S - 1 && shared_cap >= 0) {
      cap[s] = shared_cap;
      continue;
    }
    const double dur = ends[s] - (s == 0 ? 0.0 : ends[s - 1]);
    const int64_t c = plan_time2bs(P, dur, 0);
    if (c < 0) err = 1;
    cap[s] = imin(c, P.max_batch);
  }
  __syncwarp();
  return warp_or(err);
}

// ---- per-anchor cache ----------------------------------------------------------
// Everything about a gap that depends only on its start a = t_j (the anchor) and
// not on the chain item i that ends it: the exact census members_at(a), the census
// facts, t0_first for the exact census' tightest tier, the slot grid
// e_k = t0_first + k*t0 (repeated addition, batch_planner.cpp:241) up to the
// longest gap this anchor can see, its per-slot capacities, and the grid slot of
// every canonical due time. Built once per anchor (one new anchor per DP level);
// every (level, anchor) group then derives its variant with lane-parallel copies.
struct AnchorFacts {
  double a;
  double t0;
  double t0_first;
  double min_phase;      // over members with remaining > 0
  int64_t per_tier[kMaxTiers];
  unsigned exact_mask;
  int n_exact;
  int has_backlog;       // any member backlog > 0 (tile_gap :321-322)
  int any_bl;            // any member with remaining > 0 and backlog > 0 (:160)
  int Kg;                // grid points stored (may exceed Sc -> overflow)
  int grid_ok;           // grid strictly increasing and complete
  int cap_uniform_err;
  int dues_ok;           // the anchor due pass below ran: groups skip E2
  int64_t Lx;            // exact late dues (backlog issued + dues at d <= eps)
};

// Per (anchor j, chain item i) result of the anchor due pass: the exact dues of the
// group's tail cells (grid cells >= Sp-1 up to the group's due horizon), which are
// the only ones whose slot or inclusion depends on i.
struct GroupTail {
  int32_t tA;     // dues placed in slot Sp-1
  int32_t tB;     // dues placed in the appended slot Sp
  int32_t td;     // non-late dues counted in the tail
  int16_t fail;   // a tail due with jit < 0 (only when Sp == 0)
  int16_t spill;  // a tail due past the gap (within the horizon)
};

struct AnchorView {
  AnchorFacts* f;
  double* ph;
  int64_t* bl;
  int64_t* rm;
  double* ge;
  int64_t* gcap;   // -1: plan_time2bs throws for that grid slot
  int32_t* ccell;  // [L][Sc] grid jit of canonical time k of tier l
  int32_t* hcum;   // [Sc+2] cumulative exact due count over grid cells -1, 0, 1, ...
  GroupTail* gt;   // [N+1] per chain item i
};

__host__ __device__ __forceinline__ size_t anchor_stride_bytes(int R, int Sc, int L, int N) {
  size_t b = 256 + (size_t)R * 24 + (size_t)Sc * 16 + (size_t)L * Sc * 4 + (size_t)(Sc + 2) * 4;
  b = (b + 15) & ~(size_t)15;
  b += (size_t)(N + 1) * sizeof(GroupTail);
  return (b + 127) & ~(size_t)127;
}

__device__ __forceinline__ AnchorView anchor_view(unsigned char* base, int R, int Sc, int L) {
  AnchorView v;
  v.f = (AnchorFacts*)base;
  unsigned char* p = base + 256;
  v.ph = (double*)p; p += (size_t)R * 8;
  v.bl = (int64_t*)p; p += (size_t)R * 8;
  v.rm = (int64_t*)p; p += (size_t)R * 8;
  v.ge = (double*)p; p += (size_t)Sc * 8;
  v.gcap = (int64_t*)p; p += (size_t)Sc * 8;
  v.ccell = (int32_t*)p; p += (size_t)L * Sc * 4;
  v.hcum = (int32_t*)p; p += (size_t)(Sc + 2) * 4;
  p = (unsigned char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
  v.gt = (GroupTail*)p;
  return v;
}

// Derive a (level, anchor) group's variant from the anchor cache (warp).
// `ctime/ccnt` is the instance's canonical due-time list per tier.
__device__ inline void warp_group_from_anchor(const PlannerDev& P, const AnchorView& av, GapGroup& g,
                                              Variant& v, const GroupVar& ga, int Sc, double min_slot,
                                              const double* ctime, const int* ccnt, int item) {
  const int lane = lane_id();
  const AnchorFacts& F = *av.f;
  g.exact_mask = F.exact_mask;
  for (int l = 0; l < kMaxTiers; ++l) g.exact_per_tier[l] = F.per_tier[l];
  g.n_exact = F.n_exact;
  g.has_backlog = F.has_backlog != 0;
  g.min_phase = F.min_phase;
  g.any_due = F.any_bl || (g.horizon > kTimeEps && time_le(F.min_phase, g.horizon));
  g.po_state = 0;
  g.po_budget = 0;
  v.valid = 0;
  v.S = 0;
  v.Lx = 0;
  v.Dx = 0;
  v.exact_fail = 0;
  v.spill = 0;
  v.cap_err = 0;
  v.cfail = 0;
  v.inc = 0;
  v.dues_done = 0;
  v.packed = 0;
  for (int l = 0; l < kMaxTiers; ++l) v.q[l] = 0;
  if (g.gap <= kTimeEps || !F.exact_mask) return;
  v.t0 = F.t0;
  v.t0_first = F.t0_first;
  // canonical due counts (batch_planner.cpp:216): prefix of the canonical list
  {
    int q = 0;
    if (lane < P.L) {
      int lo = 0, hi = ccnt[lane];
      while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (time_le(ctime[lane * Sc + mid], g.gap)) lo = mid + 1; else hi = mid;
      }
      q = lo;
    }
    for (int l = 0; l < P.L; ++l) v.q[l] = __shfl_sync(0xffffffffu, q, l);
  }
  if (!F.grid_ok) {  // degenerate grid: slow path per key
    v.valid = 0;
    v.inc = -1;
    return;
  }
  // prefix of the grid inside the gap (:241): first k with !time_le(e_k, gap)
  int Sp;
  {
    int lo = 0, hi = F.Kg;
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      if (time_le(av.ge[mid], g.gap)) lo = mid + 1; else hi = mid;
    }
    Sp = lo;
  }
  int app;
  if (Sp == 0) app = time_le(min_slot, g.gap) ? 1 : 0;
  else app = (g.gap - av.ge[Sp - 1] >= min_slot - kTimeEps) ? 1 : 0;
  const int S = Sp + app;
  v.S = S;
  v.valid = 1;
  if (Sp >= F.Kg && F.Kg >= Sc) { v.S = Sc + 1; return; }  // grid truncated: capacity
  for (int l = 0; l < P.L; ++l)
    if (v.q[l] >= ccnt[l] && ccnt[l] >= Sc) { v.S = Sc + 1; return; }  // canonical list truncated
  if (S > Sc) return;
  int err = 0;
  for (int s = lane; s < S; s += 32) {
    if (s < Sp) {
      ga.ends[s] = av.ge[s];
      const int64_t c = av.gcap[s];
      if (c < 0) err = 1;
      ga.cap[s] = c;
    } else {
      ga.ends[s] = g.gap;
      const int64_t c = plan_time2bs(P, g.gap - (Sp == 0 ? 0.0 : av.ge[Sp - 1]), 0);
      if (c < 0) err = 1;
      ga.cap[s] = imin(c, P.max_batch);
    }
    ga.nx[s] = 0;
  }
  for (int x = lane; x < S * P.L; x += 32) ga.hc[x] = 0;
  v.cap_err = warp_or(err);
  // strictly increasing ends (the appended end may not exceed the grid when min_slot ~ 0)
  const int inc = app == 0 || Sp == 0 || av.ge[Sp - 1] < g.gap;
  v.inc = inc;
  if (F.dues_ok && inc) {
    // exact dues from the anchor due pass: grid cells below Sp-1 keep their counts,
    // the group's tail (slots Sp-1 and Sp) comes from its GroupTail
    const GroupTail t = av.gt[item];
    __syncwarp();
    for (int s = lane; s < S; s += 32) {
      int32_t n;
      if (s < Sp - 1) n = av.hcum[s + 2] - av.hcum[s + 1];
      else if (s == Sp - 1) n = t.tA;
      else n = t.tB;
      ga.nx[s] = n;
    }
    const int64_t pre = av.hcum[Sp];  // grid cells -1 .. Sp-2
    v.Lx = F.Lx;
    v.Dx = F.Lx + pre + t.td;
    v.exact_fail = Sp >= 1 ? (av.hcum[1] > 0 ? 1 : 0) : (t.fail ? 1 : 0);
    v.spill = t.spill ? 1 : 0;
    v.dues_done = 1;
  }
  __syncwarp();
  // canonical dues -> slots: grid jit clipped to the prefix, or the appended slot
  int cf = 0;
  for (int l = 0; l < P.L; ++l) {
    const int ql = v.q[l];
    for (int k = lane; k < ql; k += 32) {
      const double d = ctime[l * Sc + k];
      int jit;
      if (inc) {
        jit = av.ccell[l * Sc + k];
        if (jit > Sp - 1) jit = Sp - 1;
        if (app && time_le(g.gap, d)) jit = Sp;
      } else {
        jit = jit_search(ga.ends, S, d);
      }
      if (jit < 0) cf |= 1 << l;
      else atomicAdd(&ga.hc[l * S + jit], 1);
    }
  }
  v.cfail = __reduce_or_sync(0xffffffffu, (unsigned)cf);
  __syncwarp();
}

struct EvalOut {
  int status;     // 0 ok, else SLOS_ERR_*
  bool has;       // optional<int64_t>
  int64_t budget;
  int64_t dues;   // reference work counters (D, S)
  int64_t slots;
};

// ---- group setup: one pass over members (lanes over decoders) ----------------
__device__ inline void warp_group_setup(const PlannerDev& P, const DecView& D, GapGroup& g) {
  const int lane = lane_id();
  unsigned mask = 0;
  int64_t per[kMaxTiers];
  for (int l = 0; l < kMaxTiers; ++l) per[l] = 0;
  int n_valid = 0, any_due = 0, bl = 0;
  double minph = INFINITY;
  if (g.exact) {
    for (int k = lane; k < D.n; k += 32) {
      const Member m = member_at(P, D.next[k], D.backlog[k], D.rem[k], D.tier[k], g.now, g.a, g.pull);
      if (!m.valid) continue;
      ++n_valid;
      per[m.tier] += 1;
      if (m.backlog > 0) bl = 1;
      if (m.rem > 0) {
        mask |= 1u << m.tier;
        if (m.backlog > 0) any_due = 1;
        if (g.horizon > kTimeEps && time_le(m.phase, g.horizon)) any_due = 1;
        minph = dmin(minph, m.phase);
      }
    }
  }
  g.exact_mask = __reduce_or_sync(0xffffffffu, mask);
  for (int l = 0; l < P.L; ++l) g.exact_per_tier[l] = warp_sum(per[l]);
  g.n_exact = warp_sum(n_valid);
  g.any_due = warp_or(any_due) != 0;
  g.has_backlog = warp_or(bl) != 0;
  g.min_phase = warp_min(minph);
  g.po_state = 0;
  g.po_budget = 0;
}

// Ordered t0_first scan (batch_planner.cpp:234-239) without serialising the warp:
// cur only decreases, so each round finds the first lane (in member order) that
// still qualifies against the current value.
__device__ inline double warp_t0_first(const PlannerDev& P, const DecView& D, const GapGroup& g,
                                       double t0, double min_slot) {
  const int lane = lane_id();
  double cur = t0;
  if (!g.exact) return cur;
  for (int base = 0; base < D.n; base += 32) {
    const int k = base + lane;
    double ph = 0.0;
    bool ok = false;
    if (k < D.n) {
      const Member m = member_at(P, D.next[k], D.backlog[k], D.rem[k], D.tier[k], g.now, g.a, g.pull);
      ok = m.valid && m.rem > 0 && m.phase > kTimeEps;
      ph = m.phase;
    }
    unsigned above = 0xffffffffu;
    for (;;) {
      const unsigned q = __ballot_sync(0xffffffffu, ok && ph < cur - kTimeEps) & above;
      if (!q) break;
      const int f = __ffs(q) - 1;
      const double pf = __shfl_sync(0xffffffffu, ph, f);
      cur = dmax(pf, min_slot);
      above = (f == 31) ? 0u : (0xffffffffu << (f + 1));
    }
  }
  return cur;
}

// Slot ends (batch_planner.cpp:240-248) on lane 0; returns S (may exceed Sc).
__device__ inline int warp_slot_ends(double* ends, int Sc, double t0_first, double t0, double gap,
                                     double min_slot) {
  int S = 0;
  if (lane_id() == 0) {
    double last = 0.0;
    for (double e = t0_first; time_le(e, gap); e += t0) {
      if (S < Sc) ends[S] = e;
      last = e;
      ++S;
    }
    if (S == 0) {
      if (time_le(min_slot, gap)) { if (S < Sc) ends[S] = gap; ++S; }
    } else if (gap - last >= min_slot - kTimeEps) {
      if (S < Sc) ends[S] = gap;
      ++S;
    }
  }
  S = __shfl_sync(0xffffffffu, S, 0);
  __syncwarp();
  return S;
}

// Build the exact-member variant for tightest tier t0 (lanes over members).
__device__ inline void warp_build_variant(const PlannerDev& P, const DecView& D, const GapGroup& g,
                                          double t0, double min_slot, const WarpScr& w, Variant& v) {
  const int lane = lane_id();
  v.t0 = t0;
  v.t0_first = warp_t0_first(P, D, g, t0, min_slot);
  v.S = warp_slot_ends(w.ends, w.Sc, v.t0_first, t0, g.gap, min_slot);
  v.valid = 1;
  const int S = v.S;
  const bool fits = S <= w.Sc;
  int cap_err = 0;
  if (fits) {
    for (int s = lane; s < S; s += 32) w.nx[s] = 0;
    for (int x = lane; x < S * P.L; x += 32) w.hc[x] = 0;  // layout hc[l*S + s]
    cap_err = warp_slot_caps(P, w.ends, S, w.cap);
  }
  v.cap_err = cap_err;
  __syncwarp();
  int inc = 1;
  if (fits && lane_id() == 0)
    for (int x = 1; x < S; ++x) if (!(w.ends[x - 1] < w.ends[x])) inc = 0;
  v.inc = __shfl_sync(0xffffffffu, inc, 0);
  int64_t late = 0, dues = 0;
  int fail = 0, spill = 0;
  if (g.exact) {
    for (int k = lane; k < D.n; k += 32) {
      const Member m = member_at(P, D.next[k], D.backlog[k], D.rem[k], D.tier[k], g.now, g.a, g.pull);
      if (!m.valid || m.rem <= 0) continue;
      member_dues(P, m, g, w.ends, S, fits, v.inc != 0, w.nx, late, dues, fail, spill);
    }
  }
  v.Lx = warp_sum(late);
  v.Dx = warp_sum(dues) + v.Lx;
  v.exact_fail = warp_or(fail);
  v.spill = warp_or(spill);
  // canonical dues per tier (batch_planner.cpp:214-220): lane l owns tier l
  int q = 0, cf = 0;
  if (lane < P.L) {
    const double tpot = P.tpot[lane];
    for (double d = tpot; time_le(d, g.gap); d += tpot) {
      ++q;
      if (fits) {
        const int jit = jit_search(w.ends, S, d);
        if (jit < 0) cf = 1; else w.hc[lane * S + jit] += 1;
      }
    }
  }
  for (int l = 0; l < P.L; ++l) v.q[l] = __shfl_sync(0xffffffffu, q, l);
  v.cfail = __ballot_sync(0xffffffffu, cf != 0);
  __syncwarp();
}

// Group setup (E1 of a DP level): group facts + the shared variant's slot grid,
// capacities and canonical histogram for the exact census' tightest tier. The
// member-due histogram (nx, Lx, Dx, flags) is filled afterwards by block-wide
// member-chunk tasks (E2), see dp_kernel.
__device__ inline void warp_group_init(const PlannerDev& P, const DecView& D, GapGroup& g,
                                       Variant& v, const GroupVar& ga, int Sc, double min_slot) {
  const int lane = lane_id();
  warp_group_setup(P, D, g);
  v.valid = 0;
  v.S = 0;
  v.Lx = 0;
  v.Dx = 0;
  v.exact_fail = 0;
  v.spill = 0;
  v.cap_err = 0;
  v.cfail = 0;
  v.inc = 0;
  for (int l = 0; l < kMaxTiers; ++l) v.q[l] = 0;
  if (g.gap <= kTimeEps || !g.exact_mask) return;
  const double t0 = P.tpot[__ffs(g.exact_mask) - 1];
  v.t0 = t0;
  v.t0_first = warp_t0_first(P, D, g, t0, min_slot);
  v.S = warp_slot_ends(ga.ends, Sc, v.t0_first, t0, g.gap, min_slot);
  v.valid = 1;
  const int S = v.S;
  {
    int q = 0;
    if (lane < P.L)
      for (double d = P.tpot[lane]; time_le(d, g.gap); d += P.tpot[lane]) ++q;
    for (int l = 0; l < P.L; ++l) v.q[l] = __shfl_sync(0xffffffffu, q, l);
  }
  if (S > Sc) return;  // surfaces as SLOS_ERR_CAPACITY when a key reaches the slots
  for (int s = lane; s < S; s += 32) ga.nx[s] = 0;
  for (int x = lane; x < S * P.L; x += 32) ga.hc[x] = 0;
  v.cap_err = warp_slot_caps(P, ga.ends, S, ga.cap);
  int inc = 1;
  if (lane == 0)
    for (int x = 1; x < S; ++x) if (!(ga.ends[x - 1] < ga.ends[x])) inc = 0;
  v.inc = __shfl_sync(0xffffffffu, inc, 0);
  __syncwarp();
  int cf = 0;
  if (lane < P.L) {
    const double tpot = P.tpot[lane];
    for (double d = tpot; time_le(d, g.gap); d += tpot) {
      const int jit = jit_search(ga.ends, S, d);
      if (jit < 0) cf = 1; else ga.hc[lane * S + jit] += 1;
    }
  }
  v.cfail = __ballot_sync(0xffffffffu, cf != 0);
  __syncwarp();
}

// Canonical-only variant (no exact members) for the speculative remainder
// tile_gap_ar(gap - used, rest) (batch_planner.cpp:390-395).
__device__ inline void warp_build_canon_variant(const PlannerDev& P, double gap, double t0,
                                                double min_slot, double* ends, int64_t* cap,
                                                int32_t* hc, int Sc, Variant& v) {
  const int lane = lane_id();
  v.t0 = t0;
  v.t0_first = t0;
  v.S = warp_slot_ends(ends, Sc, t0, t0, gap, min_slot);
  v.valid = 1;
  const int S = v.S;
  const bool fits = S <= Sc;
  int cap_err = 0;
  if (fits) {
    for (int x = lane; x < S * P.L; x += 32) hc[x] = 0;
    cap_err = warp_slot_caps(P, ends, S, cap);
  }
  v.cap_err = cap_err;
  v.Lx = 0;
  v.Dx = 0;
  v.exact_fail = 0;
  v.spill = 0;
  v.inc = 0;
  __syncwarp();
  int q = 0, cf = 0;
  if (lane < P.L) {
    const double tpot = P.tpot[lane];
    for (double d = tpot; time_le(d, gap); d += tpot) {
      ++q;
      if (fits) {
        const int jit = jit_search(ends, S, d);
        if (jit < 0) cf = 1; else hc[lane * S + jit] += 1;
      }
    }
  }
  for (int l = 0; l < P.L; ++l) v.q[l] = __shfl_sync(0xffffffffu, q, l);
  v.cfail = __ballot_sync(0xffffffffu, cf != 0);
  __syncwarp();
}

// prefill_only lambda (batch_planner.cpp:177-195), budget only. status!=0 on throw.
// While the remaining budget fits a full chunk C = min(max_chunk, max_batch), the
// step is exactly (C, plan_predict(C)): predict is monotone in the token count
// (coefficients are validated nonnegative), so time2bs's binary search returns
// >= C whenever predict(C) fits, and min(., max_chunk) = C. Only the tail steps
// binary-search.
__device__ inline int64_t prefill_only_budget(const PlannerDev& P, double gap, double min_slot,
                                              int* status) {
  double t = 0.0;
  int64_t budget = 0;
  const int64_t C = imin(P.max_chunk, P.max_batch);
  const double predC = predict(P, C, 0);
  const double durC = predC * P.margin1;  // plan_predict(P, C, 0)
  for (long guard = 0; gap - t >= min_slot - kTimeEps; ++guard) {
    if (time_le(predC, (gap - t) / P.margin1)) {  // plan_time2bs(gap - t) >= C
      if (guard > 100000000L) { *status = SLOS_ERR_INTERNAL_INCONSISTENCY; return 0; }
      budget += C;
      t += durC;
      continue;
    }
    int64_t size = plan_time2bs(P, gap - t, 0);
    if (size < 0) { *status = SLOS_ERR_INFEASIBLE_BUDGET; return 0; }
    if (guard > 100000000L) { *status = SLOS_ERR_INTERNAL_INCONSISTENCY; return 0; }
    size = imin(size, P.max_chunk);
    const double dur = plan_predict(P, size, 0);
    budget += size;
    t += dur;
  }
  *status = 0;
  return budget;
}

// Latest-fit placement budget for counts c over a built variant (warp, lanes over
// slots). Returns 1 = feasible (*budget set), 0 = nullopt.
__device__ inline int warp_place_budget(const PlannerDev& P, const Variant& v, const double* ends,
                                        const int64_t* cap, const int32_t* nx, const int32_t* hc,
                                        int64_t* tmp, const int64_t* c, int64_t* budget) {
  (void)ends;
  const int lane = lane_id();
  const int S = v.S;
  const int L = P.L;
  if (v.Lx == 0) {
    // fast path: no late dues and every jit group fits its own slot -> latest-fit
    // places each group in its jit slot and free_s = cap_s - n_s.
    bool ok = true;
    int64_t b = 0;
    for (int base = 0; base < S; base += 32) {
      const int s = base + lane;
      if (s < S) {
        int64_t n = nx ? nx[s] : 0;
        for (int l = 0; l < L; ++l)
          if (c[l] > 0) n += c[l] * (int64_t)hc[l * S + s];
        const int64_t f = cap[s] - n;
        if (f < 0) ok = false;
        b += imin(f, P.max_chunk);
      }
    }
    if (__all_sync(0xffffffffu, ok)) {
      *budget = warp_sum(b);
      return 1;
    }
  }
  // forward pass: free capacity after late dues, F - D prefix
  int64_t carry_cap = 0, carry_F = 0, carry_D = 0, min_diff = INT64_MAX;
  for (int base = 0; base < S; base += 32) {
    const int s = base + lane;
    int64_t capv = 0, n = 0;
    if (s < S) {
      capv = cap[s];
      n = nx ? nx[s] : 0;
      for (int l = 0; l < L; ++l)
        if (c[l] > 0) n += c[l] * (int64_t)hc[l * S + s];
    }
    const int64_t cc = warp_incl_scan(capv) + carry_cap;
    const int64_t before = cc - capv;
    int64_t used = v.Lx - before;
    used = used < 0 ? 0 : (used > capv ? capv : used);
    const int64_t free0 = capv - used;
    const int64_t F = warp_incl_scan(free0) + carry_F;
    const int64_t Dn = warp_incl_scan(n) + carry_D;
    const int64_t diff = F - Dn;
    if (s < S) tmp[s] = diff;
    min_diff = imin(min_diff, s < S ? diff : INT64_MAX);
    carry_cap = __shfl_sync(0xffffffffu, cc, 31);
    carry_F = __shfl_sync(0xffffffffu, F, 31);
    carry_D = __shfl_sync(0xffffffffu, Dn, 31);
  }
  min_diff = warp_min(min_diff);
  if (v.Lx > carry_cap) return 0;  // a late due finds every slot full
  if (min_diff < 0) return 0;      // some jit group overflows
  __syncwarp();
  // suffix minima G(s) = min_{u>=s} diff(u), stored in place (backwards chunks)
  int64_t carry_min = INT64_MAX;
  const int nch = (S + 31) / 32;
  for (int ch = nch - 1; ch >= 0; --ch) {
    const int s = ch * 32 + lane;
    int64_t x = s < S ? tmp[s] : INT64_MAX;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // suffix min within the chunk
      const int64_t y = __shfl_down_sync(0xffffffffu, x, o);
      if (lane + o < 32) x = imin(x, y);
    }
    x = imin(x, carry_min);
    __syncwarp();
    if (s < S) tmp[s] = x;
    carry_min = __shfl_sync(0xffffffffu, x, 0);
  }
  __syncwarp();
  int64_t b = 0;
  for (int base = 0; base < S; base += 32) {
    const int s = base + lane;
    if (s < S) {
      const int64_t f = tmp[s] - (s > 0 ? tmp[s - 1] : 0);
      b += imin(f, P.max_chunk);
    }
  }
  *budget = warp_sum(b);
  __syncwarp();
  return 1;
}

}  // namespace slos

namespace slos {

// One-thread form of warp_place_budget (same arithmetic, same result): a forward
// pass for the totals and min_u (F(u) - D(u)), then a backward pass that rebuilds
// F and D from the totals, keeps the suffix minimum G(u) and sums
// min(G(s) - G(s-1), max_chunk). No per-slot storage, so 32 count vectors of a
// DP level are placed per warp at once (lanes over memo keys).
__device__ inline int thread_place_budget(const PlannerDev& P, const Variant& v, const int64_t* cap,
                                          const int32_t* nx, const int32_t* hc, const int64_t* c,
                                          int64_t* budget, const int64_t* cnx = nullptr,
                                          const uint32_t* hcp = nullptr) {
  const int S = v.S;
  const int L = P.L;
  if (v.packed && cnx && hcp) {
    // n(s) = nx(s) + sum_l c_l * hc_l(s): one __dp4a over 8-bit lanes (L <= 4,
    // canonical per-slot counts <= 255 and tier counts <= 250 both fit a byte)
    uint32_t cpk = 0;
#pragma unroll
    for (int l = 0; l < 4; ++l) if (l < L) cpk |= (uint32_t)c[l] << (8 * l);
    if (v.Lx == 0) {
      bool ok = true;
      int64_t b = 0;
#pragma unroll 4
      for (int s = 0; s < S; ++s) {
        const int64_t f = cnx[s] - (int64_t)__dp4a(hcp[s], cpk, 0u);
        ok = ok && f >= 0;
        b += imin(f, P.max_chunk);
      }
      if (ok) { *budget = b; return 1; }
    }
    int64_t capT = 0, F = 0, Dn = 0, min_diff = INT64_MAX;
    for (int s = 0; s < S; ++s) {
      const int64_t capv = cap[s];
      int64_t used = v.Lx - capT;
      used = used < 0 ? 0 : (used > capv ? capv : used);
      capT += capv;
      F += capv - used;
      Dn += capv - cnx[s] + (int64_t)__dp4a(hcp[s], cpk, 0u);
      min_diff = imin(min_diff, F - Dn);
    }
    if (v.Lx > capT) return 0;
    if (min_diff < 0) return 0;
    int64_t cap_after = 0, G_next = INT64_MAX, b = 0;
    for (int u = S - 1; u >= 0; --u) {
      const int64_t capv = cap[u];
      const int64_t before = capT - cap_after - capv;
      int64_t used = v.Lx - before;
      used = used < 0 ? 0 : (used > capv ? capv : used);
      const int64_t Gu = imin(F - Dn, G_next);
      if (u + 1 < S) b += imin(G_next - Gu, P.max_chunk);
      G_next = Gu;
      F -= capv - used;
      Dn -= capv - cnx[u] + (int64_t)__dp4a(hcp[u], cpk, 0u);
      cap_after += capv;
    }
    b += imin(G_next, P.max_chunk);
    *budget = b;
    return 1;
  }
  // the count vector stays in registers: every tier loop is unrolled to kMaxTiers
  // with constant indices (a runtime-bounded loop would index it in local memory)
  int64_t cr[kMaxTiers];
#pragma unroll
  for (int l = 0; l < kMaxTiers; ++l) cr[l] = l < L ? c[l] : 0;
  auto dues_at = [&](int s) -> int64_t {
    int64_t n = nx ? nx[s] : 0;
#pragma unroll
    for (int l = 0; l < kMaxTiers; ++l)
      if (cr[l] > 0) n += cr[l] * (int64_t)hc[l * S + s];
    return n;
  };
  if (v.Lx == 0) {
    bool ok = true;
    int64_t b = 0;
#pragma unroll 4
    for (int s = 0; s < S; ++s) {
      const int64_t f = cap[s] - dues_at(s);
      ok = ok && f >= 0;
      b += imin(f, P.max_chunk);
    }
    if (ok) { *budget = b; return 1; }
  }
  int64_t capT = 0, F = 0, Dn = 0, min_diff = INT64_MAX;
  for (int s = 0; s < S; ++s) {
    const int64_t capv = cap[s];
    int64_t used = v.Lx - capT;
    used = used < 0 ? 0 : (used > capv ? capv : used);
    capT += capv;
    F += capv - used;
    Dn += dues_at(s);
    min_diff = imin(min_diff, F - Dn);
  }
  if (v.Lx > capT) return 0;
  if (min_diff < 0) return 0;
  int64_t cap_after = 0, G_next = INT64_MAX, b = 0;
  for (int u = S - 1; u >= 0; --u) {
    const int64_t capv = cap[u];
    const int64_t before = capT - cap_after - capv;
    int64_t used = v.Lx - before;
    used = used < 0 ? 0 : (used > capv ? capv : used);
    const int64_t Gu = imin(F - Dn, G_next);
    if (u + 1 < S) b += imin(G_next - Gu, P.max_chunk);
    G_next = Gu;
    F -= capv - used;
    Dn -= dues_at(u);
    cap_after += capv;
  }
  b += imin(G_next, P.max_chunk);
  *budget = b;
  return 1;
}

// One-thread form of warp_eval_counts for the autoregressive budget when the
// group's shared variant applies (the common case). Returns 1 when the key needs
// the warp path instead (speculative planner, or a tightest tier that differs from
// the group variant's and so needs a private variant).
__device__ inline int thread_eval_counts(const PlannerDev& P, const GapGroup& g, const Variant& gv,
                                         const GroupVar& ga, int Sc, const int64_t* c, double min_slot,
                                         EvalOut& o) {
  o.status = 0; o.has = false; o.budget = 0; o.dues = 0; o.slots = 0;
  if (P.speculative) return 1;
  const int L = P.L;
  unsigned cmask = 0;
#pragma unroll
  for (int l = 0; l < kMaxTiers; ++l) if (l < L && c[l] > 0) cmask |= 1u << l;
  if (g.gap <= kTimeEps) { o.has = !g.any_due; return 0; }
  const unsigned present = g.exact_mask | cmask;
  auto prefill_only = [&]() {
    int st = 0;
    const int64_t b = prefill_only_budget(P, g.gap, min_slot, &st);
    if (st) { o.status = SLOS_ERR_INFEASIBLE_BUDGET; return; }
    o.has = true;
    o.budget = b;
  };
  if (!present) { prefill_only(); return 0; }
  const double t0 = P.tpot[__ffs(present) - 1];
  if (!(gv.valid && gv.t0 == t0)) return 1;
  if (gv.S > Sc) { o.status = SLOS_ERR_CAPACITY; return 0; }
  int64_t Dtot = gv.Dx;
#pragma unroll
  for (int l = 0; l < kMaxTiers; ++l) if (l < L) Dtot += c[l] * (int64_t)gv.q[l];
  o.dues = Dtot;
  if (Dtot == 0) { prefill_only(); return 0; }
  if (min_slot > t0 + kTimeEps) return 0;
  o.slots = gv.S;
  if (gv.S == 0) return 0;
  if (gv.cap_err) { o.status = SLOS_ERR_INFEASIBLE_BUDGET; return 0; }
  if (gv.exact_fail || (gv.cfail & cmask)) return 0;
  int64_t b = 0;
  o.has = thread_place_budget(P, gv, ga.cap, ga.nx, ga.hc, c, &b, ga.cnx, ga.hcp) != 0;
  o.budget = o.has ? b : 0;
  return 0;
}

}  // namespace slos
