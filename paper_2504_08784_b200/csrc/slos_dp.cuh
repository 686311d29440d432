// Admission DP kernel (K3 + terminal selection of K4): SloScheduler::run's DP,
// dp_scheduler.cpp:438-544, one CTA per planning instance.
//
// The reference walks (item i, source item j, surviving source state) in order,
// memoising gap budgets and inserting candidates into eps-Pareto buckets one by
// one. Here each chain item i is one block-synchronous LEVEL:
//   1. enumerate the level's candidates (j ascending, then source creation order:
//      exactly the reference traversal, dp_scheduler.cpp:467-478);
//   2. find-or-insert every memo key (a_us, raw_us, counts) in a per-instance HBM
//      hash table; a key new to this level keeps its FIRST candidate (atomicMin),
//      i.e. the reference's first-computed value under µs key collisions (:423-435);
//   3. evaluate the new keys grouped by anchor j, one warp per group, with the
//      warp Δpb engine (slos_gapwarp.cuh) sharing the exact census across counts;
//   4. form candidate states (:479-498);
//   5. group candidates by Pareto bucket (item, counts) with a stable multi-split,
//      then one thread per bucket replays try_insert (:445-465) in candidate order;
//   6. arena ids = rank among accepted candidates (creation order), survivors =
//      accepted and not later pruned, stored level by level (states_at).
// Terminal selection (:504-522) is a parallel lexicographic argmax when every
// value is integral (eps ties impossible), otherwise the reference's sequential
// scan; backtracking and the admitted/declined lists follow :532-544.
#pragma once

#include "slos_gapwarp.cuh"

namespace slos {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#ifndef SLOS_DP_THREADS
#define SLOS_DP_THREADS 256
#endif
constexpr int kDpThreads = SLOS_DP_THREADS;
constexpr int kNumPhases = 12;

// Optional per-phase cycle accounting (DpParams.phase_cycles != nullptr): thread 0
// reads clock64() at block-synchronous phase boundaries.
#define SLOS_PHASE(k)                                                          \
  do {                                                                         \
    if (prm.phase_cycles && threadIdx.x == 0) {                                \
      const long long now_ = clock64();                                        \
      atomicAdd(&prm.phase_cycles[(k)], (unsigned long long)(now_ - ph_t0_));  \
      ph_t0_ = now_;                                                           \
    }                                                                          \
  } while (0)
constexpr int kDpWarps = kDpThreads / 32;


__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

// ---- block-wide helpers (kDpThreads threads) --------------------------------
template <int NW>
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* wsum, int64_t* total) {
  const int lane = lane_id(), w = warp_id();
  const int64_t inc = warp_incl_scan(v);
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    int64_t x = lane < NW ? wsum[lane] : 0;
    const int64_t xi = warp_incl_scan(x);
    if (lane < NW) wsum[lane] = xi - x;
    if (lane == NW - 1) wsum[NW] = xi;
  }
  __syncthreads();
  const int64_t r = inc - v + wsum[w];
  *total = wsum[NW];
  __syncthreads();
  return r;
}

// memo find-or-insert; returns slot or -1 on overflow.
__device__ inline int memo_find_insert(MemoEnt* T, int64_t cap, uint64_t k0, uint64_t k1,
                                       uint64_t k2, int c, int32_t* new_list, int* n_new,
                                       int* n_used, int* overflow) {
  uint64_t h = mix64(k0 * 0x9E3779B97F4A7C15ULL ^ mix64(k1 + 0x632BE59BD9B4E019ULL) ^
                     mix64(k2 ^ 0x85EBCA77C2B2AE63ULL)) & (uint64_t)(cap - 1);
  for (int64_t probe = 0; probe < cap; ++probe) {
    MemoEnt* e = &T[h];
    int st = atomicAdd(&e->state, 0);
    if (st == 0) {
      if (atomicCAS(&e->state, 0, 1) == 0) {
        e->k0 = k0; e->k1 = k1; e->k2 = k2;
        e->first = c; e->has = 0; e->val = 0;
        __threadfence();
        atomicExch(&e->state, 2);
        if (atomicAdd(n_used, 1) * 2 >= cap) atomicExch(overflow, 1);
        const int idx = atomicAdd(n_new, 1);
        new_list[idx] = (int32_t)h;
        return (int)h;
      }
      st = atomicAdd(&e->state, 0);
    }
    while (st == 1) st = atomicAdd(&e->state, 0);
    __threadfence();
    const volatile MemoEnt* ve = e;
    if (ve->k0 == k0 && ve->k1 == k1 && ve->k2 == k2) {
      if (st == 2) atomicMin(&e->first, c);
      return (int)h;
    }
    h = (h + 1) & (uint64_t)(cap - 1);
  }
  atomicExch(overflow, 1);
  return -1;
}

// Evaluate one memo key (counts c) of a group: tile_gap(gap, census, dh).prefill_budget.
// `gv`/`ga` is the group's shared exact-census variant (built by the block); a
// count vector whose tightest tier differs builds a private variant in `w`.
__device__ __noinline__ EvalOut warp_eval_counts(const PlannerDev& P, const DecView& D, const GapGroup& g,
                                           const Variant& gv, const GroupVar& ga, int Sc,
                                           const WarpScr& w, const int64_t* c, double min_slot,
                                           int* spill_out) {
  EvalOut o;
  o.status = 0; o.has = false; o.budget = 0; o.dues = 0; o.slots = 0;
  const int L = P.L;
  unsigned cmask = 0;
  for (int l = 0; l < L; ++l) if (c[l] > 0) cmask |= 1u << l;
  *spill_out = gv.valid ? gv.spill : 0;
  // ---------------- tile_gap_ar (budget) ----------------
  bool ar_has = false;
  int64_t ar_budget = 0;
  if (g.gap <= kTimeEps) {
    ar_has = !g.any_due;
  } else {
    const unsigned present = g.exact_mask | cmask;
    if (!present) {
      int st = 0;
      int64_t b = 0;
      if (lane_id() == 0) b = prefill_only_budget(P, g.gap, min_slot, &st);
      st = __shfl_sync(0xffffffffu, st, 0);
      b = __shfl_sync(0xffffffffu, b, 0);
      if (st) { o.status = SLOS_ERR_INFEASIBLE_BUDGET; return o; }
      ar_has = true;
      ar_budget = b;
    } else {
      const double t0 = P.tpot[__ffs(present) - 1];
      Variant vp;
      const Variant* v;
      const double* ends;
      const int64_t* cap;
      const int32_t* nx;
      const int32_t* hc;
      int scap;
      if (gv.valid && gv.t0 == t0) {
        v = &gv; ends = ga.ends; cap = ga.cap; nx = ga.nx; hc = ga.hc; scap = Sc;
        if (gv.S > Sc) { o.status = SLOS_ERR_CAPACITY; return o; }  // histogram was not built
      } else {
        warp_build_variant(P, D, g, t0, min_slot, w, vp);
        v = &vp; ends = w.ends; cap = w.cap; nx = w.nx; hc = w.hc; scap = w.Sc;
        *spill_out = vp.spill;
      }
      int64_t Dtot = v->Dx;
      for (int l = 0; l < L; ++l) Dtot += c[l] * (int64_t)v->q[l];
      o.dues += Dtot;
      if (Dtot == 0) {
        int st = 0;
        int64_t b = 0;
        if (lane_id() == 0) b = prefill_only_budget(P, g.gap, min_slot, &st);
        st = __shfl_sync(0xffffffffu, st, 0);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (st) { o.status = SLOS_ERR_INFEASIBLE_BUDGET; return o; }
        ar_has = true;
        ar_budget = b;
      } else if (min_slot > t0 + kTimeEps) {
        ar_has = false;
      } else {
        o.slots += v->S;
        if (v->S == 0) {
          ar_has = false;
        } else if (v->S > scap) {
          o.status = SLOS_ERR_CAPACITY;
          return o;
        } else if (v->cap_err) {
          o.status = SLOS_ERR_INFEASIBLE_BUDGET;
          return o;
        } else if (v->exact_fail || (v->cfail & cmask)) {
          ar_has = false;
        } else {
          ar_has = warp_place_budget(P, *v, ends, cap, nx, hc, w.tmp, c, &ar_budget) != 0;
        }
      }
    }
  }
  o.has = ar_has;
  o.budget = ar_budget;
  // ---------------- tile_gap speculative branch (batch_planner.cpp:318-405) -----
  if (!P.speculative) return o;
  if (g.n_exact == 0 && cmask == 0) return o;  // census.empty()
  const bool spill = *spill_out != 0;
  if (g.has_backlog) return o;
  if (g.dh > g.gap + kTimeEps && spill) return o;
  int64_t merged[kMaxTiers];
  for (int l = 0; l < L; ++l) merged[l] = c[l] + g.exact_per_tier[l];
  SpecSol sp;
  if (lane_id() == 0) sp = solve_spec(P, merged);
  sp.ok = __shfl_sync(0xffffffffu, sp.ok, 0);
  if (!sp.ok) return o;
  sp.bt = __shfl_sync(0xffffffffu, sp.bt, 0);
  sp.cap = __shfl_sync(0xffffffffu, sp.cap, 0);
  for (int l = 0; l < kMaxTiers; ++l) sp.lengths[l] = __shfl_sync(0xffffffffu, sp.lengths[l], 0);
  if (g.n_exact > 0 && g.min_phase < sp.bt - kTimeEps) return o;
  const int full = (int)floor(g.gap / sp.bt + kTimeEps);
  if (full == 0) return o;
  if (full + 2 > w.Sc + 2) { o.status = SLOS_ERR_CAPACITY; return o; }
  int64_t canon_dec = 0;
  for (int l = 0; l < L; ++l) canon_dec += c[l] * (int64_t)sp.lengths[l];
  for (int k = lane_id(); k <= full; k += 32) w.kh[k] = 0;
  __syncwarp();
  if (g.exact) {
    for (int k = lane_id(); k < D.n; k += 32) {
      const Member m = member_at(P, D.next[k], D.backlog[k], D.rem[k], D.tier[k], g.now, g.a, g.pull);
      if (!m.valid || m.rem <= 0) continue;
      const int64_t sl = sp.lengths[m.tier];
      const int64_t q = m.rem / sl, r = m.rem % sl;
      atomicAdd((unsigned long long*)&w.kh[0], (unsigned long long)sl);
      if (q < full) {
        atomicAdd((unsigned long long*)&w.kh[q], (unsigned long long)(r - sl));
        atomicAdd((unsigned long long*)&w.kh[q + 1], (unsigned long long)(-r));
      }
    }
  }
  __syncwarp();
  int64_t spec_budget = 0, carry = 0;
  for (int base = 0; base < full; base += 32) {
    const int k = base + lane_id();
    const int64_t x = k < full ? w.kh[k] : 0;
    const int64_t e = warp_incl_scan(x) + carry;
    carry = __shfl_sync(0xffffffffu, e, 31);
    if (k < full) {
      const int64_t decode = canon_dec + e;
      spec_budget += imax(0, imin(sp.cap - decode, P.max_chunk));
    }
  }
  spec_budget = warp_sum(spec_budget);
  const double used = full * sp.bt;
  if (g.gap - used > kTimeEps) {
    const double gap2 = g.gap - used;
    unsigned pm = 0;
    for (int l = 0; l < L; ++l) if (merged[l] > 0) pm |= 1u << l;
    bool tail_has = false;
    int64_t tail_budget = 0;
    // tile_gap_ar(gap2, rest): gap2 > eps; rest is canonical only
    if (!pm) {
      int st = 0;
      if (lane_id() == 0) tail_budget = prefill_only_budget(P, gap2, min_slot, &st);
      st = __shfl_sync(0xffffffffu, st, 0);
      tail_budget = __shfl_sync(0xffffffffu, tail_budget, 0);
      if (st) { o.status = SLOS_ERR_INFEASIBLE_BUDGET; return o; }
      tail_has = true;
    } else {
      const double t0 = P.tpot[__ffs(pm) - 1];
      Variant v2;
      warp_build_canon_variant(P, gap2, t0, min_slot, w.ends2, w.cap2, w.hc2, w.Sc, v2);
      int64_t Dt = 0;
      for (int l = 0; l < L; ++l) Dt += merged[l] * (int64_t)v2.q[l];
      o.dues += Dt;
      if (Dt == 0) {
        int st = 0;
        if (lane_id() == 0) tail_budget = prefill_only_budget(P, gap2, min_slot, &st);
        st = __shfl_sync(0xffffffffu, st, 0);
        tail_budget = __shfl_sync(0xffffffffu, tail_budget, 0);
        if (st) { o.status = SLOS_ERR_INFEASIBLE_BUDGET; return o; }
        tail_has = true;
      } else if (min_slot > t0 + kTimeEps) {
        tail_has = false;
      } else {
        o.slots += v2.S;
        if (v2.S == 0) tail_has = false;
        else if (v2.S > w.Sc) { o.status = SLOS_ERR_CAPACITY; return o; }
        else if (v2.cap_err) { o.status = SLOS_ERR_INFEASIBLE_BUDGET; return o; }
        else if (v2.cfail & pm) tail_has = false;
        else tail_has = warp_place_budget(P, v2, w.ends2, w.cap2, nullptr, w.hc2, w.tmp, merged,
                                          &tail_budget) != 0;
      }
    }
    if (!tail_has) return o;
    spec_budget += tail_budget;
  }
  if (o.has && o.budget >= spec_budget) return o;
  o.has = true;
  o.budget = spec_budget;
  return o;
}


// Build the anchor cache of anchor j (gap start a) for this instance: block-wide.
// gmax: the longest gap any later chain item can open from this anchor.
template <int NT>
__device__ inline void block_build_anchor(const PlannerDev& P, const DecView& D, const AnchorView& av,
                                          double a, double now, double pull, double gmax, int Sc,
                                          const double* ctime, const int* ccnt, double min_slot,
                                          int64_t* s_red) {
  const int tid = threadIdx.x;
  const int lane = lane_id(), w = warp_id();
  __shared__ unsigned s_mask;
  __shared__ int s_nex, s_hb, s_abl;
  __shared__ unsigned s_pt[kMaxTiers];
  __shared__ double s_minph[(NT / 32)];
  if (tid == 0) {
    s_mask = 0; s_nex = 0; s_hb = 0; s_abl = 0;
    for (int l = 0; l < kMaxTiers; ++l) s_pt[l] = 0;
  }
  __syncthreads();
  double minph = INFINITY;
  unsigned mask = 0;
  int nex = 0, hb = 0, abl = 0;
  uint64_t pt8 = 0;  // per-thread member count per tier, 8 bits each (<= 255 members per thread)
  int it = 0;
  for (int k = tid; k < D.n; k += NT) {
    if ((++it & 0xff) == 0) {  // keep every 8-bit tier count below 256
      for (int l = 0; l < P.L; ++l)
        if ((pt8 >> (8 * l)) & 0xffu) atomicAdd(&s_pt[l], (unsigned)((pt8 >> (8 * l)) & 0xffu));
      pt8 = 0;
    }
    const Member m = member_at(P, D.next[k], D.backlog[k], D.rem[k], D.tier[k], now, a, pull);
    av.ph[k] = m.valid ? m.phase : 0.0;
    av.bl[k] = m.valid ? m.backlog : 0;
    av.rm[k] = m.valid ? m.rem : 0;
    if (!m.valid) continue;
    ++nex;
    pt8 += 1ull << (8 * m.tier);
    if (m.backlog > 0) hb = 1;
    if (m.rem > 0) {
      mask |= 1u << m.tier;
      if (m.backlog > 0) abl = 1;
      minph = dmin(minph, m.phase);
    }
  }
  for (int l = 0; l < P.L; ++l) {
    const unsigned cl = __reduce_add_sync(0xffffffffu, (unsigned)((pt8 >> (8 * l)) & 0xffu));
    if (lane == 0 && cl) atomicAdd(&s_pt[l], cl);
  }
  mask = __reduce_or_sync(0xffffffffu, mask);
  nex = __reduce_add_sync(0xffffffffu, (unsigned)nex);
  hb = warp_or(hb);
  abl = warp_or(abl);
  minph = warp_min(minph);
  if (lane == 0) {
    atomicOr(&s_mask, mask);
    atomicAdd(&s_nex, nex);
    if (hb) atomicOr(&s_hb, 1);
    if (abl) atomicOr(&s_abl, 1);
    s_minph[w] = minph;
  }
  __syncthreads();
  AnchorFacts* F = av.f;
  if (tid == 0) {
    F->a = a;
    F->exact_mask = s_mask;
    F->n_exact = s_nex;
    F->has_backlog = s_hb;
    F->any_bl = s_abl;
    double mp = s_minph[0];
    for (int x = 1; x < (NT / 32); ++x) mp = dmin(mp, s_minph[x]);
    F->min_phase = mp;
    for (int l = 0; l < kMaxTiers; ++l) F->per_tier[l] = (int64_t)s_pt[l];
    F->t0 = s_mask ? P.tpot[__ffs(s_mask) - 1] : 0.0;
    F->Kg = 0;
    F->grid_ok = 0;
    F->cap_uniform_err = 0;
  }
  __syncthreads();
  const unsigned emask = F->exact_mask;
  if (!emask) return;
  const double t0 = F->t0;
  // t0_first (batch_planner.cpp:234-239): ordered scan, warp 0
  if (w == 0) {
    double cur = t0;
    for (int base = 0; base < D.n; base += 32) {
      const int k = base + lane;
      const bool ok = k < D.n && av.rm[k] > 0 && av.ph[k] > kTimeEps;
      const double ph = ok ? av.ph[k] : 0.0;
      unsigned above = 0xffffffffu;
      for (;;) {
        const unsigned q = __ballot_sync(0xffffffffu, ok && ph < cur - kTimeEps) & above;
        if (!q) break;
        const int f = __ffs(q) - 1;
        cur = dmax(__shfl_sync(0xffffffffu, ph, f), min_slot);
        above = (f == 31) ? 0u : (0xffffffffu << (f + 1));
      }
    }
    if (lane == 0) {
      F->t0_first = cur;
      // grid e_k = t0_first + k*t0 by repeated addition (:241) up to the longest gap
      int K = 0, ok = 1;
      double prev = -INFINITY;
      for (double e = cur; time_le(e, gmax) && K < Sc; e += t0) {
        if (!(prev < e)) ok = 0;
        av.ge[K++] = e;
        prev = e;
      }
      F->Kg = K;
      F->grid_ok = ok;
    }
  }
  __syncthreads();
  const int Kg = F->Kg;
  // grid slot capacities (duration e_k - e_{k-1}); -1 where time2bs throws
  for (int s = tid; s < Kg; s += NT) {
    const double dur = av.ge[s] - (s == 0 ? 0.0 : av.ge[s - 1]);
    const int64_t c = plan_time2bs(P, dur, 0);
    av.gcap[s] = c < 0 ? -1 : imin(c, P.max_batch);
  }
  // canonical due times -> grid jit
  for (int l = 0; l < P.L; ++l)
    for (int k = tid; k < ccnt[l]; k += NT) av.ccell[l * Sc + k] = jit_search(av.ge, Kg, ctime[l * Sc + k]);
  __syncthreads();
  (void)s_red;
}

// Cooperative copy of a plain struct into shared memory (8-byte words, all threads).

// Anchor due pass (replaces the per-group member walks of E2): every exact member's
// due line from anchor a is walked ONCE, up to the longest due horizon of any group
// (j, i) this anchor opens, exactly as member_dues_warp walks it (same repeated
// additions, the same jit on the strictly increasing anchor grid). Dues land in a
// per-grid-cell histogram; a group's slots below Sp_i-1 are exactly those cells.
// Only the dues in a group's TAIL cells (>= Sp_i-1, up to its horizon) depend on i
// (slot Sp_i-1 vs the appended slot, inclusion, spill), so each due also visits the
// few groups whose tail covers its cell and accumulates their GroupTail.
// Runs only when the anchor grid is usable (grid_ok) and no member has a negative
// backlog (tile_gap's second spill scan); otherwise the groups fall back to E2.
template <int NT>
__device__ inline void block_anchor_dues(const PlannerDev& P, const DecView& D, const AnchorView& av,
                                         int j, int N, const double* ch_dl, const int32_t* ch_fl,
                                         double a, double pull, double min_slot, int Sc,
                                         unsigned char* scr, size_t scr_bytes) {
  const int tid = threadIdx.x;
  AnchorFacts* F = av.f;
  __shared__ int s_ok, s_nl;
  __shared__ unsigned long long s_lx;
  __shared__ double s_hmax;
  const int Kg = F->Kg;
  const int nG = N - j - 1;  // chain items i = j+1 .. N-1 (group index i-j-1)
  // scratch carve (overlay area, free at this point of the level)
  unsigned char* p = scr;
  double* sge = (double*)p; p += 8 * (size_t)Kg;
  double* g_gap = (double*)p; p += 8 * (size_t)nG;
  double* g_hor = (double*)p; p += 8 * (size_t)nG;
  int32_t* g_Sp = (int32_t*)p; p += 4 * (size_t)nG;
  int32_t* g_lo = (int32_t*)p; p += 4 * (size_t)nG;
  int32_t* g_hi = (int32_t*)p; p += 4 * (size_t)nG;
  int32_t* g_acc = (int32_t*)p; p += 4 * 5 * (size_t)nG;  // tA, tB, td, fail, spill
  int32_t* sHc = (int32_t*)p; p += 4 * (size_t)(Kg + 1);
  int32_t* l_off = (int32_t*)p; p += 4 * (size_t)(Kg + 2);
  const size_t used = (size_t)(p - scr);
  const int lcap = used < scr_bytes ? (int)((scr_bytes - used) / 4) : 0;
  int32_t* l_item = (int32_t*)p;
  if (tid == 0) {
    s_ok = (F->grid_ok && F->exact_mask && Kg > 0 && nG > 0 && used <= scr_bytes) ? 1 : 0;
    s_lx = 0;
    s_nl = 0;
    s_hmax = 0.0;
  }
  __syncthreads();
  if (!s_ok) {
    if (tid == 0) F->dues_ok = 0;
    return;
  }
  for (int k = tid; k < Kg; k += NT) sge[k] = av.ge[k];
  for (int k = tid; k <= Kg; k += NT) sHc[k] = 0;
  for (int k = tid; k < 5 * nG; k += NT) g_acc[k] = 0;
  int neg = 0;
  for (int k = tid; k < D.n; k += NT)
    if (av.rm[k] > 0 && av.bl[k] < 0) neg = 1;
  __syncthreads();
  // per group: gap, horizon, Sp, tail cell range [lo, hi] (cells -1 .. Kg-1)
  double hloc = 0.0;
  for (int gi = tid; gi < nG; gi += NT) {
    const int i = j + 1 + gi;
    if (ch_fl[i] > j) {  // (j, i) is never a DP transition
      g_lo[gi] = 1; g_hi[gi] = 0; g_Sp[gi] = 0; g_gap[gi] = 0.0; g_hor[gi] = 0.0;
      continue;
    }
    const double raw = dmax(0.0, ch_dl[i] - a);
    const double gap = quantize_gap(raw);
    const double hor = dmax(gap, raw + pull);
    int lo = 0, hi = Kg;
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      if (time_le(sge[mid], gap)) lo = mid + 1; else hi = mid;
    }
    const int Sp = lo;
    // last cell whose start can be <= a due within the horizon (superset; every tail
    // due is tested exactly below)
    int c_hi = -1;
    {
      int l2 = 0, h2 = Kg;
      const double lim = hor + 3e-9;
      while (l2 < h2) {
        const int mid = (l2 + h2) / 2;
        if (sge[mid] <= lim) l2 = mid + 1; else h2 = mid;
      }
      c_hi = l2 - 1;
    }
    g_gap[gi] = gap;
    g_hor[gi] = hor;
    // Sp and whether the gap end is appended as a slot (batch_planner.cpp:242-247)
    const bool app = Sp == 0 ? time_le(min_slot, gap) : (gap - sge[Sp - 1] >= min_slot - kTimeEps);
    g_Sp[gi] = 2 * Sp + (app ? 1 : 0);
    g_lo[gi] = Sp - 1;
    g_hi[gi] = c_hi < Sp - 1 ? Sp - 1 : c_hi;
    hloc = dmax(hloc, hor);
  }
  for (int o = 16; o; o >>= 1) hloc = dmax(hloc, __shfl_xor_sync(0xffffffffu, hloc, o));
  neg = warp_or(neg);
  if (lane_id() == 0) {
    if (neg) atomicExch(&s_ok, 0);
    // non-negative doubles order like their bit patterns
    atomicMax((unsigned long long*)&s_hmax, (unsigned long long)__double_as_longlong(hloc));
  }
  __syncthreads();
  if (!s_ok) {
    if (tid == 0) F->dues_ok = 0;
    return;
  }
  // per-cell group lists (cell y = c+1): counts, exclusive offsets, items
  for (int y = tid; y <= Kg; y += NT) {
    int n = 0;
    for (int gi = 0; gi < nG; ++gi) n += (g_lo[gi] <= y - 1 && y - 1 <= g_hi[gi]) ? 1 : 0;
    l_off[y + 1] = n;
  }
  __syncthreads();
  if (tid < 32) {  // list offsets: a warp scan over the cells
    const int lane = lane_id();
    int carry = 0;
    for (int base = 0; base <= Kg; base += 32) {
      const int y = base + lane;
      const int n = y <= Kg ? l_off[y + 1] : 0;
      const int inc = warp_incl_scan(n);
      if (y <= Kg) l_off[y + 1] = carry + inc;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      l_off[0] = 0;
      s_nl = carry;
      if (carry > lcap) s_ok = 0;
    }
  }
  __syncthreads();
  if (!s_ok) {
    if (tid == 0) F->dues_ok = 0;
    return;
  }
  for (int y = tid; y <= Kg; y += NT) {
    int pos = l_off[y];
    for (int gi = 0; gi < nG; ++gi)
      if (g_lo[gi] <= y - 1 && y - 1 <= g_hi[gi]) l_item[pos++] = gi;
  }
  __syncthreads();
  const double hmax = s_hmax;
  // the walk: lanes over members in lockstep (one due per lane per round)
  unsigned long long lx = 0;
  for (int base = 0; base < D.n; base += NT) {
    const int k = base + tid < D.n ? D.bytier[base + tid] : D.n;  // members grouped by tier
    int64_t rem = 0, issued = 0;
    double d = 0.0, tpot = 0.0;
    bool act = false;
    if (k < D.n) {
      rem = av.rm[k];
      act = rem > 0;
      if (act) {
        const int64_t bl = av.bl[k];
        issued = bl > 0 ? imin(bl, rem) : 0;
        lx += (unsigned long long)issued;
        tpot = P.tpot[D.tier[k]];
        d = dmax(av.ph[k], 0.0);
      }
    }
    int cell = -2;  // grid cell of the previous due (-1: before e_0); -2: none yet
    double nb = 0.0;  // the next cell boundary sge[cell + 1] (+inf past the grid)
    int l0 = 0, l1 = 0;  // the group list of cell y = cell + 1
    for (;;) {
      act = act && time_le(d, hmax) && issued < rem;
      if (!__any_sync(0xffffffffu, act)) break;
      int y = -1;
      if (act) {
        if (d <= kTimeEps) {
          ++lx;
        } else {
          // the cell only moves forward: its boundary and group list stay in
          // registers until a due crosses it
          if (cell == -2) {
            cell = jit_search(sge, Kg, d);
            nb = cell + 1 < Kg ? sge[cell + 1] : INFINITY;
            l0 = l_off[cell + 1];
            l1 = l_off[cell + 2];
          } else if (time_le(nb, d)) {
            do {
              ++cell;
              nb = cell + 1 < Kg ? sge[cell + 1] : INFINITY;
            } while (time_le(nb, d));
            l0 = l_off[cell + 1];
            l1 = l_off[cell + 2];
          }
          y = cell + 1;
          for (int q = l0; q < l1; ++q) {
            const int gi = l_item[q];
            if (!time_le(d, g_hor[gi])) continue;
            const double gap = g_gap[gi];
            const int Sp = g_Sp[gi] >> 1;
            const bool app = (g_Sp[gi] & 1) != 0;
            int32_t* acc = g_acc + 5 * gi;
            atomicAdd(&acc[2], 1);
            if (!time_le(d, gap)) acc[4] = 1;
            // slot: Sp-1 (Sp >= 1), or the appended slot when time_le(gap, d)
            if (app && time_le(gap, d)) atomicAdd(&acc[1], 1);
            else if (Sp >= 1) atomicAdd(&acc[0], 1);
            else acc[3] = 1;
          }
        }
        d += tpot;
        ++issued;
      }
      // per-lane shared-memory atomics: same-cell lanes resolve in the atomic unit
      // (a match_any + leader add measured ~2% slower over the whole anchor stage)
      if (y >= 0) atomicAdd(&sHc[y], 1);
    }
  }
  lx = warp_sum(lx);
  if (lane_id() == 0 && lx) atomicAdd(&s_lx, lx);
  __syncthreads();
  // publish: cumulative histogram, per-group tails, facts
  if (tid < 32) {  // cumulative histogram: a warp scan over the cells
    const int lane = lane_id();
    int carry = 0;
    for (int base = 0; base <= Kg; base += 32) {
      const int y = base + lane;
      const int inc = warp_incl_scan(y <= Kg ? sHc[y] : 0);
      if (y <= Kg) av.hcum[y + 1] = carry + inc;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      av.hcum[0] = 0;
      F->Lx = (int64_t)s_lx;
      F->dues_ok = 1;
    }
  }
  for (int gi = tid; gi < nG; gi += NT) {
    GroupTail t;
    t.tA = g_acc[5 * gi + 0];
    t.tB = g_acc[5 * gi + 1];
    t.td = g_acc[5 * gi + 2];
    t.fail = (int16_t)(g_acc[5 * gi + 3] ? 1 : 0);
    t.spill = (int16_t)(g_acc[5 * gi + 4] ? 1 : 0);
    av.gt[j + 1 + gi] = t;
  }
  __syncthreads();
  (void)Sc;
}

// Anchor caches (prologue of the admission DP). Everything about a gap that depends
// only on its start a = t_j -- the exact census members_at(a), the slot grid and its
// capacities, the canonical due cells and the exact-due histogram with every later
// group's tail (block_anchor_dues) -- is independent of the DP's states, so all
// anchors of all instances are built up front, one CTA per (instance, anchor),
// instead of on the DP's level-sequential critical path.
// 64 threads at 16 CTAs per SM: more anchors in flight (each CTA's serial sections
// and barriers cost less SM time); measured C2 x 1024 anchor stage 1.11 -> 1.07 ms
// against 128 threads at 8 per SM (256 at 4: 1.26; 32 at 32: 1.12), C1 0.90 -> 0.80.
#ifndef SLOS_ANCHOR_THREADS
#define SLOS_ANCHOR_THREADS 64
#endif
constexpr int kAnchorThreads = SLOS_ANCHOR_THREADS;
#ifndef SLOS_ANCHOR_MIN_BLOCKS
#define SLOS_ANCHOR_MIN_BLOCKS 16
#endif
template <int NT>
__device__ __forceinline__ void anchor_body(const DpParams& prm) {
  extern __shared__ __align__(16) unsigned char asm_[];
  __shared__ PlannerDev sP;
  __shared__ InstDev sI;
  __shared__ int ccnt[kMaxTiers];
  __shared__ double s_maxdl, s_minA;
  __shared__ int64_t s_wsum[NT / 32 + 1];
  const BatchArgs& A = prm.a;
  const int tid = threadIdx.x;
  const int task = prm.task0 + blockIdx.x;
  const int v = A.atask[2 * task], j = A.atask[2 * task + 1];
  block_copy_struct(sI, A.inst[v], tid, NT);
  block_copy_struct(sP, A.planners[A.inst[v].planner], tid, NT);
  __syncthreads();
  const PlannerDev& P = sP;
  const InstDev& I = sI;
  const int N = I.N;
  const int L = P.L;
  const int Sc = prm.Sc;
  const double* ch_dl = A.ch_deadline + I.off_chain;
  const int32_t* ch_fl = A.ch_floor + I.off_chain;
  DecView D;
  D.n = I.have_running_decode ? I.n_dec : 0;
  D.next = A.dec_next + I.off_dec;
  D.backlog = A.dec_backlog + I.off_dec;
  D.rem = A.dec_rem + I.off_dec;
  D.tier = A.dec_tier + I.off_dec;
  D.bytier = A.dec_bytier + I.off_dec;
  double* ctime = (double*)asm_;
  unsigned char* scr = asm_ + sizeof(double) * (size_t)prm.Lmax * Sc;
  if (tid < 32) {  // deadline range: a warp reduction (max / min are order-free)
    double mx = I.now, mn = I.now;
    for (int k = tid; k < N; k += 32) { mx = dmax(mx, ch_dl[k]); mn = dmin(mn, ch_dl[k]); }
    for (int o = 16; o; o >>= 1) {
      mx = dmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = dmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (tid == 0) {
      s_maxdl = mx;
      s_minA = mn;
    }
  }
  __syncthreads();
  if (tid < L) {  // instance-wide canonical due times per tier (batch_planner.cpp:216)
    const double gall = quantize_gap(dmax(0.0, s_maxdl - s_minA));
    const double tp = P.tpot[tid];
    int k = 0;
    for (double d = tp; time_le(d, gall) && k < Sc; d += tp) ctime[tid * Sc + k++] = d;
    ccnt[tid] = k;
  }
  __syncthreads();
  const double min_slot = plan_predict(P, 1, 0);  // BatchPlanner::min_slot_s
  const double pull = min_slot;
  const double a = (j < 0) ? I.now : ch_dl[j];
  const AnchorView av = anchor_view(A.anchors + I.off_anchor + (size_t)(j + 1) * I.anchor_stride, D.n, Sc, L);
  block_build_anchor<NT>(P, D, av, a, I.now, pull, quantize_gap(dmax(0.0, s_maxdl - a)), Sc, ctime, ccnt,
                     min_slot, s_wsum);
  block_anchor_dues<NT>(P, D, av, j, N, ch_dl, ch_fl, a, pull, min_slot, Sc, scr, prm.anchor_scr_bytes);
  if (j < 0) {  // the instance's canonical due times, for group_kernel
    double* gct = A.ctime + (size_t)v * prm.Lmax * Sc;
    for (int x = tid; x < L * Sc; x += NT) gct[x] = ctime[x];
    if (tid < kMaxTiers) A.ccnt[v * kMaxTiers + tid] = tid < L ? ccnt[tid] : 0;
  }
}

__global__ void __launch_bounds__(kAnchorThreads, SLOS_ANCHOR_MIN_BLOCKS) anchor_kernel(DpParams prm) {
  anchor_body<kAnchorThreads>(prm);
}

// Anchors of the large-instance class (thousands of decoders: each anchor walks
// every decoder's dues): 512 threads per anchor, since a few dozen such instances
// fill the GPU with one wave of anchors and the walk's length is the stage.
#ifndef SLOS_ANCHOR_BIG_THREADS
#define SLOS_ANCHOR_BIG_THREADS 512
#endif
constexpr int kAnchorBigThreads = SLOS_ANCHOR_BIG_THREADS;
__global__ void __launch_bounds__(kAnchorBigThreads, 2) anchor_kernel_big(DpParams prm) {
  anchor_body<kAnchorBigThreads>(prm);
}

// Gap group records (the DP's E1/E2, off its critical path): one warp per pair
// (j, i), i > j >= floor_at[i], built from anchor j's cache and written to HBM.
#ifndef SLOS_GROUP_WARPS
#define SLOS_GROUP_WARPS 4
#endif
constexpr int kGroupWarps = SLOS_GROUP_WARPS;
__global__ void __launch_bounds__(32 * kGroupWarps, 32 / kGroupWarps) group_kernel(DpParams prm) {
  __shared__ PlannerDev sP;
  __shared__ InstDev sI;
  const BatchArgs& A = prm.a;
  const int task = prm.task0 + blockIdx.x;
  const int vi = A.atask[2 * task], j = A.atask[2 * task + 1];
  // the grid is sized for the longest chain: a CTA past this anchor's pairs exits
  // before staging the headers (about half of them for anchors late in the chain)
  if ((int)blockIdx.y * kGroupWarps >= A.inst[vi].N - j - 1) return;
  block_copy_struct(sI, A.inst[vi], threadIdx.x, 32 * kGroupWarps);
  block_copy_struct(sP, A.planners[A.inst[vi].planner], threadIdx.x, 32 * kGroupWarps);
  __syncthreads();
  const PlannerDev& P = sP;
  const InstDev& I = sI;
  const int N = I.N;
  const int L = P.L;
  const int Sc = prm.Sc;
  const int gi = blockIdx.y * kGroupWarps + warp_id();
  if (gi >= N - j - 1) return;
  const int i = j + 1 + gi;
  const double* ch_dl = A.ch_deadline + I.off_chain;
  if (A.ch_floor[I.off_chain + i] > j) return;  // never a DP transition
  DecView D;
  D.n = I.have_running_decode ? I.n_dec : 0;
  D.next = A.dec_next + I.off_dec;
  D.backlog = A.dec_backlog + I.off_dec;
  D.rem = A.dec_rem + I.off_dec;
  D.tier = A.dec_tier + I.off_dec;
  const double* ctime = A.ctime + (size_t)vi * prm.Lmax * Sc;
  const int* ccnt = A.ccnt + vi * kMaxTiers;
  const double min_slot = plan_predict(P, 1, 0);
  const double pull = min_slot;
  const double a = (j < 0) ? I.now : ch_dl[j];
  const AnchorView av = anchor_view(A.anchors + I.off_anchor + (size_t)(j + 1) * I.anchor_stride, D.n, Sc, L);
  {
    unsigned char* rec = A.groups + I.off_group + (size_t)pair_index(N, j + 1, i) * prm.grec_stride;
    GroupHdr* H = (GroupHdr*)rec;
    const GroupVar ga = group_var_carve(rec + prm.grec_hdr, Sc, L);
    GapGroup g;
    g.a = a;
    const double raw = dmax(0.0, ch_dl[i] - g.a);
    const double len = quantize_gap(raw);
    g.now = I.now;
    g.pull = pull;
    g.exact = I.have_running_decode != 0;
    if (g.exact) { g.gap = len; g.dh = raw + pull; }
    else { g.gap = quantize_gap(len); g.dh = 0.0; }
    g.horizon = dmax(g.gap, g.dh);
    Variant v;
    warp_group_from_anchor(P, av, g, v, ga, Sc, min_slot, ctime, ccnt, i);
    if (v.valid && v.S <= Sc && !v.dues_done) {
      // no anchor due pass: walk the members for this group (lanes in lockstep)
      int64_t late = 0, dues = 0;
      int fail = 0, spill = 0;
      for (int base = 0; base < D.n; base += 32) {
        const int k = base + lane_id();
        Member m;
        m.valid = false;
        if (k < D.n) {
          m.rem = av.rm[k];
          m.valid = m.rem > 0;
          m.phase = av.ph[k];
          m.backlog = av.bl[k];
          m.tier = D.tier[k];
        }
        member_dues_warp(P, m, g, ga.ends, v.S, v.inc != 0, ga.nx, late, dues, fail, spill);
      }
      late = warp_sum(late);
      dues = warp_sum(dues);
      v.Lx = late;
      v.Dx = late + dues;
      v.exact_fail = warp_or(fail);
      v.spill = warp_or(spill);
      v.dues_done = 1;
    }
    __syncwarp();
    // packed form for the DP's thread-per-key placement (thread_place_budget)
    if (v.valid && v.S <= Sc && L <= 4) {
      int big = 0;
      for (int s = lane_id(); s < v.S; s += 32) {
        uint32_t pk = 0;
        for (int l = 0; l < L; ++l) {
          const int32_t h = ga.hc[l * v.S + s];
          if (h > 255) big = 1;
          pk |= (uint32_t)(h & 0xff) << (8 * l);
        }
        ga.hcp[s] = pk;
        ga.cnx[s] = ga.cap[s] - ga.nx[s];
      }
      v.packed = warp_or(big) ? 0 : 1;
    }
    __syncwarp();
    if (lane_id() == 0) { H->g = g; H->v = v; H->j = j; }
  }
}


// try_insert's closed form for one bucket of n <= 64 candidates held by a warp
// (lane r: members r and 32 + r; cn = candidate index * 256 + n_admitted): member
// x is rejected iff an EARLIER candidate y weakly dominates it, unless they are
// equal in (value, memory, budget) and y admits fewer; pm[k] collects the LATER
// candidates that weakly dominate member k (it is pruned iff one is accepted).
template <int K, typename TV, typename TM>
__device__ __forceinline__ void bucket_pair_tests(int n, const int (&cn)[2], const TV (&v)[2], const TM (&m)[2],
                                                  const TM (&p)[2], bool (&acc)[2], uint64_t (&pm)[2]) {
  for (int y = 0; y < n; ++y) {
    const int src = y & 31;
    const bool hi = K > 1 && y >= 32;  // warp-uniform
    const int ycn = __shfl_sync(0xffffffffu, hi ? cn[1] : cn[0], src);
    const TV yv = __shfl_sync(0xffffffffu, hi ? v[1] : v[0], src);
    const TM ym = __shfl_sync(0xffffffffu, hi ? m[1] : m[0], src);
    const TM yp = __shfl_sync(0xffffffffu, hi ? p[1] : p[0], src);
    const int yc = ycn >> 8;
#pragma unroll
    for (int k = 0; k < K; ++k) {  // predicated, no branches
      const int c = cn[k] >> 8;
      const bool w = (yv >= v[k]) & (ym <= m[k]) & (yp >= p[k]);
      const bool equal = (yv == v[k]) & (ym == m[k]) & (yp == p[k]);
      const bool rej = w & (yc < c) & (!equal | ((ycn & 255) >= (cn[k] & 255)));
      acc[k] = acc[k] & !rej;
      pm[k] |= (uint64_t)(w & (yc > c)) << y;
    }
  }
}

#ifndef SLOS_DP_MIN_BLOCKS
#define SLOS_DP_MIN_BLOCKS 4
#endif
// NT threads per CTA, chain levels up to MAXC. dp_kernel is the 256-thread form;
// dp_kernel_small (64 threads, 16 CTAs per SM) takes instances whose levels are a
// few dozen candidates (the C5 sweep family): the DP is a level-sequential latency
// chain, so throughput follows the instances resident per SM, not threads per instance.
template <int NT, int MINB, int MAXC>
__device__ __forceinline__ void dp_body(const DpParams& prm) {
  constexpr int kDpThreads = NT;
  constexpr int kDpWarps = NT / 32;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ PlannerDev sP;
  __shared__ InstDev sI;
  __shared__ int64_t lvl_off[MAXC + 2];
  __shared__ int32_t lvl_cnt[MAXC + 2];
  __shared__ int32_t lvl_boff[MAXC + 2];  // per level: first surviving-bucket slot
  __shared__ int32_t lvl_nsb[MAXC + 2];   // per level: surviving buckets
  __shared__ int32_t s_pre[MAXC + 2];     // candidate prefix over source levels
  __shared__ int32_t s_kpre[MAXC + 2];    // fresh-key prefix over source levels
  __shared__ uint8_t s_sh[MAXC + 2];      // source level's pair is memo-shared
  __shared__ int64_t s_wsum[kDpWarps + 1];
  __shared__ unsigned long long s_ctr[5];
  __shared__ int s_err, s_n_new, s_n_used, s_ovf, s_nb, s_best, s_nw, s_bovf, s_anysh, s_nsb, s_bkinit;
  __shared__ __align__(8) uint64_t s_mbar;  // completion of a level's record staging (TMA bulk copies)

  const BatchArgs& A = prm.a;
  const int tid = threadIdx.x;
  const int inst = A.order[prm.blk0 + blockIdx.x];
  OutHdr* out = &A.out[inst];
  block_copy_struct(sI, A.inst[inst], tid, kDpThreads);  // 8-byte words, every thread
  block_copy_struct(sP, A.planners[A.inst[inst].planner], tid, kDpThreads);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_mbar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // visible to the async proxy
    s_err = 0;
    s_ovf = 0;
    s_n_used = 0;
    s_bkinit = 0;
    for (int k = 0; k < 5; ++k) s_ctr[k] = 0;
  }
  __syncthreads();
  const PlannerDev& P = sP;
  const InstDev& I = sI;
  const int N = I.N;
  const int L = P.L;
  const double min_slot = plan_predict(P, 1, 0);  // BatchPlanner::min_slot_s
  const double pull = min_slot;

  // ---- dynamic smem: chain, decoders, warp scratch ----
  // The chain's request descriptors (deadline, prefill, memory, value, suffix budget,
  // tier, forced, floor: N + 1 entries each, 16-byte aligned slices padded to 4
  // entries by the host) arrive by TMA bulk copies on the staging mbarrier.
  unsigned char* p = dsm;
  const uint32_t b8 = (uint32_t)((8 * (N + 1) + 15) & ~15), b4 = (uint32_t)((4 * (N + 1) + 15) & ~15);
  double* ch_dl = (double*)p; p += b8;
  int64_t* ch_pf = (int64_t*)p; p += b8;
  int64_t* ch_mm = (int64_t*)p; p += b8;
  double* ch_vl = (double*)p; p += b8;
  int64_t* ch_sf = (int64_t*)p; p += b8;
  int32_t* ch_tr = (int32_t*)p; p += b4;
  int32_t* ch_fc = (int32_t*)p; p += b4;
  int32_t* ch_fl = (int32_t*)p; p += b4;
  if (tid == 0) {
    const uint32_t mb = smem_u32(&s_mbar);
    const int64_t o = I.off_chain;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(5 * b8 + 3 * b4) : "memory");
    auto bulk = [&](void* dst, const void* src, uint32_t bytes) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(dst)), "l"(src), "r"(bytes), "r"(mb)
                   : "memory");
    };
    bulk(ch_dl, A.ch_deadline + o, b8);
    bulk(ch_pf, A.ch_prefill + o, b8);
    bulk(ch_mm, A.ch_memory + o, b8);
    bulk(ch_vl, A.ch_value + o, b8);
    bulk(ch_sf, A.ch_suffix + o, b8);
    bulk(ch_tr, A.ch_tier + o, b4);
    bulk(ch_fc, A.ch_forced + o, b4);
    bulk(ch_fl, A.ch_floor + o, b4);
  }
  // decoders: only the private-variant / speculative warp path reads them
  DecView D;
  D.n = I.have_running_decode ? I.n_dec : 0;
  if (I.n_dec <= prm.dec_smem_max) {
    double* dn = (double*)p; p += sizeof(double) * I.n_dec;
    int64_t* db = (int64_t*)p; p += sizeof(int64_t) * I.n_dec;
    int64_t* dr = (int64_t*)p; p += sizeof(int64_t) * I.n_dec;
    int32_t* dt = (int32_t*)p; p += sizeof(int32_t) * I.n_dec;
    p = (unsigned char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    for (int k = tid; k < I.n_dec; k += kDpThreads) {
      dn[k] = A.dec_next[I.off_dec + k];
      db[k] = A.dec_backlog[I.off_dec + k];
      dr[k] = A.dec_rem[I.off_dec + k];
      dt[k] = A.dec_tier[I.off_dec + k];
    }
    D.next = dn; D.backlog = db; D.rem = dr; D.tier = dt;
  } else {
    D.next = A.dec_next + I.off_dec;
    D.backlog = A.dec_backlog + I.off_dec;
    D.rem = A.dec_rem + I.off_dec;
    D.tier = A.dec_tier + I.off_dec;
  }
  // per-warp scratch for the rare private-variant / speculative paths (global);
  // the placement temporaries live in shared memory
  // (slot = launch-order position: CTAs of concurrent launches never share one)
  unsigned char* wbase =
      prm.wscr_global + ((size_t)(prm.blk0 + blockIdx.x) * prm.wscr_warps + warp_id()) * prm.wscr_stride;
  WarpScr W = warp_scr_carve(wbase, prm.Sc, prm.Lmax);
  W.tmp = (int64_t*)p + (size_t)warp_id() * prm.Sc;
  p += sizeof(int64_t) * (size_t)prm.Sc * kDpWarps;
  p = (unsigned char*)(((uintptr_t)p + 127) & ~(uintptr_t)127);
  unsigned char* ovl = p;  // the level's candidate states
  p += prm.overlay_bytes;
  p = (unsigned char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
  const int Tsm = prm.Tsm;
  int32_t* k_src = (int32_t*)p; p += 4 * (size_t)Tsm;
  int32_t* k_j = (int32_t*)p; p += 4 * (size_t)Tsm;
  int32_t* k_me = (int32_t*)p; p += 4 * (size_t)Tsm;
  int32_t* k_new = (int32_t*)p; p += 4 * (size_t)Tsm;
  int32_t* k_grp = (int32_t*)p; p += 4 * (size_t)Tsm;  // direct instances: bucket sizes of a level
  // direct count-vector -> bucket table (instances whose count space is small)
  int32_t* dtab = (int32_t*)p; p += 4 * (size_t)prm.dtab;
  for (int x = tid; x < prm.dtab; x += kDpThreads) dtab[x] = -1;
  // overlay layout: 8-byte arrays first
  uint64_t* o_cn = (uint64_t*)ovl;
  int64_t* o_mm = (int64_t*)(ovl + 8 * (size_t)Tsm);
  int64_t* o_pb = (int64_t*)(ovl + 16 * (size_t)Tsm);
  double* o_vl = (double*)(ovl + 24 * (size_t)Tsm);
  uint64_t* o_bkey = (uint64_t*)(ovl + 32 * (size_t)Tsm);           // 2*Tsm
  int32_t* o_na = (int32_t*)(ovl + 48 * (size_t)Tsm);
  int32_t* o_fl = (int32_t*)(ovl + 52 * (size_t)Tsm);
  int32_t* o_bk = (int32_t*)(ovl + 56 * (size_t)Tsm);
  int32_t* o_aux = (int32_t*)(ovl + 60 * (size_t)Tsm);
  int32_t* o_lst = (int32_t*)(ovl + 64 * (size_t)Tsm);
  int32_t* o_bval = (int32_t*)(ovl + 68 * (size_t)Tsm);              // 2*Tsm

  // ---- scratch slices ----
  uint64_t* Sc_ = A.s_counts + I.off_surv;
  int64_t* Sm_ = A.s_mem + I.off_surv;
  int64_t* Sp_ = A.s_pb + I.off_surv;
  double* Sv_ = A.s_value + I.off_surv;
  int32_t* Sn_ = A.s_nadm + I.off_surv;
  int32_t* Spar = A.s_parent + I.off_surv;
  int32_t* Sar = A.s_arena + I.off_surv;
  int32_t* Sit = A.s_level + I.off_surv;
  int32_t* Ssb = A.s_sb + I.off_surv;
  uint64_t* Bc = A.s_bcnt + I.off_surv;
  int64_t* Kv = A.k_val + I.off_cand;
  MemoEnt* Memo = A.memo + I.off_memo;
  const uint8_t* PS = A.pair_shared + I.off_pair;
  unsigned char* GR = A.groups + I.off_group;
  const int64_t capC = I.cap_cand;

  if (I.has_shared) {  // the instance's memo table starts empty (state 0), 8-byte words
    uint64_t* mw = (uint64_t*)Memo;
    const int64_t nw = I.cap_memo * (int64_t)(sizeof(MemoEnt) / 8);
    for (int64_t x = tid; x < nw; x += kDpThreads) mw[x] = 0ull;
  }
  if (tid == 0) {
    Sc_[0] = 0; Sm_[0] = 0; Sp_[0] = 0; Sv_[0] = 0.0; Sn_[0] = 0; Spar[0] = -1; Sar[0] = 0; Sit[0] = -1;
    Ssb[0] = 0; Bc[0] = 0;
    lvl_off[0] = 0;
    lvl_cnt[0] = 1;
    lvl_boff[0] = 0;
    lvl_nsb[0] = 1;
  }
  __syncthreads();
  // arena bookkeeping: block-uniform, advanced identically by every thread
  int64_t r_next_free = 1, r_arena_next = 1, r_bnext = 1;

  long long ph_t0_ = clock64();
  const long long ph_start_ = ph_t0_;
  {  // the chain descriptors have landed (phase 0 of the staging barrier)
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(smem_u32(&s_mbar)), "r"(0u)
                   : "memory");
  }
  uint32_t mb_phase = 1;  // parity of the staging barrier's current phase (levels)
  SLOS_PHASE(0);  // 0: instance load / setup
  for (int i = 0; i < N && !s_err; ++i) {
    const int jlo = ch_fl[i];
    const int nlev = i - jlo;  // source levels jlo+1 .. i (anchor j = level - 1)
    if (warp_id() == 0) {  // level prefixes, lanes over source levels
      const int lane = lane_id();
      int acc = 0, kacc = 0;
      unsigned anysh = 0;
      for (int base = 0; base < nlev; base += 32) {
        const int k = base + lane;
        int cnt = 0, kc = 0;
        if (k < nlev) {
          const int lv = jlo + 1 + k;
          const uint8_t sh = PS[pair_index(N, lv, i)];
          s_sh[k] = sh;
          cnt = lvl_cnt[lv];
          kc = sh ? 0 : lvl_nsb[lv];
          anysh |= sh ? 1u : 0u;
        }
        const int ic = warp_incl_scan(cnt), ik = warp_incl_scan(kc);
        if (k < nlev) { s_pre[k] = acc + ic - cnt; s_kpre[k] = kacc + ik - kc; }
        acc += __shfl_sync(0xffffffffu, ic, 31);
        kacc += __shfl_sync(0xffffffffu, ik, 31);
      }
      anysh = __reduce_or_sync(0xffffffffu, anysh);
      if (lane == 0) {
        s_pre[nlev] = acc;
        s_kpre[nlev] = kacc;
        s_anysh = anysh != 0;
        s_n_new = 0;
        s_nb = 0;
        s_nw = 0;
        if (acc > Tsm && acc > capC) { s_err = SLOS_ERR_CAPACITY; out->need_cand = acc; }
        else if (kacc > capC) { s_err = SLOS_ERR_CAPACITY; out->need_cand = kacc; }
      }
    }
    __syncthreads();
    if (s_err) break;
    const int T = s_pre[nlev];
    const int KF = s_kpre[nlev];
    // level arrays: shared memory when the level fits, else the HBM slice
    const bool sm = T <= Tsm;
    int32_t* Csrc = sm ? k_src : A.c_src + I.off_cand;
    int32_t* Cj = sm ? k_j : A.c_j + I.off_cand;
    int32_t* Cme = sm ? k_me : A.c_memo + I.off_cand;
    int32_t* X0 = sm ? k_new : A.c_pos + I.off_cand;
    uint64_t* Ccn = sm ? o_cn : A.c_counts + I.off_cand;
    int64_t* Cmm = sm ? o_mm : A.c_mem + I.off_cand;
    int64_t* Cpb = sm ? o_pb : A.c_pb + I.off_cand;
    double* Cvl = sm ? o_vl : A.c_value + I.off_cand;
    int32_t* Cna = sm ? o_na : A.c_nadm + I.off_cand;
    int32_t* Cfl = sm ? o_fl : A.c_flag + I.off_cand;
    int32_t* Cbk = sm ? o_bk : A.c_bucket + I.off_cand;
    int32_t* Caux = sm ? o_aux : A.c_aux + I.off_cand;
    int32_t* Blst = sm ? o_lst : A.c_pos + I.off_cand;
    uint64_t* Bkey = sm ? o_bkey : A.c_bkey + 2 * I.off_cand;
    int32_t* Bval = sm ? o_bval : A.c_bval + 2 * I.off_cand;
    const int64_t capB = sm ? 2 * (int64_t)Tsm : 2 * capC;
    const bool direct = I.direct != 0;
    int32_t* Bcnt = sm ? k_grp : A.c_bval + 2 * I.off_cand;                   // direct: bucket sizes
    int32_t* hsbA = sm ? k_new : (int32_t*)(A.k_val + I.off_cand);           // per bucket: keeps a survivor
    if (tid == 0) s_ctr[0] += (unsigned long long)T;
    const double t_i = ch_dl[i];
    // source level index of candidate c: last k with s_pre[k] <= c
    auto level_of = [&](int c) {
      int lo = 0, hi = nlev - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (s_pre[mid] <= c) lo = mid; else hi = mid - 1;
      }
      return lo;
    };
    // the level's gap group records (pairs (jlo .. i-1, i), contiguous) staged into
    // the candidate-state overlay, which is free until step 4
    // (header + cap/nx/hc of each record; the slot ends are not read by E3)
    const bool staged = (size_t)nlev * prm.grec_stage <= prm.overlay_bytes;
    const unsigned char* GRl = GR + (size_t)pair_index(N, jlo + 1, i) * prm.grec_stride;
    if (staged && tid == 0) {
      // one TMA bulk copy per record (global -> shared, completion on s_mbar); it runs
      // under the candidate enumeration below, which does not read the records. The
      // overlay's last generic-proxy use is behind the level barrier above.
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t mb = smem_u32(&s_mbar);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                   "r"((uint32_t)((size_t)nlev * prm.grec_stage))
                   : "memory");
      for (int r = 0; r < nlev; ++r)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(ovl + (size_t)r * prm.grec_stage)),
                     "l"(GRl + (size_t)r * prm.grec_stride), "r"((uint32_t)prm.grec_stage), "r"(mb)
                     : "memory");
    }
    auto rec_of = [&](int j) -> const unsigned char* {
      return staged ? (const unsigned char*)ovl + (size_t)(j - jlo) * prm.grec_stage
                    : GRl + (size_t)(j - jlo) * prm.grec_stride;
    };
    // a group's variant arrays: the staged prefix (cnx, hcp, cap) and, from the
    // HBM record, the unpacked nx / hc / ends
    auto var_of = [&](int j) -> GroupVar {
      GroupVar g = group_var_carve((unsigned char*)GRl + (size_t)(j - jlo) * prm.grec_stride + prm.grec_hdr,
                                   prm.Sc, L);
      if (staged) {
        const GroupVar st = group_var_carve((unsigned char*)rec_of(j) + prm.grec_hdr, prm.Sc, L);
        g.cnx = st.cnx;
        g.hcp = st.hcp;
        g.cap = st.cap;
      }
      return g;
    };
    // ---- 1: memo keys. A pair whose key (a_us, raw_us) is unique to it (host
    // flag) has one key per surviving source bucket: key s_kpre[k] + bucket id,
    // no table. Shared pairs use the instance's hash memo, whose first-inserted
    // candidate decides under µs key collisions (dp_scheduler.cpp:423-435). ----
    for (int c = tid; c < T; c += kDpThreads) {
      if (direct) Bcnt[c] = 0;  // step 5's bucket sizes (no other use of the array this level)
      const int k = level_of(c);
      const int lv = jlo + 1 + k;
      const int src = (int)(lvl_off[lv] + (c - s_pre[k]));
      Csrc[c] = src;
      if (!s_sh[k]) {  // fresh pair: the key is (level, surviving source bucket)
        Cme[c] = -(s_kpre[k] + Ssb[src]) - 1;
        continue;
      }
      const int j = lv - 1;
      const double a = (j < 0) ? I.now : ch_dl[j];
      const double raw = dmax(0.0, t_i - a);
      uint64_t k0, k1;
      if (I.have_running_decode) {
        k0 = (uint64_t)llround(a * 1e6);
        k1 = (uint64_t)llround(raw * 1e6);
      } else {
        const double gap = quantize_gap(quantize_gap(raw));
        k0 = 0xFFFFFFFFFFFFFFFFULL;
        k1 = (uint64_t)llround(gap * 1000.0);
      }
      Cme[c] = memo_find_insert(Memo, I.cap_memo, k0, k1, Sc_[src], c, X0, &s_n_new, &s_n_used, &s_ovf);
    }
    if (staged) {  // the level's records have landed (every thread waits: no copy outlives the level)
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_u32(&s_mbar)), "r"(mb_phase)
                     : "memory");
      mb_phase ^= 1u;
    }
    __syncthreads();
    if (s_ovf) {
      if (tid == 0) { s_err = SLOS_ERR_CAPACITY; out->need_memo = 2 * I.cap_memo; }
      __syncthreads();
      break;
    }
    const int n_new = s_n_new;
    const int nkeys = KF + n_new;
    if (tid == 0) s_ctr[1] += (unsigned long long)nkeys;
    SLOS_PHASE(3);  // 3: candidate enumeration + memo keys
    // key q -> (anchor j, counts, result slot)
    auto key_of = [&](int q, int& j, uint64_t& cw, MemoEnt*& e) {
      if (q < KF) {
        int lo = 0, hi = nlev - 1;  // last k with s_kpre[k] <= q
        while (lo < hi) {
          const int mid = (lo + hi + 1) / 2;
          if (s_kpre[mid] <= q) lo = mid; else hi = mid - 1;
        }
        const int lv = jlo + 1 + lo;
        j = lv - 1;
        cw = Bc[lvl_boff[lv] + (q - s_kpre[lo])];
        e = nullptr;
      } else {
        e = &Memo[X0[q - KF]];
        cw = e->k2;
        j = jlo + level_of(e->first);
      }
    };
    // ---- 2: E3a, lanes over keys (thread_eval_counts on the pair's group record);
    // keys that need a private variant or the speculative branch go to E3b ----
    {
      unsigned long long td = 0, tsl = 0;
      for (int q = tid; q < nkeys; q += kDpThreads) {
        int j;
        uint64_t cw;
        MemoEnt* e;
        const long long dbg0 = prm.phase_cycles ? clock64() : 0;
        key_of(q, j, cw, e);
        const unsigned char* rec = rec_of(j);
        const GroupHdr& H = *(const GroupHdr*)rec;
        const GroupVar ga = var_of(j);
        int64_t cv[kMaxTiers];
#pragma unroll
        for (int l = 0; l < kMaxTiers; ++l) cv[l] = l < L ? pack_get(cw, l) : 0;
        EvalOut r;
        const long long dbg1 = prm.phase_cycles ? clock64() : 0;
        const int fb = thread_eval_counts(P, H.g, H.v, ga, prm.Sc, cv, min_slot, r);
        if (prm.phase_cycles) {
          const long long dbg2 = clock64();
          atomicAdd(&prm.phase_cycles[24], (unsigned long long)(dbg2 - dbg1));
          atomicAdd(&prm.phase_cycles[25], 1ull);
          atomicMax(&prm.phase_cycles[26], (unsigned long long)(dbg2 - dbg1));
          atomicAdd(&prm.phase_cycles[27], (unsigned long long)(dbg1 - dbg0));
          if (r.dues == 0) atomicAdd(&prm.phase_cycles[28], 1ull);
          if (H.v.Lx > 0) atomicAdd(&prm.phase_cycles[29], 1ull);
        }
        if (fb) {
          Cj[atomicAdd(&s_nw, 1)] = q;
          continue;
        }
        td += (unsigned long long)r.dues;
        tsl += (unsigned long long)r.slots;
        if (r.status) {
          atomicCAS(&s_err, 0, r.status);
          if (r.status == SLOS_ERR_CAPACITY) out->need_work = 2 * prm.Sc;
          continue;
        }
        if (e) { e->has = r.has ? 1 : 0; e->val = r.budget; }
        else Kv[q] = r.has ? r.budget : -1;
      }
      td = warp_sum(td);
      tsl = warp_sum(tsl);
      if (lane_id() == 0 && (td | tsl)) {
        atomicAdd(&s_ctr[2], td);
        atomicAdd(&s_ctr[3], tsl);
      }
    }
    __syncthreads();
    if (s_nw) {  // ---- E3b: one warp per queued key ----
      const int nw = s_nw;
      unsigned long long wd = 0, wsl = 0;
      for (int x = warp_id(); x < nw; x += kDpWarps) {
        if (s_err) break;
        const int q = Cj[x];
        int j;
        uint64_t cw;
        MemoEnt* e;
        key_of(q, j, cw, e);
        const unsigned char* rec = rec_of(j);
        const GroupHdr& H = *(const GroupHdr*)rec;
        const GroupVar ga = var_of(j);
        int64_t cv[kMaxTiers];
#pragma unroll
        for (int l = 0; l < kMaxTiers; ++l) cv[l] = l < L ? pack_get(cw, l) : 0;
        int spill = 0;
        const EvalOut r = warp_eval_counts(P, D, H.g, H.v, ga, prm.Sc, W, cv, min_slot, &spill);
        wd += (unsigned long long)r.dues;
        wsl += (unsigned long long)r.slots;
        if (r.status) {
          if (lane_id() == 0) {
            atomicCAS(&s_err, 0, r.status);
            if (r.status == SLOS_ERR_CAPACITY) out->need_work = 2 * prm.Sc;
          }
          break;
        }
        if (lane_id() == 0) {
          if (e) { e->has = r.has ? 1 : 0; e->val = r.budget; }
          else Kv[q] = r.has ? r.budget : -1;
        }
      }
      if (lane_id() == 0 && (wd | wsl)) {
        atomicAdd(&s_ctr[2], wd);
        atomicAdd(&s_ctr[3], wsl);
      }
      __syncthreads();
    }
    SLOS_PHASE(7);  // 7: E3 placements
    if (s_err) break;
    for (int q = tid; q < n_new; q += kDpThreads) Memo[X0[q]].state = 3;
    // ---- 4: candidate states ----
    const int tier_i = ch_tr[i];
    const bool forced = ch_fc[i] != 0;
    for (int c = tid; c < T; c += kDpThreads) {
      if (!direct) Cj[c] = 0;  // bucket sizes of step 5 (the E3b key list is consumed)
      const int src = Csrc[c];
      const int me = Cme[c];
      bool has;
      int64_t val;
      if (me >= 0) {
        const MemoEnt* e = &Memo[me];
        has = e->has != 0;
        val = e->val;
      } else {
        val = Kv[-me - 1];
        has = val >= 0;
      }
      int flag = 0;
      uint64_t nc = 0;
      if (has) {
        const int64_t avail = Sp_[src] + val;
        if (avail >= ch_pf[i]) {
          nc = pack_add(Sc_[src], tier_i);
          if (pack_get(nc, tier_i) > 250) atomicCAS(&s_err, 0, SLOS_ERR_INTERNAL_INCONSISTENCY);
          int64_t mem = Sm_[src];
          bool ok = true;
          if (!forced) {
            mem = mem + ch_mm[i];
            if (mem > I.mem_budget) ok = false;
          }
          if (ok) {
            flag = 1;
            Ccn[c] = nc;
            Cmm[c] = mem;
            Cpb[c] = imin(avail - ch_pf[i], ch_sf[i + 1]);
            Cvl[c] = Sv_[src] + (forced ? 0.0 : ch_vl[i]);
            Cna[c] = Sn_[src] + (forced ? 0 : 1);
          }
        }
      }
      Cfl[c] = flag;
      if (direct) {  // ---- 5 (fused): count vector -> dense index -> bucket id (shared-memory 32-bit atomics)
        int b = -1;
        if (flag) {
          int idx = 0;
#pragma unroll
          for (int l = 0; l < kMaxTiers; ++l) if (l < L) idx += (int)pack_get(nc, l) * I.dstride[l];
          int v = atomicCAS(&dtab[idx], -1, -2);
          if (v == -1) {
            b = atomicAdd(&s_nb, 1);
            Caux[b] = idx;
            atomicExch(&dtab[idx], b);
          } else {
            while (v < 0) v = atomicAdd(&dtab[idx], 0);
            b = v;
          }
          atomicAdd(&Bcnt[b], 1);  // bucket size (Bcnt zeroed in step 1)
        }
        Cbk[c] = b;
      }
    }
    if (!direct) {
      if (sm) {  // fresh level-local bucket table
        for (int x = tid; x < capB; x += kDpThreads) { Bkey[x] = 0ull; Bval[x] = -1; }
      } else if (!s_bkinit) {  // first HBM level: clear the instance's hash once
        for (int64_t x = tid; x < capB; x += kDpThreads) { Bkey[x] = 0ull; Bval[x] = -1; }
      }
      __syncthreads();
      if (!sm && tid == 0) s_bkinit = 1;  // later HBM levels reset the slots they claim
      SLOS_PHASE(8);  // 8: candidate states
      // ---- 5: Pareto buckets (hash of the count vector) ----
      for (int c = tid; c < T; c += kDpThreads) {
        int b = -1;
        if (Cfl[c] & 1) {
          const uint64_t key = Ccn[c];
          uint64_t h = mix64(key) & (uint64_t)(capB - 1);
          for (;;) {
            const unsigned long long old = atomicCAS((unsigned long long*)&Bkey[h], 0ull,
                                                     (unsigned long long)key);
            if (old == 0ull) {
              b = atomicAdd(&s_nb, 1);
              Caux[b] = (int32_t)h;
              atomicExch(&Bval[h], b);
              break;
            }
            if (old == key) {
              int x;
              do { x = atomicAdd(&Bval[h], 0); } while (x < 0);
              b = x;
              break;
            }
            h = (h + 1) & (uint64_t)(capB - 1);
          }
          atomicAdd(&Cj[b], 1);  // bucket size (Cj zeroed in step 4)
        }
        Cbk[c] = b;
      }
    }
    __syncthreads();
    if (s_err) break;
    const int NB = s_nb;
    for (int b = tid; b < NB; b += kDpThreads) hsbA[b] = 0;  // read after the next barrier
    SLOS_PHASE(12);  // 12 (sub of buckets): bucket hashing
    // try_insert replay (dp_scheduler.cpp:445-465). Fast path: one warp per bucket
    // finds its candidates in creation order by ballots over the level and keeps
    // the bucket's Pareto frontier in registers (lane r, slot k holds frontier
    // entry 32k+r; up to kFront entries); dominance tests are warp votes. The
    // frontier is a set: rejection is an any-vote and pruning a per-entry test, so
    // its order never matters. Big levels or frontiers take the list path below.
    // Integral values make the eps tests exact, so dominance is transitive and the
    // sequential replay has a closed form: c is accepted iff no EARLIER candidate of
    // its bucket rejects it, and an accepted c is pruned iff a LATER accepted
    // candidate of its bucket weakly dominates it: decided pairwise, one thread per
    // candidate over its bucket's list.
    // Why: let W(x,y) = x.v>=y.v && x.mem<=y.mem && x.pb>=y.pb (transitive when the
    // comparisons are exact) and rej(x,y) = W(x,y) && (x != y in (v,mem,pb) ||
    // x.n >= y.n). If an earlier y rejects c but is not on the frontier when c
    // arrives, y was rejected by, or later pruned by, some frontier member f with
    // W(f,y); then W(f,c), and if f equals c in (v,mem,pb) so do y and c, with
    // f.n >= y.n >= c.n (rejection) or f.n > y.n (f was accepted while y was on the
    // frontier). By induction some member on c's frontier rejects c. Conversely a
    // rejecting frontier member is an earlier candidate. Pruning removes exactly
    // the accepted entries weakly dominated by a later accepted candidate.
    const bool pairwise = I.values_integral != 0;
    bool fastB = !pairwise && NB <= 64;
    if (pairwise) {
      // unordered bucket lists (counting sort without stability: "earlier" is the
      // candidate index itself)
      int32_t* cntB = direct ? Bcnt : Cj;   // bucket sizes, counted while the buckets were assigned
      int32_t* offB = Cme;  // memo slots are no longer needed after step 4
      if (warp_id() == 0) {  // bucket offsets: one warp (NB is small), sizes reset for the scatter
        const int lane = lane_id();
        int carry = 0;
        for (int base = 0; base < NB; base += 32) {
          const int b = base + lane;
          const int x = b < NB ? cntB[b] : 0;
          const int inc = warp_incl_scan(x);
          if (b < NB) { offB[b] = carry + inc - x; cntB[b] = 0; }
          carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) s_bovf = 0;  // reused below: a bucket of more than 32 candidates exists
      }
      __syncthreads();
      for (int c = tid; c < T; c += kDpThreads) {
        const int b = Cbk[c];
        if (b >= 0) {
          const int pos = atomicAdd(&cntB[b], 1);
          Blst[offB[b] + pos] = c;
          if (pos == 64) s_bovf = 1;
        }
      }
      __syncthreads();
      // buckets of <= 64 candidates: one warp each, members in registers (lane r
      // holds members r and 32 + r), every pair tested once over shuffles (no
      // memory traffic in the loop); 32-bit operands whenever the bucket's values,
      // memory and budgets fit (4 shuffles per member instead of 7)
      {
        const int lane = lane_id();
        for (int b = warp_id(); b < NB; b += kDpWarps) {
          const int n = cntB[b];
          if (n > 64) continue;
          int cc[2] = {-1, -1}, cn[2] = {-1, -1};
          double xv[2] = {0.0, 0.0};
          int64_t xm[2] = {0, 0}, xp[2] = {0, 0};
          bool fit = true;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (32 * k + lane < n) {
              const int c = Blst[offB[b] + 32 * k + lane];
              cc[k] = c;
              xv[k] = Cvl[c]; xm[k] = Cmm[c]; xp[k] = Cpb[c];
              cn[k] = c * 256 + Cna[c];  // candidate index (< 2^23) and n_admitted (<= 250)
              fit = fit && fabs(xv[k]) < 2147483647.0 && xm[k] >= INT32_MIN && xm[k] <= INT32_MAX &&
                    xp[k] >= INT32_MIN && xp[k] <= INT32_MAX;
            }
          }
          bool acc[2] = {true, true};
          uint64_t pm[2] = {0ull, 0ull};
          if (__all_sync(0xffffffffu, fit)) {
            const int v32[2] = {(int)xv[0], (int)xv[1]};
            const int m32[2] = {(int)xm[0], (int)xm[1]};
            const int p32[2] = {(int)xp[0], (int)xp[1]};
            if (n <= 32) bucket_pair_tests<1>(n, cn, v32, m32, p32, acc, pm);
            else bucket_pair_tests<2>(n, cn, v32, m32, p32, acc, pm);
          } else {
            bucket_pair_tests<2>(n, cn, xv, xm, xp, acc, pm);
          }
          const uint64_t Am = (uint64_t)__ballot_sync(0xffffffffu, acc[0] && lane < n) |
                              ((uint64_t)__ballot_sync(0xffffffffu, acc[1] && 32 + lane < n) << 32);
          bool surv = false;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (32 * k + lane < n && acc[k]) {
              const bool pr = (pm[k] & Am) != 0;
              Cfl[cc[k]] |= pr ? 6 : 2;
              surv = surv || !pr;
            }
          }
          if (__any_sync(0xffffffffu, surv) && lane == 0) hsbA[b] = 1;
        }
      }
      if (s_bovf) {  // larger buckets: one thread per candidate over the bucket list
      for (int c = tid; c < T; c += kDpThreads) {
        const int b = Cbk[c];
        if (b < 0 || cntB[b] <= 64) continue;
        const double xv = Cvl[c];
        const int64_t xm = Cmm[c], xp = Cpb[c];
        const int xn = Cna[c];
        const int32_t* lst = Blst + offB[b];
        const int n = cntB[b];
        bool acc = true;
        for (int q = 0; q < n; ++q) {
          const int y = lst[q];
          if (y >= c) continue;
          const double yv = Cvl[y];
          const int64_t ym = Cmm[y], yp = Cpb[y];
          if (yv >= xv && ym <= xm && yp >= xp) {
            const bool equal = yv == xv && ym == xm && yp == xp;
            if (!equal || Cna[y] >= xn) { acc = false; break; }
          }
        }
        if (acc) Cfl[c] |= 2;
      }
      __syncthreads();
      // pruned marks (bit 4) are held back until every thread has read the accepted
      // marks (bit 2) of its bucket: no thread writes a flag word another reads
      uint32_t pm = 0;
      int it = 0;
      for (int c = tid; c < T; c += kDpThreads, ++it) {
        if (!(Cfl[c] & 2)) continue;
        const int b = Cbk[c];
        if (cntB[b] <= 64) continue;
        const double xv = Cvl[c];
        const int64_t xm = Cmm[c], xp = Cpb[c];
        const int32_t* lst = Blst + offB[b];
        const int n = cntB[b];
        bool pruned = false;
        for (int q = 0; q < n; ++q) {
          const int y = lst[q];
          if (y <= c || !(Cfl[y] & 2)) continue;
          if (Cvl[y] >= xv && Cmm[y] <= xm && Cpb[y] >= xp) {
            if (it < 32) pm |= 1u << it;
            else Cfl[c] |= 4;  // levels beyond 32 x kDpThreads (HBM arrays): bit 2 is never cleared
            pruned = true;
            break;
          }
        }
        if (!pruned) hsbA[b] = 1;
      }
      __syncthreads();
      for (int k = 0; pm; ++k, pm >>= 1)
        if (pm & 1u) Cfl[tid + k * kDpThreads] |= 4;
      }
    }
    if (fastB) {
      if (tid == 0) s_bovf = 0;
      __syncthreads();
      constexpr int kFront = 4;
      const int lane = lane_id();
      for (int b = warp_id(); b < NB; b += kDpWarps) {
        double fv[kFront];
        int64_t fm[kFront], fp[kFront];
        int fn[kFront], fc[kFront];
        unsigned A[kFront];
#pragma unroll
        for (int k = 0; k < kFront; ++k) { A[k] = 0u; fv[k] = 0.0; fm[k] = 0; fp[k] = 0; fn[k] = 0; fc[k] = 0; }
        bool ovf = false;
        for (int base = 0; base < T && !ovf; base += 32) {
          const int c = base + lane;
          const bool in = c < T && Cbk[c] == b;
          unsigned mm = __ballot_sync(0xffffffffu, in);
          if (!mm) continue;
          double xv = 0.0;
          int64_t xm = 0, xp = 0;
          int xn = 0;
          if (in) { xv = Cvl[c]; xm = Cmm[c]; xp = Cpb[c]; xn = Cna[c]; }
          while (mm) {
            const int src = __ffs(mm) - 1;
            mm &= mm - 1;
            const double sv = __shfl_sync(0xffffffffu, xv, src);
            const int64_t smm = __shfl_sync(0xffffffffu, xm, src);
            const int64_t spb = __shfl_sync(0xffffffffu, xp, src);
            const int sn = __shfl_sync(0xffffffffu, xn, src);
            bool rj = false;
#pragma unroll
            for (int k = 0; k < kFront; ++k) {
              if ((A[k] >> lane) & 1u) {
                if (fv[k] >= sv - kValueEps && fm[k] <= smm && fp[k] >= spb) {
                  const bool equal = fabs(fv[k] - sv) <= kValueEps && fm[k] == smm && fp[k] == spb;
                  if (!equal || fn[k] >= sn) rj = true;
                }
              }
            }
            if (__any_sync(0xffffffffu, rj)) continue;
#pragma unroll
            for (int k = 0; k < kFront; ++k) {
              bool pr = false;
              if ((A[k] >> lane) & 1u) {
                if (sv >= fv[k] - kValueEps && smm <= fm[k] && spb >= fp[k]) {
                  pr = true;
                  Cfl[fc[k]] |= 4;  // pruned (this lane accepted it earlier)
                }
              }
              A[k] &= ~__ballot_sync(0xffffffffu, pr);
            }
            int ks = -1;
#pragma unroll
            for (int k = kFront - 1; k >= 0; --k) if (A[k] != 0xffffffffu) ks = k;
            if (ks < 0) { ovf = true; break; }
            const int slot = __ffs(~A[ks]) - 1;
#pragma unroll
            for (int k = 0; k < kFront; ++k) {
              if (k == ks) {
                if (lane == slot) {
                  fv[k] = sv; fm[k] = smm; fp[k] = spb; fn[k] = sn; fc[k] = base + src;
                  Cfl[base + src] |= 2;  // accepted
                }
                A[k] |= 1u << slot;
              }
            }
          }
        }
        if (ovf && lane == 0) s_bovf = 1;
      }
      __syncthreads();
      if (s_bovf) {  // some frontier outgrew the registers: redo the level on the list path
        for (int c = tid; c < T; c += kDpThreads) Cfl[c] &= 1;
        fastB = false;
        __syncthreads();
      }
    }
    SLOS_PHASE(13);  // 13 (sub): fast try_insert
    if (!fastB && !pairwise) {
      int32_t* cntB = Cj;   // anchors are no longer needed this level
      int32_t* offB = Cme;  // memo slots are no longer needed after step 4
      for (int b = tid; b < NB; b += kDpThreads) cntB[b] = 0;
      __syncthreads();
      for (int c = tid; c < T; c += kDpThreads)
        if (Cbk[c] >= 0) atomicAdd(&cntB[Cbk[c]], 1);
      __syncthreads();
      {
        int64_t carry = 0;
        for (int base = 0; base < NB; base += kDpThreads) {
          const int b = base + tid;
          const int64_t x = b < NB ? cntB[b] : 0;
          int64_t tot;
          const int64_t ex = block_excl_scan<kDpWarps>(x, s_wsum, &tot);
          if (b < NB) { offB[b] = (int32_t)(carry + ex); cntB[b] = 0; }
          carry += tot;
        }
      }
      __syncthreads();
      // stable multi-split: chunk by chunk, warp by warp, candidate order preserved
      for (int base = 0; base < T; base += kDpThreads) {
        const int c = base + tid;
        const int b = c < T ? Cbk[c] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int lane = lane_id();
        const int rank = __popc(peers & ((1u << lane) - 1));
        const int leader = __ffs(peers) - 1;
        for (int w = 0; w < kDpWarps; ++w) {
          if (warp_id() == w) {
            int basepos = 0;
            if (b >= 0 && lane == leader) {
              basepos = cntB[b];
              cntB[b] = basepos + __popc(peers);
            }
            basepos = __shfl_sync(0xffffffffu, basepos, leader);
            if (b >= 0) Blst[offB[b] + basepos + rank] = c;
          }
          __syncthreads();
        }
      }
      // one warp per bucket: try_insert replay (dp_scheduler.cpp:445-465) in candidate
      // order; the frontier scan of each step is lane-parallel (ballots).
      for (int b = warp_id(); b < NB; b += kDpWarps) {
        int32_t* lst = Blst + offB[b];
        const int n = cntB[b];
        const int lane = lane_id();
        int f = 0;  // frontier lst[0..f)
        for (int q = 0; q < n; ++q) {
          const int c = lst[q];
          const double sv = Cvl[c];
          const int64_t smm = Cmm[c], spb = Cpb[c];
          const int sn = Cna[c];
          bool reject = false;
          for (int r0 = 0; r0 < f && !reject; r0 += 32) {
            bool rj = false;
            if (r0 + lane < f) {
              const int e = lst[r0 + lane];
              if (Cvl[e] >= sv - kValueEps && Cmm[e] <= smm && Cpb[e] >= spb) {
                const bool equal = fabs(Cvl[e] - sv) <= kValueEps && Cmm[e] == smm && Cpb[e] == spb;
                rj = !equal || Cna[e] >= sn;
              }
            }
            reject = __any_sync(0xffffffffu, rj);
          }
          if (reject) continue;
          int wq = 0;
          for (int r0 = 0; r0 < f; r0 += 32) {
            int e = -1;
            bool keep = false;
            if (r0 + lane < f) {
              e = lst[r0 + lane];
              if (sv >= Cvl[e] - kValueEps && smm <= Cmm[e] && spb >= Cpb[e]) Cfl[e] |= 4;  // pruned
              else keep = true;
            }
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            __syncwarp();
            if (keep) lst[wq + __popc(km & ((1u << lane) - 1))] = e;
            wq += __popc(km);
            __syncwarp();
          }
          if (lane == 0) {
            lst[wq] = c;
            Cfl[c] |= 2;  // accepted
          }
          f = wq + 1;
          __syncwarp();
        }
      }
    }
    __syncthreads();
    if (!pairwise) {  // register / list paths: mark the buckets that keep a survivor
      for (int c = tid; c < T; c += kDpThreads) {
        const int fl = Cfl[c];
        if ((fl & 2) && !(fl & 4)) hsbA[Cbk[c]] = 1;
      }
      __syncthreads();
    }
    // reset the bucket-table entries claimed by this level (read again only after
    // the level's last barrier)
    if (direct) {
      for (int b = tid; b < NB; b += kDpThreads) dtab[Caux[b]] = -1;
    } else if (!sm) {
      for (int b = tid; b < NB; b += kDpThreads) {
        Bkey[Caux[b]] = 0ull;
        Bval[Caux[b]] = -1;
      }
    }
    SLOS_PHASE(9);  // 9: Pareto buckets
    // ---- 6: arena ids, survivors and their surviving-bucket ids ----
    {
      const int32_t* hsb = hsbA;  // per bucket: has a survivor -> dense id
      int32_t* sbid = Cme;
      const int lane = lane_id(), w = warp_id();
      if (w == 0) {  // surviving-bucket dense ids: one warp (NB is small)
        int carry = 0;
        for (int base = 0; base < NB; base += 32) {
          const int b = base + lane;
          const int x = b < NB ? hsb[b] : 0;
          const int inc = warp_incl_scan(x);
          if (b < NB) sbid[b] = carry + inc - x;
          carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) s_nsb = carry;
      }
      // accepted / surviving ranks in candidate order: every warp scans a contiguous
      // range (one barrier for the whole level instead of one scan per 256 candidates);
      // packed value: accepted in the low, surviving in the high word
      const int per = (T + kDpWarps - 1) / kDpWarps;
      const int lo = min(T, w * per), hi = min(T, lo + per);
      auto packed = [&](int c) -> int64_t {
        const int fl = c < hi ? Cfl[c] : 0;
        return (int64_t)((fl & 2) ? 1 : 0) | ((int64_t)(((fl & 2) && !(fl & 4)) ? 1 : 0) << 32);
      };
      int64_t wt = 0;
      for (int base = lo; base < hi; base += 32) wt += warp_sum(packed(base + lane));
      if (lane == 0) s_wsum[w] = wt;
      __syncthreads();
      int64_t carry = 0, total = 0;
      for (int x = 0; x < kDpWarps; ++x) {
        if (x < w) carry += s_wsum[x];
        total += s_wsum[x];
      }
      const int64_t bbase = r_bnext;
      const int64_t base_free = r_next_free;
      for (int base = lo; base < hi; base += 32) {
        const int c = base + lane;
        const int64_t v = packed(c);
        const int64_t inc = warp_incl_scan(v);
        const int64_t ex = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
        if (v >> 32) {  // a survivor
          const int64_t dst = base_free + (ex >> 32);
          if (dst < I.cap_surv) {
            const int sb = sbid[Cbk[c]];
            Sc_[dst] = Ccn[c];
            Sm_[dst] = Cmm[c];
            Sp_[dst] = Cpb[c];
            Sv_[dst] = Cvl[c];
            Sn_[dst] = Cna[c];
            Spar[dst] = Csrc[c];
            Sar[dst] = (int32_t)(r_arena_next + (ex & 0xffffffffLL));
            Sit[dst] = i;
            Ssb[dst] = sb;
            Bc[bbase + sb] = Ccn[c];  // every survivor of the bucket writes the same counts
          }
        }
      }
      // level bookkeeping: every thread advances its copies, thread 0 publishes the
      // level's ranges (read after the barrier below)
      const int64_t tot_acc = total & 0xffffffffLL, tot_sv = total >> 32;
      const int nsb = s_nsb;
      r_bnext = bbase + nsb;
      r_next_free = base_free + tot_sv;
      r_arena_next += tot_acc;
      if (tid == 0) {
        lvl_off[i + 1] = base_free;
        lvl_cnt[i + 1] = (int32_t)tot_sv;
        lvl_boff[i + 1] = (int32_t)bbase;
        lvl_nsb[i + 1] = nsb;
        if (r_next_free > I.cap_surv) { s_err = SLOS_ERR_CAPACITY; out->need_surv = 2 * r_next_free; }
      }
    }
    __syncthreads();
    SLOS_PHASE(10);  // 10: arena ids + survivors
  }
  __syncthreads();
  if (s_err) {
    if (tid == 0) {
      out->status = s_err;
      build_queue_push(A, inst, I.part, I.build_kind, false);
    }
    return;
  }
  // ---- terminal selection (dp_scheduler.cpp:504-522) ----
  const int lv0 = I.last_forced + 1;
  const int64_t t_lo = lvl_off[lv0];
  const int64_t t_hi = r_next_free;
  if (I.values_integral) {
    // total order: value desc, n_admitted desc, mem asc, pb desc, arena asc
    int64_t best = -1;
    for (int64_t x = t_lo + tid; x < t_hi; x += kDpThreads) {
      if (best < 0) { best = x; continue; }
      const double vx = Sv_[x], vb = Sv_[best];
      bool bt;
      if (vx != vb) bt = vx > vb;
      else if (Sn_[x] != Sn_[best]) bt = Sn_[x] > Sn_[best];
      else if (Sm_[x] != Sm_[best]) bt = Sm_[x] < Sm_[best];
      else if (Sp_[x] != Sp_[best]) bt = Sp_[x] > Sp_[best];
      else bt = Sar[x] < Sar[best];
      if (bt) best = x;
    }
    // block argmax under the same order
    for (int o = 16; o; o >>= 1) {
      const int64_t y = __shfl_xor_sync(0xffffffffu, best, o);
      if (y >= 0) {
        bool bt;
        if (best < 0) bt = true;
        else {
          const double vy = Sv_[y], vb = Sv_[best];
          if (vy != vb) bt = vy > vb;
          else if (Sn_[y] != Sn_[best]) bt = Sn_[y] > Sn_[best];
          else if (Sm_[y] != Sm_[best]) bt = Sm_[y] < Sm_[best];
          else if (Sp_[y] != Sp_[best]) bt = Sp_[y] > Sp_[best];
          else bt = Sar[y] < Sar[best];
        }
        if (bt) best = y;
      }
    }
    if (lane_id() == 0) s_wsum[warp_id()] = best;
    __syncthreads();
    if (tid == 0) {
      int64_t b = -1;
      for (int w = 0; w < kDpWarps; ++w) {
        const int64_t y = s_wsum[w];
        if (y < 0) continue;
        bool bt;
        if (b < 0) bt = true;
        else {
          const double vy = Sv_[y], vb = Sv_[b];
          if (vy != vb) bt = vy > vb;
          else if (Sn_[y] != Sn_[b]) bt = Sn_[y] > Sn_[b];
          else if (Sm_[y] != Sm_[b]) bt = Sm_[y] < Sm_[b];
          else if (Sp_[y] != Sp_[b]) bt = Sp_[y] > Sp_[b];
          else bt = Sar[y] < Sar[b];
        }
        if (bt) b = y;
      }
      s_best = (int)b;
    }
  } else if (tid == 0) {
    int64_t b = -1;
    for (int64_t x = t_lo; x < t_hi; ++x) {
      bool bt;
      if (b < 0) bt = true;
      else if (fabs(Sv_[x] - Sv_[b]) > kValueEps) bt = Sv_[x] > Sv_[b];
      else if (Sn_[x] != Sn_[b]) bt = Sn_[x] > Sn_[b];
      else if (Sm_[x] != Sm_[b]) bt = Sm_[x] < Sm_[b];
      else if (Sp_[x] != Sp_[b]) bt = Sp_[x] > Sp_[b];
      else bt = Sar[x] < Sar[b];
      if (bt) b = x;
    }
    s_best = (int)b;
  }
  __syncthreads();
  if (tid == 0) {
    const int best = s_best;
    int32_t* sel = A.sel + I.off_sel;
    int32_t* adm = A.ids + I.off_ids;
    int32_t* dec = adm + I.n_pending;
    out->best = best;
    out->ctr[0] = (int64_t)s_ctr[0];
    out->ctr[1] = (int64_t)s_ctr[1];
    out->ctr[2] = (int64_t)s_ctr[2];
    out->ctr[3] = (int64_t)s_ctr[3];
    out->ctr[4] = r_arena_next - 1;
    if (best < 0) {  // dp_scheduler.cpp:525-530
      out->infeasible = 1;
      out->n_sel = 0;
      out->n_admitted = 0;
      out->n_declined = I.n_pending;
      for (int q = 0; q < I.n_pending; ++q) dec[q] = q;
      out->value = 0.0;
    } else {  // :532-544
      int n = 0;
      for (int s = best; s > 0; s = Spar[s]) sel[n++] = Sit[s];
      for (int a = 0, b = n - 1; a < b; ++a, --b) { const int t = sel[a]; sel[a] = sel[b]; sel[b] = t; }
      double value = 0.0;
      int na = 0, nd = 0;
      int k = 0;
      for (int q = 0; q < n; ++q) {
        const int ci = sel[q];
        if (!ch_fc[ci]) {
          adm[na++] = -A.ch_ref[I.off_chain + ci] - 1;
          value += ch_vl[ci];
        }
      }
      for (int ci = 0; ci < N; ++ci) {  // sel is ascending: merge-walk
        while (k < n && sel[k] < ci) ++k;
        const bool in_chain = k < n && sel[k] == ci;
        if (!ch_fc[ci] && !in_chain) dec[nd++] = -A.ch_ref[I.off_chain + ci] - 1;
      }
      out->infeasible = 0;
      out->n_sel = n;
      out->n_admitted = na;
      out->n_declined = nd;
      out->value = value;
    }
    out->status = 0;
    // plan-reconstruction queue: instances that fall back (a long sequential batch
    // loop) are queued from the front, the rest from the back
    // (a batch mixing speculative and autoregressive planners -- the C5 sweep --
    // queues the speculative instances from the front and the rest from the back:
    // the reconstruction CTAs then run one code path at a time, which halves the
    // instruction footprint the SMs share; otherwise long fallbacks go first)
    build_queue_push(A, inst, I.part, I.build_kind, A.mixed_spec ? P.speculative != 0 : best < 0);
  }
  SLOS_PHASE(11);  // 11: terminal selection + backtrack
  if (prm.phase_cycles && tid == 0) out->dbg_dp_cycles = clock64() - ph_start_;
}


__global__ void __launch_bounds__(kDpThreads, SLOS_DP_MIN_BLOCKS) dp_kernel(DpParams prm) {
  dp_body<kDpThreads, SLOS_DP_MIN_BLOCKS, SLOS_MAX_CHAIN>(prm);
}

#ifndef SLOS_DP_SMALL_THREADS
#define SLOS_DP_SMALL_THREADS 64
#endif
#ifndef SLOS_DP_SMALL_MIN_BLOCKS
#define SLOS_DP_SMALL_MIN_BLOCKS 16
#endif
constexpr int kDpSmallThreads = SLOS_DP_SMALL_THREADS;
#ifndef SLOS_DP_BIG_THREADS
#define SLOS_DP_BIG_THREADS 512
#endif
// dp_kernel_big: 512 threads (one CTA per SM, up to 128 registers, no spills) for
// the instances whose levels carry the most candidates and buckets (thousands of
// running decoders, the C4 family: a few dozen instances leave most SMs idle, so
// the per-instance latency is the whole stage).
constexpr int kDpBigThreads = SLOS_DP_BIG_THREADS;
__global__ void __launch_bounds__(kDpBigThreads, 1) dp_kernel_big(DpParams prm) {
  dp_body<kDpBigThreads, 1, SLOS_MAX_CHAIN>(prm);
}
constexpr int kDpSmallMaxChain = 16;  // chain items of a small-kernel instance (host: cost < 2048)
__global__ void __launch_bounds__(kDpSmallThreads, SLOS_DP_SMALL_MIN_BLOCKS) dp_kernel_small(DpParams prm) {
  dp_body<kDpSmallThreads, SLOS_DP_SMALL_MIN_BLOCKS, kDpSmallMaxChain>(prm);
}

}  // namespace slos
