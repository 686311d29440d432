// Plan reconstruction kernel (K4): build_plan (dp_scheduler.cpp:196-354) and the
// EDF fallback (:96-188), one CTA per instance, after the DP kernel.
// Gaps are sequential (chain lines carry decode_assigned from gap to gap, :244,
// :287); inside a gap everything is block-parallel (slos_gapblock.cuh).
// Output batches are written in slos_batch layout and entries in slos_entry
// layout so the host hands them to the caller without conversion.
#pragma once

#include "slos_gapblock.cuh"

namespace slos {


#define SLOS_BPHASE(k)                                                         \
  do {                                                                         \
    if (phase_cycles && G::rank() == 0) {                                      \
      const long long now_ = clock64();                                        \
      atomicAdd(&phase_cycles[(k)], (unsigned long long)(now_ - bph_t0_));     \
      bph_t0_ = now_;                                                          \
    }                                                                          \
  } while (0)

// A plan token count as a 32-bit entry field (flags values that do not fit).
// Plan entries (include/slos_planner.h): a range violation flags the plan
// (SLOS_ERR_INVALID_PARAMETERS) instead of truncating.
__device__ __forceinline__ int32_t tok32(int64_t v, int* err);
__device__ __forceinline__ slos_entry entry_prefill(int32_t req, int64_t tok, int* err) {
  return slos_entry_prefill(req, tok32(tok, err));
}
__device__ __forceinline__ slos_entry entry_decode(int32_t req, int64_t tok, int spec, int* err) {
  if (spec < 0 || spec > SLOS_ENTRY_MAX_SPEC) *err = 1;
  return slos_entry_decode(req, tok32(tok, err), spec);
}
__device__ __forceinline__ int32_t tok32(int64_t v, int* err) {
  if (v > 2147483647LL || v < -2147483647LL - 1) *err = 1;
  return (int32_t)v;
}

struct BuildShared {
  BlockShared bs;
  GapPlanBuf o, tmp;
  PlannerDev P;
  InstDev I;
  // per selected chain item (N + 2 entries; carved from the group's arena, so the
  // static shared footprint of a reconstruction warp does not scale with the
  // longest chain the ABI allows)
  double* bounds;
  int64_t* m_left;
  unsigned long long* m_asg;
  int32_t* m_item;
  int nb, nsel, edf, fill_late, err, m1;
  int range_err;  // a plan token count outside the 32-bit entry range
  int64_t n_batch, n_entry;
  double tail_len;
};

// members_at(running, now, at, pull) compacted in decoder (= owner) order.
template <class G>
__device__ inline int build_members_at(const BatchArgs& A, BuildShared& sh, double at, double pull,
                                       const MemBuf& E) {
  const InstDev& I = sh.I;
  int64_t carry = 0;
  for (int base = 0; base < I.n_dec; base += G::kSize) {
    const int k = base + G::rank();
    Member m;
    m.valid = false;
    if (k < I.n_dec) {
      const int64_t o = I.off_dec + k;
      m = member_at(sh.P, A.dec_next[o], A.dec_backlog[o], A.dec_rem[o], A.dec_tier[o], I.now, at, pull);
    }
    int64_t tot;
    const int64_t ex = G::excl(sh.bs, m.valid ? 1 : 0, &tot);
    if (m.valid) {
      const int64_t d = carry + ex;
      E.ph[d] = m.phase;
      E.bl[d] = m.backlog;
      E.rm[d] = m.rem;
      E.tr[d] = m.tier;
      E.ow[d] = A.dec_idx[I.off_dec + k];
    }
    carry += tot;
  }
  return (int)carry;
}

// chain_member lambda (dp_scheduler.cpp:238-252) for selected member mi.
__device__ inline void chain_member(const BatchArgs& A, BuildShared& sh, int mi, double a,
                                    double span, double pull, const MemBuf& E, int at) {
  const PlannerDev& P = sh.P;
  const int ci = sh.m_item[mi];
  const int64_t o = sh.I.off_chain + ci;
  const int tier = A.ch_tier[o];
  const double tpot = P.tpot[tier];
  const int64_t remaining = (int64_t)ceil(span / tpot) + 2;
  double next = A.ch_deadline[o] + (double)((int64_t)sh.m_asg[mi] + 1) * tpot;
  int64_t backlog = 0;
  while (backlog < remaining && time_lt(next - a, pull)) {
    backlog += 1;
    next += tpot;
  }
  E.ph[at] = next - a;
  E.bl[at] = backlog;
  E.rm[at] = remaining;
  E.tr[at] = tier;
  E.ow[at] = sh.I.R_total + mi;
}

__device__ __forceinline__ int32_t owner_ref(const BatchArgs& A, const BuildShared& sh, int64_t owner) {
  if (owner < sh.I.R_total) return (int32_t)owner;
  return A.ch_ref[sh.I.off_chain + sh.m_item[owner - sh.I.R_total]];
}
__device__ __forceinline__ int owner_tier(const BatchArgs& A, const BuildShared& sh, int64_t owner) {
  if (owner < sh.I.R_total) return A.run_tier[sh.I.off_run + owner];
  return A.ch_tier[sh.I.off_chain + sh.m_item[owner - sh.I.R_total]];
}

// Emit one tiled gap (offset `a`): decode entries per owner, then EDF prefill
// fill (fill_prefill, dp_scheduler.cpp:220-232). track=true updates
// decode_assigned of chain owners (the gap loop, :287; not the tail, :341-344).
template <class G>
__device__ inline int emit_gap(const BatchArgs& A, BuildShared& sh, double a, bool track, Arena ar) {
  const int tid = G::rank();
  const InstDev& I = sh.I;
  GapPlanBuf& o = sh.o;
  slos_batch* OB = A.batches + I.off_batch;
  slos_entry* OE = A.entries + I.off_entry;
  int64_t* bpos = (int64_t*)ar.take(sizeof(int64_t) * (o.n_b + 1));
  // (1) one thread: EDF prefill fill (fill_prefill, dp_scheduler.cpp:220-232) and
  //     the batch records; each batch's decode entries are reserved ahead of its
  //     prefill entries.
  if (tid == 0) {
    int64_t ne = sh.n_entry;
    for (int k = 0; k < o.n_b; ++k) {
      const GapBatchOut& gb = o.b[k];
      const int64_t e0 = ne;
      bpos[k] = e0;
      ne += gb.n_owner;
      const double end_abs = a + gb.end_s;
      int64_t budget = gb.prefill_budget;
      while (budget > 0) {
        while (sh.edf < sh.nsel && sh.m_left[sh.edf] == 0) ++sh.edf;
        if (sh.edf == sh.nsel) break;
        const int mi = sh.edf;
        const int64_t spend = imin(budget, sh.m_left[mi]);
        sh.m_left[mi] -= spend;
        budget -= spend;
        const int64_t o2 = I.off_chain + sh.m_item[mi];
        if (sh.m_left[mi] == 0 && end_abs > A.ch_deadline[o2] + kTimeEps) sh.fill_late = 1;
        if (ne < I.cap_entry) {
          OE[ne] = entry_prefill(A.ch_ref[o2], spend, &sh.range_err);
        }
        ++ne;
      }
      if (sh.n_batch < I.cap_batch) {
        slos_batch bt;
        bt.start_s = a + gb.start_s;
        bt.end_s = a + gb.end_s;
        bt.capacity_tokens = gb.capacity;
        bt.spec_step = gb.spec_step;
        bt.prefill_budget_left = budget;
        bt.first_entry = e0;
        bt.n_entries = ne - e0;
        OB[sh.n_batch] = bt;
      }
      sh.n_batch++;
    }
    sh.n_entry = ne;
  }
  G::sync();
  // (2) decode entries, one warp per batch, lanes over owners
  const int nw = G::kSize / 32, wr = tid / 32, lane = lane_id();
  for (int k = wr; k < o.n_b; k += nw) {
    const GapBatchOut& gb = o.b[k];
    const bool spec_batch = gb.spec_step > 0 && o.n_spec > 0;
    const int64_t e0 = bpos[k];
    for (int q = lane; q < gb.n_owner; q += 32) {
      const int64_t owner = o.own[2 * (gb.first_owner + q)];
      const int64_t t = o.own[2 * (gb.first_owner + q) + 1];
      const int64_t at = e0 + q;
      if (at < I.cap_entry) {
        OE[at] = entry_decode(owner_ref(A, sh, owner), t, spec_batch ? o.spec[owner_tier(A, sh, owner)] : 0,
                              &sh.range_err);
      }
      if (track && owner >= I.R_total) atomicAdd(&sh.m_asg[owner - I.R_total], (unsigned long long)t);
    }
  }
  G::sync();
  return 0;
}

// edf_fallback dp_scheduler.cpp:96-188. The batch loop is inherently sequential
// (hundreds of batches until every line completes); inside a batch every thread of
// the group owns a contiguous range of decoders (and of prefills), so entry order
// (decoder order, then EDF prefill order) is rank-major and one group scan per batch
// places every entry.
template <class G>
__device__ __noinline__ void group_edf_fallback(const BatchArgs& A, BuildShared& sh, Arena ar, OutHdr* out) {
  const int lane = G::rank();
  constexpr int NT = G::kSize;
  const InstDev& I = sh.I;
  const PlannerDev& P = sh.P;
  const int nd = I.n_dec, np = I.n_pre;
  double* dnext = (double*)ar.take(sizeof(double) * (nd + 1));
  double* dtp = (double*)ar.take(sizeof(double) * (nd + 1));
  int64_t* dbl = (int64_t*)ar.take(sizeof(int64_t) * (nd + 1));
  int64_t* dleft = (int64_t*)ar.take(sizeof(int64_t) * (nd + 1));
  int64_t* ddue = (int64_t*)ar.take(sizeof(int64_t) * (nd + 1));
  int32_t* didx = (int32_t*)ar.take(sizeof(int32_t) * (nd + 1));
  int64_t* pleft = (int64_t*)ar.take(sizeof(int64_t) * (np + 1));
  int32_t* pidx = (int32_t*)ar.take(sizeof(int32_t) * (np + 1));
  if (ar.over()) {
    if (lane == 0) { sh.err = SLOS_ERR_CAPACITY; out->need_work = ar.need(); }
    G::sync();
    return;
  }
  const int dper = (nd + NT - 1) / NT, d0 = min(nd, lane * dper), d1 = min(nd, d0 + dper);
  const int pper = (np + NT - 1) / NT, p0 = min(np, lane * pper), p1 = min(np, p0 + pper);
  double tmin = INFINITY;
  int act = 0;
  for (int k = d0; k < d1; ++k) {
    const int64_t o = I.off_dec + k;
    dnext[k] = A.dec_next[o];
    dleft[k] = A.dec_rem[o];
    dbl[k] = imin(A.dec_backlog[o], A.dec_rem[o]);
    dtp[k] = P.tpot[A.dec_tier[o]];
    didx[k] = A.dec_idx[o];
    tmin = dmin(tmin, dtp[k]);
    if (dleft[k] > 0) act = 1;
  }
  int64_t lsum = 0;  // prefill tokens still pending in this lane's range
  for (int k = p0; k < p1; ++k) {
    pleft[k] = A.pre_left[I.off_pre + k];
    pidx[k] = A.pre_idx[I.off_pre + k];
    if (pleft[k] > 0) lsum += pleft[k];
  }
  G::sync();
  const double t0 = nd > 0 ? G::min(sh.bs, tmin) : 0.0;  // :125-126
  slos_batch* OB = A.batches + I.off_batch;
  slos_entry* OE = A.entries + I.off_entry;
  const int64_t chunk_cap = P.max_chunk;
  int64_t nb = 0, ne = 0, cap_t0 = -2;
  double t = I.now;
  bool decodes = G::or_(sh.bs, act) != 0;
  bool prefills = G::or_(sh.bs, lsum > 0 ? 1 : 0) != 0;
  int par = 0;  // mscan buffer parity (uniform across the group)
  // per-lane decoder state in registers when the lane owns at most kR decoders
  constexpr int kR = 4;
  const bool regs = d1 - d0 <= kR;
  double rn[kR], rt[kR];
  int64_t rb[kR], rl[kR], rd[kR];
  int32_t ri[kR];
#pragma unroll
  for (int q = 0; q < kR; ++q) {
    const int k = d0 + q;
    const bool in = regs && k < d1;
    rn[q] = in ? dnext[k] : 0.0;
    rt[q] = in ? dtp[k] : 0.0;
    rb[q] = in ? dbl[k] : 0;
    rl[q] = in ? dleft[k] : 0;
    rd[q] = 0;
    ri[q] = in ? didx[k] : 0;
  }
  bool tail_try = true;
  for (int guard = 0; guard < 100000; ++guard) {
    if (!prefills && !decodes) break;
    if (!prefills && tail_try) {
      tail_try = false;
      // ---- the decode-only tail in closed time (dp_scheduler.cpp:138-169 with no
      // prefill left). While every batch lasts exactly t0 (predict(decode tokens) <=
      // t0), batch k starts at t + t0 + ... + t0 (the sequential loop's own additions),
      // so each decoder's dues per batch follow from its own state alone: decoders in
      // parallel over all batches, then batches in parallel for the totals, entry
      // positions and records. A batch that would outlast t0 (or no room for the due
      // matrix) voids the attempt and the sequential loop below runs unchanged. ----
      if (cap_t0 == -2) cap_t0 = plan_time2bs(P, t0, 0);
      auto st_get = [&](int k, int q, double& n_, double& tp_, int64_t& b_, int64_t& l_) {
        if (regs) {  // constant register indices (a runtime index would demote them to local memory)
#pragma unroll
          for (int qq = 0; qq < kR; ++qq)
            if (qq == q) { n_ = rn[qq]; tp_ = rt[qq]; b_ = rb[qq]; l_ = rl[qq]; }
        } else {
          n_ = dnext[k]; tp_ = dtp[k]; b_ = dbl[k]; l_ = dleft[k];
        }
      };
      // the per-batch dues of one decoder, batch by batch (exactly the sequential step)
      auto step = [&](double tt, double& n_, double tp_, int64_t& b_, int64_t& l_) -> int64_t {
        if (l_ <= 0) return 0;
        int64_t due = imin(b_, l_);
        b_ -= due;
        const double slot_end = tt + t0;
        while (l_ - due > 0 && time_le(n_, slot_end)) { ++due; n_ += tp_; }
        if (due > 0) l_ -= due;
        return due;
      };
      const int64_t left_guard = 100000 - guard;
      int64_t klast = -1;  // last batch with a due, over this lane's decoders
#pragma unroll 1
      for (int k = d0; k < d1; ++k) {
        double n_, tp_;
        int64_t b_, l_;
        st_get(k, k - d0, n_, tp_, b_, l_);
        double tt = t;
        for (int64_t kb = 0; l_ > 0 && kb <= left_guard; ++kb) {
          step(tt, n_, tp_, b_, l_);
          if (l_ <= 0) klast = kb > klast ? kb : klast;
          tt = tt + t0;
        }
        if (l_ > 0) klast = left_guard + 1;  // never finishes inside the guard
      }
      const int64_t K = (int64_t)(-G::min(sh.bs, -(double)klast)) + 1;
      Arena a2 = ar;
      // dues per (decoder, batch) as bytes (a due above 255 voids the attempt)
      uint8_t* Dm = (uint8_t*)a2.take((int64_t)nd * (K > 0 ? K : 1));
      int64_t* Bt = (int64_t*)a2.take(sizeof(int64_t) * 3 * (size_t)(K > 0 ? K : 1));
      const bool room = !a2.over() && K > 0 && K <= left_guard && cap_t0 >= 0;
      if (room) {
        // pass 1: the due matrix, decoder-major
        int wide = 0;
#pragma unroll 1
        for (int k = d0; k < d1; ++k) {
          double n_, tp_;
          int64_t b_, l_;
          st_get(k, k - d0, n_, tp_, b_, l_);
          double tt = t;
          uint8_t* row = Dm + (size_t)k * (size_t)K;
          for (int64_t kb = 0; kb < K; ++kb) {
            const int64_t due = step(tt, n_, tp_, b_, l_);
            if (due > 255) wide = 1;
            row[kb] = (uint8_t)due;
            tt = tt + t0;
          }
        }
        G::sync();
        // pass 2: per batch (contiguous batch ranges per lane): tokens, entries, and
        // whether the batch outlasts t0
        const int64_t kper = (K + NT - 1) / NT, k0 = imin(K, (int64_t)lane * kper), k1 = imin(K, k0 + kper);
        int bad = 0;
        int64_t lcnt = 0;
        for (int64_t kb = k0; kb < k1; ++kb) {
          int64_t tok = 0, cnt = 0;
          for (int d = 0; d < nd; ++d) {
            const int64_t x = (int64_t)Dm[(size_t)d * (size_t)K + kb];
            tok += x;
            cnt += x > 0 ? 1 : 0;
          }
          if (tok > 0 && plan_predict(P, tok, 0) > t0) bad = 1;
          if (wide) bad = 1;
          Bt[3 * kb] = tok;
          Bt[3 * kb + 1] = cnt;
          lcnt += cnt;
        }
        if (!G::or_(sh.bs, bad)) {
          int64_t cv[1] = {lcnt}, cex[1], ctot[1];
          G::template mscan<1>(sh.bs, cv, cex, ctot, par);
          // pass 3: entries and batch records of this lane's batches
          double tt = t;
          for (int64_t kb = 0; kb < k0; ++kb) tt = tt + t0;
          int64_t pos = ne + cex[0];
          for (int64_t kb = k0; kb < k1; ++kb) {
            const int64_t first = pos;
            for (int d = 0; d < nd; ++d) {
              const int64_t x = (int64_t)Dm[(size_t)d * (size_t)K + kb];
              if (x <= 0) continue;
              if (pos < I.cap_entry) OE[pos] = entry_decode(didx[d], x, 0, &sh.range_err);
              ++pos;
            }
            const int64_t tok = Bt[3 * kb];
            slos_batch b;
            b.start_s = tt;
            b.end_s = tt + t0;
            b.capacity_tokens = imax(cap_t0, tok);
            b.spec_step = 0;
            b.prefill_budget_left = imax(0, imin(cap_t0 - tok, chunk_cap));
            b.first_entry = first;
            b.n_entries = pos - first;
            if (nb + kb < I.cap_batch) OB[nb + kb] = b;
            tt = b.end_s;
          }
          // every lane advances the same sequence to the tail's end
          double te = t;
          for (int64_t kb = 0; kb < K; ++kb) te = te + t0;
          t = te;
          nb += K;
          ne += ctot[0];
          decodes = false;
          G::sync();
          break;
        }
      }
      G::sync();  // the attempt is void: the due matrix is scratch, the state untouched
    }
    const bool dec_branch = decodes;
    const int64_t e0 = ne;
    int64_t pre_before = 0, pre_tot = 0;
    bool have_pre = false;
    int64_t free, dtok = 0, cap = 0;
    if (dec_branch) {
      const double slot_end = t + t0;
      int cnt = 0, still = 0;
      int64_t tok = 0;
      if (regs) {  // the lane's decoders live in registers (no shared-memory round trips)
#pragma unroll
        for (int q = 0; q < kR; ++q) {
          if (q >= d1 - d0) break;
          int64_t due = 0;
          if (rl[q] > 0) {
            due = imin(rb[q], rl[q]);
            rb[q] -= due;
            while (rl[q] - due > 0 && time_le(rn[q], slot_end)) {
              ++due;
              rn[q] += rt[q];
            }
            if (due > 0) {
              rl[q] -= due;
              ++cnt;
              tok += due;
            }
          }
          rd[q] = due;
          if (rl[q] > 0) still = 1;
        }
      } else {
      for (int k = d0; k < d1; ++k) {
        int64_t due = 0;
        if (dleft[k] > 0) {
          due = imin(dbl[k], dleft[k]);
          dbl[k] -= due;
          while (dleft[k] - due > 0 && time_le(dnext[k], slot_end)) {
            ++due;
            dnext[k] += dtp[k];
          }
          if (due > 0) {
            dleft[k] -= due;
            ++cnt;
            tok += due;
          }
        }
        ddue[k] = due;
        if (dleft[k] > 0) still = 1;
      }
      }
      // one scan for entry positions, the batch's decode tokens, "still decoding" and
      // the prefill EDF prefix (pending prefill before this lane's range)
      int64_t mv[4] = {(int64_t)cnt, tok, (int64_t)still, lsum}, mex[4], mtot[4];
      G::template mscan<4>(sh.bs, mv, mex, mtot, par);
      pre_before = mex[3];
      pre_tot = mtot[3];
      have_pre = true;
      int64_t pos = e0 + mex[0];
      if (regs) {
#pragma unroll
        for (int q = 0; q < kR; ++q) {
          if (q >= d1 - d0) break;
          if (rd[q] <= 0) continue;
          if (pos < I.cap_entry) {
            OE[pos] = entry_decode(ri[q], rd[q], 0, &sh.range_err);
          }
          ++pos;
        }
      } else {
      for (int k = d0; k < d1; ++k) {
        if (ddue[k] <= 0) continue;
        if (pos < I.cap_entry) {
          OE[pos] = entry_decode(didx[k], ddue[k], 0, &sh.range_err);
        }
        ++pos;
      }
      }
      ne += mtot[0];
      dtok = mtot[1];
      decodes = mtot[2] != 0;
      if (cap_t0 == -2) cap_t0 = plan_time2bs(P, t0, 0);  // loop-invariant: t0 is fixed
      cap = cap_t0;
      if (cap < 0) {
        if (lane == 0) sh.err = SLOS_ERR_INFEASIBLE_BUDGET;
        G::sync();
        return;
      }
      free = imax(0, imin(cap - dtok, chunk_cap));
    } else {
      free = chunk_cap;
    }
    // EDF prefill in order: take_k = min(left_k, max(0, free - sum_{k'<k} left_k'))
    int64_t spent = 0;
    if (prefills) {
      if (!have_pre) {
        int64_t pv[1] = {lsum}, pex[1], ptot[1];
        G::template mscan<1>(sh.bs, pv, pex, ptot, par);
        pre_before = pex[0];
        pre_tot = ptot[0];
      }
      const int64_t before = pre_before, tot0 = pre_tot;
      int cnt = 0;
      int64_t run = before, mine = 0;
      for (int k = p0; k < p1; ++k) {
        const int64_t lk = pleft[k] > 0 ? pleft[k] : 0;
        const int64_t take = imin(lk, imax(0, free - run));
        run += lk;
        if (take > 0) ++cnt;
        mine += take;
      }
      int64_t cv[2] = {(int64_t)cnt, mine}, cex[2], ctot[2];
      G::template mscan<2>(sh.bs, cv, cex, ctot, par);
      const int64_t totc = ctot[0];
      int64_t pos = ne + cex[0];
      run = before;
      for (int k = p0; k < p1; ++k) {
        const int64_t lk = pleft[k] > 0 ? pleft[k] : 0;
        const int64_t take = imin(lk, imax(0, free - run));
        run += lk;
        if (take <= 0) continue;
        pleft[k] -= take;
        if (pos < I.cap_entry) {
          OE[pos] = entry_prefill(pidx[k], take, &sh.range_err);
        }
        ++pos;
      }
      ne += totc;
      spent = ctot[1];
      lsum -= mine;
      prefills = tot0 - spent > 0;  // every lane's pending prefill is >= 0
    }
    slos_batch b;
    b.start_s = t;
    b.spec_step = 0;
    b.first_entry = e0;
    b.n_entries = ne - e0;
    if (dec_branch) {  // :138-169
      const int64_t total = dtok + spent;
      const double dur = dmax(t0, total > 0 ? plan_predict(P, total, 0) : 0.0);
      b.end_s = t + dur;
      b.capacity_tokens = imax(cap, total);
      b.prefill_budget_left = imax(0, free - spent);
    } else {  // :170-182
      b.end_s = t + plan_predict(P, spent, 0);
      b.capacity_tokens = spent;
      b.prefill_budget_left = 0;
    }
    if (lane == 0 && nb < I.cap_batch) OB[nb] = b;
    ++nb;
    t = b.end_s;
  }
  if (lane == 0) {
    sh.n_batch = nb;
    sh.n_entry = ne;
    out->exact_until = t;
  }
  G::sync();
}

template <class G>
__device__ inline void build_instance(const BatchArgs& A, BuildShared& sh, int inst,
                                      unsigned char* smem_buf, int64_t smem_cap,
                                      unsigned long long* phase_cycles) {
  long long bph_t0_ = clock64();
  const long long bph_start_ = bph_t0_;
  struct EndTimer {
    unsigned long long* pc;
    long long t0;
    OutHdr* o;
    __device__ ~EndTimer() {
      if (pc && G::rank() == 0) {
        const unsigned long long d = (unsigned long long)(clock64() - t0);
        atomicMax(&pc[6], d);
        atomicAdd(&pc[7], 1ull);
        o->dbg_cycles = (int64_t)d;
      }
    }
  } end_timer_{phase_cycles, bph_start_, &A.out[inst]};
  const int tid = G::rank();
  OutHdr* out = &A.out[inst];
  if (out->status != 0) return;
  block_copy_struct(sh.P, A.planners[A.inst[inst].planner], tid, G::kSize);
  block_copy_struct(sh.I, A.inst[inst], tid, G::kSize);
  if (tid == 0) {
    sh.err = 0;
    sh.n_batch = 0;
    sh.n_entry = 0;
    sh.edf = 0;
    sh.fill_late = 0;
    sh.range_err = 0;
  }
  G::sync();
  const InstDev& I = sh.I;
  const PlannerDev& P = sh.P;
  const double pull = plan_predict(P, 1, 0);
  // global work area: plan outputs of a gap; the per-gap working set goes to
  // shared memory first (smem_buf), overflowing into the rest of the work area
  Arena ga;
  ga.base = A.work + I.off_work;
  ga.cap = I.cap_work;
  ga.used = 0;
  ga.base2 = nullptr;
  ga.cap2 = 0;
  ga.used2 = 0;
  GapBatchOut* gb = (GapBatchOut*)ga.take(sizeof(GapBatchOut) * I.cap_gb);
  int64_t* go = (int64_t*)ga.take(sizeof(int64_t) * 2 * I.cap_go);
  GapBatchOut* tb = (GapBatchOut*)ga.take(sizeof(GapBatchOut) * I.cap_gb);
  Arena ar;
  ar.base = smem_buf;
  ar.cap = smem_cap;
  ar.used = 0;
  ar.base2 = ga.base + ((ga.used + 255) & ~(int64_t)255);
  ar.cap2 = ga.cap - ((ga.used + 255) & ~(int64_t)255);
  ar.used2 = 0;
  const int Mmax = I.n_dec + I.N + 1;
  MemBuf E;
  E.ph = (double*)ar.take(sizeof(double) * Mmax);
  E.bl = (int64_t*)ar.take(sizeof(int64_t) * Mmax);
  E.rm = (int64_t*)ar.take(sizeof(int64_t) * Mmax);
  E.tr = (int32_t*)ar.take(sizeof(int32_t) * Mmax);
  double* ch_bounds = (double*)ar.take(sizeof(double) * (I.N + 2));
  int64_t* ch_left = (int64_t*)ar.take(sizeof(int64_t) * (I.N + 2));
  unsigned long long* ch_asg = (unsigned long long*)ar.take(sizeof(unsigned long long) * (I.N + 2));
  int32_t* ch_item = (int32_t*)ar.take(sizeof(int32_t) * (I.N + 2));
  E.ow = (int32_t*)ar.take(sizeof(int32_t) * Mmax);
  if (ga.over() || ar.over()) {
    if (tid == 0) { out->status = SLOS_ERR_CAPACITY; out->need_work = ar.need(); }
    return;
  }
  if (tid == 0) {
    sh.bounds = ch_bounds; sh.m_left = ch_left; sh.m_asg = ch_asg; sh.m_item = ch_item;
    sh.o.b = gb; sh.o.cap_b = (int32_t)I.cap_gb; sh.o.own = go; sh.o.cap_own = (int32_t)I.cap_go;
    sh.tmp.b = tb; sh.tmp.cap_b = (int32_t)I.cap_gb; sh.tmp.own = nullptr; sh.tmp.cap_own = 0;
  }
  int64_t zero[kMaxTiers];
  for (int l = 0; l < kMaxTiers; ++l) zero[l] = 0;
  bool fallback = out->best < 0;
  if (!fallback) {
    const int32_t* sel = A.sel + I.off_sel;
    if (tid == 0) {
      sh.nsel = out->n_sel;
      for (int k = 0; k < sh.nsel; ++k) {
        sh.m_item[k] = sel[k];
        sh.m_left[k] = A.ch_prefill[I.off_chain + sel[k]];
        sh.m_asg[k] = 0;
      }
      int nb = 0;
      sh.bounds[nb++] = I.now;
      for (int k = 0; k < sh.nsel; ++k) {
        const double dl = A.ch_deadline[I.off_chain + sel[k]];
        if (dl > sh.bounds[nb - 1] + kTimeEps) sh.bounds[nb++] = dl;
      }
      sh.nb = nb;
    }
    G::sync();
    for (int k = 0; k + 1 < sh.nb && !fallback; ++k) {  // :262-293
      const double a = sh.bounds[k];
      const double raw = sh.bounds[k + 1] - a;
      const double len = quantize_gap(raw);
      SLOS_BPHASE(0);  // 0: setup / previous gap bookkeeping
      int m = build_members_at<G>(A, sh, a, pull, E);
      if (tid == 0) {
        int mm = m;
        for (int mi = 0; mi < sh.nsel; ++mi)
          if (A.ch_deadline[I.off_chain + sh.m_item[mi]] <= a + kTimeEps)
            chain_member(A, sh, mi, a, raw + pull, pull, E, mm++);
        sh.m1 = mm;
      }
      G::sync();
      SLOS_BPHASE(1);  // 1: census (members_at + chain lines)
      MemBuf EE = E;
      EE.M = sh.m1;
      Arena ar2 = ar;
      block_tile_gap<G>(P, sh.bs, len, raw + pull, zero, EE, true, ar2, sh.o, sh.tmp);
      SLOS_BPHASE(2);  // 2: tile_gap
      if (sh.o.status) {
        if (tid == 0) { out->status = sh.o.status; out->need_work = sh.o.need_work; }
        return;
      }
      if (sh.o.n_b > sh.o.cap_b || sh.o.n_own > sh.o.cap_own) {
        if (tid == 0) { out->status = SLOS_ERR_CAPACITY; out->need_work = 2 * ar.cap; }
        return;
      }
      if (!sh.o.feasible) { fallback = true; break; }
      emit_gap<G>(A, sh, a, true, ar);
      SLOS_BPHASE(3);  // 3: emission
    }
    if (!fallback) {
      if (tid == 0) {  // :294-300
        int shortfall = sh.fill_late;
        for (int k = 0; k < sh.nsel; ++k) if (sh.m_left[k] > 0) shortfall = 1;
        sh.err = shortfall;
      }
      G::sync();
      if (sh.err) fallback = true;
      G::sync();
      if (tid == 0) sh.err = 0;
    }
    if (!fallback) {  // decode tail :302-349
      SLOS_BPHASE(0);  // 0: setup / previous gap bookkeeping
      const double t_last = sh.bounds[sh.nb - 1];
      const int m = build_members_at<G>(A, sh, t_last, pull, E);
      double tl = 0.0, capv = 0.0;
      for (int q = tid; q < m; q += G::kSize) {
        const double tpot = P.tpot[E.tr[q]];
        tl = dmax(tl, E.ph[q] + (double)E.rm[q] * tpot);
        if (E.rm[q] > 0) capv = dmax(capv, E.ph[q] + tpot);
      }
      double tail_len = G::max(sh.bs, tl);
      const double capm = G::max(sh.bs, capv);
      if (sh.nsel > 0 || I.tail_horizon > kTimeEps) {
        double max_tpot = 0.0;
        for (int l = 0; l < P.L; ++l) max_tpot = dmax(max_tpot, P.tpot[l]);
        double cp = dmax(2.0 * max_tpot, I.tail_horizon);
        cp = dmax(cp, capm);
        tail_len = dmin(tail_len, cp);
      }
      if (tid == 0) {
        int mm = m;
        for (int mi = 0; mi < sh.nsel; ++mi) chain_member(A, sh, mi, t_last, tail_len, pull, E, mm++);
        sh.m1 = mm;
      }
      G::sync();
      SLOS_BPHASE(1);  // 1: census (members_at + chain lines)
      const double tlen = quantize_gap(tail_len);
      if (tlen > kTimeEps && sh.m1 > 0) {
        MemBuf EE = E;
        EE.M = sh.m1;
        Arena ar2 = ar;
        block_tile_gap<G>(P, sh.bs, tlen, tail_len, zero, EE, true, ar2, sh.o, sh.tmp);
        SLOS_BPHASE(2);  // 2: tile_gap
        if (sh.o.status) {
          if (tid == 0) { out->status = sh.o.status; out->need_work = sh.o.need_work; }
          return;
        }
        if (sh.o.n_b > sh.o.cap_b || sh.o.n_own > sh.o.cap_own) {
          if (tid == 0) { out->status = SLOS_ERR_CAPACITY; out->need_work = 2 * ar.cap; }
          return;
        }
        if (!sh.o.feasible) fallback = true;
        else emit_gap<G>(A, sh, t_last, false, ar);
        SLOS_BPHASE(3);  // 3: emission
      }
    }
    SLOS_BPHASE(4);  // 4: decode tail
    if (!fallback && tid == 0) {
      const slos_batch* OB = A.batches + I.off_batch;
      out->exact_until = sh.n_batch == 0 ? I.now
                         : (sh.n_batch <= I.cap_batch ? OB[sh.n_batch - 1].end_s : 0.0);
    }
  }
  if (fallback) {  // :525-530 / :546-556
    if (tid == 0) {
      out->infeasible = 1;
      out->n_admitted = 0;
      out->value = 0.0;
      int32_t* dec = A.ids + I.off_ids + I.n_pending;
      for (int q = 0; q < I.n_pending; ++q) dec[q] = q;
      out->n_declined = I.n_pending;
    }
    G::sync();
    const long long fb0 = clock64();
    group_edf_fallback<G>(A, sh, ar, out);
    if (phase_cycles && tid == 0) {  // debug: fallback wall cycles and batches
      atomicAdd(&phase_cycles[14], (unsigned long long)(clock64() - fb0));
      atomicAdd(&phase_cycles[15], (unsigned long long)sh.n_batch);
    }
    SLOS_BPHASE(5);  // 5: fallback
    if (sh.err) {
      if (tid == 0) out->status = sh.err;
      return;
    }
  }
  G::sync();
  if (tid == 0) {
    out->n_batches = sh.n_batch;
    out->n_entries = sh.n_entry;
    if (sh.n_batch > I.cap_batch || sh.n_entry > I.cap_entry) {
      out->status = SLOS_ERR_CAPACITY;
      out->need_batch = 2 * sh.n_batch;
      out->need_entry = 2 * sh.n_entry;
    } else if (sh.range_err) {
      out->status = SLOS_ERR_INVALID_PARAMETERS;
    }
  }
}

// Plan reconstruction granularity, chosen per instance by the host: small
// instances (few decoders) are built by one warp each, four per CTA, without CTA
// barriers (build_kernel_warp, queue 0); large ones by a 128-thread CTA each
// (build_kernel, queue 1).
constexpr int kBuildWarps = 4;
constexpr int kBuildThreads = 128;
#ifndef SLOS_BUILD_MIN_BLOCKS
#define SLOS_BUILD_MIN_BLOCKS 4  // <= 128 registers: a C2 part's 512 instances build in one wave
#endif
#ifndef SLOS_BUILD_WARP_MIN_BLOCKS
#define SLOS_BUILD_WARP_MIN_BLOCKS 4
#endif

__global__ void __launch_bounds__(32 * kBuildWarps, SLOS_BUILD_WARP_MIN_BLOCKS) build_kernel_warp(BuildParams prm) {
  const BatchArgs& A = prm.a;
  __shared__ BuildShared shs[kBuildWarps];
  extern __shared__ __align__(16) unsigned char bsm[];
  const int idx = blockIdx.x * kBuildWarps + warp_id();
  const int q = kBuildKinds * prm.part;
  if (idx >= A.qn[q]) return;  // whole warp; the engine never uses CTA barriers here
  const int64_t per = (int64_t)(prm.smem_warp / kBuildWarps) & ~(int64_t)255;
  build_instance<WarpGrp>(A, shs[warp_id()], A.bq[A.qbase[q] + idx], bsm + per * warp_id(), per,
                          prm.phase_cycles);
}

__global__ void __launch_bounds__(kBuildThreads, SLOS_BUILD_MIN_BLOCKS) build_kernel(BuildParams prm) {
  const BatchArgs& A = prm.a;
  __shared__ BuildShared sh;
  extern __shared__ __align__(16) unsigned char bsm[];
  build_instance<BlockGrpT<kBuildThreads>>(A, sh, A.bq[A.qbase[kBuildKinds * prm.part + 1] + blockIdx.x], bsm,
                                           (int64_t)prm.smem_bytes, prm.phase_cycles);
}

// Larger instances get wider CTAs, one per SM: build_kernel_big (256 threads: the
// latency mode's choice below a thousand decoders) and build_kernel_huge (512
// threads: thousands of running decoders, the C4 family; C4 x 64 1.35 -> 1.21 ms
// against 256 threads, while 256 stays faster for a single C2-sized plan).
#ifndef SLOS_BUILD_BIG_THREADS
#define SLOS_BUILD_BIG_THREADS (2 * kBuildThreads)
#endif
#ifndef SLOS_BUILD_HUGE_THREADS
#define SLOS_BUILD_HUGE_THREADS (4 * kBuildThreads)
#endif
static_assert(SLOS_BUILD_HUGE_THREADS <= kBT, "BlockShared holds groups of at most kBT threads");
__global__ void __launch_bounds__(SLOS_BUILD_BIG_THREADS, 1) build_kernel_big(BuildParams prm) {
  const BatchArgs& A = prm.a;
  __shared__ BuildShared sh;
  extern __shared__ __align__(16) unsigned char bsm[];
  build_instance<BlockGrpT<SLOS_BUILD_BIG_THREADS>>(A, sh, A.bq[A.qbase[kBuildKinds * prm.part + 2] + blockIdx.x], bsm,
                                               (int64_t)prm.smem_big, prm.phase_cycles);
}
__global__ void __launch_bounds__(SLOS_BUILD_HUGE_THREADS, 1) build_kernel_huge(BuildParams prm) {
  const BatchArgs& A = prm.a;
  __shared__ BuildShared sh;
  extern __shared__ __align__(16) unsigned char bsm[];
  build_instance<BlockGrpT<SLOS_BUILD_HUGE_THREADS>>(A, sh, A.bq[A.qbase[kBuildKinds * prm.part + 3] + blockIdx.x],
                                                     bsm, (int64_t)prm.smem_big, prm.phase_cycles);
}

// ---- standalone gap queries (slos_tile_gap_batch) ----------------------------
struct GapParams {
  const PlannerDev* planner;
  const GapQueryDev* q;
  const double* ph;
  const int64_t* bl;
  const int64_t* rm;
  const int32_t* tr;
  const int32_t* ow;
  GapBatchOut* ob;
  int64_t* oo;
  unsigned char* work;
  GapOutDev* out;
};

__global__ void __launch_bounds__(kBT) gap_kernel(GapParams prm) {
  __shared__ BlockShared bs;
  __shared__ GapPlanBuf o, tmp;
  __shared__ PlannerDev P;
  const int tid = threadIdx.x;
  const GapQueryDev q = prm.q[blockIdx.x];
  if (tid == 0) P = *prm.planner;
  __syncthreads();
  Arena ar;
  ar.base = prm.work + q.off_work;
  ar.cap = q.cap_work;
  ar.used = 0;
  ar.base2 = nullptr;
  ar.cap2 = 0;
  ar.used2 = 0;
  MemBuf E;
  E.ph = const_cast<double*>(prm.ph) + q.off_exact;
  E.bl = const_cast<int64_t*>(prm.bl) + q.off_exact;
  E.rm = const_cast<int64_t*>(prm.rm) + q.off_exact;
  E.tr = const_cast<int32_t*>(prm.tr) + q.off_exact;
  E.ow = const_cast<int32_t*>(prm.ow) + q.off_exact;
  E.M = q.n_exact;
  GapBatchOut* tb = (GapBatchOut*)ar.take(sizeof(GapBatchOut) * q.cap_batch);
  if (tid == 0) {
    o.b = prm.ob + q.off_out_batch; o.cap_b = (int32_t)q.cap_batch;
    o.own = prm.oo + 2 * q.off_out_owner; o.cap_own = (int32_t)q.cap_owner;
    tmp.b = tb; tmp.cap_b = (int32_t)q.cap_batch; tmp.own = nullptr; tmp.cap_own = 0;
  }
  __syncthreads();
  int64_t c[kMaxTiers];
  for (int l = 0; l < kMaxTiers; ++l) c[l] = q.counts[l];
  bool sorted = true;
  for (int m = 1; m < E.M; ++m) if (E.ow[m] <= E.ow[m - 1]) { sorted = false; break; }
  if (q.mode == SLOS_GAP_TILE_AR) {
    block_tile_gap_ar<BlockGrp>(P, bs, q.gap_s, q.horizon, c, E, sorted, ar, o);
  } else if (q.mode == SLOS_GAP_TILE) {
    block_tile_gap<BlockGrp>(P, bs, q.gap_s, q.horizon, c, E, sorted, ar, o, tmp);
  } else {  // prefill_budget: quantised gap, canonical census, due_horizon 0
    MemBuf none = E;
    none.M = 0;
    block_tile_gap<BlockGrp>(P, bs, quantize_gap(q.gap_s), 0.0, c, none, true, ar, o, tmp);
  }
  if (tid == 0) {
    GapOutDev r;
    r.status = o.status;
    r.feasible = o.feasible;
    r.budget = o.budget;
    r.n_spec = o.n_spec;
    for (int l = 0; l < kMaxTiers; ++l) r.spec_lengths[l] = o.spec[l];
    r.n_batches = o.n_b;
    r.n_owner_pairs = o.n_own;
    r.need_batch = o.n_b;
    r.need_owner = o.n_own;
    r.need_work = o.need_work;
    if (!r.status && (o.n_b > o.cap_b || o.n_own > o.cap_own)) r.status = SLOS_ERR_CAPACITY;
    prm.out[blockIdx.x] = r;
  }
}

// ---- PerfModel primitives (slos_time2bs_batch / slos_predict_batch) --------
__global__ void time2bs_kernel(const PlannerDev* P, int n, const double* budget, const int64_t* spec,
                               int64_t max_tokens, int64_t* out, int32_t* status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t s = spec ? spec[k] : 0;
  if (max_tokens < 1 || s < 0) { out[k] = 0; status[k] = SLOS_ERR_INVALID_PARAMETERS; return; }
  const int64_t r = time2bs(*P, budget[k], s, max_tokens);
  out[k] = r < 0 ? 0 : r;
  status[k] = r < 0 ? SLOS_ERR_INFEASIBLE_BUDGET : SLOS_OK;
}

__global__ void predict_kernel(const PlannerDev* P, int n, const int64_t* tokens, const int64_t* spec,
                               double* out, int32_t* status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t s = spec ? spec[k] : 0;
  if (tokens[k] < 0 || s < 0) { out[k] = 0.0; status[k] = SLOS_ERR_INVALID_PARAMETERS; return; }
  out[k] = predict(*P, tokens[k], s);
  status[k] = SLOS_OK;
}

}  // namespace slos
