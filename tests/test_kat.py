"""The reference's own unit-test known answers (proj/tests/test_perf_model.cpp,
test_batch_planner.cpp, test_dp_scheduler.cpp), restated against the C-ABI and run
on every backend: the C oracle and the compiled reference on CPU, the product on
the B200 (marked gpu)."""
import math
import os
import random

import pytest

from conftest import HAS_GPU
from paper_2504_08784_b200 import abi
from paper_2504_08784_b200 import workload as W
from paper_2504_08784_b200.planner import (BatchPlanner, DecodeCensus, DecodeMember, Error,
                                           PendingRequest, PerfModel, PerfTerm, PlannerConfig,
                                           ScheduleInput, SloConfig, SloScheduler)

BACKENDS = [
    pytest.param("oracle", id="oracle"),
    pytest.param("reference", id="reference",
                 marks=pytest.mark.skipif(not os.path.exists(abi.REF_LIB), reason="no oracle/_ref")),
    pytest.param("product", id="product", marks=pytest.mark.gpu),
]


def lib_of(name):
    return {"oracle": abi.oracle, "reference": abi.reference, "product": abi.product}[name]()


def two_tier(t0, t1):
    return SloConfig([t0, t1], [3.0, 5.0])


# ---- test_perf_model.cpp -----------------------------------------------------

@pytest.mark.parametrize("b", BACKENDS)
def test_predict_takes_max_across_terms(b):  # :45-52
    m = PerfModel([PerfTerm(1e-4, 0.0, 0.02), PerfTerm(0.0, 0.0, 0.03)], lib=lib_of(b))
    assert m.predict(50) == pytest.approx(0.03, rel=1e-12)
    assert m.predict(200) == pytest.approx(0.04, rel=1e-12)
    assert m.predict(100) == pytest.approx(0.03, rel=1e-12)
    assert m.predict(101) == pytest.approx(0.0301, rel=1e-12)


@pytest.mark.parametrize("b", BACKENDS)
def test_predict_charges_spec_steps(b):  # :54-58
    m = PerfModel([PerfTerm(1e-4, 5e-4, 0.02)], lib=lib_of(b))
    assert m.predict(100, 4) == pytest.approx(0.032, rel=1e-12)
    assert m.predict(100, 0) == pytest.approx(0.03, rel=1e-12)


@pytest.mark.parametrize("b", BACKENDS)
def test_time2bs_inverts_predict(b):  # :60-67
    m = PerfModel([PerfTerm(1e-4, 0.0, 0.02)], lib=lib_of(b))
    assert m.time2bs(0.05) == 300
    assert m.predict(300) <= 0.05 + 1e-9
    assert m.predict(301) > 0.05
    with pytest.raises(Error) as e:
        m.time2bs(0.019)
    assert e.value.code == "infeasible-budget"


@pytest.mark.parametrize("b", BACKENDS)
def test_time2bs_cap_and_spec(b):  # :69-77
    m = PerfModel([PerfTerm(1e-5, 1e-3, 0.005)], lib=lib_of(b))
    assert m.time2bs(10.0, 0, 512) == 512
    ws, wo = m.time2bs(0.05, 8), m.time2bs(0.05, 0)
    assert ws < wo
    assert m.predict(ws, 8) <= 0.05 + 1e-9 and m.predict(ws + 1, 8) > 0.05


@pytest.mark.parametrize("b", BACKENDS)
def test_time2bs_monotone(b):  # :79-88 (draws from std::mt19937_64(7) are not needed: property)
    m = PerfModel(W.DESK_MODEL, lib=lib_of(b))
    rng = random.Random(7)
    pairs = [sorted((rng.uniform(0.021, 0.4), rng.uniform(0.021, 0.4))) for _ in range(200)]
    lo = m.time2bs_many([p[0] for p in pairs])
    hi = m.time2bs_many([p[1] for p in pairs])
    assert (lo <= hi).all()


# ---- test_batch_planner.cpp --------------------------------------------------

@pytest.mark.parametrize("b", BACKENDS)
def test_expected_accepted(b):  # :75-80
    lib = lib_of(b)
    from paper_2504_08784_b200.planner import expected_accepted as ea
    assert ea(0.5, 1, lib) == pytest.approx(1.0, rel=1e-12)
    assert ea(0.5, 4, lib) == pytest.approx(1.875, rel=1e-12)
    assert ea(1.0, 6, lib) == pytest.approx(6.0, rel=1e-12)
    assert ea(0.0, 3, lib) == pytest.approx(1.0, rel=1e-12)


@pytest.mark.parametrize("b", BACKENDS)
def test_ar_tiling_serves_jit_members(b):  # :105-132
    lib = lib_of(b)
    p = BatchPlanner(PerfModel([PerfTerm(1 / 6, 0, 0)], lib=lib), two_tier(1.0, 2.0), lib=lib)
    plan = p.tile_gap_ar(4.0, DecodeCensus([1, 0]))
    assert plan is not None and len(plan.batches) == 4
    assert plan.prefill_budget == 20
    for i, bt in enumerate(plan.batches):
        assert bt.end_s == pytest.approx(i + 1.0, rel=1e-9)
        assert bt.capacity_tokens == 6 and bt.decode_tokens == 1
    assert p.tile_gap_ar(4.0, DecodeCensus([1, 1])).prefill_budget == 18
    assert p.prefill_budget(4.0, [1, 0]) == 20
    assert p.prefill_budget(4.0, [1, 1]) == 18
    assert p.prefill_budget(4.0004, [1, 1]) == 18


@pytest.mark.parametrize("b", BACKENDS)
def test_empty_census_prefill_chunks(b):  # :134-146
    lib = lib_of(b)
    p = BatchPlanner(PerfModel([PerfTerm(1 / 6, 0, 0)], lib=lib), two_tier(1.0, 2.0),
                     PlannerConfig(max_chunk_tokens=6), lib=lib)
    plan = p.tile_gap_ar(4.0, DecodeCensus([0, 0]))
    assert plan.prefill_budget == 24
    assert all(bt.decode_tokens == 0 for bt in plan.batches)


@pytest.mark.parametrize("b", BACKENDS)
def test_overloaded_census_infeasible(b):  # :148-156
    lib = lib_of(b)
    p = BatchPlanner(PerfModel([PerfTerm(1 / 6, 0, 0)], lib=lib), two_tier(1.0, 2.0), lib=lib)
    assert p.tile_gap_ar(4.0, DecodeCensus([7, 0])) is None
    assert p.prefill_budget(4.0, [7, 0]) is None


@pytest.mark.parametrize("b", BACKENDS)
def test_exact_members_served_on_their_lines(b):  # :158-197
    lib = lib_of(b)
    p = BatchPlanner(PerfModel([PerfTerm(1 / 6, 0, 0)], lib=lib), two_tier(1.0, 2.0), lib=lib)
    plan = p.tile_gap_ar(3.0, DecodeCensus([0, 0], [DecodeMember(0, 1.0, 0, 100, 5)]))
    served = sum(t for bt in plan.batches for (o, t) in bt.decode_by_owner if o == 5)
    assert served == 3 and plan.prefill_budget == 15
    plan2 = p.tile_gap_ar(2.0, DecodeCensus([0, 0], [DecodeMember(0, 0.5, 2, 10, 9)]))
    assert sum(t for (o, t) in plan2.batches[0].decode_by_owner if o == 9) >= 2


def _brute_spec(counts, alpha, max_len, model, slo, cfg, lib):  # test_batch_planner.cpp:30-71
    from itertools import product as iprod
    from paper_2504_08784_b200.planner import expected_accepted as ea
    present = [l for l in range(slo.num_tiers()) if counts[l] > 0]
    best = None
    margin = 1.0 + cfg.plan_margin
    for sl in iprod(range(1, max_len + 1), repeat=len(present)):
        t_batch = min(slo.tpot_tiers_s[l] * ea(alpha, s, lib) for l, s in zip(present, sl))
        step = max(sl)
        dec = sum(counts[l] * s for l, s in zip(present, sl))
        if model.predict(1, step) * margin <= t_batch + 1e-9:
            lo, hi = 1, cfg.max_batch_tokens
            while lo < hi:
                mid = lo + (hi - lo + 1) // 2
                if model.predict(mid, step) * margin <= t_batch + 1e-9:
                    lo = mid
                else:
                    hi = mid - 1
            if lo >= dec:
                tpt = min(lo - dec, cfg.max_chunk_tokens) / t_batch
                best = tpt if best is None else max(best, tpt)
    return best


@pytest.mark.parametrize("b", BACKENDS)
def test_spec_solver_matches_exhaustive(b):  # :199-240 (draws via the same mt19937_64(2024))
    lib = lib_of(b)
    u = iter(W.uniforms(2024, 4000))
    checked = 0
    for it in range(60):
        nt = 1 + int(next(u) * 2.0)
        t0 = 0.02 + 0.08 * next(u)
        tp = [t0] + ([t0 * (1.5 + next(u))] if nt == 2 else [])
        slo = SloConfig(tp, [3.0, 5.0][:nt])
        model = PerfModel([PerfTerm(1e-5 + 2e-4 * next(u), 1e-4 + 2e-3 * next(u), 1e-3 + 2e-2 * next(u))], lib=lib)
        cfg = PlannerConfig(plan_margin=0.0 if next(u) < 0.5 else 0.1)
        counts = [int(next(u) * 7.0) for _ in range(nt)]
        if not any(counts):
            counts[0] = 1
        alpha = 0.1 + 0.85 * next(u)
        got = BatchPlanner(model, slo, cfg, lib=lib).solve_spec_lengths(counts, alpha, 8)
        want = _brute_spec(counts, alpha, 8, model, slo, cfg, lib)
        assert (got is not None) == (want is not None)
        if got is not None:
            assert got.prefill_throughput == pytest.approx(want, rel=1e-9)
            assert sum(c * l for c, l in zip(counts, got.lengths)) == got.decode_tokens
            assert got.batch_capacity >= got.decode_tokens
            checked += 1
    assert checked >= 20


@pytest.mark.parametrize("b", BACKENDS)
def test_spec_tiling_never_loses(b):  # :279-305
    lib = lib_of(b)
    rng = random.Random(77)
    for _ in range(80):
        slo = two_tier(0.04 + 0.03 * rng.random(), 0.1 + 0.1 * rng.random())
        cfg = PlannerConfig(speculative=True, spec_alpha=0.6 + 0.35 * rng.random(), spec_max_len=8,
                            max_chunk_tokens=16384)
        p = BatchPlanner(PerfModel(W.DESK_MODEL, lib=lib), slo, cfg, lib=lib)
        c = DecodeCensus([int(rng.random() * 4), int(rng.random() * 4)])
        if not any(c.counts_per_tier):
            c.counts_per_tier[1] = 2
        gap = BatchPlanner.quantize_gap(1.0 + 3.0 * rng.random())
        ar, sp = p.tile_gap_ar(gap, c), p.tile_gap(gap, c)
        if ar is None:
            continue
        assert sp is not None and sp.prefill_budget >= ar.prefill_budget


def test_quantize_gap():  # :307-312
    q = BatchPlanner.quantize_gap
    assert q(0.0015) == pytest.approx(0.001, rel=1e-12)
    assert q(1.9999) == pytest.approx(1.999, rel=1e-12)
    assert q(-3.0) == 0.0
    assert q(2.0) == pytest.approx(2.0, rel=1e-12)


@pytest.mark.parametrize("b", BACKENDS)
def test_planner_rejects_invalid_configuration(b):  # :314-325
    lib = lib_of(b)
    with pytest.raises(Error) as e:
        BatchPlanner(PerfModel([PerfTerm(1e-4, 0, 0.01)], lib=lib), two_tier(0.05, 0.1),
                     PlannerConfig(max_chunk_tokens=0), lib=lib)
    assert e.value.code == "invalid-parameters"


# ---- test_dp_scheduler.cpp ---------------------------------------------------

def _sched(inst_fields, lib):
    f = inst_fields
    p = BatchPlanner(PerfModel(W.oracle_model(f), lib=lib), W.oracle_slo(f), PlannerConfig(), lib=lib)
    return SloScheduler(p), W.oracle_input(f)


def _fields(cap, tpots, runners, cands, mem, horizon):
    return dict(cap=cap, tpots=tpots, runners=runners, candidates=cands, memory_total=mem, horizon=horizon)


@pytest.mark.parametrize("b", BACKENDS)
def test_tight_budget_admits_affordable_subset(b):  # :86-110
    s, inp = _sched(_fields(6, [1], [0, 0, 0], [(6, 6, 0, 1, 1)] * 4, 100, 12), lib_of(b))
    r = s.schedule(inp)
    assert len(r.admitted) == 3 and r.admitted_value == pytest.approx(3.0)
    assert len(r.declined) + len(r.deferred) == 1


@pytest.mark.parametrize("b", BACKENDS)
def test_memory_caps_admission(b):  # :112-127
    s, inp = _sched(_fields(8, [1], [], [(8, 2, 0, 3, 1)] * 4, 7, 14), lib_of(b))
    assert s.schedule(inp).admitted_value == pytest.approx(2.0)


@pytest.mark.parametrize("b", BACKENDS)
def test_value_vs_throughput_exact_sets(b):  # :146-175
    f = _fields(2, [1], [], [(2, 4, 0, 1, 9), (1, 2, 0, 1, 1), (3, 2, 0, 1, 1)], 10, 10)
    s, inp = _sched(f, lib_of(b))
    byv = s.schedule(inp)
    assert byv.admitted_value == pytest.approx(9.0) and byv.admitted == ["cand-0"]
    byc = s.schedule_throughput(inp)
    assert sorted(byc.admitted) == ["cand-1", "cand-2"]


@pytest.mark.parametrize("b", BACKENDS)
def test_unsustainable_running_set_surfaced(b):  # :192-210
    s, inp = _sched(_fields(2, [1], [0, 0, 0], [(4, 2, 0, 1, 1)], 10, 10), lib_of(b))
    r = s.schedule(inp)
    assert r.running_set_infeasible and not r.admitted and r.plan.batches


@pytest.mark.parametrize("b", BACKENDS)
def test_scheduling_is_deterministic(b):  # :212-225
    lib = lib_of(b)
    F = W.FAMILIES["C1"]
    inp = W.stress_instance(F["spec"], 5)
    s = SloScheduler(BatchPlanner(PerfModel(F["model"], lib=lib), W.TWO_TIER_SLO, F["cfg"], lib=lib))
    a, c = s.schedule(inp), s.schedule(inp)
    assert a == c


@pytest.mark.parametrize("b", BACKENDS)
def test_reconstruction_meets_deadlines(b):  # :52-84 on the golden 171717 draws
    from golden_io import load
    lib = lib_of(b)
    for item in load("oracle_instances")["171717"]["items"][:30]:
        f = W.oracle_fields(item["rec"])
        s, inp = _sched(f, lib)
        r = s.schedule(inp)
        for cid in r.admitted:
            cand = f["candidates"][int(cid[5:])]
            placed, last = 0, 0.0
            for bt in r.plan.batches:
                for e in bt.entries:
                    if e.id == cid and e.prefill_tokens > 0:
                        placed += e.prefill_tokens
                        last = max(last, bt.end_s)
            assert placed == cand[1] and last <= cand[0] + 1e-9
        prev = 0.0
        for bt in r.plan.batches:
            assert bt.start_s >= prev - 1e-9 and bt.end_s > bt.start_s - 1e-9
            prev = bt.start_s
