"""Host-side mirror of the reference planner interface, backed by the C-ABI.

Names, argument meaning and error behaviour follow the reference so that the
parity tests read like its doctest suite:

  reference (proj/include/slosim/...)               here
  PerfModel::predict / time2bs  perf_model.hpp:32-37    PerfModel.predict / time2bs
  SloConfig                     workload.hpp:14-21      SloConfig
  PlannerConfig                 batch_planner.hpp:57-66 PlannerConfig
  BatchPlanner::tile_gap_ar / tile_gap / prefill_budget BatchPlanner.*
                                batch_planner.hpp:110-122
  solve_spec_lengths / expected_accepted  batch_planner.hpp:70-85
  Scheduler / SloScheduler::schedule / schedule_throughput  dp_scheduler.hpp:81-106
  slosim::Error{code()}         common.hpp:12-21        Error(.code)

Every call goes through a library exporting include/slos_planner.h. The default
is the product library (libslos_b200.so, sm_100a kernels); it raises if that
library or a B200 is missing -- there is no CPU fallback. Tests pass
``lib=abi.oracle()`` / ``lib=abi.reference()`` to drive the checkers through the
very same code.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import abi


class Error(RuntimeError):
    """slosim::Error: a stable machine-checkable code slug plus a message."""

    def __init__(self, code: str, message: str = ""):
        super().__init__(f"{code}: {message}" if message else code)
        self.code = code


def _raise(lib, status: int) -> None:
    if status == abi.SLOS_OK:
        return
    slug = lib.slos_status_slug(status).decode()
    raise Error(slug, lib.slos_last_error().decode(errors="replace"))


# ---------------------------------------------------------------- config ---


@dataclass
class PerfTerm:
    k1: float = 0.0
    k2: float = 0.0
    b: float = 0.0


DEFAULT_MAX_TOKENS = 16384  # PerfModel::kDefaultMaxTokens perf_model.hpp:57


@dataclass
class SloConfig:
    tpot_tiers_s: list = field(default_factory=list)
    ttft_slowdowns: list = field(default_factory=list)
    tpot_window: int = 10

    def num_tiers(self) -> int:
        return len(self.tpot_tiers_s)


@dataclass
class PlannerConfig:
    max_chunk_tokens: int = 2048
    max_batch_tokens: int = DEFAULT_MAX_TOKENS
    speculative: bool = False
    spec_alpha: float = 0.8
    spec_max_len: int = 8
    plan_margin: float = 0.0

    def to_c(self) -> abi.PlannerConfigC:
        return abi.PlannerConfigC(int(self.max_chunk_tokens), int(self.max_batch_tokens),
                                  1 if self.speculative else 0, int(self.spec_max_len),
                                  float(self.spec_alpha), float(self.plan_margin))


class _Handle:
    """Owns one slos_planner* in one library."""

    def __init__(self, lib, terms, slo: SloConfig, cfg: PlannerConfig):
        self.lib = lib
        tarr = (abi.PerfTerm * max(1, len(terms)))(*[abi.PerfTerm(t.k1, t.k2, t.b) for t in terms])
        n = len(slo.tpot_tiers_s)
        tp = (C.c_double * max(1, n))(*slo.tpot_tiers_s)
        sl = (C.c_double * max(1, len(slo.ttft_slowdowns)))(*slo.ttft_slowdowns)
        if len(slo.ttft_slowdowns) != n:
            raise Error("invalid-parameters", "tpot tier and slowdown lists must align")
        c = cfg.to_c()
        h = C.c_void_p()
        _raise(lib, lib.slos_planner_create(tarr, len(terms), tp, sl, n, int(slo.tpot_window),
                                            C.byref(c), C.byref(h)))
        self.ptr = h

    def __del__(self):
        try:
            if self.ptr:
                self.lib.slos_planner_destroy(self.ptr)
        except Exception:
            pass


class PerfModel:
    """Max-of-affine batch latency model (perf_model.hpp:27-61)."""

    kDefaultMaxTokens = DEFAULT_MAX_TOKENS

    def __init__(self, terms: Sequence, lib=None):
        self.terms = [t if isinstance(t, PerfTerm) else PerfTerm(*t) for t in terms]
        if not self.terms:
            raise Error("invalid-parameters", "perf model needs at least one term")
        for t in self.terms:
            if t.k1 < 0 or t.k2 < 0 or t.b < 0:
                raise Error("invalid-parameters", "perf model coefficients must be nonnegative")
        self._lib = lib
        self._h = None

    def _handle(self):
        if self._h is None:
            self._h = _Handle(self._lib or abi.product(), self.terms, SloConfig([1.0], [1.0]),
                              PlannerConfig())
        return self._h

    def predict(self, num_tokens: int, spec_step: int = 0) -> float:
        h = self._handle()
        n = (C.c_int64 * 1)(num_tokens)
        s = (C.c_int64 * 1)(spec_step)
        out = (C.c_double * 1)()
        _raise(h.lib, h.lib.slos_predict_batch(h.ptr, 1, n, s, out))
        return out[0]

    def time2bs(self, budget_s: float, spec_step: int = 0,
                max_tokens: int = DEFAULT_MAX_TOKENS) -> int:
        return int(self.time2bs_many([budget_s], [spec_step], max_tokens)[0])

    def time2bs_many(self, budgets, spec_steps=None, max_tokens: int = DEFAULT_MAX_TOKENS):
        h = self._handle()
        b = np.ascontiguousarray(budgets, dtype=np.float64)
        s = np.zeros(len(b), np.int64) if spec_steps is None else np.ascontiguousarray(
            spec_steps, dtype=np.int64)
        out = np.zeros(len(b), np.int64)
        st = np.zeros(len(b), np.int32)
        h.lib.slos_time2bs_batch(h.ptr, len(b), b.ctypes.data_as(C.POINTER(C.c_double)),
                                 s.ctypes.data_as(C.POINTER(C.c_int64)), int(max_tokens),
                                 out.ctypes.data_as(C.POINTER(C.c_int64)),
                                 st.ctypes.data_as(C.POINTER(C.c_int32)))
        for k in range(len(b)):
            _raise(h.lib, int(st[k]))
        return out


# ---------------------------------------------------------- batch planner ---


@dataclass
class DecodeMember:
    tier: int = 0
    phase_s: float = 0.0
    backlog: int = 0
    remaining: int = 0
    owner: int = -1


@dataclass
class DecodeCensus:
    counts_per_tier: list = field(default_factory=list)
    exact: list = field(default_factory=list)


@dataclass
class PlannedBatch:
    start_s: float = 0.0
    end_s: float = 0.0
    capacity_tokens: int = 0
    spec_step: int = 0
    decode_by_owner: list = field(default_factory=list)
    decode_per_tier: list = field(default_factory=list)
    decode_tokens: int = 0
    prefill_budget: int = 0


@dataclass
class GapPlan:
    batches: list = field(default_factory=list)
    prefill_budget: int = 0
    spec_lengths: list = field(default_factory=list)


@dataclass
class SpecPlan:
    lengths: list
    batch_time_s: float
    batch_capacity: int
    decode_tokens: int
    prefill_throughput: float


def expected_accepted(alpha: float, sl: int, lib=None) -> float:
    if sl < 1:
        raise Error("invalid-parameters", "speculation length must be >= 1")
    return (lib or abi.product()).slos_expected_accepted(alpha, sl)


class BatchPlanner:
    """PB* gap tiling + speculative solver (batch_planner.hpp:87-134)."""

    def __init__(self, model: PerfModel, slo: SloConfig, cfg: Optional[PlannerConfig] = None,
                 lib=None):
        self.lib = lib or abi.product()
        self.model_ = model
        self.slo_ = slo
        self.cfg_ = cfg or PlannerConfig()
        self._h = _Handle(self.lib, model.terms, slo, self.cfg_)

    def config(self) -> PlannerConfig:
        return self.cfg_

    def slo(self) -> SloConfig:
        return self.slo_

    def model(self) -> PerfModel:
        return self.model_

    @property
    def handle(self):
        return self._h.ptr

    @staticmethod
    def quantize_gap(gap_s: float) -> float:  # batch_planner.cpp:136-139
        import math
        if gap_s <= 0:
            return 0.0
        return math.floor(gap_s * 1000.0 + 1e-6) / 1000.0

    def plan_time2bs(self, budget_s: float, spec_step: int = 0) -> int:  # batch_planner.cpp:131
        b = (C.c_double * 1)(budget_s / (1.0 + self.cfg_.plan_margin))
        s = (C.c_int64 * 1)(spec_step)
        out = (C.c_int64 * 1)()
        st = (C.c_int32 * 1)()
        self.lib.slos_time2bs_batch(self.handle, 1, b, s, int(self.cfg_.max_batch_tokens), out, st)
        _raise(self.lib, st[0])
        return int(out[0])

    def _gap(self, mode: int, queries) -> list:
        n = len(queries)
        qs = (abi.GapQuery * max(1, n))()
        keep = []
        for k, (gap, census, horizon) in enumerate(queries):
            q = qs[k]
            q.mode = mode
            q.gap_s = gap
            q.due_horizon_s = horizon
            for l, c in enumerate(census.counts_per_tier[: abi.MAX_TIERS]):
                q.counts_per_tier[l] = int(c)
            ex = (abi.DecodeMemberC * max(1, len(census.exact)))(*[
                abi.DecodeMemberC(m.tier, m.owner, m.phase_s, m.backlog, m.remaining)
                for m in census.exact])
            keep.append(ex)
            q.exact = ex
            q.n_exact = len(census.exact)
        outs = (abi.GapResult * max(1, n))()
        _raise(self.lib, self.lib.slos_tile_gap_batch(self.handle, n, qs, outs))
        res = []
        for k in range(n):
            o = outs[k]
            if o.status != abi.SLOS_OK:
                self.lib.slos_gap_result_free(C.byref(o))
                res.append(Error(self.lib.slos_status_slug(o.status).decode()))
                continue
            if not o.feasible:
                res.append(None)
                continue
            if mode == abi.GAP_PREFILL_BUDGET:
                res.append(int(o.prefill_budget))
                continue
            gp = GapPlan(prefill_budget=int(o.prefill_budget),
                         spec_lengths=[o.spec_lengths[l] for l in range(o.n_spec_lengths)])
            L = self.slo_.num_tiers()
            for b in range(o.n_batches):
                gb = o.batches[b]
                own = [(int(o.owner_tokens[2 * (gb.first_owner + q)]),
                        int(o.owner_tokens[2 * (gb.first_owner + q) + 1]))
                       for q in range(gb.n_owners)]
                gp.batches.append(PlannedBatch(gb.start_s, gb.end_s, int(gb.capacity_tokens),
                                               int(gb.spec_step), own,
                                               [int(gb.decode_per_tier[l]) for l in range(L)],
                                               int(gb.decode_tokens), int(gb.prefill_budget)))
            self.lib.slos_gap_result_free(C.byref(o))
            res.append(gp)
        return res

    @staticmethod
    def _unwrap(r):
        if isinstance(r, Error):
            raise r
        return r

    def tile_gap_ar(self, gap_s: float, census: DecodeCensus, due_horizon_s: float = 0.0):
        return self._unwrap(self._gap(abi.GAP_TILE_AR, [(gap_s, census, due_horizon_s)])[0])

    def tile_gap(self, gap_s: float, census: DecodeCensus, due_horizon_s: float = 0.0):
        return self._unwrap(self._gap(abi.GAP_TILE, [(gap_s, census, due_horizon_s)])[0])

    def tile_gap_many(self, queries, speculative_entry: bool = True):
        return self._gap(abi.GAP_TILE if speculative_entry else abi.GAP_TILE_AR, queries)

    def prefill_budget(self, gap_s: float, counts_per_tier) -> Optional[int]:
        c = DecodeCensus(list(counts_per_tier), [])
        return self._unwrap(self._gap(abi.GAP_PREFILL_BUDGET, [(gap_s, c, 0.0)])[0])

    def solve_spec_lengths(self, decoders_per_tier, alpha: float, max_len: int):
        n = len(decoders_per_tier)
        arr = (C.c_int64 * max(1, n))(*decoders_per_tier)
        out = abi.SpecPlanC()
        _raise(self.lib, self.lib.slos_solve_spec_lengths(self.handle, arr, n, alpha, max_len,
                                                          C.byref(out)))
        if not out.feasible:
            return None
        L = self.slo_.num_tiers()
        return SpecPlan([out.lengths[l] for l in range(L)], out.batch_time_s,
                        int(out.batch_capacity), int(out.decode_tokens), out.prefill_throughput)


def solve_spec_lengths(decoders_per_tier, alpha, max_len, model: PerfModel, slo: SloConfig,
                       cfg: PlannerConfig, lib=None):
    """batch_planner.cpp:51-115."""
    return BatchPlanner(model, slo, cfg, lib=lib).solve_spec_lengths(decoders_per_tier, alpha,
                                                                     max_len)


# -------------------------------------------------------------- scheduler ---


@dataclass
class PendingRequest:
    id: str = ""
    prefill_deadline: float = 0.0
    prefill_tokens: int = 0
    decode_tier: int = 0
    memory_units: int = 0
    value: float = 1.0


@dataclass
class RunningRequest:
    id: str = ""
    prefill_remaining: int = 0
    prefill_deadline: float = 0.0
    decode_tier: int = 0
    next_due_s: float = 0.0
    backlog: int = 0
    decode_remaining: int = 0


@dataclass
class ScheduleInput:
    now: float = 0.0
    running: list = field(default_factory=list)
    pending: list = field(default_factory=list)
    memory_total: int = 0
    memory_standard_resident: int = 0
    tail_horizon_s: float = 0.0


@dataclass
class PlanEntry:
    id: str = ""
    prefill_tokens: int = 0
    decode_tokens: int = 0
    spec_len: int = 0


@dataclass
class PlanBatch:
    start_s: float = 0.0
    end_s: float = 0.0
    capacity_tokens: int = 0
    spec_step: int = 0
    entries: list = field(default_factory=list)
    prefill_budget_left: int = 0


@dataclass
class SchedulePlan:
    batches: list = field(default_factory=list)
    exact_until_s: float = 0.0


@dataclass
class ScheduleResult:
    admitted: list = field(default_factory=list)
    declined: list = field(default_factory=list)
    deferred: list = field(default_factory=list)
    admitted_value: float = 0.0
    running_set_infeasible: bool = False
    plan: SchedulePlan = field(default_factory=SchedulePlan)
    counters: dict = field(default_factory=dict)


class _CInput:
    """Keeps the ctypes arrays of one ScheduleInput alive."""

    def __init__(self, inp: ScheduleInput):
        self.ids = [r.id.encode() for r in inp.running] + [p.id.encode() for p in inp.pending]
        R, Pn = len(inp.running), len(inp.pending)
        self.run = (abi.Running * max(1, R))()
        for k, r in enumerate(inp.running):
            self.run[k] = abi.Running(self.ids[k], int(r.prefill_remaining),
                                      float(r.prefill_deadline), int(r.decode_tier), 0,
                                      float(r.next_due_s), int(r.backlog),
                                      int(r.decode_remaining))
        self.pen = (abi.Pending * max(1, Pn))()
        for k, p in enumerate(inp.pending):
            self.pen[k] = abi.Pending(self.ids[R + k], float(p.prefill_deadline),
                                      int(p.prefill_tokens), int(p.decode_tier), 0,
                                      int(p.memory_units), float(p.value))
        self.c = abi.Input(float(inp.now), self.run, R, Pn, self.pen, int(inp.memory_total),
                           int(inp.memory_standard_resident), float(inp.tail_horizon_s))


def _convert(inp: ScheduleInput, r: abi.Result) -> ScheduleResult:
    def rid(ref: int) -> str:
        return inp.running[ref].id if ref >= 0 else inp.pending[-ref - 1].id

    out = ScheduleResult()
    out.admitted = [inp.pending[r.admitted[k]].id for k in range(r.n_admitted)]
    out.declined = [inp.pending[r.declined[k]].id for k in range(r.n_declined)]
    out.deferred = [inp.pending[r.deferred[k]].id for k in range(r.n_deferred)]
    out.admitted_value = r.admitted_value
    out.running_set_infeasible = bool(r.running_set_infeasible)
    out.plan.exact_until_s = r.exact_until_s
    for b in range(r.n_batches):
        cb = r.batches[b]
        pb = PlanBatch(cb.start_s, cb.end_s, int(cb.capacity_tokens), int(cb.spec_step), [],
                       int(cb.prefill_budget_left))
        for e in range(cb.first_entry, cb.first_entry + cb.n_entries):
            ce = r.entries[e]
            pb.entries.append(PlanEntry(rid(ce.req), ce.prefill_tokens, ce.decode_tokens, ce.spec_len))
        out.plan.batches.append(pb)
    c = r.counters
    out.counters = dict(transitions=c.transitions, gap_evals=c.gap_evals, dues=c.dues,
                        slots=c.slots, states=c.states)
    return out


class Scheduler:
    """dp_scheduler.hpp:81-86."""

    def schedule(self, inp: ScheduleInput) -> ScheduleResult:  # pragma: no cover
        raise NotImplementedError

    def name(self) -> str:  # pragma: no cover
        raise NotImplementedError


class SloScheduler(Scheduler):
    """Value-optimal admission DP + plan reconstruction (dp_scheduler.hpp:92-106)."""

    def __init__(self, planner: BatchPlanner):
        self.planner_ = planner

    def name(self) -> str:
        return "slos"

    def _run(self, inp: ScheduleInput, unit_value: bool) -> ScheduleResult:
        lib = self.planner_.lib
        ci = _CInput(inp)
        res = abi.Result()
        st = lib.slos_plan(self.planner_.handle, C.byref(ci.c), 1 if unit_value else 0,
                           C.byref(res))
        try:
            _raise(lib, st)
            return _convert(inp, res)
        finally:
            lib.slos_result_free(C.byref(res))

    def schedule(self, inp: ScheduleInput) -> ScheduleResult:
        return self._run(inp, False)

    def schedule_throughput(self, inp: ScheduleInput) -> ScheduleResult:
        return self._run(inp, True)

    def schedule_batch(self, inputs: Sequence[ScheduleInput], unit_value: bool = False):
        """Many independent instances in one slos_plan_batch launch."""
        lib = self.planner_.lib
        cis = [_CInput(i) for i in inputs]
        n = len(cis)
        arr = (abi.Input * max(1, n))(*[c.c for c in cis])
        hs = (C.c_void_p * max(1, n))(*([self.planner_.handle] * n))
        outs = (abi.Result * max(1, n))()
        _raise(lib, lib.slos_plan_batch(hs, n, C.cast(arr, C.c_void_p), 1 if unit_value else 0,
                                        outs, None))
        res = []
        for k in range(n):
            if outs[k].status != abi.SLOS_OK:
                res.append(Error(lib.slos_status_slug(outs[k].status).decode()))
            else:
                res.append(_convert(inputs[k], outs[k]))
            lib.slos_result_free(C.byref(outs[k]))
        return res


def make_scheduler(name: str, planner: BatchPlanner) -> Scheduler:
    """Registration point (baselines.cpp:175-180): "slos" is this planner."""
    if name == "slos":
        return SloScheduler(planner)
    raise Error("invalid-parameters", "unknown scheduler: " + name)
