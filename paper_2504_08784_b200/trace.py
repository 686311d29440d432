"""Batched synthetic trace generation (include/slos_trace.h).

Python mirror of the reference's scenario loading and trace generation for many
(scenario, rate scale, seed) points at once:
  scenario_from_json   ~ slosim::load_scenario_file   (proj/src/workload.cpp:294-338)
  generate_traces      ~ slosim::scale_scenario + slosim::generate_trace, batched
                         (proj/src/metrics.cpp:214-221, proj/src/workload.cpp:159-206)
The work runs in libslos_b200.so's host thread pool (slos_trace_batch); request k
of a trace has the reference id "<name>-<k:06d>".
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

import numpy as np

from . import abi

SHAPES = {"single": 0, "reasoning": 1, "tool": 2}
PROCESSES = {"poisson": 0, "bursty": 1}
ERR_SLUGS = {0: "ok", 1: "invalid-parameters", 2: "internal-inconsistency", 13: "alloc",
             20: "invalid-distribution-parameters", 21: "invariant-violation"}


class Scenario(C.Structure):
    _fields_ = [("shape", C.c_int32), ("process", C.c_int32),
                ("rate_per_s", C.c_double), ("on_multiplier", C.c_double),
                ("mean_on_s", C.c_double), ("mean_off_s", C.c_double),
                ("prompt_mean", C.c_double), ("prompt_std", C.c_double),
                ("output_mean", C.c_double), ("output_std", C.c_double),
                ("think_mean", C.c_double), ("think_std", C.c_double),
                ("response_mean", C.c_double), ("response_std", C.c_double),
                ("prefill_tier", C.c_int32), ("decode_tier", C.c_int32),
                ("think_tier", C.c_int32), ("response_tier", C.c_int32),
                ("value", C.c_double),
                ("tool_pairs_mean", C.c_double), ("tool_pairs_std", C.c_double),
                ("tool_delay_min_s", C.c_double), ("tool_delay_max_s", C.c_double),
                ("memory_overprovision", C.c_double),
                ("tpot_tiers_s", C.POINTER(C.c_double)), ("ttft_slowdowns", C.POINTER(C.c_double)),
                ("n_tiers", C.c_int32), ("tpot_window", C.c_int32)]


class TraceJob(C.Structure):
    _fields_ = [("scenario", C.POINTER(Scenario)), ("rate_scale", C.c_double),
                ("seed", C.c_uint64), ("duration_s", C.c_double)]


class TraceStage(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("external_delay_s", C.c_double),
                ("kind", C.c_int32), ("slo_tier", C.c_int32)]


class TraceRequest(C.Structure):
    _fields_ = [("arrival_s", C.c_double), ("value", C.c_double), ("memory_units", C.c_int64),
                ("first_stage", C.c_int32), ("n_stages", C.c_int32)]


class Trace(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_requests", C.c_int32), ("n_stages", C.c_int64),
                ("requests", C.POINTER(TraceRequest)), ("stages", C.POINTER(TraceStage))]


STAGE_DTYPE = np.dtype([("tokens", "<i8"), ("external_delay_s", "<f8"), ("kind", "<i4"), ("slo_tier", "<i4")])
REQUEST_DTYPE = np.dtype([("arrival_s", "<f8"), ("value", "<f8"), ("memory_units", "<i8"),
                          ("first_stage", "<i4"), ("n_stages", "<i4")])


@dataclass
class ScenarioSpec:
    """A ScenarioConfig with its SLO arrays kept alive for the C struct."""
    name: str
    c: Scenario
    tiers: object
    slow: object


def scenario_from_json(d: dict) -> ScenarioSpec:
    """The reference's load_scenario_file defaults (workload.cpp:303-332); an
    unknown shape / process is passed through as an invalid code (the generator
    reports it like ScenarioConfig::validate)."""
    slo = d["slo"]
    tiers = (C.c_double * len(slo["tpot_tiers_s"]))(*slo["tpot_tiers_s"])
    slow = (C.c_double * len(slo["ttft_slowdowns"]))(*slo["ttft_slowdowns"])
    a = d.get("arrival")
    s = Scenario()
    s.shape = SHAPES.get(d.get("shape", "single"), -1)
    if a is not None:
        s.process = PROCESSES.get(a.get("process", "poisson"), -1)
        s.rate_per_s = a.get("rate_per_s", 1.0)
        s.on_multiplier = a.get("on_multiplier", 4.0)
        s.mean_on_s = a.get("mean_on_s", 20.0)
        s.mean_off_s = a.get("mean_off_s", 60.0)
    else:
        s.process, s.rate_per_s, s.on_multiplier, s.mean_on_s, s.mean_off_s = 0, 1.0, 4.0, 20.0, 60.0

    def dist(key):
        v = d.get(key)
        return (0.0, 0.0) if v is None else (float(v.get("mean", 0.0)), float(v.get("std", 0.0)))

    s.prompt_mean, s.prompt_std = dist("prompt_tokens")
    s.output_mean, s.output_std = dist("output_tokens")
    s.think_mean, s.think_std = dist("think_tokens")
    s.response_mean, s.response_std = dist("response_tokens")
    s.prefill_tier = d.get("prefill_tier", 0)
    s.decode_tier = d.get("decode_tier", 0)
    s.value = d.get("value", 1.0)
    s.think_tier = d.get("think_tier", 0)
    s.response_tier = d.get("response_tier", len(slo["tpot_tiers_s"]) - 1)
    s.tool_pairs_mean = d.get("tool_pairs_mean", 2.7)
    s.tool_pairs_std = d.get("tool_pairs_std", 1.1)
    s.tool_delay_min_s = d.get("tool_delay_min_s", 0.05)
    s.tool_delay_max_s = d.get("tool_delay_max_s", 0.2)
    s.memory_overprovision = d.get("memory_overprovision", 1.0)
    s.tpot_tiers_s = C.cast(tiers, C.POINTER(C.c_double))
    s.ttft_slowdowns = C.cast(slow, C.POINTER(C.c_double))
    s.n_tiers = len(slo["tpot_tiers_s"])
    s.tpot_window = slo.get("tpot_window", 10)
    return ScenarioSpec(d.get("name", "scenario"), s, tiers, slow)


def load_scenario(path: str) -> ScenarioSpec:
    with open(path) as f:
        return scenario_from_json(json.load(f))


def _bind(lib):
    if not getattr(lib, "_trace_bound", False):
        lib.slos_trace_batch.argtypes = [C.POINTER(TraceJob), C.c_int32, C.c_int32, C.POINTER(Trace)]
        lib.slos_trace_batch.restype = C.c_int
        lib.slos_trace_free.argtypes = [C.POINTER(Trace)]
        lib.slos_trace_free.restype = None
        lib._trace_bound = True
    return lib


def make_jobs(points):
    """points: iterable of (ScenarioSpec, rate_scale, seed, duration_s)."""
    pts = list(points)
    jobs = (TraceJob * len(pts))()
    for k, (sc, scale, seed, dur) in enumerate(pts):
        jobs[k].scenario = C.pointer(sc.c)
        jobs[k].rate_scale = scale
        jobs[k].seed = seed
        jobs[k].duration_s = dur
    return jobs, pts


def to_numpy(t: Trace):
    """(status, requests, stages) of one trace as numpy copies."""
    if t.status != 0:
        return t.status, np.zeros(0, REQUEST_DTYPE), np.zeros(0, STAGE_DTYPE)
    nr, ns = int(t.n_requests), int(t.n_stages)
    req = np.frombuffer(C.string_at(t.requests, nr * REQUEST_DTYPE.itemsize), REQUEST_DTYPE).copy() \
        if nr else np.zeros(0, REQUEST_DTYPE)
    st = np.frombuffer(C.string_at(t.stages, ns * STAGE_DTYPE.itemsize), STAGE_DTYPE).copy() \
        if ns else np.zeros(0, STAGE_DTYPE)
    return int(t.status), req, st


def generate_traces(points, threads: int = 0, lib=None):
    """Batched generate_trace over (scenario, rate_scale, seed, duration_s) points
    -> list of (status, requests, stages) numpy triples."""
    lib = _bind(lib or abi.product())
    jobs, pts = make_jobs(points)
    outs = (Trace * len(pts))()
    st = lib.slos_trace_batch(jobs, len(pts), threads, outs)
    if st != 0:
        raise RuntimeError(f"slos_trace_batch failed: {st}")
    res = [to_numpy(outs[k]) for k in range(len(pts))]
    for k in range(len(pts)):
        lib.slos_trace_free(C.byref(outs[k]))
    return res


def reference_traces(points, timed: bool = False):  # test infrastructure only: the reference's generate_trace
    lib = abi.reference()
    if not getattr(lib, "_trace_ref_bound", False):
        lib.slos_ref_trace.argtypes = [C.POINTER(TraceJob), C.POINTER(Trace)]
        lib.slos_ref_trace.restype = C.c_int32
        lib.slos_ref_trace_free.argtypes = [C.POINTER(Trace)]
        lib.slos_ref_trace_free.restype = None
        lib._trace_ref_bound = True
    import time
    jobs, pts = make_jobs(points)
    res, dt = [], 0.0
    for k in range(len(pts)):
        t = Trace()
        t0 = time.perf_counter()
        lib.slos_ref_trace(C.byref(jobs[k]), C.byref(t))
        dt += time.perf_counter() - t0
        res.append(to_numpy(t))
        lib.slos_ref_trace_free(C.byref(t))
    return (res, dt) if timed else res


def bench_points(root: str, seeds: int = 16, horizon_s: float = 60.0):
    """The C5 sweep's trace grid: every scenario file under
    tests/golden/scenarios with bursty arrivals (coder.json's burst parameters) x
    4 rate scales x `seeds` seeds."""
    import glob
    import os
    pts = []
    for p in sorted(glob.glob(os.path.join(root, "tests", "golden", "scenarios", "*.json"))):
        d = json.load(open(p))
        d["arrival"] = dict(d.get("arrival", {}), process="bursty", on_multiplier=4.0, mean_on_s=10.0,
                            mean_off_s=30.0)
        sc = scenario_from_json(d)
        for scale in (0.5, 1.0, 2.0, 4.0):
            for seed in range(seeds):
                pts.append((sc, scale, seed, horizon_s))
    return pts


def bench_leg(root: str, steps: int, warmup: int, with_cpu: bool):
    """f3 leg of bench.py: the whole trace grid per step through slos_trace_batch
    (all host threads) and, beside it, the reference's generate_trace looped over a
    bounded sample on one thread (it has no batched entry point)."""
    import os
    import time
    pts = bench_points(root)
    lib = _bind(abi.product())
    jobs, _ = make_jobs(pts)
    outs = (Trace * len(pts))()
    dts = []
    for it in range(max(1, warmup) + steps):  # timed: the C-ABI call (generation + result arrays)
        t0 = time.perf_counter()
        lib.slos_trace_batch(jobs, len(pts), 0, outs)
        dt = time.perf_counter() - t0
        if it >= max(1, warmup):
            dts.append(dt)
        if it + 1 < max(1, warmup) + steps:
            for k in range(len(pts)):
                lib.slos_trace_free(C.byref(outs[k]))
    res = [to_numpy(outs[k]) for k in range(len(pts))]
    for k in range(len(pts)):
        lib.slos_trace_free(C.byref(outs[k]))
    dt = sum(dts) / len(dts)
    n_req = sum(len(r[1]) for r in res)
    leg = {"workload": f"f3: batched trace generation, {len(pts)} traces (6 scenarios, bursty, 4 rate scales x "
                       f"16 seeds, 60 s) = {n_req} requests per step",
           "value": len(pts) / dt, "unit": "traces/s", "requests_per_s": n_req / dt, "ms_per_step": dt * 1e3,
           "threads": os.cpu_count(), "statuses_ok": all(r[0] == 0 for r in res)}
    if with_cpu:
        idx = list(range(0, len(pts), 8))  # every 8th point: the grid's mix, bounded
        sample = [pts[k] for k in idx]
        ref, rdt = reference_traces(sample, timed=True)
        n_ref = sum(len(r[1]) for r in ref)
        leg["cpu_baseline"] = {"value": len(sample) / rdt, "unit": "traces/s", "requests_per_s": n_ref / rdt,
                               "cores": 1, "kind": "reference",
                               "sample": f"every 8th grid point ({len(sample)} traces, {n_ref} requests) through "
                                         f"the reference's generate_trace, {rdt:.2f} s wall"}
        leg["identical_to_reference"] = all(res[k][1].tobytes() == b[1].tobytes() and res[k][2].tobytes() == b[2].tobytes()
                                            for k, b in zip(idx, ref))
    return leg
