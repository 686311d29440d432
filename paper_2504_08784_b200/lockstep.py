"""Batched routing rounds and lockstep simulation lanes (include/slos_lockstep.h).

ctypes wrapper of integration/_build/libslos_lockstep.so: the reference's own
replica simulator driven in conservative-lookahead windows, many simulations as
concurrent lanes, every waiting schedule() served by the product's plan broker in
one batched launch. Results are identical to the
reference's sequential ClusterSim / simulate_scenario / capacity_search.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

from . import abi

LOCKSTEP_LIB = os.path.join(abi.ROOT, "integration", "_build", "libslos_lockstep.so")
SCENARIOS = os.path.join(abi.ROOT, "tests", "golden", "scenarios")
DESK = [(2.5e-5, 2e-3, 0.006), (0.0, 0.0, 0.02)]  # the desk perf model


class SimConfig(C.Structure):  # slos_sim_config
    _fields_ = [("speculative", C.c_int32), ("spec_max_len", C.c_int32), ("spec_alpha", C.c_double),
                ("noise", C.c_double), ("memory_units", C.c_int64), ("max_chunk_tokens", C.c_int64),
                ("max_batch_tokens", C.c_int64), ("replicas", C.c_int32), ("routing_limit", C.c_int32),
                ("backup_best_effort", C.c_int32), ("reserved0", C.c_int32), ("net_delay_s", C.c_double)]


class SimSummary(C.Structure):  # slos_sim_summary
    _fields_ = [("requests", C.c_int64), ("standard", C.c_int64), ("attained", C.c_int64),
                ("best_effort", C.c_int64), ("dropped", C.c_int64), ("total_hops", C.c_int64),
                ("plans", C.c_int64), ("tokens_out", C.c_int64), ("attainment", C.c_double),
                ("overall_attainment", C.c_double), ("digest", C.c_uint64)]


class CapacityResult(C.Structure):  # slos_capacity_result
    _fields_ = [("scale", C.c_double), ("per_gpu_rate", C.c_double), ("attainment", C.c_double),
                ("evaluations", C.c_int32), ("reserved0", C.c_int32)]


class Stats(C.Structure):  # slos_lockstep_stats
    _fields_ = [("plans", C.c_int64), ("flushes", C.c_int64), ("windows", C.c_int64), ("wall_s", C.c_double)]


@dataclass
class Sim:
    """ExecConfig + ClusterConfig knobs (sim_executor.hpp:24-41, tiers_router.hpp:14-21)."""
    speculative: bool = False
    spec_max_len: int = 8
    spec_alpha: float = 0.8
    noise: float = 0.0
    memory_units: int = 8192
    max_chunk_tokens: int = 2048
    max_batch_tokens: int = 16384
    replicas: int = 1
    routing_limit: int = 3
    backup_best_effort: bool = True
    net_delay_s: float = 0.001

    def c(self) -> SimConfig:
        return SimConfig(int(self.speculative), self.spec_max_len, self.spec_alpha, self.noise,
                         self.memory_units, self.max_chunk_tokens, self.max_batch_tokens, self.replicas,
                         self.routing_limit, int(self.backup_best_effort), 0, self.net_delay_s)


def available() -> bool:
    return os.path.exists(LOCKSTEP_LIB)


def _terms(model):
    arr = (abi.PerfTerm * len(model))(*[abi.PerfTerm(*t) for t in model])
    return arr, len(model)


def scenario_path(name: str) -> str:
    return name if os.path.sep in name else os.path.join(SCENARIOS, name + ".json")


class Lockstep:
    def __init__(self, backend: str | None = None):
        lib = C.CDLL(LOCKSTEP_LIB)
        lib.slos_lockstep_set_backend.argtypes = [C.c_char_p]
        lib.slos_lockstep_last_error.restype = C.c_char_p
        lib.slos_lockstep_simulate.argtypes = [C.c_int32, C.POINTER(C.c_char_p), C.c_void_p, C.c_int32,
                                               C.POINTER(SimConfig), C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                               C.POINTER(C.c_double), C.POINTER(SimSummary), C.POINTER(Stats)]
        lib.slos_lockstep_capacity.argtypes = [C.c_int32, C.POINTER(C.c_char_p), C.c_void_p, C.c_int32,
                                               C.POINTER(SimConfig), C.c_double, C.c_double, C.c_double,
                                               C.c_double, C.c_int32, C.c_uint64, C.c_double,
                                               C.POINTER(CapacityResult), C.POINTER(Stats)]
        self.lib = lib
        self.backend(backend)

    def _check(self, st):
        if st != 0:
            raise RuntimeError(f"lockstep status {st}: {self.lib.slos_lockstep_last_error().decode()}")

    def backend(self, path):
        """None: the reference SloScheduler per replica; else a library exporting
        slos_planner.h (the product libslos_b200.so), served through its broker."""
        self._check(self.lib.slos_lockstep_set_backend(path.encode() if path else None))

    def simulate(self, lanes, model=DESK):
        """lanes: list of (scenario, Sim, seed, horizon_s, scale). Returns (summaries, stats)."""
        n = len(lanes)
        paths = (C.c_char_p * n)(*[scenario_path(l[0]).encode() for l in lanes])
        cfgs = (SimConfig * n)(*[l[1].c() for l in lanes])
        seeds = (C.c_uint64 * n)(*[l[2] for l in lanes])
        hor = (C.c_double * n)(*[l[3] for l in lanes])
        sc = (C.c_double * n)(*[l[4] for l in lanes])
        outs = (SimSummary * n)()
        st = Stats()
        t, nt = _terms(model)
        self._check(self.lib.slos_lockstep_simulate(n, paths, C.cast(t, C.c_void_p), nt, cfgs, seeds, hor, sc,
                                                    outs, C.byref(st)))
        res = [{f: getattr(o, f) for f, _ in SimSummary._fields_} for o in outs]
        return res, {f: getattr(st, f) for f, _ in Stats._fields_}

    def capacity(self, searches, seeds=2, horizon_s=10.0, target=0.9, lo=0.25, hi=8.0, rel_tol=0.1, base_seed=1,
                 model=DESK):
        """searches: list of (scenario, Sim). Returns (results, stats)."""
        n = len(searches)
        paths = (C.c_char_p * n)(*[scenario_path(s[0]).encode() for s in searches])
        cfgs = (SimConfig * n)(*[s[1].c() for s in searches])
        outs = (CapacityResult * n)()
        st = Stats()
        t, nt = _terms(model)
        self._check(self.lib.slos_lockstep_capacity(n, paths, C.cast(t, C.c_void_p), nt, cfgs, target, lo, hi,
                                                    rel_tol, seeds, base_seed, horizon_s, outs, C.byref(st)))
        res = [{"scale": o.scale, "per_gpu_rate": o.per_gpu_rate, "attainment": o.attainment,
                "evaluations": o.evaluations} for o in outs]
        return res, {f: getattr(st, f) for f, _ in Stats._fields_}
