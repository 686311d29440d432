"""TEST INFRASTRUCTURE: ctypes wrapper of oracle/_ref/libslos_refsim.so -- the
reference's own simulator (ReplicaSim / ClusterSim) and capacity sweep
(simulate_scenario / capacity_search) with its scheduler factory hooked, so the
planner behind `Scheduler::schedule` can be the reference SloScheduler or any
library exporting include/slos_planner.h (see oracle/ref_sim.cpp).

Scenario and model fixtures live in tests/golden/scenarios/ (our own
parameterisations in the reference's scenario-file format, workload.cpp:294-338).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

from paper_2504_08784_b200 import abi

REFSIM_LIB = os.path.join(abi.ROOT, "oracle", "_ref", "libslos_refsim.so")
SCEN = os.path.join(abi.ROOT, "tests", "golden", "scenarios")
# the desk perf model, passed as terms
DESK = [(2.5e-5, 2e-3, 0.006), (0.0, 0.0, 0.02)]


def _terms(model):
    arr = (abi.PerfTerm * len(model))(*[abi.PerfTerm(*t) for t in model])
    return arr, len(model)


class SimConfig(C.Structure):
    _fields_ = [("speculative", C.c_int32), ("spec_max_len", C.c_int32), ("spec_alpha", C.c_double),
                ("noise", C.c_double), ("memory_units", C.c_int64), ("max_chunk_tokens", C.c_int64),
                ("max_batch_tokens", C.c_int64), ("replicas", C.c_int32), ("routing_limit", C.c_int32),
                ("backup_best_effort", C.c_int32), ("reserved0", C.c_int32), ("net_delay_s", C.c_double)]


class SimSummary(C.Structure):
    _fields_ = [("requests", C.c_int64), ("standard", C.c_int64), ("attained", C.c_int64),
                ("best_effort", C.c_int64), ("dropped", C.c_int64), ("total_hops", C.c_int64),
                ("plans", C.c_int64), ("tokens_out", C.c_int64), ("attainment", C.c_double),
                ("overall_attainment", C.c_double), ("digest", C.c_uint64)]


@dataclass
class Sim:
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
    return os.path.exists(REFSIM_LIB)


class RefSim:
    def __init__(self):
        lib = C.CDLL(REFSIM_LIB)
        lib.slos_sim_set_backend.argtypes = [C.c_char_p]
        lib.slos_sim_set_recording.argtypes = [C.c_int32]
        lib.slos_sim_recorded_count.restype = C.c_int64
        lib.slos_sim_recorded_write.argtypes = [C.c_char_p]
        lib.slos_sim_last_error.restype = C.c_char_p
        lib.slos_sim_scenario.argtypes = [C.c_char_p, C.c_void_p, C.c_int32, C.POINTER(SimConfig), C.c_uint64,
                                          C.c_double, C.c_double, C.POINTER(SimSummary)]
        lib.slos_sim_capacity.argtypes = [C.c_char_p, C.c_void_p, C.c_int32, C.POINTER(SimConfig), C.c_double,
                                          C.c_double, C.c_double, C.c_double, C.c_int32, C.c_uint64,
                                          C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        self.lib = lib

    def _check(self, st):
        if st != 0:
            raise RuntimeError(f"refsim status {st}: {self.lib.slos_sim_last_error().decode()}")

    def backend(self, path):
        """None: the reference SloScheduler; else a library exporting slos_planner.h."""
        self._check(self.lib.slos_sim_set_backend(path.encode() if path else None))

    def run(self, scenario: str, sim: Sim, seed: int = 1, horizon_s: float = 20.0,
            scale: float = 1.0, model=DESK) -> dict:
        cfg = sim.c()
        out = SimSummary()
        t, n = _terms(model)
        self._check(self.lib.slos_sim_scenario(os.path.join(SCEN, scenario + ".json").encode(),
                                               C.cast(t, C.c_void_p), n, C.byref(cfg), seed, horizon_s, scale,
                                               C.byref(out)))
        return {f: getattr(out, f) for f, _ in SimSummary._fields_}

    def capacity(self, scenario: str, sim: Sim, seeds: int = 2, horizon_s: float = 10.0,
                 target: float = 0.9, lo: float = 0.25, hi: float = 8.0, rel_tol: float = 0.1,
                 base_seed: int = 1, model=DESK) -> dict:
        cfg = sim.c()
        t, nt = _terms(model)
        s, r, a = C.c_double(), C.c_double(), C.c_double()
        n = C.c_int32()
        self._check(self.lib.slos_sim_capacity(os.path.join(SCEN, scenario + ".json").encode(),
                                               C.cast(t, C.c_void_p), nt, C.byref(cfg), target, lo, hi, rel_tol, seeds, base_seed,
                                               horizon_s, C.byref(s), C.byref(r), C.byref(a), C.byref(n)))
        return {"scale": s.value, "per_gpu_rate": r.value, "attainment": a.value, "evaluations": n.value}

    def record(self, on: bool):
        self.lib.slos_sim_set_recording(1 if on else 0)

    def recorded(self) -> int:
        return int(self.lib.slos_sim_recorded_count())

    def write_recorded(self, path: str):
        self._check(self.lib.slos_sim_recorded_write(path.encode()))
