"""Batched multi-replica routing rounds (include/slos_route.h).

`route_rounds` runs the product's slos_route_rounds: many clusters of R replica
snapshots; every round plans every replica that was offered requests, across all
clusters, in one slos_plan_batch, then re-offers the declines to the next replica
of the ring (ClusterSim::on_decline, tiers_router.cpp:80-108). `bench_leg` is
bench.py's C3 leg (BASELINE configs[2]: reasoning with speculative decoding,
4-replica routing).
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from . import abi
from . import workload as W

ROUTE_OUTCOME_DTYPE = np.dtype([("fate", "<i4"), ("replica", "<i4"), ("hops", "<i4"), ("round", "<i4")])
ADMITTED, BEST_EFFORT, DROPPED = 0, 1, 2


class RouteConfig(C.Structure):  # slos_route_config
    _fields_ = [("replicas", C.c_int32), ("routing_limit", C.c_int32), ("backup_best_effort", C.c_int32),
                ("unit_value", C.c_int32), ("net_delay_s", C.c_double)]


class RouteStats(C.Structure):  # slos_route_stats
    _fields_ = [("rounds", C.c_int64), ("plans", C.c_int64), ("admitted", C.c_int64),
                ("best_effort", C.c_int64), ("dropped", C.c_int64)]


def _bind(lib):
    f = lib.slos_route_rounds
    f.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(RouteConfig), C.c_void_p, C.c_void_p,
                  C.POINTER(RouteStats)]
    f.restype = C.c_int
    return f


def route_rounds(lib, handles, n_clusters: int, snapshots: W.InstanceBatch, replicas: int = 4,
                 routing_limit: int = 3, backup_best_effort: bool = True, net_delay_s: float = 0.001,
                 unit_value: bool = False):
    """Returns (outcomes[structured array, one per pending entry], stats dict)."""
    f = _bind(lib)
    n = n_clusters * replicas
    assert snapshots.n == n and len(handles) == n
    hs = (C.c_void_p * n)(*handles)
    cfg = RouteConfig(replicas, routing_limit, int(backup_best_effort), int(unit_value), net_delay_s)
    n_out = int(snapshots.inputs["n_pending"].sum())
    out = np.zeros(max(1, n_out), ROUTE_OUTCOME_DTYPE)
    st = RouteStats()
    r = f(hs, n_clusters, C.byref(cfg), C.c_void_p(snapshots.inputs_ptr()), C.c_void_p(out.ctypes.data),
          C.byref(st))
    if r != abi.SLOS_OK:
        raise RuntimeError(f"slos_route_rounds: status {r}: {lib.slos_last_error().decode()}")
    return out[:n_out], {f_: getattr(st, f_) for f_, _ in RouteStats._fields_}


def c3_snapshots(n_clusters: int, replicas: int = 4, seed0: int = 0, gen=None):
    """each replica a G(124, 4) snapshot (reasoning + speculative
    decoding, desk model), replica r of cluster c drawn with seed seed0 + c*R + r;
    request ids are unique across the cluster (routed requests move)."""
    F = W.FAMILIES["C3"]
    return W.InstanceBatch.stress(F["spec"], range(seed0, seed0 + n_clusters * replicas), gen=gen,
                                  unique_ids=True), F


def bench_leg(lib, stream, steps, warmup, with_cpu, n_clusters: int = 256):
    """C3 leg: n_clusters 4-replica clusters (1024 replica snapshots G(124, 4), spec
    on), routing rounds end to end through slos_route_rounds (host inputs, every
    round's plans in one launch); the reference planner on all host cores runs the
    same rounds (tests/route_oracle.py's restatement over oracle/_ref)."""
    from .planner import _Handle
    snaps, F = c3_snapshots(n_clusters)
    h = _Handle(lib, F["model"], W.TWO_TIER_SLO, F["cfg"])
    hs = [h.ptr] * snaps.n
    for _ in range(max(2, warmup)):
        route_rounds(lib, hs, n_clusters, snaps)
    wall, plans, rounds = 0.0, 0, 0
    for _ in range(steps):
        t0 = time.perf_counter()
        out, st = route_rounds(lib, hs, n_clusters, snaps)
        wall += time.perf_counter() - t0
        plans += st["plans"]
        rounds += st["rounds"]
    fates = np.bincount(out["fate"], minlength=3)
    leg = {"workload": "C3: reasoning + speculative decoding (spec_max_len 8), 4-replica routing rounds "
                       f"(routing_limit 3, net_delay 1 ms, best_effort_on_origin), {n_clusters} clusters x 4 "
                       "replica snapshots G(124, 4) (BASELINE configs[2])",
           "value": plans / wall, "unit": "plans/s", "ms_per_step": 1e3 * wall / steps,
           "rounds_per_step": rounds / steps, "plans_per_step": plans / steps,
           "e2e": {"value": plans / wall, "unit": "plans/s",
                   "note": "host snapshots -> slos_route_rounds -> host outcomes, every round one launch"},
           "outcomes": {"admitted": int(fates[0]), "best_effort": int(fates[1]), "dropped": int(fates[2]),
                        "rerouted": int((out["hops"] > 0).sum())}}
    if with_cpu and os.path.exists(abi.REF_LIB):
        import sys
        sys.path.insert(0, os.path.join(abi.ROOT, "tests"))
        from route_oracle import route_rounds_py  # the checker / CPU baseline (oracle/_ref planner)
        ref = abi.reference()
        nc = max(4, min(n_clusters, 4 * int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))))
        sn, _ = c3_snapshots(nc, gen=abi.reference_stress_gen())
        hr = _Handle(ref, F["model"], W.TWO_TIER_SLO, F["cfg"])
        t0 = time.perf_counter()
        _, rst = route_rounds_py(ref, [hr.ptr] * sn.n, nc, sn)
        dt = time.perf_counter() - t0
        leg["cpu_baseline"] = {"value": rst["plans"] / dt, "unit": "plans/s",
                               "cores": int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1)),
                               "kind": "reference", "sample": f"{nc} clusters ({rst['plans']} plans), {dt:.2f} s"}
    return leg
