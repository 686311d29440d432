"""Batched multi-replica routing rounds (include/slos_route.h):
the product's slos_route_rounds against an independent Python restatement of the
reference's routing (tests/route_oracle.py) planning with the REFERENCE planner.

CPU: the same C++ driver (paper_2504_08784_b200/csrc/slos_route.cpp) linked over
the C oracle planner (oracle/_ref/libslos_route_oracle.so) vs the restatement
over the compiled reference. GPU: the product (every round one launch)."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2504_08784_b200 import abi
from paper_2504_08784_b200 import workload as W
from paper_2504_08784_b200.planner import _Handle
from paper_2504_08784_b200.routing import c3_snapshots, route_rounds
from route_oracle import route_rounds_py

ROUTE_ORACLE = os.path.join(abi.ROOT, "oracle", "_ref", "libslos_route_oracle.so")

CONFIGS = [dict(), dict(backup_best_effort=False), dict(routing_limit=1), dict(replicas=2),
           dict(net_delay_s=0.01, routing_limit=2)]


def _dense(n_clusters, replicas, seed0=0):
    # C1-size replicas with 16 arrivals each: many declines, so routing matters
    F = W.FAMILIES["C1"]
    return W.InstanceBatch.stress(F["spec"], range(seed0, seed0 + n_clusters * replicas), unique_ids=True), F


def _compare(lib, n_clusters=6):
    ref = abi.reference()
    for kw in CONFIGS:
        R = kw.get("replicas", 4)
        for snaps, F in (c3_snapshots(n_clusters, R), _dense(n_clusters, R, 100)):
            hp = _Handle(lib, F["model"], W.TWO_TIER_SLO, F["cfg"])
            hr = _Handle(ref, F["model"], W.TWO_TIER_SLO, F["cfg"])
            got, st = route_rounds(lib, [hp.ptr] * snaps.n, n_clusters, snaps, **kw)
            want, wst = route_rounds_py(ref, [hr.ptr] * snaps.n, n_clusters, snaps, **kw)
            assert got.tobytes() == want.tobytes(), kw
            assert st["plans"] == wst["plans"] and st["rounds"] == wst["rounds"]
            yield got, st


@pytest.mark.skipif(not (os.path.exists(ROUTE_ORACLE) and os.path.exists(abi.REF_LIB)),
                    reason="oracle/_ref not built")
def test_route_driver_over_c_oracle_matches_reference_restatement():
    lib = abi.load(ROUTE_ORACLE)
    _bind_route(lib)
    rerouted = 0
    for got, st in _compare(lib):
        rerouted += int((got["hops"] > 0).sum())
    assert rerouted > 0  # declines were re-offered around the ring


def _bind_route(lib):
    from paper_2504_08784_b200.routing import _bind
    _bind(lib)


@pytest.mark.gpu
def test_route_rounds_on_b200_match_reference_restatement():
    if not os.path.exists(abi.REF_LIB):
        pytest.skip("oracle/_ref not built")
    rerouted = 0
    for got, st in _compare(abi.product(), n_clusters=16):
        rerouted += int((got["hops"] > 0).sum())
        assert st["rounds"] >= 1
    assert rerouted > 0
