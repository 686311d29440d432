"""Batched routing rounds and lockstep simulation lanes (include/slos_lockstep.h,
SURVEY.md §8 rows a13, a14, f1).

integration/_build/libslos_lockstep.so runs the reference's own ReplicaSim in
conservative-lookahead windows (replicas of a cluster advance concurrently between
routing hops), many simulations as concurrent lanes, and serves every waiting
schedule() through the backend's plan broker in one batched launch. Each run must
be IDENTICAL to the reference's sequential ClusterSim::run / simulate_scenario /
capacity_search with the reference SloScheduler (oracle/_ref/libslos_refsim.so):
a digest over every field of every RequestRecord, and the capacity results.

CPU: the lockstep driver with the reference planner and with the C oracle.
GPU: with the product behind the broker (batched launches).
"""
import pytest

from paper_2504_08784_b200 import abi
from paper_2504_08784_b200.lockstep import Lockstep, Sim, available
from sim_harness import RefSim
from sim_harness import Sim as RSim
from sim_harness import available as ref_available

pytestmark = pytest.mark.skipif(not (available() and ref_available()), reason="lockstep or refsim not built")

# routing: 2- and 4-replica rings, both backup policies, speculative decoding,
# a zero-delay network (no lookahead: one reference iteration per window)
CASES = [
    ("chatbot", Sim(replicas=4, routing_limit=3), 3.0),
    ("reasoning", Sim(replicas=4, speculative=True), 2.0),
    ("coder", Sim(replicas=2, routing_limit=1, backup_best_effort=False), 4.0),
    ("summarizer", Sim(replicas=3, routing_limit=2, backup_best_effort=False, net_delay_s=0.005), 3.0),
    ("toolllm", Sim(replicas=4, routing_limit=2), 2.0),
    ("chatbot", Sim(replicas=2, net_delay_s=0.0), 2.0),
    ("chatbot", Sim(), 1.0),
]


def _want(cases, seed=7, horizon_s=20.0):
    rs = RefSim()
    rs.backend(None)
    return [rs.run(s, RSim(**sim.__dict__), seed=seed, horizon_s=horizon_s, scale=sc) for s, sim, sc in cases]


def _check(backend, cases=CASES, seed=7, horizon_s=20.0):
    want = _want(cases, seed, horizon_s)
    ls = Lockstep(backend)
    got, st = ls.simulate([(s, sim, seed, horizon_s, sc) for s, sim, sc in cases])
    ls.backend(None)
    for g, w, c in zip(got, want, cases):
        assert w["plans"] > 0
        assert g == w, c
    assert st["plans"] == sum(w["plans"] for w in want)
    return st


def _capacity(backend):
    rs = RefSim()
    rs.backend(None)
    searches = [("chatbot", Sim(replicas=2)), ("coder", Sim())]
    want = [rs.capacity(s, RSim(**sim.__dict__), seeds=2, horizon_s=8.0, lo=0.05, hi=4.0, target=0.9)
            for s, sim in searches]
    ls = Lockstep(backend)
    got, st = ls.capacity(searches, seeds=2, horizon_s=8.0, lo=0.05, hi=4.0, target=0.9)
    ls.backend(None)
    assert got == want
    return st


def test_lockstep_with_reference_planner_matches_sequential_clustersim():
    _check(None)


def test_lockstep_with_c_oracle_matches_reference():
    _check(abi.ORACLE_LIB)


def test_lockstep_lanes_of_one_scenario_over_seeds():
    cases = [("reasoning", Sim(replicas=4, speculative=True), 2.0)] * 3
    for seed in (1, 2):
        _check(abi.ORACLE_LIB, cases, seed=seed, horizon_s=10.0)


def test_lockstep_capacity_search_matches_reference():
    _capacity(abi.ORACLE_LIB)


@pytest.mark.gpu
def test_lockstep_with_b200_planner_matches_reference():
    st = _check(abi.PRODUCT_LIB)
    assert st["flushes"] < st["plans"]  # the broker batched concurrent replans


@pytest.mark.gpu
def test_lockstep_capacity_search_with_b200_planner_matches_reference():
    st = _capacity(abi.PRODUCT_LIB)
    assert st["flushes"] < st["plans"]
