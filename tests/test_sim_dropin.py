"""The planner as a drop-in inside the REFERENCE's own simulator, routing and
capacity sweep.

oracle/_ref/libslos_refsim.so is the reference's ReplicaSim / ClusterSim /
simulate_scenario / capacity_search compiled unmodified, with make_scheduler
hooked so `Scheduler::schedule` is served by the INTEGRATION.md adapter over a
library exporting include/slos_planner.h. Every run is compared with the same
simulation driven by the reference's own SloScheduler: identical RequestRecords
(a digest over every field and every stage), identical capacity results.

The CPU tests drive the C restatement (oracle/liboracle_slos.so) through the
adapter; the gpu tests drive the product (libslos_b200.so, sm_100a).
"""
import pytest

from paper_2504_08784_b200 import abi
from sim_harness import RefSim, Sim, available

pytestmark = pytest.mark.skipif(not available(), reason="oracle/_ref/libslos_refsim.so not built")

# (scenario, simulator/cluster config, rate scale): single replicas, speculative
# decoding, tool-calling stages, and 2/4-replica routing with both backup policies
CASES = [
    ("chatbot", Sim(), 1.0),
    ("chatbot", Sim(), 3.0),
    ("coder", Sim(), 2.0),
    ("summarizer", Sim(), 1.5),
    ("reasoning", Sim(speculative=True), 1.0),
    ("toolllm", Sim(), 2.0),
    ("chatbot", Sim(replicas=4, routing_limit=3), 3.0),
    ("coder", Sim(replicas=2, routing_limit=1, backup_best_effort=False), 4.0),
    ("reasoning", Sim(replicas=4, speculative=True), 2.0),
]


def _compare(backend, cases, seed=7, horizon_s=20.0):
    rs = RefSim()
    for scen, sim, scale in cases:
        rs.backend(None)
        want = rs.run(scen, sim, seed=seed, horizon_s=horizon_s, scale=scale)
        rs.backend(backend)
        got = rs.run(scen, sim, seed=seed, horizon_s=horizon_s, scale=scale)
        rs.backend(None)
        assert want["plans"] > 0
        assert got == want, (scen, sim, scale)


def _capacity(backend):
    rs = RefSim()
    for scen, sim in (("chatbot", Sim(replicas=2)), ("coder", Sim())):
        rs.backend(None)
        want = rs.capacity(scen, sim, seeds=2, horizon_s=8.0, lo=0.05, hi=4.0, target=0.9)
        rs.backend(backend)
        got = rs.capacity(scen, sim, seeds=2, horizon_s=8.0, lo=0.05, hi=4.0, target=0.9)
        rs.backend(None)
        assert want["evaluations"] > 1
        assert got == want, scen


def test_simulator_with_c_oracle_matches_reference():
    _compare(abi.ORACLE_LIB, CASES)


def test_capacity_search_with_c_oracle_matches_reference():
    _capacity(abi.ORACLE_LIB)


@pytest.mark.gpu
def test_simulator_with_b200_planner_matches_reference():
    _compare(abi.PRODUCT_LIB, CASES)


@pytest.mark.gpu
def test_capacity_search_with_b200_planner_matches_reference():
    _capacity(abi.PRODUCT_LIB)
