"""Pin the C oracle (oracle/slos_oracle.c) against the reference.

(1) against golden fixtures written by the compiled reference (always, CPU);
(2) against the compiled reference itself, live, when oracle/_ref is built;
(3) against the reference's own known answers (brute-force optimum, including the
    reference's documented miss on acceptance instance 102 of seed 20240817)."""
import os

import pytest

from golden_checks import check_c5, check_fuzz, check_oracle_instances, check_stress
from golden_io import load
from paper_2504_08784_b200 import abi


def test_oracle_matches_reference_on_brute_force_families():
    assert check_oracle_instances(abi.oracle()) == 811


def test_oracle_matches_reference_on_stress_families():
    check_stress(abi.oracle(), families=("C1", "LAT", "C2", "C3"))


def test_oracle_matches_reference_on_c5_simulator_corpus():
    # 4,096 inputs recorded from the reference simulator over the sweep grid
    assert check_c5(abi.oracle()) == 4096


def test_oracle_matches_reference_on_fuzz():
    check_fuzz(abi.oracle())


def test_reference_known_answers_reproduced():
    fams = load("oracle_instances")
    # test_dp_scheduler.cpp:30-50: value == brute-force optimum on the 250 draws of seed 424242
    for it in fams["424242"]["items"]:
        assert it["ref"]["value_bits"] is not None
        assert abs(_val(it) - it["best_value"]) <= 1e-12 * max(1.0, it["best_value"])
        assert it["ref_subset_feasible"] == 1
    # acceptance_main.cpp:132-167: instance 102 is a known reference miss (0 vs 29)
    miss = fams["20240817"]["items"][102]
    assert miss["best_value"] == 29.0 and _val(miss) == 0.0 and miss["ref"]["infeasible"] == 1
    bad = [i for i, it in enumerate(fams["20240817"]["items"]) if abs(_val(it) - it["best_value"]) > 1e-9]
    assert bad == [102]
    # throughput objective == unit-value optimum (test_dp_scheduler.cpp:177-190)
    for it in fams["909090"]["items"]:
        assert len(it["ref"]["admitted"]) == it["best_value"]


def _val(it):
    import struct
    return struct.unpack("<d", struct.pack("<q", it["ref"]["value_bits"]))[0]


@pytest.mark.skipif(not os.path.exists(abi.REF_LIB), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_on_fresh_fuzz():
    import ctypes as C

    from fuzz import random_case
    from parity import diff, plan_one
    from paper_2504_08784_b200.planner import _CInput, _Handle
    ref, ora = abi.reference(), abi.oracle()
    for seed in range(5000, 5400):
        terms, slo, cfg, inp = random_case(seed, max_pending=12)
        ci = _CInput(inp)
        hr, ho = _Handle(ref, terms, slo, cfg), _Handle(ora, terms, slo, cfg)
        for uv in (False, True):
            a = plan_one(ref, hr.ptr, ci.c, uv)
            b = plan_one(ora, ho.ptr, ci.c, uv)
            assert not diff(a, b), (seed, uv, diff(a, b))


def test_oracle_work_counters_equal_instrumented_reference():
    """T/G/D/S/states (the roofline numerator) of the C oracle equal
    the counters measured inside the reference itself (oracle/instrument_ref.py:
    the reference sources patched with counters in a /tmp copy)."""
    from parity import plan_many
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import _Handle
    g = load("counters")
    ora = abi.oracle()
    for fam, take in (("C1", 16), ("LAT", 16), ("C3", 16), ("C2", 8)):
        F = W.FAMILIES[fam]
        seeds = g[fam]["seeds"][:take]
        b = W.InstanceBatch.stress(F["spec"], seeds)
        h = _Handle(ora, F["model"], W.TWO_TIER_SLO, F["cfg"])
        res = plan_many(ora, h.ptr, b)
        for k, r in enumerate(res):
            assert list(r["counters"]) == g[fam]["counters"][k], (fam, seeds[k])
