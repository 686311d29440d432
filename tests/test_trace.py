"""Batched trace generation (include/slos_trace.h) against the reference's own
scale_scenario + generate_trace (metrics.cpp:214-221, workload.cpp:159-206),
compiled unmodified in oracle/_ref. Host-only code: runs in the CPU suite."""
import copy
import glob
import json
import os

import numpy as np
import pytest

from paper_2504_08784_b200 import abi
from paper_2504_08784_b200 import trace as TR

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "scenarios", "*.json")))


def _ref_available():
    return os.path.exists(abi.REF_LIB)


need_ref = pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built")


def _variants():
    """Every scenario file as given and with bursty arrivals (coder.json's burst
    parameters applied to all, as the C5 sweep does), plus edge configurations."""
    out = []
    for p in SCEN:
        d = json.load(open(p))
        out.append(d)
        b = copy.deepcopy(d)
        b["arrival"] = dict(b.get("arrival", {}), process="bursty", on_multiplier=6.0, mean_on_s=4.0,
                            mean_off_s=12.0)
        out.append(b)
    base = json.load(open(SCEN[0]))
    z = copy.deepcopy(base)  # deterministic lengths (std 0 -> llround(mean))
    z["prompt_tokens"] = {"mean": 300.4, "std": 0}
    if "output_tokens" in z:
        z["output_tokens"] = {"mean": 2.5, "std": 0}
    out.append(z)
    o = copy.deepcopy(base)
    o["memory_overprovision"] = 1.37
    o["value"] = 2.5
    out.append(o)
    return out


@need_ref
def test_traces_match_reference_bit_for_bit():
    pts = []
    for d in _variants():
        sc = TR.scenario_from_json(d)
        for scale in (0.25, 1.0, 3.5):
            for seed in (0, 1, 7, 12345, 2**63 + 5):
                pts.append((sc, scale, seed, 40.0))
    got = TR.generate_traces(pts, threads=4)
    want = TR.reference_traces(pts)
    n_req = 0
    for k, ((gs, gr, gt), (ws, wr, wt)) in enumerate(zip(got, want)):
        assert gs == ws == 0, (k, gs, ws)
        assert gr.tobytes() == wr.tobytes(), f"job {k}: requests differ"
        assert gt.tobytes() == wt.tobytes(), f"job {k}: stages differ"
        n_req += len(gr)
    assert n_req > 1000


@need_ref
def test_trace_errors_match_reference():
    base = json.load(open(SCEN[0]))
    bad = []
    d = copy.deepcopy(base); d["prompt_tokens"] = {"mean": 0.5, "std": 1}; bad.append((d, 1.0, 30.0))
    d = copy.deepcopy(base); d["arrival"] = {"process": "bursty", "rate_per_s": 1.0, "on_multiplier": 0.5}
    bad.append((d, 1.0, 30.0))
    d = copy.deepcopy(base); d["prefill_tier"] = 5; bad.append((d, 1.0, 30.0))          # invariant-violation
    d = copy.deepcopy(base); d["memory_overprovision"] = 0.5; bad.append((d, 1.0, 30.0))
    d = copy.deepcopy(base); d["shape"] = "pipeline"; bad.append((d, 1.0, 30.0))
    d = copy.deepcopy(base); d["slo"] = dict(d["slo"], tpot_tiers_s=[0.1, 0.05]); bad.append((d, 1.0, 30.0))
    bad.append((copy.deepcopy(base), 0.0, 30.0))    # rate scale must be positive
    bad.append((copy.deepcopy(base), 1.0, 0.0))     # duration must be positive
    pts = [(TR.scenario_from_json(d), s, 3, dur) for d, s, dur in bad]
    got = TR.generate_traces(pts)
    want = TR.reference_traces(pts)
    for k, (g, w) in enumerate(zip(got, want)):
        assert g[0] == w[0] != 0, (k, TR.ERR_SLUGS.get(g[0]), TR.ERR_SLUGS.get(w[0]))


def test_trace_batch_deterministic_across_thread_counts():
    sc = TR.scenario_from_json(json.load(open(SCEN[0])))
    pts = [(sc, 1.0 + 0.1 * k, k, 20.0) for k in range(24)]
    a = TR.generate_traces(pts, threads=1)
    b = TR.generate_traces(pts, threads=8)
    for x, y in zip(a, b):
        assert x[0] == y[0] == 0
        assert x[1].tobytes() == y[1].tobytes() and x[2].tobytes() == y[2].tobytes()
