"""TEST INFRASTRUCTURE: the C5 sweep corpus -- every
`Scheduler::schedule` input the REFERENCE simulator produces over a capacity-
sweep grid, recorded by oracle/_ref/libslos_refsim.so (the reference's
simulate_scenario / ClusterSim with a recording SloScheduler), plus the reference
planner's result on each recorded input as the golden.

Grid: scenarios {chatbot, coder, summarizer, toolllm, reasoning (speculative)} x
clusters {1 replica, 4 replicas with ring routing} x rate scales {0.5, 1, 2, 4} x
seeds {1, 2}, bursty arrivals, memory_units 8192, 20 s horizon. The recorded
inputs are subsampled with a fixed stride to at most PER_GROUP instances per
planner configuration (speculative off / on) and written to
tests/golden/c5_{ar,spec}.bin.gz; tests/golden/c5.json.gz holds the planner
configurations, the provenance and the reference summaries.

  python oracle/make_corpus.py        (needs /root/reference built: make -C oracle ref)
"""
from __future__ import annotations

import gzip
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.planner import PerfTerm, PlannerConfig, _Handle  # noqa: E402
from parity import plan_many, summary  # noqa: E402
from sim_harness import DESK, RefSim, Sim  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
PER_GROUP = 2048
SCALES = (0.5, 1.0, 2.0, 4.0)
SEEDS = (1, 2)
HORIZON = 20.0


def planner_cfg(spec: bool) -> PlannerConfig:
    # ReplicaSim's PlannerConfig (sim_executor.cpp:52-58) for Sim() defaults
    return PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=spec, spec_alpha=0.8,
                         spec_max_len=8, plan_margin=0.0)


def record_group(rs: RefSim, scenarios, spec: bool, path: str) -> list:
    prov = []
    if os.path.exists(path):
        os.remove(path)
    for scen in scenarios:
        for reps in (1, 4):
            for scale in SCALES:
                for seed in SEEDS:
                    rs.record(True)
                    r = rs.run(scen, Sim(speculative=spec, replicas=reps), seed=seed, horizon_s=HORIZON,
                               scale=scale)
                    n = rs.recorded()
                    rs.write_recorded(path)
                    rs.record(False)
                    prov.append(dict(scenario=scen, replicas=reps, scale=scale, seed=seed, plans=n,
                                     requests=r["requests"]))
    return prov


def main():
    rs = RefSim()
    rs.backend(None)
    ref = abi.reference()
    meta = {"model": DESK, "slo": {"tpot_tiers_s": [0.05, 0.1], "ttft_slowdowns": [3.0, 5.0], "tpot_window": 10},
            "horizon_s": HORIZON, "groups": {}}
    for name, scens, spec in (("ar", ("chatbot", "coder", "summarizer", "toolllm"), False),
                              ("spec", ("reasoning",), True)):
        with tempfile.TemporaryDirectory() as td:
            raw = os.path.join(td, "c.bin")
            prov = record_group(rs, scens, spec, raw)
            buf = open(raw, "rb").read()
        full = W.InstanceBatch.from_corpus(buf)
        stride = max(1, full.n // PER_GROUP)
        keep = np.arange(0, full.n, stride)[:PER_GROUP]
        # re-serialise only the kept instances: re-record from the parsed arrays
        sub = full.subset(keep)
        blob = serialise(sub)
        with gzip.open(os.path.join(OUT, f"c5_{name}.bin.gz"), "wb", compresslevel=9) as f:
            f.write(blob)
        cfg = planner_cfg(spec)
        h = _Handle(ref, [PerfTerm(*t) for t in DESK], W.TWO_TIER_SLO, cfg)
        chk = W.InstanceBatch.from_corpus(blob)
        res = plan_many(ref, h.ptr, chk)
        meta["groups"][name] = {"speculative": spec, "recorded": int(full.n), "stride": int(stride),
                                "count": int(chk.n), "provenance": prov,
                                "ref": [summary(r) for r in res]}
        print(name, "recorded", full.n, "kept", chk.n, "bytes", len(blob))
    with gzip.open(os.path.join(OUT, "c5.json.gz"), "wt", compresslevel=9) as f:
        json.dump(meta, f)


def serialise(b: W.InstanceBatch) -> bytes:
    """Back to the recorder's binary layout (oracle/ref_sim.cpp slos_sim_recorded_write)."""
    import ctypes as C
    import struct
    out = []
    rsz, psz = b.running.itemsize, b.pending.itemsize
    rbase, pbase = b.running.ctypes.data, b.pending.ctypes.data
    for inp in b.inputs:
        nr, npn = int(inp["n_running"]), int(inp["n_pending"])
        out.append(struct.pack("<ddqqii", inp["now"], inp["tail_horizon_s"], inp["memory_total"],
                               inp["memory_standard_resident"], nr, npn))
        r0 = (int(inp["running"]) - rbase) // rsz
        p0 = (int(inp["pending"]) - pbase) // psz
        ids = []
        for r in b.running[r0:r0 + nr]:
            out.append(struct.pack("<qdiidqq", r["prefill_remaining"], r["prefill_deadline"], r["decode_tier"], 0,
                                   r["next_due_s"], r["backlog"], r["decode_remaining"]))
            ids.append(C.string_at(int(r["id"])))
        for p in b.pending[p0:p0 + npn]:
            out.append(struct.pack("<dqiiqd", p["prefill_deadline"], p["prefill_tokens"], p["decode_tier"], 0,
                                   p["memory_units"], p["value"]))
            ids.append(C.string_at(int(p["id"])))
        for s in ids:
            out.append(struct.pack("<H", len(s)) + s)
    return b"".join(out)


if __name__ == "__main__":
    main()
