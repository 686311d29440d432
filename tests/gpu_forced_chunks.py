"""The host chunk pipeline with three chunks forced (SLOS_PIPELINE_CHUNKS=3, read once
per process, hence a script of its own: tests/test_parity_gpu.py runs it in a
subprocess) so the split collection, the three rotating workspaces and the chunked
upload reductions all run on small batches -- C5 corpus instances against the
reference's goldens, C2 stress instances (12, four per chunk) against the C oracle."""
import gzip
import json
import os
import sys

os.environ["SLOS_PIPELINE_CHUNKS"] = "3"  # read once, at the library's first batch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_checks import _cmp  # noqa: E402
from parity import diff, plan_many  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.planner import PerfTerm, PlannerConfig, _Handle  # noqa: E402

prod, ora = abi.product(), abi.oracle()
GOLDEN = os.path.join(ROOT, "tests", "golden")
meta = json.load(gzip.open(os.path.join(GOLDEN, "c5.json.gz"), "rt"))
for g in ("ar", "spec"):
    G = meta["groups"][g]
    b = W.load_corpus(os.path.join(GOLDEN, f"c5_{g}.bin.gz")).subset(range(1536))
    cfg = PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=G["speculative"],
                        spec_alpha=0.8, spec_max_len=8, plan_margin=0.0)
    h = _Handle(prod, [PerfTerm(*t) for t in meta["model"]], W.TWO_TIER_SLO, cfg)
    res = plan_many(prod, h.ptr, b)
    for k, got in enumerate(res):
        _cmp(got, G["ref"][k], f"c5 {g} instance {k}")
    print("C5", g, b.n, "match", flush=True)
F = W.FAMILIES["C2"]
b = W.InstanceBatch.stress(F["spec"], range(200, 212))
hp = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"])
ho = _Handle(ora, F["model"], W.TWO_TIER_SLO, F["cfg"])
P, O = plan_many(prod, hp.ptr, b), plan_many(ora, ho.ptr, b)
print("C2", b.n, "mismatches", [k for k in range(b.n) if diff(P[k], O[k], counters=True)], flush=True)
print("forced chunks done")
