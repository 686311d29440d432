"""compute-sanitizer target (run under gpurun): a small mixed workload through every
kernel -- C2 / C1 stress instances (block- and warp-built reconstruction, fallback),
C4 (256-thread reconstruction), C3 (speculative), C5 corpus instances -- checked
against the C oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from parity import diff, plan_many  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.planner import _Handle  # noqa: E402

prod, ora = abi.product(), abi.oracle()
for fam, seeds in (("C2", range(120, 136)), ("C1", range(0, 24)), ("C3", range(0, 16)), ("C4", range(0, 2)),
                   ("LAT", range(0, 8))):
    F = W.FAMILIES[fam]
    b = W.InstanceBatch.stress(F["spec"], seeds)
    hp = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"])  # handles must outlive the calls
    ho = _Handle(ora, F["model"], W.TWO_TIER_SLO, F["cfg"])
    P = plan_many(prod, hp.ptr, b)
    O = plan_many(ora, ho.ptr, b)
    bad = [k for k in range(b.n) if diff(P[k], O[k], counters=True)]
    print(fam, b.n, "mismatches", bad, flush=True)
print("sanitize workload done")
