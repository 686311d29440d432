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
# the device PerfModel::fit: one set staged in shared memory, one read from HBM
from paper_2504_08784_b200 import fit as FT  # noqa: E402
import numpy as np  # noqa: E402
rng = np.random.default_rng(5)
sets = []
for cnt in (300, 6000):
    n = rng.integers(1, 8193, cnt)
    s_ = rng.choice([0, 2, 5], cnt)
    lat = np.maximum(2.5e-5 * n + 2e-3 * s_ + 0.006, 0.02) * (1 + rng.uniform(-0.01, 0.01, cnt))
    sets.append(FT.as_samples(n, s_, lat))
got, st = FT.fit_batch(sets, 2)
ok = all(got[k].tobytes() == FT.reference_fit(sets[k], 2)[0].tobytes() for k in range(2)) \
    if os.path.exists(abi.REF_LIB) else None
print("fit", list(st), "identical to reference:", ok, flush=True)
print("sanitize workload done")
