"""GPU bring-up diagnostics (run directly under gpurun): per-family mismatch
counts of product vs oracle, with the first differing batch/entry spelled out."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from fuzz import random_case  # noqa: E402
from golden_io import load  # noqa: E402
from parity import diff, plan_many, plan_one  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.planner import PlannerConfig, _CInput, _Handle  # noqa: E402


def explain(a, b):
    out = []
    for k in ("status", "infeasible", "value", "admitted", "declined", "exact_until_bits", "counters"):
        if a.get(k) != b.get(k):
            out.append(f"{k}: prod={a.get(k)} oracle={b.get(k)}")
    if a.get("status") == 0 and b.get("status") == 0:
        x, y = a["batches"], b["batches"]
        out.append(f"n_batches prod={len(x)} oracle={len(y)}; n_entries prod={len(a['entries'])} oracle={len(b['entries'])}")
        for i in range(min(len(x), len(y))):
            if x[i].tobytes() != y[i].tobytes():
                out.append(f"batch {i}: prod={x[i]} oracle={y[i]}")
                break
        ex, ey = a["entries"], b["entries"]
        for i in range(min(len(ex), len(ey))):
            if ex[i].tobytes() != ey[i].tobytes():
                out.append(f"entry {i}: prod={ex[i]} oracle={ey[i]}")
                break
    return "\n    ".join(out)


def main():
    prod, ora = abi.product(), abi.oracle()
    print("backend", prod.slos_backend())
    for fam, seeds in (("C1", range(16)), ("LAT", range(8)), ("C3", range(16)), ("C2", range(8))):
        F = W.FAMILIES[fam]
        b = W.InstanceBatch.stress(F["spec"], list(seeds))
        hp, ho = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"]), _Handle(ora, F["model"], W.TWO_TIER_SLO, F["cfg"])
        t = time.time()
        P = plan_many(prod, hp.ptr, b)
        tp = time.time() - t
        O = plan_many(ora, ho.ptr, b)
        bad = [k for k in range(b.n) if diff(P[k], O[k], counters=True)]
        print(f"{fam}: {len(bad)}/{b.n} mismatches ({tp*1e3:.1f} ms product)", flush=True)
        for k in bad[:2]:
            print("  seed", list(seeds)[k], "\n    " + explain(P[k], O[k]), flush=True)
    fams = load("oracle_instances")
    nb = 0
    for name, fam in fams.items():
        for idx, item in enumerate(fam["items"]):
            f = W.oracle_fields(item["rec"])
            ci = _CInput(W.oracle_input(f))
            hp = _Handle(prod, W.oracle_model(f), W.oracle_slo(f), PlannerConfig())
            ho = _Handle(ora, W.oracle_model(f), W.oracle_slo(f), PlannerConfig())
            a = plan_one(prod, hp.ptr, ci.c, fam["unit_value"])
            o = plan_one(ora, ho.ptr, ci.c, fam["unit_value"])
            if diff(a, o, counters=True):
                nb += 1
                if nb <= 3:
                    print(f"  oracle-family {name}#{idx}\n    " + explain(a, o), flush=True)
    print("brute-force families mismatches:", nb, flush=True)
    nb = 0
    for seed in range(400):
        terms, slo, cfg, inp = random_case(seed)
        ci = _CInput(inp)
        hp, ho = _Handle(prod, terms, slo, cfg), _Handle(ora, terms, slo, cfg)
        for uv in (False, True):
            a, o = plan_one(prod, hp.ptr, ci.c, uv), plan_one(ora, ho.ptr, ci.c, uv)
            if diff(a, o, counters=True):
                nb += 1
                if nb <= 4:
                    print(f"  fuzz {seed} uv={uv} L={slo.num_tiers()} spec={cfg.speculative}\n    " + explain(a, o), flush=True)
    print("fuzz mismatches:", nb, flush=True)
    # a first throughput number
    F = W.FAMILIES["C2"]
    b = W.InstanceBatch.stress(F["spec"], range(1024))
    hp = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"])
    for rep in range(3):
        t = time.time()
        P = plan_many(prod, hp.ptr, b)
        print(f"C2 x1024 wall {time.time()-t:.3f}s  statuses {set(p['status'] for p in P)}", flush=True)


if __name__ == "__main__":
    main()
