"""Golden-fixture checks shared by the oracle pinning tests (CPU) and the product
parity tests (GPU). Every fixture was produced by the UNMODIFIED reference
(oracle/make_golden.py); comparisons are bit-exact via canonical-byte digests."""
import numpy as np

from golden_io import load
from parity import plan_many, plan_one, summary
from paper_2504_08784_b200 import workload as W
from paper_2504_08784_b200.planner import PlannerConfig, _CInput, _Handle
from fuzz import random_case


def _cmp(got, want, what):
    g, w = summary(got), want
    if g != w:
        keys = [k for k in set(g) | set(w) if g.get(k) != w.get(k)]
        raise AssertionError(f"{what}: mismatch in {sorted(keys)}: got {({k: g.get(k) for k in keys})} "
                             f"want {({k: w.get(k) for k in keys})}")


def check_oracle_instances(lib, batched=False):
    fams = load("oracle_instances")
    n = 0
    for name, fam in fams.items():
        unit = fam["unit_value"]
        for idx, item in enumerate(fam["items"]):
            f = W.oracle_fields(item["rec"])
            h = _Handle(lib, W.oracle_model(f), W.oracle_slo(f), PlannerConfig())
            ci = _CInput(W.oracle_input(f))
            got = plan_one(lib, h.ptr, ci.c, unit_value=unit)
            _cmp(got, item["ref"], f"oracle family {name} instance {idx}")
            n += 1
    return n


def check_stress(lib, families=("C1", "LAT", "C2", "C3", "C4")):
    st = load("stress")
    for fam in families:
        F = W.FAMILIES[fam]
        b = W.InstanceBatch.stress(F["spec"], st[fam]["seeds"])
        h = _Handle(lib, F["model"], W.TWO_TIER_SLO, F["cfg"])
        res = plan_many(lib, h.ptr, b)
        for k, (got, want) in enumerate(zip(res, st[fam]["ref"])):
            _cmp(got, want, f"{fam} seed {st[fam]['seeds'][k]}")


def check_fuzz(lib, seeds=None):
    fz = load("fuzz")
    for case in fz:
        if seeds is not None and case["seed"] not in seeds:
            continue
        terms, slo, cfg, inp = random_case(case["seed"])
        ci = _CInput(inp)
        h = _Handle(lib, terms, slo, cfg)
        _cmp(plan_one(lib, h.ptr, ci.c, False), case["value"], f"fuzz {case['seed']} value")
        _cmp(plan_one(lib, h.ptr, ci.c, True), case["throughput"], f"fuzz {case['seed']} throughput")


def check_c5(lib, groups=("ar", "spec"), limit=None):
    """The C5 sweep corpus: inputs recorded from the reference simulator
    (oracle/make_corpus.py), reference results as goldens."""
    import os
    from golden_io import GOLDEN
    from paper_2504_08784_b200.planner import PerfTerm
    meta = load("c5")
    n = 0
    for g in groups:
        G = meta["groups"][g]
        b = W.load_corpus(os.path.join(GOLDEN, f"c5_{g}.bin.gz"))
        if limit:
            b = b.subset(range(min(limit, b.n)))
        cfg = PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=G["speculative"],
                            spec_alpha=0.8, spec_max_len=8, plan_margin=0.0)
        h = _Handle(lib, [PerfTerm(*t) for t in meta["model"]], W.TWO_TIER_SLO, cfg)
        res = plan_many(lib, h.ptr, b)
        for k, got in enumerate(res):
            _cmp(got, G["ref"][k], f"c5 {g} instance {k}")
        n += len(res)
    return n
