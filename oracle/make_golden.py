"""TEST INFRASTRUCTURE: writes tests/golden/*.json.gz from the UNMODIFIED reference
planner compiled in oracle/_ref/ (make -C oracle ref). Run in the container that
has /root/reference; the fixtures are committed and the GPU box only reads them.

  python oracle/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import gzip
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.planner import PlannerConfig, _CInput, _Handle  # noqa: E402
from parity import plan_many, plan_one, summary  # noqa: E402
from fuzz import random_case  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
REC = W.ORACLE_REC_LEN


def reflib():
    lib = abi.reference()
    raw = C.CDLL(abi.REF_LIB)
    raw.slos_ref_uniforms.argtypes = [C.c_uint64, C.c_int32, C.POINTER(C.c_double)]
    raw.slos_ref_oracle_instances.argtypes = [C.c_uint64, C.c_int32, C.POINTER(C.c_int64)]
    raw.slos_ref_oracle_best_value.argtypes = [C.POINTER(C.c_int64)]
    raw.slos_ref_oracle_best_value.restype = C.c_double
    raw.slos_ref_oracle_subset_feasible.argtypes = [C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_int32]
    raw.slos_ref_oracle_subset_feasible.restype = C.c_int32
    return lib, raw


def dump(name, obj):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


def main():
    only = set(sys.argv[1:])  # optional section filter: uniforms oracle stress fuzz
    lib, raw = reflib()
    # 1. RNG pin (acceptance_main.cpp:577 draws)
    if not only or "uniforms" in only:
        _uniforms(raw)
    if not only or "oracle" in only:
        _oracle(lib, raw)
    if not only or "stress" in only:
        _stress(lib)
    if not only or "fuzz" in only:
        _fuzz(lib)


def _uniforms(raw):
    uni = {}
    for seed in (88, 0, 1, 2024, 123456789):
        a = np.zeros(600)
        raw.slos_ref_uniforms(seed, 600, a.ctypes.data_as(C.POINTER(C.c_double)))
        uni[str(seed)] = [int(x) for x in a.view(np.uint64)]
    dump("uniforms", uni)


def _oracle(lib, raw):
    # 2. brute-force oracle instance families (test_dp_scheduler.cpp / acceptance_main.cpp)
    fams = {}
    for seed, count, unit in ((424242, 250, False), (20240817, 300, False), (171717, 60, False),
                              (555, 80, False), (909090, 120, True), (31337, 1, False)):
        recs = np.zeros(count * REC, np.int64)
        raw.slos_ref_oracle_instances(seed, count, recs.ctypes.data_as(C.POINTER(C.c_int64)))
        recs = recs.reshape(count, REC)
        items = []
        for r in recs:
            f = W.oracle_fields(r)
            if unit:
                f["candidates"] = [(d, p, t, m, 1) for (d, p, t, m, v) in f["candidates"]]
                r = r.copy()
                for i in range(len(f["candidates"])):
                    r[9 + 5 * i + 4] = 1
            rr = np.ascontiguousarray(r, np.int64)
            best = raw.slos_ref_oracle_best_value(rr.ctypes.data_as(C.POINTER(C.c_int64)))
            h = _Handle(lib, W.oracle_model(f), W.oracle_slo(f), PlannerConfig())
            ci = _CInput(W.oracle_input(f))
            res = plan_one(lib, h.ptr, ci.c, unit_value=unit)
            item = dict(rec=[int(x) for x in r], best_value=best, ref=summary(res))
            if res["status"] == 0:
                adm = np.asarray(res["admitted"], np.int32)
                item["ref_subset_feasible"] = int(raw.slos_ref_oracle_subset_feasible(
                    rr.ctypes.data_as(C.POINTER(C.c_int64)), adm.ctypes.data_as(C.POINTER(C.c_int32)),
                    len(adm)))
            items.append(item)
        fams[f"{seed}"] = dict(seed=seed, unit_value=unit, items=items)
    dump("oracle_instances", fams)


def _stress(lib):
    # 3. stress families C1-C4 + the reference latency criterion
    stress = {}
    # C4 (2032 decoders, the 256-thread reconstruction and HBM-spill DP levels) on 32
    # seeds: ~3 s per plan in the reference, ~15 s on 8 host threads
    for fam, seeds in (("C1", range(16)), ("LAT", range(16)), ("C2", range(6)), ("C3", range(16)),
                       ("C4", range(32))):
        F = W.FAMILIES[fam]
        b = W.InstanceBatch.stress(F["spec"], list(seeds))
        h = _Handle(lib, F["model"], W.TWO_TIER_SLO, F["cfg"])
        res = plan_many(lib, h.ptr, b)
        stress[fam] = dict(seeds=list(seeds), ref=[summary(r) for r in res])
        print(fam, "admitted", [len(r["admitted"]) for r in res][:8])
    dump("stress", stress)


def _fuzz(lib):
    # 4. structural fuzz (tests/fuzz.py), value and throughput objectives
    fz = []
    for seed in range(1000):
        terms, slo, cfg, inp = random_case(seed)
        ci = _CInput(inp)
        h = _Handle(lib, terms, slo, cfg)
        fz.append(dict(seed=seed, value=summary(plan_one(lib, h.ptr, ci.c, False)),
                       throughput=summary(plan_one(lib, h.ptr, ci.c, True))))
    dump("fuzz", fz)


if __name__ == "__main__":
    main()
