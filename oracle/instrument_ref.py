"""TEST INFRASTRUCTURE: pin the T/G/D/S/states work counters to the REFERENCE.

The roofline numerator (B_smem = 80·T + 32·D + 48·S per plan) is
defined on the reference's own traversal. The product and the C oracle both report
these counters; this script measures them on the reference itself:

  1. copy /root/reference/proj/{src,include,tests} to a scratch dir under /tmp
     (the reference tree is read-only; nothing is copied into this repo);
  2. insert thread-local counter increments at exactly the statements SURVEY.md §8
     names -- T after the pruned-source skip (dp_scheduler.cpp:475-479), G on each
     memo miss (dp_scheduler.cpp:427, batch_planner.cpp:414), D = dues materialised
     (batch_planner.cpp:223, before the empty check), S = slots built
     (batch_planner.cpp:247), states = arena size - 1 -- snapshotted when the DP
     loop ends (dp_scheduler.cpp:502), so build_plan's re-tiling is excluded;
  3. compile those sources with oracle/ref_capi.cpp (-DSLOS_REF_INSTR: a fresh
     BatchPlanner per plan, counters copied into slos_result.counters) into
     oracle/_ref/libslos_ref_instr.so;
  4. write tests/golden/counters.json.gz: the reference counters of the C2 bench
     seeds 0..63, the C1 / LAT / C3 stress seeds and C4 seeds 0..7.

  python oracle/instrument_ref.py
"""
from __future__ import annotations

import ctypes as C
import gzip
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

REF = os.environ.get("SLOS_REF", "/root/reference/proj")
SCRATCH = "/tmp/slos_ref_instr"
OUT_LIB = os.path.join(ROOT, "oracle", "_ref", "libslos_ref_instr.so")
NLOH = os.path.join(ROOT, "oracle", "_ref", "inc")

DECL = ("namespace slos_instr { extern thread_local long long T, G, D, S, snap[5]; "
        "extern thread_local int on; }\n")

# (file, anchor text that must occur exactly once, text inserted after it)
PATCHES = [
    ("src/batch_planner.cpp",
     "  // No due lands in the gap or its pull window: cadence is vacuous and\n",
     "  if (slos_instr::on) slos_instr::D += (long long)dues.size();\n"),
    ("src/batch_planner.cpp",
     "  const int num_slots = static_cast<int>(ends.size());\n",
     "  if (slos_instr::on) slos_instr::S += num_slots;\n"),
    ("src/batch_planner.cpp",
     "  if (it != memo_.end()) return it->second;\n",
     "  if (slos_instr::on) ++slos_instr::G;\n"),
    ("src/dp_scheduler.cpp",
     "    if (itf != memo.end()) return itf->second;\n",
     "    if (slos_instr::on) ++slos_instr::G;\n"),
    ("src/dp_scheduler.cpp",
     "          if (std::find(bv.begin(), bv.end(), src[si]) == bv.end()) continue;\n        }\n",
     "        ++slos_instr::T;\n"),
    ("src/dp_scheduler.cpp",
     "  std::vector<std::vector<int>> states_at(chain.size() + 1);\n  states_at[0] = {0};\n",
     "  slos_instr::T = slos_instr::G = slos_instr::D = slos_instr::S = 0;\n  slos_instr::on = 1;\n"),
    ("src/dp_scheduler.cpp",
     "  // Terminal states: chains that passed every forced item.\n",
     "  slos_instr::on = 0;\n  slos_instr::snap[0] = slos_instr::T; slos_instr::snap[1] = slos_instr::G;\n"
     "  slos_instr::snap[2] = slos_instr::D; slos_instr::snap[3] = slos_instr::S;\n"
     "  slos_instr::snap[4] = (long long)arena.size() - 1;\n"),
]

DEFN = ("namespace slos_instr { thread_local long long T = 0, G = 0, D = 0, S = 0, snap[5] = {0, 0, 0, 0, 0}; "
        "thread_local int on = 0; }\n")


def patch_tree():
    if os.path.isdir(SCRATCH):
        shutil.rmtree(SCRATCH)
    for d in ("src", "include", "tests"):
        shutil.copytree(os.path.join(REF, d), os.path.join(SCRATCH, d))
    for rel, head in (("src/batch_planner.cpp", DECL + DEFN), ("src/dp_scheduler.cpp", DECL)):
        p = os.path.join(SCRATCH, rel)
        s = open(p).read()
        s = s.replace("namespace slosim {", head + "namespace slosim {", 1)
        open(p, "w").write(s)
    for rel, anchor, ins in PATCHES:
        p = os.path.join(SCRATCH, rel)
        s = open(p).read()
        assert s.count(anchor) == 1, (rel, anchor)
        s = s.replace(anchor, anchor + ins, 1)
        open(p, "w").write(s)


def build():
    os.makedirs(os.path.dirname(OUT_LIB), exist_ok=True)
    if not os.path.exists(os.path.join(NLOH, "json.hpp")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    srcs = [os.path.join(SCRATCH, "src", f + ".cpp") for f in
            ("perf_model", "workload", "batch_planner", "dp_scheduler", "baselines")]
    srcs.append(os.path.join(ROOT, "oracle", "ref_capi.cpp"))
    cmd = ["g++", "-std=gnu++20", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-shared",
           "-DSLOS_REF_INSTR", "-I" + os.path.join(SCRATCH, "include"), "-I" + os.path.join(SCRATCH, "tests"),
           "-I" + NLOH, "-I" + os.path.join(ROOT, "include"), *srcs, "-o", OUT_LIB, "-lpthread"]
    # ref_capi.cpp also wraps ref_tools entry points; they are not needed here
    subprocess.run(cmd, check=True)
    return OUT_LIB


def golden():
    from paper_2504_08784_b200 import abi
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import _Handle
    from parity import plan_many
    lib = abi.load(OUT_LIB)
    out = {}
    for fam, seeds in (("C2", range(64)), ("C1", range(16)), ("LAT", range(16)), ("C3", range(16)),
                       ("C4", range(8))):
        F = W.FAMILIES[fam]
        b = W.InstanceBatch.stress(F["spec"], list(seeds))
        h = _Handle(lib, F["model"], W.TWO_TIER_SLO, F["cfg"])
        res = plan_many(lib, h.ptr, b)
        out[fam] = dict(seeds=list(seeds), counters=[list(r["counters"]) for r in res])
        print(fam, "T/G/D/S/states of seed", seeds[0], out[fam]["counters"][0])
    path = os.path.join(ROOT, "tests", "golden", "counters.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path)


if __name__ == "__main__":
    patch_tree()
    build()
    golden()
