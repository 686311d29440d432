"""The drop-in boundary: every function include/slos_planner.h declares is exported
by the product and by both CPU checkers; the product refuses to run without a
B200 (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import HAS_GPU
from paper_2504_08784_b200 import abi

HEADER = os.path.join(abi.ROOT, "include", "slos_planner.h")


# headers whose functions libslos_b200.so implements (slos_lockstep.h belongs to the
# reference-side integration library, integration/)
PRODUCT_HEADERS = ["slos_planner.h", "slos_plan_json.h", "slos_route.h", "slos_trace.h", "slos_fit.h"]


def declared(header=HEADER):
    # header-only inline accessors (SLOS_ENTRY_FN) are not exported symbols
    src = "\n".join(l for l in open(header).read().splitlines() if not l.startswith("SLOS_ENTRY_FN") and "return " not in l)
    return sorted(set(re.findall(r"^[a-z_ ]*?[\w\*]+\s+\**(slos_\w+)\(", src, re.M)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    return {l.split()[-1] for l in out.splitlines() if " T " in l}


def test_header_declares_the_abi():
    names = declared()
    for must in ("slos_plan", "slos_plan_batch", "slos_planner_create", "slos_tile_gap_batch",
                 "slos_workspace_solve", "slos_workspace_records"):
        assert must in names
    assert len(names) >= 20


@pytest.mark.parametrize("path", [abi.PRODUCT_LIB, abi.ORACLE_LIB, abi.REF_LIB])
def test_every_declared_symbol_is_exported(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built")
    missing = [n for n in declared() if n not in exported(path)]
    assert not missing, missing


@pytest.mark.parametrize("header", PRODUCT_HEADERS)
def test_product_exports_every_header(header):
    names = declared(os.path.join(abi.ROOT, "include", header))
    assert names, header
    missing = [n for n in names if n not in exported(abi.PRODUCT_LIB)]
    assert not missing, (header, missing)


def test_product_library_loads_and_identifies():
    lib = abi.product()
    assert lib.slos_backend() == b"b200-cuda"


@pytest.mark.skipif(HAS_GPU, reason="only meaningful without a GPU")
def test_product_fails_loudly_without_device():
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import BatchPlanner, Error, PerfModel, SloScheduler
    lib = abi.product()
    bp = BatchPlanner(PerfModel(W.DESK_MODEL, lib=lib), W.TWO_TIER_SLO, lib=lib)
    with pytest.raises(Error) as e:
        SloScheduler(bp).schedule(W.stress_instance(W.FAMILIES["C1"]["spec"], 0))
    assert e.value.code == "no-device"


def test_record_layout_matches_header():
    assert C.sizeof(abi.Record) == abi.RECORD_DTYPE.itemsize == 88
