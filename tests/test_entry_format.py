"""The 8-byte plan entry (include/slos_planner.h slos_entry): the packing is
lossless over the documented ranges, the Python accessors agree with the
vectorised canonical form, and the planners reject configurations the format
cannot carry (speculative spec_max_len above SLOS_ENTRY_MAX_SPEC) the same way."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2504_08784_b200 import abi
from paper_2504_08784_b200 import workload as W
from paper_2504_08784_b200.planner import Error, PlannerConfig, _Handle

MAX_REQS = 1 << 23


def pack(req, tokens, decode, spec):
    ref = (req & 0xFFFFFF) | ((spec & 0x7F) << 24) | (0x80000000 if decode else 0)
    return abi.Entry(ref, tokens)


CASES = [(0, 1, False, 0), (5, 2048, False, 0), (-1, 7, False, 0), (-MAX_REQS, 2**31 - 1, False, 0),
         (MAX_REQS - 1, 3, True, 0), (12, 9, True, 127), (-3, 1, True, 8), (0, -2**31, True, 1),
         (7, 0, True, 0), (-MAX_REQS, 0, False, 0)]


@pytest.mark.parametrize("req,tokens,decode,spec", CASES)
def test_entry_round_trip(req, tokens, decode, spec):
    e = pack(req, tokens, decode, spec)
    assert C.sizeof(e) == 8
    assert e.req == req and e.is_decode == decode and e.spec_len == spec
    assert e.prefill_tokens == (0 if decode else tokens)
    assert e.decode_tokens == (tokens if decode else 0)


def test_canonical_form_matches_accessors():
    arr = (abi.Entry * len(CASES))(*[pack(*c) for c in CASES])
    raw = np.frombuffer(bytes(arr), dtype=abi.ENTRY_DTYPE)
    canon = abi.canon_entries(raw)
    for k, c in enumerate(CASES):
        e = arr[k]
        assert (int(canon["req"][k]), int(canon["spec_len"][k]), int(canon["prefill_tokens"][k]),
                int(canon["decode_tokens"][k])) == (e.req, e.spec_len, e.prefill_tokens, e.decode_tokens)


@pytest.mark.parametrize("which", ["oracle", "reference", "product"])
def test_spec_len_beyond_entry_format_is_rejected(which):
    lib = {"oracle": abi.oracle, "reference": abi.reference, "product": abi.product}[which]
    path = {"oracle": abi.ORACLE_LIB, "reference": abi.REF_LIB, "product": abi.PRODUCT_LIB}[which]
    if not os.path.exists(path):
        pytest.skip(f"{path} not built")
    lib = lib()
    ok = _Handle(lib, W.DESK_MODEL, W.TWO_TIER_SLO, PlannerConfig(speculative=True, spec_max_len=127))
    assert ok.ptr
    _Handle(lib, W.DESK_MODEL, W.TWO_TIER_SLO, PlannerConfig(speculative=False, spec_max_len=500))
    with pytest.raises(Error) as ei:
        _Handle(lib, W.DESK_MODEL, W.TWO_TIER_SLO, PlannerConfig(speculative=True, spec_max_len=128))
    assert ei.value.code == "invalid-parameters"
