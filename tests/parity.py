"""Bit-exact comparison helpers for ScheduleResult-shaped outputs of any library
exporting include/slos_planner.h (product, oracle, reference)."""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from paper_2504_08784_b200 import abi


def bits(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", x))[0]


def canon_c(r: abi.Result) -> dict:
    """Canonical, bit-exact view of a C slos_result."""
    d = dict(status=int(r.status))
    if r.status != abi.SLOS_OK:
        return d
    d["infeasible"] = int(r.running_set_infeasible)
    d["value_bits"] = bits(r.admitted_value)
    d["value"] = r.admitted_value
    d["admitted"] = [int(r.admitted[k]) for k in range(r.n_admitted)]
    d["declined"] = [int(r.declined[k]) for k in range(r.n_declined)]
    d["deferred"] = [int(r.deferred[k]) for k in range(r.n_deferred)]
    d["exact_until_bits"] = bits(r.exact_until_s)
    nb, ne = int(r.n_batches), int(r.n_entries)
    if nb:
        bb = np.ctypeslib.as_array(C.cast(r.batches, C.POINTER(C.c_uint8)), (nb * C.sizeof(abi.Batch),))
        d["batches"] = bb.view(abi.BATCH_DTYPE).copy()
    else:
        d["batches"] = np.zeros(0, abi.BATCH_DTYPE)
    # entries in the canonical int64 layout (digests are independent of the wire form)
    ent = np.zeros(ne, abi.CANON_ENTRY_DTYPE)
    if ne:
        eb = np.ctypeslib.as_array(C.cast(r.entries, C.POINTER(C.c_uint8)), (ne * C.sizeof(abi.Entry),))
        ent = abi.canon_entries(eb.view(abi.ENTRY_DTYPE))
    d["entries"] = ent
    d["counters"] = (r.counters.transitions, r.counters.gap_evals, r.counters.dues,
                     r.counters.slots, r.counters.states)
    return d


def diff(a: dict, b: dict, counters: bool = False) -> list:
    """Return the list of fields that differ (empty = bit-exact)."""
    out = []
    keys = ["status", "infeasible", "value_bits", "admitted", "declined", "deferred",
            "exact_until_bits"]
    for k in keys:
        if a.get(k) != b.get(k):
            out.append(k)
    if a.get("status") == 0 and b.get("status") == 0:
        for k in ("batches", "entries"):
            x, y = a[k], b[k]
            if x.shape != y.shape or x.tobytes() != y.tobytes():
                out.append(k)
        if counters and a["counters"] != b["counters"]:
            out.append("counters")
    return out


def plan_many(lib, handle, batch, unit_value=False) -> list:
    """Run slos_plan_batch over an InstanceBatch with one planner handle."""
    n = batch.n
    hs = (C.c_void_p * n)(*([handle] * n))
    outs = (abi.Result * n)()
    st = lib.slos_plan_batch(hs, n, C.c_void_p(batch.inputs_ptr()), 1 if unit_value else 0, outs,
                             None)
    assert st == abi.SLOS_OK, lib.slos_last_error()
    res = [canon_c(outs[k]) for k in range(n)]
    for k in range(n):
        lib.slos_result_free(C.byref(outs[k]))
    return res


def plan_one(lib, handle, cinput, unit_value=False) -> dict:
    out = abi.Result()
    lib.slos_plan(handle, C.byref(cinput), 1 if unit_value else 0, C.byref(out))
    d = canon_c(out)
    lib.slos_result_free(C.byref(out))
    return d


def digest(d: dict) -> str:
    """sha256 over the canonical bytes of a result (used to pin goldens)."""
    import hashlib
    h = hashlib.sha256()
    h.update(struct.pack("<i", d["status"]))
    if d["status"] == 0:
        h.update(struct.pack("<iqq", d["infeasible"], d["value_bits"], d["exact_until_bits"]))
        for k in ("admitted", "declined", "deferred"):
            h.update(struct.pack("<i", len(d[k])))
            h.update(np.asarray(d[k], np.int32).tobytes())
        h.update(d["batches"].tobytes())
        h.update(d["entries"].tobytes())
    return h.hexdigest()


def summary(d: dict) -> dict:
    s = dict(status=d["status"])
    if d["status"] == 0:
        s.update(infeasible=d["infeasible"], value_bits=d["value_bits"], admitted=d["admitted"],
                 declined=d["declined"], n_batches=int(len(d["batches"])),
                 n_entries=int(len(d["entries"])), exact_until_bits=d["exact_until_bits"],
                 digest=digest(d))
    return s
