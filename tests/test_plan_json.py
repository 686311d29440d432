"""plan_to_json (dp_scheduler.cpp:560-589), the reference's canonical
result serialisation, from include/slos_plan_json.h. The product's serialiser
(libslos_b200.so, host code) must write exactly the bytes the reference's own
plan_to_json writes (oracle/_ref/libslos_ref.so wraps it) for the same result:
over planned results of the golden families and the recorded C5 corpus, over
crafted results that stress the number and string rules, and (gpu) for the
product planner's own plans against the reference planner's plans."""
import ctypes as C
import json
import math
import os
import random
import struct

import pytest

from paper_2504_08784_b200 import abi
from paper_2504_08784_b200 import workload as W
from paper_2504_08784_b200.planner import PerfTerm, PlannerConfig, _Handle

pytestmark = pytest.mark.skipif(not os.path.exists(abi.REF_LIB), reason="oracle/_ref not built")

GOLDEN = os.path.join(abi.ROOT, "tests", "golden")
ISZ = C.sizeof(abi.Input)


def _jsons(plan_lib, handle, batch, serialisers):
    """Plan `batch` with plan_lib; serialise every result with each serialiser."""
    n = batch.n
    hs = (C.c_void_p * n)(*([handle] * n))
    outs = (abi.Result * n)()
    assert plan_lib.slos_plan_batch(hs, n, C.c_void_p(batch.inputs_ptr()), 0, outs, None) == abi.SLOS_OK
    try:
        res = []
        for k in range(n):
            assert outs[k].status == abi.SLOS_OK
            now = float(batch.inputs["now"][k])
            res.append([abi.plan_to_json(s, batch.inputs_ptr() + k * ISZ, outs[k], now) for s in serialisers])
        return res
    finally:
        for k in range(n):
            plan_lib.slos_result_free(C.byref(outs[k]))


def _c5(group, limit):
    meta = json.load(__import__("gzip").open(os.path.join(GOLDEN, "c5.json.gz"), "rt"))
    G = meta["groups"][group]
    b = W.load_corpus(os.path.join(GOLDEN, f"c5_{group}.bin.gz")).subset(range(limit))
    cfg = PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=G["speculative"],
                        spec_alpha=0.8, spec_max_len=8, plan_margin=0.0)
    return b, [PerfTerm(*t) for t in meta["model"]], cfg


@pytest.mark.parametrize("fam,seeds", [("C1", range(0, 6)), ("LAT", range(0, 2)), ("C3", range(0, 2))])
def test_product_json_matches_reference_plan_to_json(fam, seeds):
    ref, prod = abi.reference(), abi.product()
    F = W.FAMILIES[fam]
    b = W.InstanceBatch.stress(F["spec"], seeds)
    h = _Handle(ref, F["model"], W.TWO_TIER_SLO, F["cfg"])
    for ours, theirs in _jsons(ref, h.ptr, b, [prod, ref]):
        assert ours == theirs
        json.loads(ours)


@pytest.mark.parametrize("group", ["ar", "spec"])
def test_product_json_matches_reference_on_corpus(group):
    ref, prod = abi.reference(), abi.product()
    b, model, cfg = _c5(group, 256)
    h = _Handle(ref, model, W.TWO_TIER_SLO, cfg)
    for ours, theirs in _jsons(ref, h.ptr, b, [prod, ref]):
        assert ours == theirs


def _result_bytes(n_pending, doubles, rng):
    nb = len(doubles) // 2
    batches = (abi.Batch * max(1, nb))()
    entries = (abi.Entry * max(1, 2 * nb))()
    for b in range(nb):
        batches[b].start_s = doubles[2 * b]
        batches[b].end_s = doubles[2 * b + 1]
        batches[b].capacity_tokens = rng.randrange(-2**62, 2**62)
        batches[b].spec_step = rng.randrange(0, 9)
        batches[b].prefill_budget_left = rng.randrange(-5, 2**40)
        batches[b].first_entry = 2 * b
        batches[b].n_entries = 2
        entries[2 * b] = abi.Entry((0 & 0xFFFFFF) | (rng.randrange(128) << 24) | 0x80000000,
                                   rng.randrange(-2**31, 2**31))
        entries[2 * b + 1] = abi.Entry((-(1 + rng.randrange(n_pending))) & 0xFFFFFF, rng.randrange(0, 2**31))
    adm = (C.c_int32 * n_pending)(*range(n_pending))
    r = abi.Result()
    r.status = 0
    r.running_set_infeasible = rng.randrange(2)
    r.admitted_value = doubles[-1]
    r.n_admitted = n_pending // 2
    r.n_declined = n_pending - n_pending // 2
    r.admitted = C.cast(adm, C.POINTER(C.c_int32))
    r.declined = C.cast(C.byref(adm, 4 * (n_pending // 2)), C.POINTER(C.c_int32))
    r.deferred = C.cast(adm, C.POINTER(C.c_int32))
    r.n_batches = nb
    r.batches = C.cast(batches, C.POINTER(abi.Batch))
    r.n_entries = 2 * nb
    r.entries = C.cast(entries, C.POINTER(abi.Entry))
    r.exact_until_s = doubles[-2]
    return r, (batches, entries, adm)


def _input(ids_running, ids_pending):
    run = (abi.Running * len(ids_running))()
    pen = (abi.Pending * len(ids_pending))()
    keep = []
    for k, s in enumerate(ids_running):
        keep.append(C.create_string_buffer(s))
        run[k].id = C.cast(keep[-1], C.c_char_p)
    for k, s in enumerate(ids_pending):
        keep.append(C.create_string_buffer(s))
        pen[k].id = C.cast(keep[-1], C.c_char_p)
    inp = abi.Input()
    inp.now = 0.0
    inp.running = C.cast(run, C.POINTER(abi.Running))
    inp.n_running = len(ids_running)
    inp.pending = C.cast(pen, C.POINTER(abi.Pending))
    inp.n_pending = len(ids_pending)
    return inp, (run, pen, keep)


def _rand_double(rng):
    k = rng.randrange(6)
    if k == 0:
        return 100.0 + rng.random() * 50.0
    if k == 1:
        x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
        return x if math.isfinite(x) else 1.5
    if k == 2:
        return rng.random() * 1e-3
    if k == 3:
        return math.ldexp(rng.random(), rng.randrange(-1075, 1024))
    if k == 4:
        return rng.randrange(100000) / 8.0
    return rng.choice([0.0, -0.0, 1e15, 1e16, 1e-4, 1e-5, 5e-324, 1.7976931348623157e308, float("nan"),
                       float("inf"), -float("inf"), 0.1, 123456789012345678.0])


def test_crafted_results_numbers_and_strings():
    ref, prod = abi.reference(), abi.product()
    rng = random.Random(11)
    id_pool = [b"r0", b"p\"q", b"back\\slash", b"tab\there", b"nl\n\r\b\f", b"ctl\x01\x1f\x7f", b"utf8-\xc3\xa9\xe2\x82\xac",
               b"emoji\xf0\x9f\x98\x80", b"", b"plain-id-123"]
    for trial in range(300):
        ids_p = [rng.choice(id_pool) for _ in range(rng.randrange(1, 6))]
        inp, keep_in = _input([rng.choice(id_pool)], ids_p)
        doubles = [_rand_double(rng) for _ in range(2 * rng.randrange(0, 6) + 2)]
        r, keep_r = _result_bytes(len(ids_p), doubles, rng)
        now = _rand_double(rng)
        a = abi.plan_to_json(prod, C.addressof(inp), r, now)
        b = abi.plan_to_json(ref, C.addressof(inp), r, now)
        assert a == b, (trial, a, b)


def test_ill_formed_utf8_is_rejected_by_both():
    ref, prod = abi.reference(), abi.product()
    inp, keep_in = _input([b"r0"], [b"bad\xff", b"ok"])
    r, keep_r = _result_bytes(2, [1.0, 2.0, 3.0, 4.0], random.Random(1))
    for lib in (prod, ref):
        n = C.c_int64()
        st = lib.slos_plan_to_json(C.c_void_p(C.addressof(inp)), C.byref(r), 0.0, None, 0, C.byref(n))
        assert lib.slos_status_slug(st) == b"invalid-parameters"


def test_buffer_contract():
    prod = abi.product()
    inp, keep_in = _input([b"r0"], [b"p0", b"p1"])
    r, keep_r = _result_bytes(2, [1.0, 2.0, 3.0, 4.0], random.Random(2))
    n = C.c_int64()
    assert prod.slos_plan_to_json(C.c_void_p(C.addressof(inp)), C.byref(r), 0.0, None, 0, C.byref(n)) == 0
    small = C.create_string_buffer(8)
    assert prod.slos_plan_to_json(C.c_void_p(C.addressof(inp)), C.byref(r), 0.0, small, 8, C.byref(n)) == 0
    full = abi.plan_to_json(prod, C.addressof(inp), r, 0.0)
    assert n.value == len(full) and small.raw[:8] == full.encode()[:8]


@pytest.mark.gpu
@pytest.mark.parametrize("fam,seeds", [("C1", range(0, 8)), ("C2", range(0, 4)), ("C3", range(0, 4))])
def test_b200_plans_serialise_like_reference_plans(fam, seeds):
    """The product planner's plans, serialised, equal the reference planner's plans
    serialised by the reference's own plan_to_json (the determinism test's form)."""
    ref, prod = abi.reference(), abi.product()
    F = W.FAMILIES[fam]
    b = W.InstanceBatch.stress(F["spec"], seeds)
    hr = _Handle(ref, F["model"], W.TWO_TIER_SLO, F["cfg"])
    hp = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"])
    want = [x[0] for x in _jsons(ref, hr.ptr, b, [ref])]
    got = [x[0] for x in _jsons(prod, hp.ptr, b, [prod])]
    assert got == want
