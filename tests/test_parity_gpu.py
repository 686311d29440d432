"""Product (sm_100a kernels via the C-ABI) vs the reference: bit-exact on every
output field of plan() -- admitted/declined id sequences, admitted_value bits,
running_set_infeasible, every batch and entry, exact_until_s."""
import pytest

from golden_checks import check_c5, check_fuzz, check_oracle_instances, check_stress
from parity import diff, plan_many, plan_one
from paper_2504_08784_b200 import abi
from paper_2504_08784_b200 import workload as W
from paper_2504_08784_b200.planner import _CInput, _Handle

pytestmark = pytest.mark.gpu


def test_product_is_the_cuda_backend():
    assert abi.product().slos_backend() == b"b200-cuda"


def test_brute_force_families_match_reference():
    assert check_oracle_instances(abi.product()) == 811


@pytest.mark.parametrize("fam", ["C1", "LAT", "C2", "C3", "C4"])
def test_stress_families_match_reference(fam):
    check_stress(abi.product(), families=(fam,))


# Batches below the SM count take the widest kernels (latency mode, the default for
# the small batches above); the same goldens through the throughput kernels (warp /
# 128-thread reconstruction, 64- / 256-thread DP) with the latency mode off:
@pytest.mark.parametrize("fam", ["C1", "LAT", "C2", "C3", "C4"])
def test_stress_families_throughput_kernels(fam, monkeypatch):
    monkeypatch.setenv("SLOS_LATENCY_BATCH", "0")
    check_stress(abi.product(), families=(fam,))


def test_brute_force_and_fuzz_throughput_kernels(monkeypatch):
    monkeypatch.setenv("SLOS_LATENCY_BATCH", "0")
    assert check_oracle_instances(abi.product()) == 811
    check_fuzz(abi.product())


@pytest.mark.parametrize("n", [1, 147, 148, 149, 300])
def test_c5_batch_sizes_around_the_latency_mode_threshold(n):
    """Batches up to the SM count (148) take the widest kernels, larger ones the
    throughput kernels: both sides of the boundary against the reference."""
    assert check_c5(abi.product(), limit=n) == 2 * n


def test_c5_simulator_corpus_matches_reference():
    # C5: inputs recorded from the reference simulator's sweep grid, batched
    assert check_c5(abi.product()) == 4096


def test_fuzz_matches_reference():
    check_fuzz(abi.product())


def test_c2_batch_matches_oracle_with_reference_counters():
    """The benchmark workload (BASELINE configs[1]) at 64 instances, one launch;
    the T/G/D/S work counters follow the reference traversal exactly."""
    F = W.FAMILIES["C2"]
    b = W.InstanceBatch.stress(F["spec"], range(100, 164))
    prod, ora = abi.product(), abi.oracle()
    hp, ho = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"]), _Handle(ora, F["model"], W.TWO_TIER_SLO, F["cfg"])
    P = plan_many(prod, hp.ptr, b)
    O = plan_many(ora, ho.ptr, b)
    bad = [(k, diff(P[k], O[k], counters=True)) for k in range(b.n) if diff(P[k], O[k], counters=True)]
    assert not bad, bad[:4]


def test_c2_1024_pipelined_matches_reference():
    """The bench batch itself: 1024 C2 instances through slos_plan_batch, which runs
    as two pipelined chunks, each solved in two stream-pipelined parts with all three
    reconstruction kinds' queues, against the compiled reference (16 host threads)."""
    import os
    if not os.path.exists(abi.REF_LIB):
        pytest.skip("oracle/_ref not built")
    F = W.FAMILIES["C2"]
    b = W.InstanceBatch.stress(F["spec"], range(5000, 6024))
    prod, ref = abi.product(), abi.reference()
    hp, hr = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"]), _Handle(ref, F["model"], W.TWO_TIER_SLO, F["cfg"])
    P = plan_many(prod, hp.ptr, b)
    R = plan_many(ref, hr.ptr, b)
    bad = [(k, diff(P[k], R[k])) for k in range(b.n) if diff(P[k], R[k])]
    assert not bad, bad[:4]


def test_fresh_fuzz_matches_oracle():
    from fuzz import random_case
    prod, ora = abi.product(), abi.oracle()
    for seed in range(20000, 20300):
        terms, slo, cfg, inp = random_case(seed, max_pending=12)
        ci = _CInput(inp)
        hp, ho = _Handle(prod, terms, slo, cfg), _Handle(ora, terms, slo, cfg)
        for uv in (False, True):
            a, o = plan_one(prod, hp.ptr, ci.c, uv), plan_one(ora, ho.ptr, ci.c, uv)
            assert not diff(a, o, counters=True), (seed, uv, diff(a, o, counters=True))


def test_errors_are_status_codes():
    from paper_2504_08784_b200.planner import (BatchPlanner, Error, PendingRequest, PerfModel,
                                               ScheduleInput, SloConfig, SloScheduler)
    slo = SloConfig([0.05, 0.1], [3.0, 5.0])
    sched = SloScheduler(BatchPlanner(PerfModel(W.DESK_MODEL), slo))
    bad = ScheduleInput(now=0.0, memory_total=100,
                        pending=[PendingRequest(id="x", prefill_deadline=1.0, prefill_tokens=10,
                                                decode_tier=5, memory_units=1)])
    with pytest.raises(Error) as e:
        sched.schedule(bad)
    assert e.value.code == "invalid-parameters"
    many = ScheduleInput(now=0.0, memory_total=100,
                         pending=[PendingRequest(id=f"p{i}", prefill_deadline=1.0, prefill_tokens=1,
                                                 decode_tier=0, memory_units=1) for i in range(251)])
    with pytest.raises(Error) as e:
        sched.schedule(many)
    assert e.value.code == "invalid-parameters"


def test_c2_bench_seeds_with_the_infeasible_instance_match_reference():
    """Seeds 0..1023 (the bench batch) include an instance whose running set is
    infeasible: its 496-batch EDF fallback takes the closed-time decode tail."""
    import os
    if not os.path.exists(abi.REF_LIB):
        pytest.skip("oracle/_ref not built")
    F = W.FAMILIES["C2"]
    b = W.InstanceBatch.stress(F["spec"], range(0, 1024))
    prod, ref = abi.product(), abi.reference()
    hp, hr = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"]), _Handle(ref, F["model"], W.TWO_TIER_SLO, F["cfg"])
    P = plan_many(prod, hp.ptr, b)
    R = plan_many(ref, hr.ptr, b)
    assert any(r["infeasible"] for r in R)
    bad = [(k, diff(P[k], R[k])) for k in range(b.n) if diff(P[k], R[k])]
    assert not bad, bad[:4]


def test_c5_corpus_tiled_matches_reference():
    """The C5 corpus tiled (65,536 AR instances: the 4-chunk host pipeline; 32,768
    speculative: 2 chunks) with per-part collection, every result against the
    reference's golden summary."""
    import gzip
    import json
    import os
    from golden_checks import _cmp
    from paper_2504_08784_b200.planner import PerfTerm, PlannerConfig
    GOLDEN = os.path.join(abi.ROOT, "tests", "golden")
    meta = json.load(gzip.open(os.path.join(GOLDEN, "c5.json.gz"), "rt"))
    prod = abi.product()
    for g in ("ar", "spec"):
        G = meta["groups"][g]
        base = W.load_corpus(os.path.join(GOLDEN, f"c5_{g}.bin.gz"))
        b = base.tiled(32 if g == "ar" else 16)
        cfg = PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=G["speculative"],
                            spec_alpha=0.8, spec_max_len=8, plan_margin=0.0)
        h = _Handle(prod, [PerfTerm(*t) for t in meta["model"]], W.TWO_TIER_SLO, cfg)
        res = plan_many(prod, h.ptr, b)
        for k, got in enumerate(res):
            _cmp(got, G["ref"][k % base.n], f"c5 {g} tiled instance {k}")


def test_work_counters_equal_instrumented_reference():
    """The product's T/G/D/S/states equal the counters measured inside the
    reference itself (tests/golden/counters.json.gz, oracle/instrument_ref.py):
    C2 bench seeds 0..63, C1/LAT/C3 stress seeds, C4 seeds 0..7."""
    from golden_io import load
    g = load("counters")
    prod = abi.product()
    for fam, G in g.items():
        F = W.FAMILIES[fam]
        b = W.InstanceBatch.stress(F["spec"], G["seeds"])
        h = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"])
        res = plan_many(prod, h.ptr, b)
        bad = [(G["seeds"][k], list(r["counters"]), G["counters"][k]) for k, r in enumerate(res)
               if list(r["counters"]) != G["counters"][k]]
        assert not bad, (fam, bad[:3])


def test_c4_32_seeds_pipelined_match_reference():
    """C4 (2032 running decoders, budget 8192, b200-synthetic model) on all 32 golden
    seeds, tiled x16 = 512 instances so slos_plan_batch runs its two-chunk pipeline
    with two stream-pipelined solve parts and the 256-thread reconstruction."""
    from golden_checks import _cmp
    from golden_io import load
    st = load("stress")["C4"]
    assert len(st["seeds"]) >= 32
    F = W.FAMILIES["C4"]
    base = W.InstanceBatch.stress(F["spec"], st["seeds"])
    b = base.tiled(16)
    prod = abi.product()
    h = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"])
    res = plan_many(prod, h.ptr, b)
    for k, got in enumerate(res):
        _cmp(got, st["ref"][k % base.n], f"C4 seed {st['seeds'][k % base.n]} (tile {k // base.n})")


def test_device_resident_workspace_path_matches_reference():
    """The path bench.py's `value` times: slos_workspace_upload once, solve twice
    (the second solve re-runs the resident batch), download -- C2 x 1024 (seeds
    0..1023) against the compiled reference, every field bit-exact, plus the
    88-byte records the multi-GPU gather carries."""
    import ctypes as C
    import os

    import torch
    from parity import canon_c
    from paper_2504_08784_b200.sweep import ShardSolver, ShardSpec, records_view
    if not os.path.exists(abi.REF_LIB):
        pytest.skip("oracle/_ref not built")
    F = W.FAMILIES["C2"]
    prod, ref = abi.product(), abi.reference()
    solver = ShardSolver(prod, ShardSpec(F["spec"], F["model"], F["cfg"]), range(1024))
    stream = torch.cuda.Stream()
    rec = torch.empty((1024, C.sizeof(abi.Record)), dtype=torch.uint8, device="cuda")
    solver.upload(stream.cuda_stream)
    solver.converge(rec, stream.cuda_stream)
    solver.solve(stream.cuda_stream)
    solver.records(rec.data_ptr(), stream.cuda_stream)
    outs = solver.download(stream.cuda_stream)
    P = [canon_c(outs[k]) for k in range(1024)]
    solver.free_results()
    solver.close()
    hr = _Handle(ref, F["model"], W.TWO_TIER_SLO, F["cfg"])
    R = plan_many(ref, hr.ptr, solver.batch)
    bad = [(k, diff(P[k], R[k])) for k in range(1024) if diff(P[k], R[k])]
    assert not bad, bad[:4]
    torch.cuda.synchronize()
    rv = records_view(rec)
    for k in (0, 1, 511, 1023):
        assert rv["n_admitted"][k] == len(R[k]["admitted"]) and rv["n_entries"][k] == len(R[k]["entries"])
        assert rv["status"][k] == 0


def test_long_deadline_span_is_isolated():
    """An instance whose pending deadline lies far in the future needs a wide slot
    grid. It is solved in its own slot class: it must not resize (or fail) the
    launch of the ordinary instances beside it. A span of 80 s (1,608 slots at the
    50 ms tier) still plans bit-exactly like the oracle; a span of 5,000 s (100k
    slots, more than a CTA's shared memory) is a per-instance SLOS_ERR_RANGE."""
    F = W.FAMILIES["C1"]
    ins = [W.stress_instance(F["spec"], s) for s in range(6)]
    ins[2].pending[3].prefill_deadline = ins[2].now + 80.0
    ins[4].pending[0].prefill_deadline = ins[4].now + 5000.0
    b = W.InstanceBatch.from_inputs(ins)
    prod, ora = abi.product(), abi.oracle()
    hp, ho = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"]), _Handle(ora, F["model"], W.TWO_TIER_SLO, F["cfg"])
    P = plan_many(prod, hp.ptr, b)
    keep = [0, 1, 2, 3, 5]
    O = plan_many(ora, ho.ptr, b.subset(keep))
    for x, k in enumerate(keep):
        assert not diff(P[k], O[x], counters=True), (k, diff(P[k], O[x], counters=True))
    assert P[4]["status"] == abi.SLOS_ERR_RANGE


def test_invalid_instances_inside_a_pipelined_batch():
    """Instances failing validation spread over the chunks of a 3-chunk pipelined batch
    (65,536 C5 instances; the upload's parallel reductions and the split collection):
    they get the status code, every other instance still matches the reference, and
    slos_last_error names the last failing instance's fault."""
    import gzip
    import json
    import os

    import numpy as np
    from golden_checks import _cmp
    from paper_2504_08784_b200.planner import PerfTerm, PlannerConfig
    GOLDEN = os.path.join(abi.ROOT, "tests", "golden")
    meta = json.load(gzip.open(os.path.join(GOLDEN, "c5.json.gz"), "rt"))
    G = meta["groups"]["ar"]
    base = W.load_corpus(os.path.join(GOLDEN, "c5_ar.bin.gz"))
    b = base.tiled(32)
    bad = np.zeros(1, abi.PENDING_DTYPE)
    bad[0]["prefill_deadline"] = 1e9
    bad[0]["prefill_tokens"] = 10
    bad[0]["decode_tier"] = 7  # out of range for two tiers
    bad[0]["memory_units"] = 1
    bad[0]["id"] = b._blob.ctypes.data  # any valid C string
    broken = [5, 21845, 21846, 40000, 65535]
    for k in broken:
        b.inputs[k]["pending"] = bad.ctypes.data
        b.inputs[k]["n_pending"] = 1
    prod = abi.product()
    cfg = PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=G["speculative"],
                        spec_alpha=0.8, spec_max_len=8, plan_margin=0.0)
    h = _Handle(prod, [PerfTerm(*t) for t in meta["model"]], W.TWO_TIER_SLO, cfg)
    res = plan_many(prod, h.ptr, b)
    assert b"tier" in prod.slos_last_error()
    for k, got in enumerate(res):
        if k in broken:
            assert got["status"] == abi.SLOS_ERR_INVALID_PARAMETERS, (k, got["status"])
        else:
            _cmp(got, G["ref"][k % base.n], f"c5 ar tiled instance {k}")


def test_forced_three_chunk_pipeline_matches_reference():
    """Small batches through three forced pipeline chunks (tests/gpu_forced_chunks.py,
    its own process: the chunk count is read once per process)."""
    import os
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(abi.ROOT, "tests", "gpu_forced_chunks.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "C2 12 mismatches []" in r.stdout and "forced chunks done" in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("n", [511, 512, 513, 39999, 40000, 40001])
def test_c5_batch_sizes_around_the_pipeline_chunk_thresholds(n):
    """Batch sizes at the chunk-count thresholds of the end-to-end pipeline (1 -> 2
    chunks at 512, 2 -> n / 20k chunks at 40,000): every instance matches the reference."""
    import gzip
    import json
    import os
    from golden_checks import _cmp
    from paper_2504_08784_b200.planner import PerfTerm, PlannerConfig
    GOLDEN = os.path.join(abi.ROOT, "tests", "golden")
    meta = json.load(gzip.open(os.path.join(GOLDEN, "c5.json.gz"), "rt"))
    G = meta["groups"]["ar"]
    base = W.load_corpus(os.path.join(GOLDEN, "c5_ar.bin.gz"))
    b = base.tiled((n + base.n - 1) // base.n).subset(range(n))
    prod = abi.product()
    cfg = PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=G["speculative"],
                        spec_alpha=0.8, spec_max_len=8, plan_margin=0.0)
    h = _Handle(prod, [PerfTerm(*t) for t in meta["model"]], W.TWO_TIER_SLO, cfg)
    res = plan_many(prod, h.ptr, b)
    assert len(res) == n
    for k, got in enumerate(res):
        _cmp(got, G["ref"][k % base.n], f"c5 ar batch of {n}, instance {k}")


def test_large_heavy_batch_equals_small_batches():
    """43,690 C2 instances (64 seeds repeated) in one slos_plan_batch: the heavy-instance
    chunking (four chunks of <= 10,923 over three rotating workspaces) returns, for every
    sampled instance, exactly the plan the same input gets in a 64-instance batch (itself
    pinned to the reference by the tests above)."""
    import ctypes as C
    from parity import canon_c
    F = W.FAMILIES["C2"]
    n = 43690
    prod = abi.product()
    h = _Handle(prod, F["model"], W.TWO_TIER_SLO, F["cfg"])
    small = plan_many(prod, h.ptr, W.InstanceBatch.stress(F["spec"], range(64)))
    b = W.InstanceBatch.stress(F["spec"], range(64)).tiled((n + 63) // 64).subset(range(n))
    hs = (C.c_void_p * n)(*([h.ptr] * n))
    outs = (abi.Result * n)()
    assert prod.slos_plan_batch(hs, n, C.c_void_p(b.inputs_ptr()), 0, outs, None) == abi.SLOS_OK
    try:
        assert all(outs[k].status == abi.SLOS_OK for k in range(n))
        for k in range(0, n, 97):
            d = diff(canon_c(outs[k]), small[k % 64], counters=True)
            assert not d, (k, d)
    finally:
        for k in range(n):
            prod.slos_result_free(C.byref(outs[k]))
