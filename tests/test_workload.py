"""Synthetic instance generator pinned to the reference's RNG draw sequence."""
import numpy as np

from golden_io import load
from paper_2504_08784_b200 import workload as W


def test_uniform_draws_match_reference_engine():
    # std::mt19937_64 + std::uniform_real_distribution<double>(0,1) (acceptance_main.cpp:577-578)
    for seed, bits in load("uniforms").items():
        got = W.uniforms(int(seed), len(bits)).view(np.uint64)
        assert [int(x) for x in got] == bits


def test_stress_instance_shape():
    spec = W.FAMILIES["C2"]["spec"]
    inp = W.stress_instance(spec, 7)
    assert len(inp.running) == 240 and len(inp.pending) == 16
    for i, r in enumerate(inp.running):
        assert r.decode_tier == i % 2
        assert inp.now <= r.next_due_s < inp.now + W.TWO_TIER_SLO.tpot_tiers_s[r.decode_tier]
        assert 50 <= r.decode_remaining < 250
    for p in inp.pending:
        assert inp.now + 0.3 <= p.prefill_deadline < inp.now + 1.2 + 1e-9
        assert 200 <= p.prefill_tokens < 900 and 20 <= p.memory_units < 80
        assert p.value == int(p.value) and 1 <= p.value <= 8


def test_batch_marshalling_matches_objects():
    spec = W.FAMILIES["C1"]["spec"]
    b = W.InstanceBatch.stress(spec, [3, 4])
    for k, seed in enumerate([3, 4]):
        inp = W.stress_instance(spec, seed)
        rr = b.running[k * spec.n_dec:(k + 1) * spec.n_dec]
        assert np.array_equal(rr["next_due_s"], [r.next_due_s for r in inp.running])
        pp = b.pending[k * spec.n_new:(k + 1) * spec.n_new]
        assert np.array_equal(pp["prefill_tokens"], [p.prefill_tokens for p in inp.pending])
