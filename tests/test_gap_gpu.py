"""K1/K2 standalone: BatchPlanner::tile_gap_ar / tile_gap / prefill_budget on the
device vs the oracle, full GapPlan (batches, per-owner and per-tier tokens,
speculative lengths), on random censuses that exercise overload, late dues,
spill past the gap, multi-tier canonical members and speculation."""
import random

import pytest

from paper_2504_08784_b200 import abi
from paper_2504_08784_b200.planner import (BatchPlanner, DecodeCensus, DecodeMember, Error,
                                           PerfModel, PerfTerm, PlannerConfig, SloConfig)

pytestmark = pytest.mark.gpu


def random_gap(rng):
    L = rng.choice([1, 2, 3])
    base = rng.uniform(0.02, 0.1)
    tp = [base]
    for _ in range(L - 1):
        tp.append(tp[-1] * rng.choice([1.0, 1.5, 2.0, rng.uniform(1.1, 3)]))
    slo = SloConfig(tp, [3.0] * L)
    terms = [PerfTerm(rng.uniform(1e-6, 2e-4), rng.uniform(0, 2e-3), rng.uniform(1e-3, 0.6 * base))]
    if rng.random() < 0.5:
        terms.append(PerfTerm(0, 0, rng.uniform(0.2, 0.9) * base))
    cfg = PlannerConfig(max_chunk_tokens=rng.choice([8, 64, 512, 2048]),
                        max_batch_tokens=rng.choice([16, 512, 16384]),
                        speculative=rng.random() < 0.4, spec_alpha=rng.choice([0.6, 0.8, 1.0]),
                        spec_max_len=rng.choice([2, 8]), plan_margin=rng.choice([0.0, 0.1]))
    counts = [rng.choice([0, 0, 1, 3, 20]) for _ in range(L)]
    ex = []
    owners = list(range(100))
    rng.shuffle(owners)
    for i in range(rng.randint(0, 30)):
        ex.append(DecodeMember(tier=rng.randrange(L), phase_s=rng.choice([0.0, rng.uniform(-0.01, 3 * base)]),
                               backlog=rng.choice([0, 0, 0, 1, 3]), remaining=rng.choice([0, 1, 5, 100]),
                               owner=owners[i] if rng.random() < 0.5 else i))
    gap = rng.choice([0.0, 5e-10, rng.uniform(0, 1.5), float(rng.randint(1, 20)) * base])
    horizon = rng.choice([0.0, gap, gap + rng.uniform(0, 0.1)])
    return PerfModel(terms), slo, cfg, DecodeCensus(counts, ex), gap, horizon


def same(a, b):
    if isinstance(a, Error) or isinstance(b, Error):
        return isinstance(a, Error) and isinstance(b, Error) and a.code == b.code
    return a == b


def test_tile_gap_matches_oracle():
    rng = random.Random(7)
    prod, ora = abi.product(), abi.oracle()
    n = 0
    for it in range(1500):
        model, slo, cfg, census, gap, hor = random_gap(rng)
        bp, bo = BatchPlanner(model, slo, cfg, lib=prod), BatchPlanner(model, slo, cfg, lib=ora)
        for mode in (abi.GAP_TILE_AR, abi.GAP_TILE, abi.GAP_PREFILL_BUDGET):
            q = [(gap, census, hor)]
            a, o = bp._gap(mode, q)[0], bo._gap(mode, q)[0]
            assert same(a, o), (it, mode, a, o)
            n += 1
    assert n == 4500
