"""Structural fuzz cases for differential parity (product vs oracle vs reference).

Each case varies the parts of plan() that the §8d stress families never reach:
forced running prefills (chain floor), decode backlog and overdue lines, 1-3
tiers, speculative decoding, planning margin, chunk/batch caps, duplicate and
near-duplicate deadlines, empty sets, memory pressure, zero tail horizon.
"""
from __future__ import annotations

import random

from paper_2504_08784_b200.planner import (PendingRequest, PerfTerm, PlannerConfig, RunningRequest,
                                           ScheduleInput, SloConfig)


def random_case(seed: int, max_pending: int = 10, max_running: int = 40):
    rng = random.Random(seed)
    L = rng.choice([1, 2, 2, 2, 3])
    base = rng.uniform(0.02, 0.1)
    tp = [base]
    for _ in range(L - 1):
        tp.append(tp[-1] * rng.choice([1.0, 1.5, 2.0, rng.uniform(1.1, 3.0)]))
    slo = SloConfig(tp, [rng.choice([1.0, 3.0, 5.0]) for _ in range(L)], 10)
    terms = [PerfTerm(rng.uniform(1e-6, 6e-5), rng.choice([0.0, rng.uniform(1e-4, 2e-3)]),
                      rng.uniform(1e-3, 0.5 * base))]
    if rng.random() < 0.6:
        terms.append(PerfTerm(0.0, 0.0, rng.uniform(0.2, 0.8) * base))
    cfg = PlannerConfig(max_chunk_tokens=rng.choice([64, 256, 512, 2048]),
                        max_batch_tokens=rng.choice([512, 2048, 16384]),
                        speculative=rng.random() < 0.35, spec_alpha=rng.choice([0.5, 0.8, 0.95, 1.0]),
                        spec_max_len=rng.choice([1, 4, 8]),
                        plan_margin=rng.choice([0.0, 0.0, 0.05, 0.1]))
    now = rng.choice([0.0, 100.0, 12345.678])
    inp = ScheduleInput(now=now, memory_total=rng.choice([50, 200, 2000, 200000]),
                        memory_standard_resident=rng.choice([0, 10, 40]),
                        tail_horizon_s=rng.choice([0.0, 0.2, 0.5]))
    nr = rng.randint(0, max_running)
    ddl_pool = [now + rng.uniform(0.05, 1.5) for _ in range(4)]
    for i in range(nr):
        tier = rng.randrange(L)
        if rng.random() < 0.15:
            inp.running.append(RunningRequest(id=f"r{i:03d}", prefill_remaining=rng.randint(1, 800),
                                              prefill_deadline=rng.choice(ddl_pool + [now + rng.uniform(0.0, 1.2)]),
                                              decode_tier=tier))
        else:
            nd = now + rng.uniform(-0.3 if rng.random() < 0.1 else 0.0, 1.0) * tp[tier]
            inp.running.append(RunningRequest(id=f"r{i:03d}", decode_tier=tier, next_due_s=nd,
                                              backlog=rng.choice([0] * 12 + [1, 2, 5]),
                                              decode_remaining=rng.choice([0, 1, 3, 20, 100, 300])))
    np_ = rng.randint(0, max_pending)
    for i in range(np_):
        if rng.random() < 0.2:
            ddl = rng.choice(ddl_pool)
        elif rng.random() < 0.1:
            ddl = rng.choice(ddl_pool) + rng.choice([1e-10, 5e-10, 2e-7, -3e-10])
        else:
            ddl = now + rng.uniform(0.0, 1.5)
        val = float(rng.randint(1, 9)) if rng.random() < 0.8 else rng.uniform(0.5, 5.0)
        inp.pending.append(PendingRequest(id=rng.choice(["n", "m"]) + f"{i:02d}", prefill_deadline=ddl,
                                          prefill_tokens=rng.randint(1, 2000), decode_tier=rng.randrange(L),
                                          memory_units=rng.randint(1, 100), value=val))
    return terms, slo, cfg, inp
