#!/usr/bin/env python
"""Benchmark: multi-SLO DP plans/sec (and p50 per-plan latency) on B200.

Workload (BASELINE.json configs[1], SURVEY.md §8 d2 "C2"): Mixed Summarizer+Coder
SLOs, 240 running decoders + 16 pending requests per instance (256 requests,
tiers i%2), desk perf model, chunked prefill 2048, batch of 1024 instances per
GPU. One "step" = one plan() pass over the whole batch. Synthetic inputs from the
reference's own stress generator (acceptance_main.cpp:577-605).

  value  : device-resident instances, kernel pipeline only (CUDA events on the
           launching stream), L2 flushed (512 MiB write) before every step.
  e2e    : the reference-facing C-ABI call slos_plan_batch with HOST inputs:
           host prep + H2D + kernels + compaction + D2H of every plan.
  multi-GPU: one process per GPU, weak scaling (1024 instances per rank), one
           all_gather of 88-byte result records per step (the only collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "multi-SLO DP plans/sec and p50 per-plan latency at 1/2/4/8 B200"
FAMILY = "C2"
PER_RANK = 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instances", type=int, default=PER_RANK)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="C2", choices=["C2", "C5"],
                    help="C2 (default, BASELINE configs[1]) or C5: the recorded capacity-sweep "
                         "corpus, 65,536 instances sharded across the ranks (configs[4])")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None
        self._t = None

    def _read(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __enter__(self):
        # nvidia-smi's own loop (-lms) samples every 50 ms while the timed steps run
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                        "--format=csv,noheader,nounits", "-lms", "50"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p:
            time.sleep(0.1)
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
        if self._t:
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() in ("active", "1", "yes")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


C5_TOTAL = 65536


def c5_shard(lib, rank: int, world: int):
    """configs[4]: the C5 corpus (tests/golden/c5_*.bin.gz, schedule() inputs recorded
    from the reference simulator's sweep grid, 2,048 per planner configuration) tiled
    to 65,536 instances, half AR (chatbot/coder/summarizer/toolllm) and half
    speculative (reasoning), sharded contiguously across the ranks (strong scaling).
    Returns (batch, per-instance handles, shard size)."""
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import PerfTerm, PlannerConfig, _Handle
    from paper_2504_08784_b200.sweep import shard_range
    gold = os.path.join(ROOT, "tests", "golden")
    model = [PerfTerm(2.5e-5, 2e-3, 0.006), PerfTerm(0.0, 0.0, 0.02)]  # the desk model
    parts, hs = [], []
    for g, spec in (("ar", False), ("spec", True)):
        b = W.load_corpus(os.path.join(gold, f"c5_{g}.bin.gz"))
        half = C5_TOTAL // 2
        parts.append(b.tiled((half + b.n - 1) // b.n).subset(range(half)))
        cfg = PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=spec, spec_alpha=0.8,
                            spec_max_len=8)
        hs.append((_Handle(lib, model, W.TWO_TIER_SLO, cfg), half))
    full = W.InstanceBatch.concat(parts)
    sh = shard_range(C5_TOTAL, rank, world)
    handles = [hs[0][0]] * hs[0][1] + [hs[1][0]] * hs[1][1]
    return full.subset(sh), [handles[k] for k in sh], len(sh)


def family():
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.sweep import ShardSpec
    F = W.FAMILIES[FAMILY]
    return ShardSpec(F["spec"], F["model"], F["cfg"]), F


def cpu_reference_rate(n_inst: int, seeds_base: int = 0):
    """The reference CPU planner (oracle/_ref, compiled from the reference sources;
    else the C oracle port) over a bounded sample of the same workload, all host
    cores. Returns (plans/sec, kind, cores, sample description)."""
    from paper_2504_08784_b200 import abi
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import _Handle
    spec, F = family()
    if os.path.exists(abi.REF_LIB):
        lib, kind = abi.reference(), "reference"
        cores = int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))
    else:
        lib, kind, cores = abi.oracle(), "port", 1
    batch = W.InstanceBatch.stress(spec.family, range(seeds_base, seeds_base + n_inst))
    h = _Handle(lib, spec.model, spec.slo, spec.cfg)
    hs = (C.c_void_p * batch.n)(*([h.ptr] * batch.n))
    outs = (abi.Result * batch.n)()
    t = time.perf_counter()
    lib.slos_plan_batch(hs, batch.n, C.c_void_p(batch.inputs_ptr()), 0, outs, None)
    dt = time.perf_counter() - t
    for k in range(batch.n):
        lib.slos_result_free(C.byref(outs[k]))
    return batch.n / dt, kind, cores, dt


def cpu_reference_rate_c5(n_inst: int = 8192):
    """The reference CPU planner over the first n_inst instances of the C5 workload
    (all host cores). Returns (plans/sec, kind, cores, seconds, n)."""
    from paper_2504_08784_b200 import abi
    if os.path.exists(abi.REF_LIB):
        lib, kind = abi.reference(), "reference"
        cores = int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))
    else:
        lib, kind, cores = abi.oracle(), "port", 1
    b, handles, _ = c5_shard(lib, 0, 1)
    idx = list(range(0, C5_TOTAL, C5_TOTAL // n_inst))  # both halves, every recorded source
    sub = b.subset(idx)
    hs = (C.c_void_p * len(idx))(*[handles[k].ptr for k in idx])
    outs = (abi.Result * len(idx))()
    t = time.perf_counter()
    lib.slos_plan_batch(hs, len(idx), C.c_void_p(sub.inputs_ptr()), 0, outs, None)
    dt = time.perf_counter() - t
    for k in range(len(idx)):
        lib.slos_result_free(C.byref(outs[k]))
    return len(idx) / dt, kind, cores, dt, len(idx)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    ncores = int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))
    if args.workload == "C5":  # configs[4] corpus: the reference over all host cores
        for _ in range(args.warmup):
            cpu_reference_rate_c5()
        rates = [cpu_reference_rate_c5() for _ in range(args.steps)]
        value = sum(r[0] for r in rates) / len(rates)
        kind, cores, n5 = rates[0][1], rates[0][2], rates[0][4]
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": "plans/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n5 / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp64+int64",
            "data": "schedule() inputs recorded from the reference simulator's capacity-sweep grid",
            "config": {"workload": "C5: bursty capacity-sweep corpus (BASELINE configs[4])",
                       "instances_per_step": n5, "parallelism": f"{cores} host threads"},
            "cpu_baseline": {"value": value, "unit": "plans/s", "cores": cores, "kind": kind,
                             "sample": f"{n5} C5 instances per step"},
            "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0
    sample = max(2 * ncores, 8)  # ~0.5 s of all-core reference work per step
    for _ in range(args.warmup):
        cpu_reference_rate(sample)
    rates, wall = [], 0.0
    for k in range(args.steps):
        r, kind, cores, dt = cpu_reference_rate(sample, seeds_base=10000 + k * sample)
        rates.append(r)
        wall += dt
    value = args.steps * sample / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "plans/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp64+int64",
        "data": "synthetic (reference stress generator G(240,16), acceptance_main.cpp:577-605)",
        "config": {"workload": "C2: Mixed Summarizer+Coder, 240 running + 16 pending per instance, "
                               "chunk 2048, desk model", "instances_per_step": sample,
                   "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "plans/s", "cores": cores, "kind": kind,
                         "sample": f"{sample} C2 instances per step"},
        "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def load_ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2504_08784_b200 import abi
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import _Handle
    from paper_2504_08784_b200.sweep import ShardSolver, gather_records, records_view, weak_seeds

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = abi.product()
    spec, F = family()
    c5 = args.workload == "C5"
    if c5:
        batch5, handles5, per = c5_shard(lib, rank, world)
        solver = ShardSolver(lib, spec, None, batch=batch5, handles=handles5)
    else:
        per = args.instances
        solver = ShardSolver(lib, spec, weak_seeds(rank, per))
    stream = torch.cuda.Stream()
    sptr = stream.cuda_stream
    rec = torch.empty((per, C.sizeof(abi.Record)), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    solver.upload(sptr)
    solver.converge(rec, sptr)
    torch.cuda.synchronize()

    def step():
        solver.solve(sptr)
        solver.records(rec.data_ptr(), sptr)
        with torch.cuda.stream(stream):
            allrec = gather_records(rec, world)
        return allrec

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    anc_ms, dp_ms, build_ms = [], [], []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            evs[k][0].record(stream)
            allrec = step()
            evs[k][1].record(stream)
            st = solver.stage_ms()
            anc_ms.append(st[0])
            dp_ms.append(st[1])
            build_ms.append(st[2])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = sum(s.elapsed_time(e) for s, e in evs)
    t = torch.tensor([total_ms, sum(anc_ms), sum(dp_ms), sum(build_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, anc_tot, dp_tot, build_tot = (float(x) for x in t.tolist())
    recs = records_view(allrec)
    n_all = per * world if not c5 else len(recs)
    assert len(recs) == n_all and (recs["status"] == 0).all(), "solve produced error records"
    value = n_all * args.steps / (total_ms / 1e3)

    # correctness spot check: download the last solve of this shard
    outs = solver.download(sptr)
    ok = all(outs[k].status == 0 for k in range(per))
    adm = sum(outs[k].n_admitted for k in range(per)) / per
    solver.free_results()

    # ---- e2e: the reference-facing C-ABI call with host inputs ----
    batch = solver.batch
    hs = solver._hs
    outs2 = (abi.Result * per)()
    for _ in range(max(3, args.warmup)):  # pinned result arenas and host pools warm
        lib.slos_plan_batch(hs, per, C.c_void_p(batch.inputs_ptr()), 0, outs2, sptr)
        for k in range(per):
            lib.slos_result_free(C.byref(outs2[k]))
    if world > 1:
        dist.barrier()
    e2e_wall = 0.0
    h2d = C.c_int64()
    d2h = C.c_int64()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        lib.slos_plan_batch(hs, per, C.c_void_p(batch.inputs_ptr()), 0, outs2, sptr)
        e2e_wall += time.perf_counter() - t0
        lib.slos_last_transfer_bytes(C.byref(h2d), C.byref(d2h))
        for k in range(per):
            lib.slos_result_free(C.byref(outs2[k]))
    te = torch.tensor([e2e_wall], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n_all * args.steps / float(te.item())

    line = None
    if rank == 0:
        # p50 per-plan latency: one C1 (ChatBot) instance per call, end to end
        F1 = W.FAMILIES["C1"]
        h1 = _Handle(lib, F1["model"], W.TWO_TIER_SLO, F1["cfg"])
        lat = []
        for s in range(34):
            b1 = W.InstanceBatch.stress(F1["spec"], [50000 + s])
            o1 = (abi.Result * 1)()
            hh = (C.c_void_p * 1)(h1.ptr)
            t0 = time.perf_counter()
            lib.slos_plan_batch(hh, 1, C.c_void_p(b1.inputs_ptr()), 0, o1, sptr)
            lat.append(time.perf_counter() - t0)
            lib.slos_result_free(C.byref(o1[0]))
        lat = sorted(lat[3:])
        p50_ms = 1e3 * lat[len(lat) // 2]
        # roofline of the dominant kernel (admission DP): algorithmic bytes per
        # plan from the reference-defined counters:
        #   B_smem = 80*T + 32*D + 48*S
        T = int(recs["transitions"][:per].sum())
        D = int(recs["dues"][:per].sum())
        S = int(recs["slots"][:per].sum())
        alg = 80 * T + 32 * D + 48 * S
        ck = clk.summary()
        f_mhz = ck.get("sm_mhz") or 1965.0
        # the admission-DP stage: anchor caches + pair groups + level DP (the
        # reference counters' work is split across these three kernels)
        dp_avg_s = ((anc_tot + dp_tot) / args.steps) / 1e3
        achieved = alg / dp_avg_s / 1e9
        peak = 148 * 128 * f_mhz * 1e6 / 1e9
        ncu = load_ncu_traffic()
        traffic = None
        if ncu and ncu.get("kernel") == "dp_stage" and ncu.get("instances") == per:
            traffic = ncu.get("dram_bytes_per_launch")
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            ncores = int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))
            if c5:
                r, kind, cores, dt, n5 = cpu_reference_rate_c5()
                cpu = {"value": r, "unit": "plans/s", "cores": cores, "kind": kind,
                       "sample": f"{n5} C5 corpus instances (mixed AR / speculative), {dt:.1f} s wall"}
            else:
                sample = max(16 * ncores, 32)
                r, kind, cores, dt = cpu_reference_rate(sample, seeds_base=0)
                cpu = {"value": r, "unit": "plans/s", "cores": cores, "kind": kind,
                       "sample": f"{sample} C2 instances (seeds 0..{sample - 1}), {dt:.1f} s wall"}
        line = {
            "metric": METRIC, "value": value, "unit": "plans/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp64+int64",
            "data": "synthetic (reference stress generator G(240,16), acceptance_main.cpp:577-605)",
            "config": {"workload": "C2: Mixed Summarizer+Coder, 240 running + 16 pending per instance, "
                                   "chunk 2048, desk model (BASELINE configs[1])",
                       "instances_per_gpu": per, "total_instances": n_all,
                       "parallelism": f"{world} GPU(s), one process each, weak scaling",
                       "l2": "flushed before every step (512 MiB write)",
                       "p50_plan_ms": {"value": p50_ms, "workload": "C1 ChatBot: 48 running + 16 pending, "
                                       "one instance per slos_plan_batch call, end to end"}},
            "e2e": {"value": e2e_value, "unit": "plans/s", "h2d_bytes_per_step": int(h2d.value),
                    "d2h_bytes_per_step": int(d2h.value)},
            "gpu_launches": 5 * args.steps,
            "kernel_ms_per_step": {"anchor_kernel+group_kernel": anc_tot / args.steps,
                                   "dp_kernel": dp_tot / args.steps, "build_kernel": build_tot / args.steps},
            "roofline": {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "dp_stage (anchor_kernel + group_kernel + dp_kernel)",
                         "alg_bytes_per_launch": alg,
                         "note": "B_smem=80T+32D+48S per plan (reference counters, SURVEY 8d6) over the "
                                 "admission-DP stage's device time; peak=148 SM x 128 B/clk x median "
                                 "SM clock under load"},
            "cpu_baseline": cpu,
            "clocks": ck,
            "check": {"statuses_ok": bool(ok), "mean_admitted": adm},
        }
        if c5:  # configs[4]: the sharded sweep corpus, strong scaling
            line["scaling"] = "strong"
            line["data"] = ("schedule() inputs recorded from the reference simulator's capacity-sweep grid "
                            "(tests/golden/c5_*.bin.gz, 4,096 distinct, tiled)")
            line["config"]["workload"] = ("C5: bursty capacity-sweep corpus, 65,536 instances (32,768 AR + "
                                          "32,768 speculative) sharded across the GPUs (BASELINE configs[4])")
            line["config"]["parallelism"] = f"{world} GPU(s), one process each, strong scaling"
            line["config"]["instances_per_gpu"] = per
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
