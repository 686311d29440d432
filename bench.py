#!/usr/bin/env python
"""Benchmark: multi-SLO DP plans/sec (and p50 per-plan latency) on B200.

Headline workload (BASELINE.json configs[1], SURVEY.md §8 d2 "C2"): Mixed
Summarizer+Coder SLOs, 240 running decoders + 16 pending requests per instance
(256 requests, tiers i%2), desk perf model, chunked prefill 2048, a batch of 1024
instances per GPU. One "step" = one plan() pass over the whole batch. Synthetic
inputs from the reference's own stress generator (acceptance_main.cpp:577-605).

  value  : device-resident instances, kernel pipeline only (CUDA events on the
           launching stream), L2 flushed (512 MiB write) before every step.
  e2e    : the reference-facing C-ABI call slos_plan_batch with HOST inputs:
           host prep + H2D + kernels + compaction + D2H of every plan.
  multi-GPU: one process per GPU, weak scaling (1024 instances per rank), one
           all_gather of 88-byte result records per step (the only collective).
           `--gpus N` without a torchrun environment re-launches itself under
           torch.distributed.run with N ranks.
  legs   : the other BASELINE configs measured in the same run (N=1): C1 (p50
           single-plan latency + plans/s), C3 (4-replica routing rounds with
           speculative decoding), C4 (2032 decoders, budget 8192) and C5 (the
           65,536-instance sweep corpus, sharded across the ranks) -- each with the
           reference CPU planner timed beside it on this box's cores.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "multi-SLO DP plans/sec and p50 per-plan latency at 1/2/4/8 B200"
FAMILY = "C2"
PER_RANK = 1024
C5_TOTAL = 65536


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instances", type=int, default=PER_RANK)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-legs", action="store_true", help="headline C2 line only")
    ap.add_argument("--workload", default="C2", choices=["C2", "C5"],
                    help="C2 (default, BASELINE configs[1]) or C5: the recorded capacity-sweep "
                         "corpus, 65,536 instances sharded across the ranks (configs[4])")
    ap.add_argument("--launch-check", action="store_true",
                    help="multi-rank launcher self-test: init the process group (gloo on CPU, nccl "
                         "on GPUs), all-gather the ranks, print one line, exit")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args) -> None:
    """`--gpus N` (N > 1) outside torchrun: re-exec under torch.distributed.run with
    one rank per GPU (127.0.0.1 rendezvous). Under torchrun WORLD_SIZE is set and
    this is a no-op."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def launch_check(args) -> int:
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    gpu = torch.cuda.is_available()
    if world > 1:
        if gpu:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = "cuda" if gpu else "cpu"
    t = torch.tensor([rank], dtype=torch.int64, device=dev)
    parts = [torch.zeros_like(t) for _ in range(world)]
    if world > 1:
        dist.all_gather(parts, t)
    else:
        parts = [t]
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "requested": args.gpus,
                          "ranks": [int(p.item()) for p in parts],
                          "backend": dist.get_backend() if world > 1 else None}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


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


def host_cpu():
    """The box's host CPU: model name and the threads this process may use."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count(),
            "threads_used": int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))}


# ------------------------------------------------------------------ workloads ---

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


def family(name=FAMILY):
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.sweep import ShardSpec
    F = W.FAMILIES[name]
    return ShardSpec(F["spec"], F["model"], F["cfg"]), F


# ------------------------------------------------- reference CPU planner arm ---

def _ref_batch_rate(lib, batch, handles):
    hs = (C.c_void_p * batch.n)(*handles)
    from paper_2504_08784_b200 import abi
    outs = (abi.Result * batch.n)()
    t = time.perf_counter()
    lib.slos_plan_batch(hs, batch.n, C.c_void_p(batch.inputs_ptr()), 0, outs, None)
    dt = time.perf_counter() - t
    for k in range(batch.n):
        lib.slos_result_free(C.byref(outs[k]))
    return batch.n / dt, dt


def cpu_reference_rate(n_inst: int, seeds_base: int = 0, fam: str = FAMILY):
    """The reference CPU planner (oracle/_ref, compiled from the reference sources;
    else the C oracle port) over a bounded sample of the family, all host cores, one
    planner per worker thread. Inputs come from the reference
    harness's own generator in oracle/_ref (no repo library is loaded).
    Returns (plans/sec, kind, cores, seconds)."""
    from paper_2504_08784_b200 import abi
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import _Handle
    spec, F = family(fam)
    if os.path.exists(abi.REF_LIB):
        lib, kind, gen = abi.reference(), "reference", abi.reference_stress_gen()
        cores = int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))
    else:
        lib, kind, cores, gen = abi.oracle(), "port", 1, None
    batch = W.InstanceBatch.stress(spec.family, range(seeds_base, seeds_base + n_inst), gen=gen)
    h = _Handle(lib, spec.model, spec.slo, spec.cfg)
    r, dt = _ref_batch_rate(lib, batch, [h.ptr] * batch.n)
    return r, kind, cores, dt


def cpu_reference_p50(fam: str, n: int = 31, seeds_base: int = 50000):
    """Single-thread p50 per plan of the reference, a fresh BatchPlanner per instance
    and only schedule() inside the clock -- the reference's own latency criterion
    (acceptance_main.cpp:573-626). Returns ms or None without oracle/_ref."""
    from paper_2504_08784_b200 import abi
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import _Handle
    if not os.path.exists(abi.REF_LIB):
        return None
    spec, F = family(fam)
    lib = abi.reference()
    timed = abi.reference_schedule_timed()
    batch = W.InstanceBatch.stress(spec.family, range(seeds_base, seeds_base + n), gen=abi.reference_stress_gen())
    h = _Handle(lib, spec.model, spec.slo, spec.cfg)
    ts = []
    for k in range(n):
        out = abi.Result()
        sec = C.c_double()
        timed(h.ptr, C.c_void_p(batch.inputs_ptr() + k * batch.inputs.itemsize), 0, C.byref(out), C.byref(sec))
        lib.slos_result_free(C.byref(out))
        ts.append(sec.value)
    ts.sort()
    return 1e3 * ts[len(ts) // 2]


def cpu_reference_rate_c5(n_inst: int = 8192):
    """The reference CPU planner over n_inst instances of the C5 workload spread over
    both halves (all host cores). Returns (plans/sec, kind, cores, seconds, n)."""
    from paper_2504_08784_b200 import abi
    if os.path.exists(abi.REF_LIB):
        lib, kind = abi.reference(), "reference"
        cores = int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))
    else:
        lib, kind, cores = abi.oracle(), "port", 1
    b, handles, _ = c5_shard(lib, 0, 1)
    idx = list(range(0, C5_TOTAL, C5_TOTAL // n_inst))  # both halves, every recorded source
    sub = b.subset(idx)
    r, dt = _ref_batch_rate(lib, sub, [handles[k].ptr for k in idx])
    return r, kind, cores, dt, len(idx)


def run_reference(args):
    """The driver's reference arm: the reference's own CPU planner (oracle/_ref) on
    this box's host cores, on our arm's workload, metric and unit. Only rank 0 works."""
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
            "host_cpu": host_cpu(),
        }
        print(json.dumps(line), flush=True)
        return 0
    # >= 16 instances per host thread per step, so a few slow instances cannot
    # dominate a step; warm-up steps are short (they only fault pages in)
    sample = max(16 * ncores, 64)
    for _ in range(args.warmup):
        cpu_reference_rate(ncores, seeds_base=90000)
    rates, wall = [], 0.0
    kind, cores = "reference", ncores
    for k in range(args.steps):
        r, kind, cores, dt = cpu_reference_rate(sample, seeds_base=10000 + k * sample)
        rates.append(r)
        wall += dt
    value = args.steps * sample / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "plans/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp64+int64",
        "data": "synthetic (reference stress generator G(240,16), acceptance_main.cpp:577-605, "
                "drawn by oracle/_ref)",
        "config": {"workload": "C2: Mixed Summarizer+Coder, 240 running + 16 pending per instance, "
                               "chunk 2048, desk model (BASELINE configs[1])", "instances_per_step": sample,
                   "parallelism": f"{cores} host threads, one reference planner per thread"},
        "cpu_baseline": {"value": value, "unit": "plans/s", "cores": cores, "kind": kind,
                         "sample": f"{sample} C2 instances per step ({sample // max(1, cores)} per thread)"},
        "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host_cpu": host_cpu(),
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ our GPU arm ---

def load_ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def smem_peak():
    """Measured shared-memory read bandwidth of this GPU (libslos_probe.so), GB/s,
    and the SM clock it ran at; None if the probe is not built."""
    path = os.path.join(ROOT, "paper_2504_08784_b200", "libslos_probe.so")
    if not os.path.exists(path):
        return None
    lib = C.CDLL(path)
    lib.slos_probe_smem.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    g, f = C.c_double(), C.c_double()
    best = None
    for _ in range(3):
        if lib.slos_probe_smem(20000, C.byref(g), C.byref(f)) == 0 and (best is None or g.value > best[0]):
            best = (g.value, f.value)
    return best


class Resident:
    """A device-resident batch behind one slos_workspace (CUDA-event timing)."""

    def __init__(self, lib, batch, handles, stream):
        import torch
        from paper_2504_08784_b200 import abi
        from paper_2504_08784_b200.sweep import ShardSolver
        self.torch = torch
        self.solver = ShardSolver(lib, None, None, batch=batch, handles=handles)
        self.stream = stream
        self.rec = torch.empty((batch.n, C.sizeof(abi.Record)), dtype=torch.uint8, device="cuda")
        self.solver.upload(stream.cuda_stream)
        self.solver.converge(self.rec, stream.cuda_stream)
        torch.cuda.synchronize()

    def time(self, steps, warmup, flush=None):
        torch = self.torch
        s = self.stream
        for _ in range(max(3, warmup)):
            self.solver.solve(s.cuda_stream)
        torch.cuda.synchronize()
        ms, launches, dp_stage = 0.0, 0, 0.0
        for _ in range(steps):
            if flush is not None:
                with torch.cuda.stream(s):
                    flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            self.solver.solve(s.cuda_stream)
            b.record(s)
            b.synchronize()
            ms += a.elapsed_time(b)
            launches += self.solver.launches()
            st = self.solver.stage_ms()
            dp_stage += st[0] + st[1]  # anchor + group + DP (the roofline's stage)
        self.solver.records(self.rec.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        self.dp_stage_ms = dp_stage / steps
        return ms / steps, launches / steps

    def records(self):
        from paper_2504_08784_b200.sweep import records_view
        return records_view(self.rec)

    def close(self):
        self.solver.close()


def e2e_rate(lib, batch, handles, steps, warmup, sptr):
    """slos_plan_batch with host inputs, wall clock per call (host prep, H2D,
    kernels, compaction, D2H of every plan). Returns (plans/s, h2d, d2h, s/call)."""
    from paper_2504_08784_b200 import abi
    n = batch.n
    hs = (C.c_void_p * n)(*handles)
    outs = (abi.Result * n)()
    for _ in range(max(3, warmup)):
        lib.slos_plan_batch(hs, n, C.c_void_p(batch.inputs_ptr()), 0, outs, sptr)
        for k in range(n):
            lib.slos_result_free(C.byref(outs[k]))
    wall = 0.0
    h2d, d2h = C.c_int64(), C.c_int64()
    for _ in range(steps):
        t0 = time.perf_counter()
        lib.slos_plan_batch(hs, n, C.c_void_p(batch.inputs_ptr()), 0, outs, sptr)
        wall += time.perf_counter() - t0
        lib.slos_last_transfer_bytes(C.byref(h2d), C.byref(d2h))
        bad = sum(1 for k in range(n) if outs[k].status != 0)
        for k in range(n):
            lib.slos_result_free(C.byref(outs[k]))
        assert bad == 0, f"{bad} instances failed"
    return n * steps / wall, int(h2d.value), int(d2h.value), wall / steps


def single_plan_p50(lib, fam, sptr, n=34, seeds_base=50000):
    """p50 end-to-end latency of ONE plan per slos_plan_batch call (ms)."""
    from paper_2504_08784_b200 import abi
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import _Handle
    spec, F = family(fam)
    h = _Handle(lib, spec.model, spec.slo, spec.cfg)
    lat = []
    for s in range(n):
        b1 = W.InstanceBatch.stress(spec.family, [seeds_base + s])
        o1 = (abi.Result * 1)()
        hh = (C.c_void_p * 1)(h.ptr)
        t0 = time.perf_counter()
        lib.slos_plan_batch(hh, 1, C.c_void_p(b1.inputs_ptr()), 0, o1, sptr)
        lat.append(time.perf_counter() - t0)
        assert o1[0].status == 0
        lib.slos_result_free(C.byref(o1[0]))
    lat = sorted(lat[3:])
    return 1e3 * lat[len(lat) // 2]


def leg_family(lib, fam, n, stream, steps, warmup, flush, cpu_sample, cpu_p50_n, with_cpu):
    """One stress family as a bench leg: device-resident and e2e plans/s on n
    instances, the reference beside it (all cores, bounded sample; single-thread p50)."""
    from paper_2504_08784_b200 import workload as W
    from paper_2504_08784_b200.planner import _Handle
    spec, F = family(fam)
    batch = W.InstanceBatch.stress(spec.family, range(n))
    h = _Handle(lib, spec.model, spec.slo, spec.cfg)
    res = Resident(lib, batch, [h] * n, stream)
    ms, launches = res.time(steps, warmup, flush)
    recs = res.records()
    res.close()
    assert (recs["status"] == 0).all()
    e2e, h2d, d2h, _ = e2e_rate(lib, batch, [h.ptr] * n, max(2, steps // 2), 2, stream.cuda_stream)
    T, D, S = int(recs["transitions"].sum()), int(recs["dues"].sum()), int(recs["slots"].sum())
    out = {"workload": F.get("desc", fam), "instances": n, "value": n / (ms / 1e3), "unit": "plans/s",
           "ms_per_step": ms, "gpu_launches_per_step": launches,
           "e2e": {"value": e2e, "unit": "plans/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
           "alg_bytes_per_plan": (80 * T + 32 * D + 48 * S) / n}
    # the same roofline as the headline: algorithmic bytes of the launch
    # over the admission-DP stage's device time, against the measured LDS peak
    probe = smem_peak()
    if probe and res.dp_stage_ms > 0:
        ach = (80 * T + 32 * D + 48 * S) / (res.dp_stage_ms / 1e3) / 1e9
        out["roofline"] = {"bound": "smem", "achieved": ach, "peak": probe[0], "unit": "GB/s",
                           "frac": ach / probe[0], "dp_stage_ms": res.dp_stage_ms,
                           "note": "algorithmic work rate (reference-defined counters), as the headline"}
    if with_cpu:
        r, kind, cores, dt = cpu_reference_rate(cpu_sample, seeds_base=0, fam=fam)
        out["cpu_baseline"] = {"value": r, "unit": "plans/s", "cores": cores, "kind": kind,
                               "sample": f"{cpu_sample} {fam} instances, {dt:.1f} s wall"}
        if cpu_p50_n:
            out["cpu_p50_plan_ms_1thread"] = cpu_reference_p50(fam, cpu_p50_n)
    return out


def leg_c5(lib, rank, world, stream, steps, warmup, with_cpu):
    """configs[4]: the 65,536-instance sweep corpus sharded across the ranks (strong
    scaling); the records of every rank are all-gathered (the only collective)."""
    import torch
    import torch.distributed as dist
    from paper_2504_08784_b200.sweep import gather_records, records_view
    b5, h5, per = c5_shard(lib, rank, world)
    res = Resident(lib, b5, h5, stream)
    if world > 1:
        dist.barrier()
    ms, launches = res.time(steps, warmup)
    with torch.cuda.stream(stream):
        allrec = gather_records(res.rec, world, n_total=C5_TOTAL)
    torch.cuda.synchronize()
    recs = records_view(allrec)
    res.close()
    e2e, h2d, d2h, sec = e2e_rate(lib, b5, [h.ptr for h in h5], max(2, steps // 2), 2, stream.cuda_stream)
    t = torch.tensor([ms, sec], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, sec = (float(x) for x in t.tolist())
    out = {"workload": "C5: bursty capacity-sweep corpus, 65,536 instances (32,768 AR + 32,768 speculative) "
                       "recorded from the reference simulator, sharded across the GPUs (BASELINE configs[4])",
           "instances": C5_TOTAL, "scaling": "strong", "value": C5_TOTAL / (ms / 1e3), "unit": "plans/s",
           "ms_per_step": ms, "gpu_launches_per_step": launches,
           "e2e": {"value": C5_TOTAL / sec, "unit": "plans/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h},
           "statuses_ok": bool(len(recs) == C5_TOTAL and (recs["status"] == 0).all())}
    if with_cpu and rank == 0:
        r, kind, cores, dt, n5 = cpu_reference_rate_c5()
        out["cpu_baseline"] = {"value": r, "unit": "plans/s", "cores": cores, "kind": kind,
                               "sample": f"{n5} C5 corpus instances (mixed AR / speculative), {dt:.2f} s wall"}
    return out


def leg_c3(lib, stream, steps, warmup, with_cpu):
    """configs[2]: reasoning + speculative decoding over 4 replicas with routing
    (paper_2504_08784_b200/routing.py). Absent until the routing driver exists."""
    try:
        from paper_2504_08784_b200 import routing
    except Exception:
        return None
    return routing.bench_leg(lib, stream, steps, warmup, with_cpu)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2504_08784_b200 import abi
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
    n_total = C5_TOTAL if c5 else per * world

    def step():
        solver.solve(sptr)
        solver.records(rec.data_ptr(), sptr)
        with torch.cuda.stream(stream):
            allrec = gather_records(rec, world, n_total=n_total)
        return allrec

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    anc_ms, dp_ms, build_ms, launches = [], [], [], 0
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            evs[k][0].record(stream)
            allrec = step()
            evs[k][1].record(stream)
            launches += solver.launches() + 1  # + records_kernel
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
    n_all = n_total
    assert len(recs) == n_all and (recs["status"] == 0).all(), "solve produced error records"
    value = n_all * args.steps / (total_ms / 1e3)

    # correctness spot check: download the last solve of this shard
    outs = solver.download(sptr)
    ok = all(outs[k].status == 0 for k in range(per))
    adm = sum(outs[k].n_admitted for k in range(per)) / per
    solver.free_results()

    # ---- e2e: the reference-facing C-ABI call with host inputs ----
    if world > 1:
        dist.barrier()
    e2e_value, h2d, d2h, sec = e2e_rate(lib, solver.batch, list(solver._hs), args.steps, args.warmup, sptr)
    te = torch.tensor([sec], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n_all / float(te.item())

    with_cpu = world == 1 and not args.no_cpu_baseline
    legs = {}
    if not args.no_legs and not c5:
        # C5 (strong scaling across every rank) first: it is collective
        legs["C5"] = leg_c5(lib, rank, world, stream, max(3, args.steps // 2), args.warmup, with_cpu)
        if rank == 0 and world == 1:
            legs["C1"] = leg_family(lib, "C1", 1024, stream, max(3, args.steps // 2), args.warmup, flush,
                                    cpu_sample=256, cpu_p50_n=31, with_cpu=with_cpu)
            legs["C1"]["p50_plan_ms"] = single_plan_p50(lib, "C1", sptr)
            legs["C4"] = leg_family(lib, "C4", 64, stream, max(3, args.steps // 2), args.warmup, flush,
                                    cpu_sample=int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1)),
                                    cpu_p50_n=0, with_cpu=with_cpu)
            c3 = leg_c3(lib, stream, max(3, args.steps // 2), args.warmup, with_cpu)
            if c3 is not None:
                legs["C3"] = c3
            # the callers either side of the planner
            from paper_2504_08784_b200 import fit as fit_mod
            from paper_2504_08784_b200 import trace as trace_mod
            legs["trace"] = trace_mod.bench_leg(ROOT, max(3, args.steps // 2), args.warmup, with_cpu)
            legs["fit"] = fit_mod.bench_leg(max(3, args.steps // 2), args.warmup, with_cpu)
        if world > 1:
            dist.barrier()

    line = None
    if rank == 0:
        p50_ms = single_plan_p50(lib, "C1", sptr)
        # roofline of the dominant stage (admission DP): algorithmic bytes per plan
        # from the reference-defined counters (pinned to the
        # instrumented reference by tests/golden/counters.json.gz):
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
        probe = smem_peak()
        nominal = 148 * 128 * f_mhz * 1e6 / 1e9
        if probe:  # measured LDS.128 bandwidth (the probe runs at the same boost clock)
            peak = probe[0]
            peak_src = (f"measured: libslos_probe.so LDS.128 stream on all SMs, {probe[0]:.0f} GB/s "
                        f"(probe SM clock estimate {probe[1]:.0f} MHz)")
        else:
            peak, peak_src = nominal, "nominal 148 SM x 128 B/clk x median SM clock (probe not built)"
        ncu = load_ncu_traffic()
        traffic, traffic_src = None, None
        if ncu and ncu.get("kernel") == "dp_stage" and ncu.get("instances") == per:
            traffic = ncu.get("dram_bytes_per_launch")
            traffic_src = "ncu --set full capture of the same workload, profiles/ncu_summary.json"
        cpu = None
        if with_cpu:
            ncores = int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))
            if c5:
                r, kind, cores, dt, n5 = cpu_reference_rate_c5()
                cpu = {"value": r, "unit": "plans/s", "cores": cores, "kind": kind,
                       "sample": f"{n5} C5 corpus instances (mixed AR / speculative), {dt:.1f} s wall"}
            else:
                sample = max(16 * ncores, 64)
                r, kind, cores, dt = cpu_reference_rate(sample, seeds_base=0)
                cpu = {"value": r, "unit": "plans/s", "cores": cores, "kind": kind,
                       "sample": f"{sample} C2 instances (seeds 0..{sample - 1}), {dt:.1f} s wall",
                       "p50_plan_ms_1thread": cpu_reference_p50("C2", 31),
                       "p50_note": "single thread, fresh BatchPlanner per instance, schedule() only "
                                   "(acceptance_main.cpp:573-626), 31 instances",
                       "host_cpu": host_cpu()}
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
            "e2e": {"value": e2e_value, "unit": "plans/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "gpu_launches_note": "kernels launched inside the timed steps, counted by the library per solve "
                                 "(anchor/group/dp per solve part, one per non-empty reconstruction queue) "
                                 "+ the records kernel",
            "kernel_ms_per_step": {"anchor_kernel+group_kernel": anc_tot / args.steps,
                                   "dp_kernel": dp_tot / args.steps, "build_kernel": build_tot / args.steps},
            "roofline": {"bound": "smem", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src, "peak_nominal": nominal,
                         "kernel": "dp_stage (anchor_kernel + group_kernel + dp_kernel)",
                         "alg_bytes_per_launch": alg,
                         "note": "ALGORITHMIC work rate, not a hardware counter: B_smem=80T+32D+48S per plan "
                                 "(reference-defined counters, SURVEY 8d6) over the admission-DP stage's "
                                 "device time; the engine shares the census across count vectors, so it "
                                 "moves far fewer bytes than this"},
            "cpu_baseline": cpu,
            "clocks": ck,
            "check": {"statuses_ok": bool(ok), "mean_admitted": adm},
        }
        if legs:
            line["legs"] = legs
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
    self_launch(args)
    if args.launch_check:
        return launch_check(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
