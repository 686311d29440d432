"""Synthetic planning instances and compact batch marshalling.

* ``stress_instance`` / ``StressSpec``: the reference stress generator G(n_dec,
  n_new, seed, tiers) (acceptance_main.cpp:577-605), computed by
  the C generator in csrc/slos_workload.c (mt19937_64 + libstdc++ uniform draw).
* ``InstanceBatch``: many ScheduleInputs laid out as numpy arrays of the C-ABI
  structs (slos_running / slos_pending / slos_input) with ids packed in one blob,
  so a 1024-instance batch crosses the ABI without per-request Python objects.
* ``oracle_input`` and friends: the reference's integer-time brute-force instance
  adapters (tests/oracle.cpp:104-145).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi
from .planner import (PendingRequest, PerfModel, PerfTerm, PlannerConfig, RunningRequest,
                      ScheduleInput, SloConfig)

# Models.
DESK_MODEL = [PerfTerm(2.5e-5, 2e-3, 0.006), PerfTerm(0.0, 0.0, 0.02)]  # configs/desk_model.txt
B200_SYNTH_MODEL = [PerfTerm(2.5e-6, 2e-4, 0.003), PerfTerm(0.0, 0.0, 0.008)]
TWO_TIER_SLO = SloConfig([0.05, 0.1], [3.0, 5.0], 10)  # configs/chatbot.json:6


@dataclass
class StressSpec:
    """One §8d family member: G(n_dec, n_new, seed, two_tier) + its planner."""
    n_dec: int
    n_new: int
    two_tier: bool = True
    now: float = 100.0
    memory_total: int = 200000
    memory_standard_resident: int = 50000
    tail_horizon_s: float = 0.5


# Benchmark families. budget -> max_batch_tokens, chunk = min(2048, B).
FAMILIES = {
    "C1": dict(spec=StressSpec(48, 16, two_tier=False), model=DESK_MODEL,
               cfg=PlannerConfig(max_chunk_tokens=512, max_batch_tokens=512)),
    "C2": dict(spec=StressSpec(240, 16), model=DESK_MODEL,
               cfg=PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=2048)),
    "C3": dict(spec=StressSpec(124, 4), model=DESK_MODEL,
               cfg=PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=True,
                                 spec_alpha=0.8, spec_max_len=8)),
    "C4": dict(spec=StressSpec(2032, 16), model=B200_SYNTH_MODEL,
               cfg=PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=8192)),
    # the reference's own latency criterion (acceptance_main.cpp:573-626)
    "LAT": dict(spec=StressSpec(200, 10), model=DESK_MODEL, cfg=PlannerConfig()),
}


def uniforms(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float64)
    abi.workload().slos_wl_uniforms(seed, n, out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def stress_arrays(spec: StressSpec, seed: int, slo: SloConfig = TWO_TIER_SLO, gen=None) -> dict:
    """G(n_dec, n_new, seed) arrays. `gen` is the generator entry point: the
    product-side slos_wl_stress by default, or abi.reference_stress_gen() (the
    reference harness's own std::mt19937_64 draws, oracle/_ref) for bench.py's
    reference arm, which must not map any repo library."""
    P = C.POINTER
    tp = (C.c_double * len(slo.tpot_tiers_s))(*slo.tpot_tiers_s)
    a = dict(dec_tier=np.zeros(spec.n_dec, np.int32), dec_next_due=np.zeros(spec.n_dec),
             dec_remaining=np.zeros(spec.n_dec, np.int64), new_deadline=np.zeros(spec.n_new),
             new_prefill=np.zeros(spec.n_new, np.int64), new_tier=np.zeros(spec.n_new, np.int32),
             new_memory=np.zeros(spec.n_new, np.int64), new_value=np.zeros(spec.n_new))
    (gen or abi.workload().slos_wl_stress)(
        seed, spec.n_dec, spec.n_new, 1 if spec.two_tier else 0, tp, spec.now,
        a["dec_tier"].ctypes.data_as(P(C.c_int32)), a["dec_next_due"].ctypes.data_as(P(C.c_double)),
        a["dec_remaining"].ctypes.data_as(P(C.c_int64)),
        a["new_deadline"].ctypes.data_as(P(C.c_double)),
        a["new_prefill"].ctypes.data_as(P(C.c_int64)), a["new_tier"].ctypes.data_as(P(C.c_int32)),
        a["new_memory"].ctypes.data_as(P(C.c_int64)), a["new_value"].ctypes.data_as(P(C.c_double)))
    return a


def stress_instance(spec: StressSpec, seed: int, slo: SloConfig = TWO_TIER_SLO) -> ScheduleInput:
    a = stress_arrays(spec, seed, slo)
    inp = ScheduleInput(now=spec.now, memory_total=spec.memory_total,
                        memory_standard_resident=spec.memory_standard_resident,
                        tail_horizon_s=spec.tail_horizon_s)
    for i in range(spec.n_dec):
        inp.running.append(RunningRequest(id=f"run-{i}", decode_tier=int(a["dec_tier"][i]),
                                          next_due_s=float(a["dec_next_due"][i]),
                                          decode_remaining=int(a["dec_remaining"][i])))
    for i in range(spec.n_new):
        inp.pending.append(PendingRequest(id=f"new-{i}", prefill_deadline=float(a["new_deadline"][i]),
                                          prefill_tokens=int(a["new_prefill"][i]),
                                          decode_tier=int(a["new_tier"][i]),
                                          memory_units=int(a["new_memory"][i]),
                                          value=float(a["new_value"][i])))
    return inp


class InstanceBatch:
    """N ScheduleInputs as contiguous C-ABI struct arrays (numpy-backed)."""

    def __init__(self, inputs_np, running_np, pending_np, blob, id_offsets):
        self.inputs = inputs_np
        self.running = running_np
        self.pending = pending_np
        self._blob = blob
        self._id_offsets = id_offsets

    @property
    def n(self) -> int:
        return len(self.inputs)

    def inputs_ptr(self) -> int:
        return self.inputs.ctypes.data

    def host_bytes(self) -> int:
        return self.inputs.nbytes + self.running.nbytes + self.pending.nbytes + len(self._blob)

    @classmethod
    def from_inputs(cls, inputs) -> "InstanceBatch":
        R = sum(len(i.running) for i in inputs)
        Pn = sum(len(i.pending) for i in inputs)
        ids = []
        for i in inputs:
            ids += [r.id.encode() + b"\0" for r in i.running]
            ids += [p.id.encode() + b"\0" for p in i.pending]
        blob = np.frombuffer(b"".join(ids) + b"\0", np.uint8).copy()
        offs = np.cumsum([0] + [len(x) for x in ids])[:-1]
        base = blob.ctypes.data
        run = np.zeros(max(1, R), abi.RUNNING_DTYPE)
        pen = np.zeros(max(1, Pn), abi.PENDING_DTYPE)
        inp = np.zeros(len(inputs), abi.INPUT_DTYPE)
        r0 = p0 = k = 0
        for n_, i in enumerate(inputs):
            for r in i.running:
                run[r0] = (base + offs[k], r.prefill_remaining, r.prefill_deadline, r.decode_tier, 0,
                           r.next_due_s, r.backlog, r.decode_remaining)
                r0 += 1
                k += 1
            for p in i.pending:
                pen[p0] = (base + offs[k], p.prefill_deadline, p.prefill_tokens, p.decode_tier, 0,
                           p.memory_units, p.value)
                p0 += 1
                k += 1
        out = cls(inp, run, pen, blob, offs)
        r0 = p0 = 0
        for n_, i in enumerate(inputs):
            inp[n_] = (i.now, run.ctypes.data + r0 * run.itemsize, len(i.running), len(i.pending),
                       pen.ctypes.data + p0 * pen.itemsize, i.memory_total,
                       i.memory_standard_resident, i.tail_horizon_s)
            r0 += len(i.running)
            p0 += len(i.pending)
        return out

    @classmethod
    def stress(cls, spec: StressSpec, seeds, slo: SloConfig = TWO_TIER_SLO, gen=None,
               unique_ids: bool = False) -> "InstanceBatch":
        """Vectorised G(...) batch: no per-request Python objects. With unique_ids
        every instance's ids carry an "i<k>/" prefix (requests that move between
        instances, e.g. routed to another replica, stay distinguishable)."""
        seeds = list(seeds)
        n = len(seeds)
        R, Pn = spec.n_dec, spec.n_new
        rid = [f"run-{i}".encode() + b"\0" for i in range(R)]
        pid = [f"new-{i}".encode() + b"\0" for i in range(Pn)]
        if unique_ids:
            names = [f"i{k}/".encode() + x for k in range(n) for x in rid + pid]
        else:  # ids are identical across instances: one copy, shared pointers
            names = rid + pid
        blob = np.frombuffer(b"".join(names) + b"\0", np.uint8).copy()
        lens = [len(x) for x in names]
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
        base = np.uint64(blob.ctypes.data)
        run = np.zeros(max(1, n * R), abi.RUNNING_DTYPE)
        pen = np.zeros(max(1, n * Pn), abi.PENDING_DTYPE)
        for k, s in enumerate(seeds):
            a = stress_arrays(spec, s, slo, gen)
            o = offs[k * (R + Pn):(k + 1) * (R + Pn)] if unique_ids else offs
            rr = run[k * R:(k + 1) * R]
            rr["id"] = base + o[:R]
            rr["decode_tier"] = a["dec_tier"]
            rr["next_due_s"] = a["dec_next_due"]
            rr["decode_remaining"] = a["dec_remaining"]
            pp = pen[k * Pn:(k + 1) * Pn]
            pp["id"] = base + o[R:]
            pp["prefill_deadline"] = a["new_deadline"]
            pp["prefill_tokens"] = a["new_prefill"]
            pp["decode_tier"] = a["new_tier"]
            pp["memory_units"] = a["new_memory"]
            pp["value"] = a["new_value"]
        inp = np.zeros(n, abi.INPUT_DTYPE)
        inp["now"] = spec.now
        inp["running"] = run.ctypes.data + np.arange(n, dtype=np.uint64) * np.uint64(R * run.itemsize)
        inp["n_running"] = R
        inp["n_pending"] = Pn
        inp["pending"] = pen.ctypes.data + np.arange(n, dtype=np.uint64) * np.uint64(Pn * pen.itemsize)
        inp["memory_total"] = spec.memory_total
        inp["memory_standard_resident"] = spec.memory_standard_resident
        inp["tail_horizon_s"] = spec.tail_horizon_s
        return cls(inp, run, pen, blob, offs)


    @classmethod
    def from_corpus(cls, buf: bytes) -> "InstanceBatch":
        """Parse a recorded-input corpus (the binary layout written by the simulator
        recorder, oracle/ref_sim.cpp slos_sim_recorded_write) into C-ABI arrays."""
        import struct
        run_rec = np.dtype([("prefill_remaining", "<i8"), ("prefill_deadline", "<f8"), ("decode_tier", "<i4"),
                            ("pad", "<i4"), ("next_due_s", "<f8"), ("backlog", "<i8"),
                            ("decode_remaining", "<i8")])
        pen_rec = np.dtype([("prefill_deadline", "<f8"), ("prefill_tokens", "<i8"), ("decode_tier", "<i4"),
                            ("pad", "<i4"), ("memory_units", "<i8"), ("value", "<f8")])
        heads, runs, pens, ids = [], [], [], []
        off = 0
        while off < len(buf):
            now, th, mt, msr, nr, npn = struct.unpack_from("<ddqqii", buf, off)
            off += 40
            runs.append(np.frombuffer(buf, run_rec, nr, off))
            off += nr * run_rec.itemsize
            pens.append(np.frombuffer(buf, pen_rec, npn, off))
            off += npn * pen_rec.itemsize
            for _ in range(nr + npn):
                (ln,) = struct.unpack_from("<H", buf, off)
                ids.append(bytes(buf[off + 2:off + 2 + ln]) + b"\0")
                off += 2 + ln
            heads.append((now, th, mt, msr, nr, npn))
        blob = np.frombuffer(b"".join(ids) + b"\0", np.uint8).copy()
        offs = np.concatenate([[0], np.cumsum([len(x) for x in ids])[:-1]]).astype(np.uint64)
        base = np.uint64(blob.ctypes.data)
        R = sum(h[4] for h in heads)
        Pn = sum(h[5] for h in heads)
        run = np.zeros(max(1, R), abi.RUNNING_DTYPE)
        pen = np.zeros(max(1, Pn), abi.PENDING_DTYPE)
        inp = np.zeros(len(heads), abi.INPUT_DTYPE)
        r0 = p0 = k = 0
        for n_, (now, th, mt, msr, nr, npn) in enumerate(heads):
            rr, pr = runs[n_], pens[n_]
            dst = run[r0:r0 + nr]
            dst["id"] = base + offs[k:k + nr]
            for f in ("prefill_remaining", "prefill_deadline", "decode_tier", "next_due_s", "backlog",
                      "decode_remaining"):
                dst[f] = rr[f]
            k += nr
            dp = pen[p0:p0 + npn]
            dp["id"] = base + offs[k:k + npn]
            for f in ("prefill_deadline", "prefill_tokens", "decode_tier", "memory_units", "value"):
                dp[f] = pr[f]
            k += npn
            inp[n_] = (now, run.ctypes.data + r0 * run.itemsize, nr, npn, pen.ctypes.data + p0 * pen.itemsize,
                       mt, msr, th)
            r0 += nr
            p0 += npn
        return cls(inp, run, pen, blob, offs)

    @classmethod
    def concat(cls, parts) -> "InstanceBatch":
        """Instances of several batches in one (the request arrays stay where they are;
        the new batch keeps the parts alive)."""
        out = cls(np.concatenate([p.inputs for p in parts]), parts[0].running, parts[0].pending,
                  parts[0]._blob, parts[0]._id_offsets)
        out._parts = list(parts)
        return out

    def tiled(self, reps: int) -> "InstanceBatch":
        """The same instances repeated `reps` times (shares every request array)."""
        out = InstanceBatch(np.tile(self.inputs, reps), self.running, self.pending, self._blob, self._id_offsets)
        out._parts = [self]
        return out

    def subset(self, idx) -> "InstanceBatch":
        out = InstanceBatch(self.inputs[np.asarray(idx)].copy(), self.running, self.pending, self._blob,
                            self._id_offsets)
        out._parts = [self]
        return out


def load_corpus(path: str) -> InstanceBatch:
    """A gzip'd recorded-input corpus (tests/golden/c5_*.bin.gz)."""
    import gzip
    with gzip.open(path, "rb") as f:
        return InstanceBatch.from_corpus(f.read())


# --------------------------------------------- brute-force oracle adapters ---

ORACLE_REC_LEN = 41  # oracle/ref_tools.cpp encode()


def oracle_fields(rec):
    """Decode a tests/oracle.hpp Instance record (oracle/ref_tools.cpp)."""
    rec = [int(x) for x in rec]
    return dict(cap=rec[0], tpots=rec[2:2 + rec[1]], runners=rec[5:5 + rec[4]],
                candidates=[tuple(rec[9 + 5 * i:14 + 5 * i]) for i in range(rec[8])],
                memory_total=rec[39], horizon=rec[40])


def oracle_model(f) -> list:  # tests/oracle.cpp:104-106
    return [PerfTerm(1.0 / float(f["cap"]), 0.0, 0.0)]


def oracle_slo(f) -> SloConfig:  # tests/oracle.cpp:108-114
    return SloConfig([float(t) for t in f["tpots"]], [1.0] * len(f["tpots"]), 10)


def oracle_input(f) -> ScheduleInput:  # tests/oracle.cpp:116-145
    inp = ScheduleInput(now=0.0, memory_total=f["memory_total"], memory_standard_resident=0)
    for j, tier in enumerate(f["runners"]):
        inp.running.append(RunningRequest(id=f"run-{j}", prefill_remaining=0, decode_tier=tier,
                                          next_due_s=float(f["tpots"][tier]), backlog=0,
                                          decode_remaining=1000))
    for i, (ddl, pre, tier, mem, val) in enumerate(f["candidates"]):
        inp.pending.append(PendingRequest(id=f"cand-{i}", prefill_deadline=float(ddl),
                                          prefill_tokens=pre, decode_tier=tier, memory_units=mem,
                                          value=float(val)))
    inp.tail_horizon_s = 2.0 * float(max(f["tpots"]))
    return inp
