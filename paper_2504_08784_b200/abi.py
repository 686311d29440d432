"""ctypes mirror of include/slos_planner.h (the C-ABI drop-in boundary).

The same declarations bind all three libraries that export the ABI:
  * the product ``libslos_b200.so`` (CUDA kernels + C++ host shim),
  * the test-only C oracle ``oracle/liboracle_slos.so``,
  * the test-only reference adapter ``oracle/_ref/libslos_ref.so``.
Only tests/, bench.py's cpu_baseline leg and __graft_entry__.smoke() ever load
the latter two.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.dirname(os.path.abspath(__file__))

PRODUCT_LIB = os.environ.get("SLOS_PRODUCT_LIB", os.path.join(PKG, "libslos_b200.so"))
WORKLOAD_LIB = os.path.join(PKG, "libslos_workload.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "liboracle_slos.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libslos_ref.so")

MAX_TIERS = 8

SLOS_OK = 0
SLOS_ERR_INVALID_PARAMETERS = 1
SLOS_ERR_INTERNAL_INCONSISTENCY = 2
SLOS_ERR_INFEASIBLE_BUDGET = 3
SLOS_ERR_CUDA = 10
SLOS_ERR_CAPACITY = 11
SLOS_ERR_NO_DEVICE = 12
SLOS_ERR_ALLOC = 13
SLOS_ERR_RANGE = 14

SLUGS = {
    SLOS_ERR_INVALID_PARAMETERS: "invalid-parameters",
    SLOS_ERR_INTERNAL_INCONSISTENCY: "internal-inconsistency",
    SLOS_ERR_INFEASIBLE_BUDGET: "infeasible-budget",
}

GAP_TILE_AR, GAP_TILE, GAP_PREFILL_BUDGET = 0, 1, 2


class PerfTerm(C.Structure):
    _fields_ = [("k1", C.c_double), ("k2", C.c_double), ("b", C.c_double)]


class PlannerConfigC(C.Structure):
    _fields_ = [
        ("max_chunk_tokens", C.c_int64),
        ("max_batch_tokens", C.c_int64),
        ("speculative", C.c_int32),
        ("spec_max_len", C.c_int32),
        ("spec_alpha", C.c_double),
        ("plan_margin", C.c_double),
    ]


class Running(C.Structure):
    _fields_ = [
        ("id", C.c_char_p),
        ("prefill_remaining", C.c_int64),
        ("prefill_deadline", C.c_double),
        ("decode_tier", C.c_int32),
        ("reserved0", C.c_int32),
        ("next_due_s", C.c_double),
        ("backlog", C.c_int64),
        ("decode_remaining", C.c_int64),
    ]


class Pending(C.Structure):
    _fields_ = [
        ("id", C.c_char_p),
        ("prefill_deadline", C.c_double),
        ("prefill_tokens", C.c_int64),
        ("decode_tier", C.c_int32),
        ("reserved0", C.c_int32),
        ("memory_units", C.c_int64),
        ("value", C.c_double),
    ]


class Input(C.Structure):
    _fields_ = [
        ("now", C.c_double),
        ("running", C.POINTER(Running)),
        ("n_running", C.c_int32),
        ("n_pending", C.c_int32),
        ("pending", C.POINTER(Pending)),
        ("memory_total", C.c_int64),
        ("memory_standard_resident", C.c_int64),
        ("tail_horizon_s", C.c_double),
    ]


class Entry(C.Structure):
    """slos_entry: 8 bytes on the wire (include/slos_planner.h). `ref` packs the
    24-bit signed request reference, the 7-bit spec_len and the decode bit; `tokens`
    is the prefill or decode count. The properties mirror the header's accessors."""
    _fields_ = [
        ("ref", C.c_uint32),
        ("tokens", C.c_int32),
    ]

    @property
    def req(self) -> int:
        r = self.ref & 0xFFFFFF
        return r - (1 << 24) if r & 0x800000 else r

    @property
    def is_decode(self) -> bool:
        return bool(self.ref >> 31)

    @property
    def spec_len(self) -> int:
        return (self.ref >> 24) & 0x7F

    @property
    def prefill_tokens(self) -> int:
        return 0 if self.is_decode else int(self.tokens)

    @property
    def decode_tokens(self) -> int:
        return int(self.tokens) if self.is_decode else 0


class Batch(C.Structure):
    _fields_ = [
        ("start_s", C.c_double),
        ("end_s", C.c_double),
        ("capacity_tokens", C.c_int64),
        ("spec_step", C.c_int64),
        ("prefill_budget_left", C.c_int64),
        ("first_entry", C.c_int64),
        ("n_entries", C.c_int64),
    ]


class Counters(C.Structure):
    _fields_ = [
        ("transitions", C.c_int64),
        ("gap_evals", C.c_int64),
        ("dues", C.c_int64),
        ("slots", C.c_int64),
        ("states", C.c_int64),
    ]


class Result(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("running_set_infeasible", C.c_int32),
        ("admitted_value", C.c_double),
        ("n_admitted", C.c_int32),
        ("n_declined", C.c_int32),
        ("n_deferred", C.c_int32),
        ("reserved0", C.c_int32),
        ("admitted", C.POINTER(C.c_int32)),
        ("declined", C.POINTER(C.c_int32)),
        ("deferred", C.POINTER(C.c_int32)),
        ("n_batches", C.c_int64),
        ("batches", C.POINTER(Batch)),
        ("n_entries", C.c_int64),
        ("entries", C.POINTER(Entry)),
        ("exact_until_s", C.c_double),
        ("counters", Counters),
        ("owner_", C.c_void_p),
    ]


class Record(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("running_set_infeasible", C.c_int32),
        ("n_admitted", C.c_int32),
        ("n_declined", C.c_int32),
        ("admitted_value", C.c_double),
        ("n_batches", C.c_int64),
        ("n_entries", C.c_int64),
        ("exact_until_s", C.c_double),
        ("counters", Counters),
    ]


RECORD_DTYPE = None  # set below


class DecodeMemberC(C.Structure):
    _fields_ = [
        ("tier", C.c_int32),
        ("owner", C.c_int32),
        ("phase_s", C.c_double),
        ("backlog", C.c_int64),
        ("remaining", C.c_int64),
    ]


class GapQuery(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("n_exact", C.c_int32),
        ("gap_s", C.c_double),
        ("due_horizon_s", C.c_double),
        ("counts_per_tier", C.c_int64 * MAX_TIERS),
        ("exact", C.POINTER(DecodeMemberC)),
    ]


class GapBatch(C.Structure):
    _fields_ = [
        ("start_s", C.c_double),
        ("end_s", C.c_double),
        ("capacity_tokens", C.c_int64),
        ("spec_step", C.c_int64),
        ("decode_tokens", C.c_int64),
        ("prefill_budget", C.c_int64),
        ("decode_per_tier", C.c_int64 * MAX_TIERS),
        ("first_owner", C.c_int64),
        ("n_owners", C.c_int64),
    ]


class GapResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("feasible", C.c_int32),
        ("prefill_budget", C.c_int64),
        ("n_spec_lengths", C.c_int32),
        ("spec_lengths", C.c_int32 * MAX_TIERS),
        ("n_batches", C.c_int64),
        ("batches", C.POINTER(GapBatch)),
        ("n_owner_pairs", C.c_int64),
        ("owner_tokens", C.POINTER(C.c_int64)),
        ("owner_", C.c_void_p),
    ]


class SpecPlanC(C.Structure):
    _fields_ = [
        ("feasible", C.c_int32),
        ("lengths", C.c_int32 * MAX_TIERS),
        ("batch_time_s", C.c_double),
        ("batch_capacity", C.c_int64),
        ("decode_tokens", C.c_int64),
        ("prefill_throughput", C.c_double),
    ]


# numpy views of the input structs (used to build large batches without
# per-request Python objects: ids are pointers into one bytes blob).
RUNNING_DTYPE = np.dtype(
    {
        "names": ["id", "prefill_remaining", "prefill_deadline", "decode_tier", "reserved0",
                  "next_due_s", "backlog", "decode_remaining"],
        "formats": [np.uint64, np.int64, np.float64, np.int32, np.int32, np.float64, np.int64,
                    np.int64],
        "offsets": [Running.id.offset, Running.prefill_remaining.offset,
                    Running.prefill_deadline.offset, Running.decode_tier.offset,
                    Running.reserved0.offset, Running.next_due_s.offset, Running.backlog.offset,
                    Running.decode_remaining.offset],
        "itemsize": C.sizeof(Running),
    }
)
PENDING_DTYPE = np.dtype(
    {
        "names": ["id", "prefill_deadline", "prefill_tokens", "decode_tier", "reserved0",
                  "memory_units", "value"],
        "formats": [np.uint64, np.float64, np.int64, np.int32, np.int32, np.int64, np.float64],
        "offsets": [Pending.id.offset, Pending.prefill_deadline.offset,
                    Pending.prefill_tokens.offset, Pending.decode_tier.offset,
                    Pending.reserved0.offset, Pending.memory_units.offset, Pending.value.offset],
        "itemsize": C.sizeof(Pending),
    }
)
INPUT_DTYPE = np.dtype(
    {
        "names": ["now", "running", "n_running", "n_pending", "pending", "memory_total",
                  "memory_standard_resident", "tail_horizon_s"],
        "formats": [np.float64, np.uint64, np.int32, np.int32, np.uint64, np.int64, np.int64,
                    np.float64],
        "offsets": [Input.now.offset, Input.running.offset, Input.n_running.offset,
                    Input.n_pending.offset, Input.pending.offset, Input.memory_total.offset,
                    Input.memory_standard_resident.offset, Input.tail_horizon_s.offset],
        "itemsize": C.sizeof(Input),
    }
)
ENTRY_DTYPE = np.dtype(
    {
        "names": ["ref", "tokens"],
        "formats": [np.uint32, np.int32],
        "offsets": [0, 4],
        "itemsize": C.sizeof(Entry),
    }
)
# The canonical (reference PlanEntry) form used by parity digests: int64 token
# counts, independent of the wire layout.
CANON_ENTRY_DTYPE = np.dtype(
    {
        "names": ["req", "spec_len", "prefill_tokens", "decode_tokens"],
        "formats": [np.int32, np.int32, np.int64, np.int64],
        "offsets": [0, 4, 8, 16],
        "itemsize": 24,
    }
)


def canon_entries(wire: np.ndarray) -> np.ndarray:
    """Wire entries (ENTRY_DTYPE) -> CANON_ENTRY_DTYPE, vectorised Entry accessors."""
    ref = wire["ref"].astype(np.uint32)
    tok = wire["tokens"].astype(np.int64)
    dec = (ref >> np.uint32(31)).astype(bool)
    out = np.zeros(len(wire), CANON_ENTRY_DTYPE)
    out["req"] = ((ref << np.uint32(8)).view(np.int32) >> 8)
    out["spec_len"] = ((ref >> np.uint32(24)) & np.uint32(0x7F)).astype(np.int32)
    out["prefill_tokens"] = np.where(dec, 0, tok)
    out["decode_tokens"] = np.where(dec, tok, 0)
    return out


BATCH_DTYPE = np.dtype(
    {
        "names": ["start_s", "end_s", "capacity_tokens", "spec_step", "prefill_budget_left",
                  "first_entry", "n_entries"],
        "formats": [np.float64, np.float64, np.int64, np.int64, np.int64, np.int64, np.int64],
        "offsets": [0, 8, 16, 24, 32, 40, 48],
        "itemsize": C.sizeof(Batch),
    }
)

RECORD_DTYPE = np.dtype(
    {
        "names": ["status", "infeasible", "n_admitted", "n_declined", "value", "n_batches",
                  "n_entries", "exact_until_s", "transitions", "gap_evals", "dues", "slots",
                  "states"],
        "formats": [np.int32, np.int32, np.int32, np.int32, np.float64, np.int64, np.int64,
                    np.float64, np.int64, np.int64, np.int64, np.int64, np.int64],
        "offsets": [0, 4, 8, 12, 16, 24, 32, 40, 48, 56, 64, 72, 80],
        "itemsize": C.sizeof(Record),
    }
)

_LIBS: dict[str, C.CDLL] = {}


def _bind(lib: C.CDLL) -> C.CDLL:
    P = C.POINTER
    lib.slos_planner_config_default.argtypes = [P(PlannerConfigC)]
    lib.slos_planner_config_default.restype = None
    lib.slos_planner_create.argtypes = [P(PerfTerm), C.c_int32, P(C.c_double), P(C.c_double),
                                        C.c_int32, C.c_int32, P(PlannerConfigC), P(C.c_void_p)]
    lib.slos_planner_create.restype = C.c_int
    lib.slos_planner_destroy.argtypes = [C.c_void_p]
    lib.slos_planner_destroy.restype = None
    lib.slos_plan.argtypes = [C.c_void_p, P(Input), C.c_int32, P(Result)]
    lib.slos_plan.restype = C.c_int
    lib.slos_plan_batch.argtypes = [P(C.c_void_p), C.c_int32, C.c_void_p, C.c_int32, P(Result),
                                    C.c_void_p]
    lib.slos_plan_batch.restype = C.c_int
    lib.slos_result_free.argtypes = [P(Result)]
    lib.slos_result_free.restype = None
    lib.slos_tile_gap_batch.argtypes = [C.c_void_p, C.c_int32, P(GapQuery), P(GapResult)]
    lib.slos_tile_gap_batch.restype = C.c_int
    lib.slos_gap_result_free.argtypes = [P(GapResult)]
    lib.slos_gap_result_free.restype = None
    lib.slos_time2bs_batch.argtypes = [C.c_void_p, C.c_int32, P(C.c_double), P(C.c_int64),
                                       C.c_int64, P(C.c_int64), P(C.c_int32)]
    lib.slos_time2bs_batch.restype = C.c_int
    lib.slos_predict_batch.argtypes = [C.c_void_p, C.c_int32, P(C.c_int64), P(C.c_int64),
                                       P(C.c_double)]
    lib.slos_predict_batch.restype = C.c_int
    lib.slos_solve_spec_lengths.argtypes = [C.c_void_p, P(C.c_int64), C.c_int32, C.c_double,
                                            C.c_int32, P(SpecPlanC)]
    lib.slos_solve_spec_lengths.restype = C.c_int
    lib.slos_expected_accepted.argtypes = [C.c_double, C.c_int32]
    lib.slos_expected_accepted.restype = C.c_double
    lib.slos_status_slug.argtypes = [C.c_int]
    lib.slos_status_slug.restype = C.c_char_p
    lib.slos_last_error.argtypes = []
    lib.slos_last_error.restype = C.c_char_p
    lib.slos_backend.argtypes = []
    lib.slos_backend.restype = C.c_char_p
    lib.slos_workspace_create.argtypes = [P(C.c_void_p)]
    lib.slos_workspace_create.restype = C.c_int
    lib.slos_workspace_destroy.argtypes = [C.c_void_p]
    lib.slos_workspace_destroy.restype = None
    lib.slos_workspace_upload.argtypes = [C.c_void_p, P(C.c_void_p), C.c_int32, C.c_void_p, C.c_int32,
                                          P(Result), C.c_void_p]
    lib.slos_workspace_upload.restype = C.c_int
    lib.slos_workspace_solve.argtypes = [C.c_void_p, C.c_void_p]
    lib.slos_workspace_solve.restype = C.c_int
    lib.slos_workspace_download.argtypes = [C.c_void_p, P(Result), C.c_void_p]
    lib.slos_workspace_download.restype = C.c_int
    lib.slos_workspace_records.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.slos_workspace_records.restype = C.c_int
    lib.slos_workspace_kernel_ms.argtypes = [C.c_void_p, P(C.c_float)]
    lib.slos_workspace_kernel_ms.restype = C.c_int
    lib.slos_workspace_launches.argtypes = [C.c_void_p, P(C.c_int64)]
    lib.slos_workspace_launches.restype = C.c_int
    lib.slos_workspace_stage_ms.argtypes = [C.c_void_p, P(C.c_float), C.c_int32]
    lib.slos_workspace_stage_ms.restype = C.c_int
    lib.slos_last_transfer_bytes.argtypes = [P(C.c_int64), P(C.c_int64)]
    lib.slos_last_transfer_bytes.restype = None
    if hasattr(lib, "slos_plan_to_json"):  # include/slos_plan_json.h (product, reference)
        lib.slos_plan_to_json.argtypes = [C.c_void_p, P(Result), C.c_double, C.c_char_p, C.c_int64,
                                          P(C.c_int64)]
        lib.slos_plan_to_json.restype = C.c_int
    return lib


def plan_to_json(lib: C.CDLL, inp, res, now_s: float) -> str:
    """include/slos_plan_json.h: plan_to_json(result, now) (dp_scheduler.cpp:560-589)
    of `res` (a Result, or a pointer to one) for the input at `inp` (an address)."""
    rp = res if isinstance(res, C._Pointer) else C.byref(res)
    n = C.c_int64()
    st = lib.slos_plan_to_json(C.c_void_p(inp), rp, now_s, None, 0, C.byref(n))
    if st != SLOS_OK:
        raise RuntimeError(f"slos_plan_to_json: {lib.slos_status_slug(st).decode()}")
    buf = C.create_string_buffer(n.value + 1)
    st = lib.slos_plan_to_json(C.c_void_p(inp), rp, now_s, buf, n.value + 1, C.byref(n))
    if st != SLOS_OK:
        raise RuntimeError(f"slos_plan_to_json: {lib.slos_status_slug(st).decode()}")
    return buf.raw[:n.value].decode()


def load(path: str) -> C.CDLL:
    """Load (once) and bind a library exporting include/slos_planner.h."""
    path = os.path.abspath(path)
    if path not in _LIBS:
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        _LIBS[path] = _bind(C.CDLL(path))
    return _LIBS[path]


def product() -> C.CDLL:
    """The product library. There is deliberately no CPU fallback: a missing
    libslos_b200.so is an error, not a reason to use the oracle."""
    return load(PRODUCT_LIB)


def oracle() -> C.CDLL:  # test infrastructure only
    return load(ORACLE_LIB)


def reference() -> C.CDLL:  # test infrastructure only
    return load(REF_LIB)


def workload() -> C.CDLL:
    path = os.path.abspath(WORKLOAD_LIB)
    if path not in _LIBS:
        lib = C.CDLL(path)
        P = C.POINTER
        lib.slos_wl_uniforms.argtypes = [C.c_uint64, C.c_int32, P(C.c_double)]
        lib.slos_wl_uniforms.restype = None
        lib.slos_wl_stress.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, P(C.c_double),
                                       C.c_double, P(C.c_int32), P(C.c_double), P(C.c_int64),
                                       P(C.c_double), P(C.c_int64), P(C.c_int32), P(C.c_int64),
                                       P(C.c_double)]
        lib.slos_wl_stress.restype = None
        _LIBS[path] = lib
    return _LIBS[path]


def reference_stress_gen():  # test infrastructure / reference bench arm only
    """slos_ref_stress from oracle/_ref/libslos_ref.so: the reference harness's
    G(...) generator (acceptance_main.cpp:577-605), same signature as slos_wl_stress."""
    lib = reference()
    f = lib.slos_ref_stress
    P = C.POINTER
    f.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, P(C.c_double), C.c_double, P(C.c_int32),
                  P(C.c_double), P(C.c_int64), P(C.c_double), P(C.c_int64), P(C.c_int32), P(C.c_int64),
                  P(C.c_double)]
    f.restype = None
    return f


def reference_schedule_timed():  # test infrastructure / reference bench arm only
    """slos_ref_schedule_timed: one reference schedule() with a fresh planner, timed
    inside (acceptance_main.cpp:606-609). Returns the bound function."""
    lib = reference()
    f = lib.slos_ref_schedule_timed
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(Result), C.POINTER(C.c_double)]
    f.restype = C.c_int
    return f
