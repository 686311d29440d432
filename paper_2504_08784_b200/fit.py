"""PerfModel::fit on the device, batched over profile sets (include/slos_fit.h,
SURVEY.md §8 f4). Mirrors slosim::PerfModel::fit (proj/src/perf_model.cpp:132-201):
same arguments, same errors ("insufficient-samples", "degenerate-samples"), same
term order (k1, k2, b)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi

SAMPLE_DTYPE = np.dtype([("num_tokens", "<i8"), ("spec_step", "<i8"), ("latency_s", "<f8")])
ERR_SLUGS = {0: "ok", 1: "invalid-parameters", 22: "insufficient-samples", 23: "degenerate-samples"}


def _bind(lib):
    if not getattr(lib, "_fit_bound", False):
        lib.slos_perf_fit_batch.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                            C.c_int32, C.POINTER(abi.PerfTerm), C.POINTER(C.c_int32)]
        lib.slos_perf_fit_batch.restype = C.c_int
        lib._fit_bound = True
    return lib


def as_samples(num_tokens, spec_step, latency_s) -> np.ndarray:
    a = np.zeros(len(num_tokens), SAMPLE_DTYPE)
    a["num_tokens"], a["spec_step"], a["latency_s"] = num_tokens, spec_step, latency_s
    return a


def fit_batch(sets, num_terms: int, max_iters: int = 100, lib=None):
    """sets: list of SAMPLE_DTYPE arrays -> (terms [n_sets, num_terms, 3] f64, status [n_sets])."""
    lib = _bind(lib or abi.product())
    arrs = [np.ascontiguousarray(s, dtype=SAMPLE_DTYPE) for s in sets]
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    ns = (C.c_int32 * len(arrs))(*[len(a) for a in arrs])
    out = (abi.PerfTerm * (len(arrs) * max(1, num_terms)))()
    st = (C.c_int32 * len(arrs))()
    r = lib.slos_perf_fit_batch(ptrs, ns, len(arrs), num_terms, max_iters, out, st)
    terms = np.array([[t.k1, t.k2, t.b] for t in out], dtype=np.float64).reshape(len(arrs), max(1, num_terms), 3)
    status = np.array(list(st), dtype=np.int32)
    if r != 0 and not status.any():
        raise RuntimeError(f"slos_perf_fit_batch failed: {r} {lib.slos_last_error()}")
    return terms, status


def reference_fit(samples: np.ndarray, num_terms: int, max_iters: int = 100):  # test infrastructure only
    lib = abi.reference()
    if not getattr(lib, "_fit_ref_bound", False):
        lib.slos_ref_perf_fit.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(abi.PerfTerm)]
        lib.slos_ref_perf_fit.restype = C.c_int32
        lib._fit_ref_bound = True
    a = np.ascontiguousarray(samples, dtype=SAMPLE_DTYPE)
    out = (abi.PerfTerm * max(1, num_terms))()
    st = lib.slos_ref_perf_fit(a.ctypes.data, len(a), num_terms, max_iters, out)
    return np.array([[t.k1, t.k2, t.b] for t in out], dtype=np.float64), int(st)
