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


def bench_sets(count: int = 64, seed: int = 7):
    """Profile sets shaped like the reference's fit criterion (acceptance_main.cpp:
    629-648): n = 8..8192 step 64 x spec_step {0,2,5,8}, +-2% noise, two regimes
    with per-set coefficients."""
    rng = np.random.default_rng(seed)
    n, s = np.meshgrid(np.arange(8, 8193, 64), [0, 2, 5, 8], indexing="ij")
    n, s = n.ravel(), s.ravel()
    out = []
    for _ in range(count):
        k1, k2, b = rng.uniform(1e-6, 5e-5), rng.uniform(1e-4, 3e-3), rng.uniform(1e-3, 1e-2)
        floor = rng.uniform(0.005, 0.03)
        lat = np.maximum(k1 * n + k2 * s + b, floor) * (1.0 + rng.uniform(-0.02, 0.02, len(n)))
        out.append(as_samples(n, s, lat))
    return out


def bench_leg(steps: int, warmup: int, with_cpu: bool):
    """f4 leg of bench.py: 64 two-regime fits per step through slos_perf_fit_batch
    (one CTA per set), the reference's PerfModel::fit looped beside it."""
    import time
    sets = bench_sets()
    for _ in range(max(1, warmup)):
        terms, st = fit_batch(sets, 2)
    t0 = time.perf_counter()
    for _ in range(steps):
        terms, st = fit_batch(sets, 2)
    dt = (time.perf_counter() - t0) / steps
    leg = {"workload": f"f4: PerfModel::fit, {len(sets)} profile sets x {len(sets[0])} samples, 2 terms, "
                       "through the C-ABI (host bands + device iterations)",
           "value": len(sets) / dt, "unit": "fits/s", "ms_per_step": dt * 1e3, "statuses_ok": bool((st == 0).all())}
    if with_cpu:
        sample = sets[:16]
        t0 = time.perf_counter()
        ref = [reference_fit(x, 2) for x in sample]
        rdt = time.perf_counter() - t0
        leg["cpu_baseline"] = {"value": len(sample) / rdt, "unit": "fits/s", "cores": 1, "kind": "reference",
                               "sample": f"{len(sample)} sets through the reference's PerfModel::fit, {rdt:.2f} s wall"}
        leg["identical_to_reference"] = all(terms[k].tobytes() == ref[k][0].tobytes() for k in range(len(sample)))
    return leg
