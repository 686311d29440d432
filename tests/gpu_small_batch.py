"""Latency of small slos_plan_batch calls (the plan broker's flush size in a live
sweep: a handful of C5-sized plans). Prints per-call wall time percentiles."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402

lib = abi.product()
b, handles, n = bench.c5_shard(lib, 0, 1)
for size in (1, 6, 32):
    hs = (C.c_void_p * size)(*[h.ptr for h in handles[:size]])
    outs = (abi.Result * size)()
    ts = []
    for it in range(300):
        t = time.perf_counter()
        lib.slos_plan_batch(hs, size, C.c_void_p(b.inputs_ptr()), 0, outs, None)
        ts.append(time.perf_counter() - t)
        for k in range(size):
            lib.slos_result_free(C.byref(outs[k]))
    ts = np.array(ts[50:]) * 1e6
    print(f"batch {size}: p50 {np.median(ts):.1f} us, p10 {np.percentile(ts, 10):.1f}, p90 {np.percentile(ts, 90):.1f}",
          flush=True)
