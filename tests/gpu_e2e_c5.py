"""e2e probe for the C5 corpus (run under gpurun): slos_plan_batch with host inputs
over 65,536 mixed AR / speculative instances."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402

lib = abi.product()
b, handles, n = bench.c5_shard(lib, 0, 1)
hs = (C.c_void_p * n)(*[h.ptr for h in handles])
outs = (abi.Result * n)()
for it in range(4):
    t = time.perf_counter()
    lib.slos_plan_batch(hs, n, C.c_void_p(b.inputs_ptr()), 0, outs, None)
    dt = time.perf_counter() - t
    for k in range(n):
        lib.slos_result_free(C.byref(outs[k]))
    print(f"C5 {n} call {it}: {dt*1e3:.2f} ms -> {n/dt:.0f} plans/s", flush=True)
