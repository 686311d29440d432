"""e2e probe (run under gpurun): slos_plan_batch with host inputs on the bench
workload; prints wall time per call (SLOS_HOST_TIMING=1 adds host phases)."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.planner import _Handle  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
F = W.FAMILIES[fam]
lib = abi.product()
b = W.InstanceBatch.stress(F["spec"], range(n))
h = _Handle(lib, F["model"], W.TWO_TIER_SLO, F["cfg"])
hs = (C.c_void_p * n)(*([h.ptr] * n))
outs = (abi.Result * n)()
for it in range(5):
    t = time.perf_counter()
    lib.slos_plan_batch(hs, n, C.c_void_p(b.inputs_ptr()), 0, outs, None)
    dt = time.perf_counter() - t
    for k in range(n):
        lib.slos_result_free(C.byref(outs[k]))
    print(fam, n, f"call {it}: {dt*1e3:.2f} ms -> {n/dt:.0f} plans/s", flush=True)
