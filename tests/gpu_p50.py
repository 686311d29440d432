"""Single-plan latency probe (run under gpurun): p50 of one C1 / C2 / C4 plan per
slos_plan_batch call, end to end, with the per-stage device times of the last call."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402,F401

import bench  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402

lib = abi.product()
s = torch.cuda.Stream()
for fam in sys.argv[1:] or ["C1", "C2"]:
    print(fam, "p50 ms", round(bench.single_plan_p50(lib, fam, s.cuda_stream), 4), flush=True)
