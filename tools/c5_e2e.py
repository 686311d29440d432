"""C5 x 65,536 end to end through slos_plan_batch (host inputs), per-call wall time;
with SLOS_HOST_TIMING=1 the library prints its per-chunk host breakdown."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402

lib = abi.product()
b5, h5, per = bench.c5_shard(lib, 0, 1)
stream = torch.cuda.Stream()
steps = int(os.environ.get("C5_STEPS", "5"))
r, h2d, d2h, sec = bench.e2e_rate(lib, b5, [h.ptr for h in h5], steps, 3, stream.cuda_stream)
print(f"C5 e2e {r / 1e6:.2f}M plans/s, {sec * 1e3:.2f} ms per call, h2d {h2d / 1e6:.1f} MB, d2h {d2h / 1e6:.1f} MB")
