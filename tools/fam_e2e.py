"""A stress family end to end through slos_plan_batch (host inputs), per-call wall
time; with SLOS_HOST_TIMING=1 the library prints its per-chunk host breakdown.
usage: python tools/fam_e2e.py [family] [n]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.planner import _Handle  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
lib = abi.product()
spec, F = bench.family(fam)
batch = W.InstanceBatch.stress(spec.family, range(n))
h = _Handle(lib, spec.model, spec.slo, spec.cfg)
stream = torch.cuda.Stream()
steps = int(os.environ.get("E2E_STEPS", "6"))
r, h2d, d2h, sec = bench.e2e_rate(lib, batch, [h.ptr] * n, steps, 3, stream.cuda_stream)
print(f"{fam} x {n} e2e {r:.0f} plans/s, {sec * 1e3:.3f} ms per call, h2d {h2d / 1e6:.1f} MB, d2h {d2h / 1e6:.1f} MB")
