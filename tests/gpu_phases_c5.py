"""Per-phase cycle breakdown (SLOS_PHASE_TIMING=1) on the C5 sweep corpus (65,536
instances, bench.py's c5_shard): DP phases, reconstruction phases, slowest instances."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SLOS_NO_PHASES") is None:
    os.environ["SLOS_PHASE_TIMING"] = "1"
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200.sweep import ShardSolver  # noqa: E402

lib = abi.product()
batch, handles, n = bench.c5_shard(lib, 0, 1)
s = ShardSolver(lib, None, None, batch=batch, handles=handles)
rec = torch.empty((n, C.sizeof(abi.Record)), dtype=torch.uint8, device="cuda")
s.upload()
s.converge(rec)
for _ in range(int(os.environ.get("SLOS_SOLVES", "2"))):
    s.solve()
    torch.cuda.synchronize()
    print("C5", n, "stage ms [anchor, dp, build]", s.stage_ms(), flush=True)
s.download()
s.free_results()
