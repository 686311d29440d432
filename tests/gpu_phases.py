"""Per-phase cycle breakdown of dp_kernel (SLOS_PHASE_TIMING=1) on the bench workload."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("SLOS_NO_PHASES") is None:
    os.environ["SLOS_PHASE_TIMING"] = "1"
import torch  # noqa: E402

from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.sweep import ShardSolver, ShardSpec  # noqa: E402

fam = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
F = W.FAMILIES[fam]
s = ShardSolver(abi.product(), ShardSpec(F["spec"], F["model"], F["cfg"]), range(n))
rec = torch.empty((n, C.sizeof(abi.Record)), dtype=torch.uint8, device="cuda")
s.upload()
s.converge(rec)
for _ in range(int(os.environ.get("SLOS_SOLVES", "3"))):
    s.solve()
    torch.cuda.synchronize()
    print(fam, n, "stage ms [anchor, dp, build]", s.stage_ms(), flush=True)
s.download()
s.free_results()
