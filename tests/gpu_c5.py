"""C5 sweep throughput probe (run under gpurun): the recorded simulator corpus
(tests/golden/c5_*.bin.gz, 2,048 instances per planner configuration) tiled to
`n` instances, device-resident solve, stage timings."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200 import workload as W  # noqa: E402
from paper_2504_08784_b200.planner import PerfTerm, PlannerConfig  # noqa: E402
from paper_2504_08784_b200.sweep import ShardSolver, ShardSpec  # noqa: E402

grp = sys.argv[1] if len(sys.argv) > 1 else "ar"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
b = W.load_corpus(os.path.join(ROOT, "tests", "golden", f"c5_{grp}.bin.gz"))
b = b.tiled((n + b.n - 1) // b.n).subset(range(n))
cfg = PlannerConfig(max_chunk_tokens=2048, max_batch_tokens=16384, speculative=(grp == "spec"),
                    spec_alpha=0.8, spec_max_len=8)
spec = ShardSpec(None, [PerfTerm(*t) for t in ((2.5e-5, 2e-3, 0.006), (0.0, 0.0, 0.02))], cfg)
s = ShardSolver(abi.product(), spec, None, batch=b)
rec = torch.empty((n, C.sizeof(abi.Record)), dtype=torch.uint8, device="cuda")
s.upload()
s.converge(rec)
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    s.solve()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    st = s.stage_ms()
    print(grp, n, f"solve {dt*1e3:.2f} ms -> {n/dt:.0f} plans/s; stage ms [anchor, dp, build] {st}", flush=True)
