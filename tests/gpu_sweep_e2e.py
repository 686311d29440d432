"""Live capacity sweep, end to end (run under gpurun): capacity_search over the C5
scenarios with the B200 planner in the loop (lockstep lanes + plan broker,
integration/) against the reference's own capacity_search with its SloScheduler,
one search per host thread. Prints one JSON line; results must be identical."""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2504_08784_b200 import abi  # noqa: E402
from paper_2504_08784_b200.lockstep import Lockstep, Sim  # noqa: E402
from sim_harness import RefSim  # noqa: E402
from sim_harness import Sim as RSim  # noqa: E402


def searches():
    out = []
    for s in ("chatbot", "coder", "summarizer", "toolllm", "reasoning"):
        for rep in ((2, 4) if s == "chatbot" else (1, 4)):
            out.append((s, Sim(replicas=rep, speculative=(s == "reasoning"))))
    return out


def main(backend=abi.PRODUCT_LIB, horizon_s=float(os.environ.get("SWEEP_HORIZON", "30")),
         seeds=int(os.environ.get("SWEEP_SEEDS", "3"))):
    S = searches()
    kw = dict(seeds=seeds, horizon_s=horizon_s, lo=0.02, hi=12.0, target=0.9, rel_tol=0.05)
    ls = Lockstep(backend)
    t0 = time.perf_counter()
    got, st = ls.capacity(S, **kw)
    t_ours = time.perf_counter() - t0
    ls.backend(None)
    rs = RefSim()
    rs.backend(None)
    threads = int(os.environ.get("SLOS_REF_THREADS", os.cpu_count() or 1))
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        want = list(ex.map(lambda x: rs.capacity(x[0], RSim(**x[1].__dict__), **kw), S))
    t_ref = time.perf_counter() - t0
    line = {"workload": f"capacity_search x {len(S)} (5 scenarios x 1/4 replicas), {seeds} seeds, {horizon_s} s horizon",
            "ours_s": t_ours, "reference_s": t_ref, "reference_threads": threads,
            "speedup": t_ref / t_ours, "identical": got == want, "plans": st.get("plans"),
            "flushes": st.get("flushes"), "backend": os.path.basename(backend)}
    print(json.dumps(line), flush=True)
    return line


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else abi.PRODUCT_LIB)
