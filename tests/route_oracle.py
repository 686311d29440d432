"""TEST INFRASTRUCTURE: an independent Python restatement of the routing rounds
(include/slos_route.h) over any library exporting slos_planner.h -- the checker
of the product's slos_route_rounds, and (with oracle/_ref) bench.py's C3 CPU
baseline. It follows the reference's routing (ClusterSim::on_decline,
tiers_router.cpp:80-108: ring re-offer while hops < min(routing_limit, R-1), then
the backup policy) and its replica bookkeeping (apply_schedule / snapshot,
sim_executor.cpp:265-340: an admitted request becomes a running prefill whose
memory joins the resident pool)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2504_08784_b200 import abi
from paper_2504_08784_b200.routing import ADMITTED, BEST_EFFORT, DROPPED, ROUTE_OUTCOME_DTYPE


def route_rounds_py(lib, handles, n_clusters, snaps, replicas=4, routing_limit=3, backup_best_effort=True,
                    net_delay_s=0.001, unit_value=False):
    R = replicas
    eff = min(routing_limit, R - 1)
    NR = n_clusters * R
    inp = snaps.inputs
    # per replica: running rows (numpy RUNNING_DTYPE), resident memory, offers
    run = []
    pend = []  # pending rows per replica (their snapshot order = outcome order)
    base_out = []
    k = 0
    for x in range(NR):
        nr, npd = int(inp["n_running"][x]), int(inp["n_pending"][x])
        r0 = (int(inp["running"][x]) - snaps.running.ctypes.data) // snaps.running.itemsize
        p0 = (int(inp["pending"][x]) - snaps.pending.ctypes.data) // snaps.pending.itemsize
        run.append(list(snaps.running[r0:r0 + nr]))
        pend.append(snaps.pending[p0:p0 + npd].copy())
        base_out.append(k)
        k += npd
    out = np.zeros(k, ROUTE_OUTCOME_DTYPE)
    out["fate"] = DROPPED
    out["replica"] = -1
    reqs = []  # (pending row, origin, hops, outcome index)
    offered = [[] for _ in range(NR)]
    for x in range(NR):
        for j in range(len(pend[x])):
            reqs.append([pend[x][j], x % R, 0, base_out[x] + j])
            offered[x].append(len(reqs) - 1)
    resident = [int(inp["memory_standard_resident"][x]) for x in range(NR)]
    stats = {"rounds": 0, "plans": 0}
    rnd = 0
    while any(offered):
        who = [x for x in range(NR) if offered[x]]
        keep = []
        arr = np.zeros(len(who), abi.INPUT_DTYPE)
        for w, x in enumerate(who):
            ra = np.array(run[x], abi.RUNNING_DTYPE) if run[x] else np.zeros(1, abi.RUNNING_DTYPE)
            pa = np.array([reqs[q][0] for q in offered[x]], abi.PENDING_DTYPE)
            keep += [ra, pa]
            arr[w] = inp[x]
            arr[w]["now"] = inp["now"][x] + rnd * net_delay_s
            arr[w]["running"] = ra.ctypes.data
            arr[w]["n_running"] = len(run[x])
            arr[w]["pending"] = pa.ctypes.data
            arr[w]["n_pending"] = len(pa)
            arr[w]["memory_standard_resident"] = resident[x]
        hs = (C.c_void_p * len(who))(*[handles[x] for x in who])
        res = (abi.Result * len(who))()
        assert lib.slos_plan_batch(hs, len(who), C.c_void_p(arr.ctypes.data), int(unit_value), res, None) == 0
        stats["rounds"] += 1
        stats["plans"] += len(who)
        nxt = [[] for _ in range(NR)]
        for w, x in enumerate(who):
            r = res[w]
            assert r.status == 0, lib.slos_last_error()
            c0 = x - x % R
            for a in range(r.n_admitted):
                q = reqs[offered[x][r.admitted[a]]]
                out[q[3]] = (ADMITTED, x % R, q[2], rnd)
                row = np.zeros(1, abi.RUNNING_DTYPE)[0]
                row["id"] = q[0]["id"]
                row["prefill_remaining"] = q[0]["prefill_tokens"]
                row["prefill_deadline"] = q[0]["prefill_deadline"]
                row["decode_tier"] = q[0]["decode_tier"]
                run[x].append(row)
                resident[x] += int(q[0]["memory_units"])
            for d in range(r.n_declined):
                qi = offered[x][r.declined[d]]
                q = reqs[qi]
                if q[2] < eff:
                    q[2] += 1
                    nxt[c0 + (x % R + 1) % R].append(qi)
                elif backup_best_effort:
                    out[q[3]] = (BEST_EFFORT, q[1], q[2], rnd)
                else:
                    out[q[3]] = (DROPPED, -1, q[2], rnd)
            lib.slos_result_free(C.byref(r))
        offered = nxt
        rnd += 1
    return out, stats
