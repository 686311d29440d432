"""Distil ncu captures (gpurun_out/*.ncu-rep + launches.csv) into profiles/.

  python tests/ncu_summary.py <tag> [report]  -> profiles/<tag>_ncu_summary.{json,md}
                                           and profiles/ncu_summary.json (read by bench.py)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warp_latency_issue_stalled_barrier",
    "launches",
]


ADDITIVE = {"gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum", "launch__grid_size"}


def raw(rep):
    """{kernel short name: {metric: {value, unit}}} over the launches in the report:
    additive metrics (time, bytes, instructions, grid) are summed over a kernel's
    launches (one solve = one launch per solve part), ratios keep the last launch."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    out = {}
    for vals in rows[2:]:
        name = vals[ki].split("(")[0].split("::")[-1]
        prev = out.get(name, {})
        d = {}
        for i, n in enumerate(hdr):
            if n in METRICS:
                v = vals[i]
                if n in ADDITIVE and n in prev:
                    try:
                        v = repr(float(prev[n]["value"].replace(",", "")) + float(v.replace(",", "")))
                    except ValueError:
                        pass
                d[n] = {"value": v, "unit": units[i]}
        d["launches"] = {"value": str(int(prev.get("launches", {"value": "0"})["value"]) + 1), "unit": ""}
        out[name] = d
    return out


def to_bytes(m):
    v = float(m["value"].replace(",", ""))
    u = m["unit"].lower()
    return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(io.StringIO("".join(lines)))
    hdr = next(rd)
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    for r in rd:
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        rows.append((r[ki].split("(")[0], v * scale))
    return rows


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "latest"
    summ = {"tag": tag, "kernels": {}}
    rep = sys.argv[2] if len(sys.argv) > 2 else os.path.join(OUT, "prof.ncu-rep")
    if os.path.exists(rep):
        for name, m in raw(rep).items():
            summ["kernels"][name] = {k: v["value"] + " " + v["unit"] for k, v in m.items()}
            if "dram__bytes_read.sum" in m:
                summ["kernels"][name]["dram_bytes_per_launch"] = to_bytes(m["dram__bytes_read.sum"]) + \
                    to_bytes(m["dram__bytes_write.sum"])
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(lp):
        rows = launches(lp)
        agg = {}
        for k, us in rows:
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += us
        tot = sum(a[1] for a in agg.values())
        summ["launch_list"] = {k: {"launches": a[0], "total_us": round(a[1], 1),
                                   "share": round(a[1] / tot, 4)} for k, a in agg.items()}
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{tag}_ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    stage = [summ["kernels"].get(k, {}).get("dram_bytes_per_launch") for k in
             ("anchor_kernel", "group_kernel", "dp_kernel")]
    with open(os.path.join(PROF, "ncu_summary.json"), "w") as f:
        json.dump({"kernel": "dp_stage", "instances": 1024,
                   "dram_bytes_per_launch": sum(stage) if all(x is not None for x in stage) else None,
                   "per_kernel": dict(zip(("anchor_kernel", "group_kernel", "dp_kernel"), stage)),
                   "source": f"{tag}_ncu_summary.json"}, f, indent=1)
    lines = [f"# ncu summary ({tag})", ""]
    for k, d in summ["kernels"].items():
        lines.append(f"## {k}")
        for m in METRICS + ["dram_bytes_per_launch"]:
            if m in d:
                lines.append(f"- `{m}`: {d[m]}")
        lines.append("")
    if "launch_list" in summ:
        lines.append("## launch list (ncu --metrics gpu__time_duration.sum, cold, serialised)")
        for k, a in sorted(summ["launch_list"].items(), key=lambda kv: -kv[1]["total_us"]):
            lines.append(f"- {k}: {a['launches']} launches, {a['total_us']} us total, share {a['share']:.1%}")
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
