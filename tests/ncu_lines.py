"""Per-CUDA-source-line hot spots from an ncu report (cuda,sass source view).

  python tests/ncu_lines.py gpurun_out/<rep>.ncu-rep [top] [kernel-regex]

Prints the source lines with the most warp-stall samples and instructions, plus
each line's dominant stall reasons (needs -lineinfo at compile time).
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
    txt = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = []
    fname = "?"
    hdr = None
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "":
            continue  # sass rows
        d = dict(zip(hdr, r))
        try:
            samp = int(d["Warp Stall Sampling (All Samples)"] or 0)
            inst = int(d["Instructions Executed"] or 0)
        except ValueError:
            continue
        stalls = []
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    stalls.append((int(v), k[6:]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        rows.append((samp, inst, fname, int(r[0]), r[1].strip()[:90], stalls[:3]))
    tot_s = sum(x[0] for x in rows) or 1
    tot_i = sum(x[1] for x in rows) or 1
    print(f"total samples {tot_s}, instructions {tot_i:.3e}")
    rows.sort(reverse=True)
    for samp, inst, f, ln, src, st in rows[:top]:
        ss = " ".join(f"{n}:{100*v/max(samp,1):.0f}%" for v, n in st if v)
        print(f"{100*samp/tot_s:5.1f}% smp {100*inst/tot_i:5.1f}% ins  {f}:{ln:<5} {src}  [{ss}]")
    byf = {}
    for samp, inst, f, *_ in rows:
        a = byf.setdefault(f, [0, 0])
        a[0] += samp
        a[1] += inst
    print("per file:", {k: f"{100*v[0]/tot_s:.1f}% smp / {100*v[1]/tot_i:.1f}% ins" for k, v in byf.items()})


if __name__ == "__main__":
    main()
