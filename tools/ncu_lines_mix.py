"""Aggregate warp-stall samples of one kernel per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass` output.
usage: python tools/ncu_lines_mix.py mix.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, cur_line, cur_src = None, None, None
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:  # a CUDA source line row
        cur_line, cur_src = r[0], r[1]
        continue
    # a SASS row under the current source line
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    k = (cur_file, cur_line)
    a = agg.setdefault(k, [0.0, cur_src, {}])
    a[0] += s
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "(Not" not in h and i < len(r):
            try:
                a[2][h] = a[2].get(h, 0.0) + float(r[i] or 0)
            except ValueError:
                pass
tot = sum(v[0] for v in agg.values()) or 1.0
for (f, ln), (s, src, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    best = sorted(st.items(), key=lambda x: -x[1])[:2]
    print(f"{100 * s / tot:5.1f}% {f}:{ln} {src.strip()[:70]!s:72} " + " ".join(f"{k[6:]}={int(v)}" for k, v in best))
