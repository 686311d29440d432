#!/bin/bash
# Round measurement on the GPU box (run under gpurun from the repo root):
#   bash tests/profile_round.sh <tag>
# 1) bench.py (N=1) and the reference arm, 2) the ncu launch list of a short bench
# run (cold, serialised: shares, not absolutes), 3) one `ncu --set full` capture of
# one solve's kernels (C2, 1024 instances: anchor + group per part, then dp + build per part). Outputs land in gpurun_out/.
tag=${1:-latest}
python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${tag}.json 2>> gpurun_out/bench_${tag}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>> gpurun_out/bench_${tag}.err
SLOS_NO_PHASES=1 SLOS_SOLVES=1 ncu --set full --clock-control none --import-source on \
    -k regex:"anchor_kernel|group_kernel|dp_kernel|build_kernel" -s 8 -c 8 -f -o gpurun_out/prof \
    python tests/gpu_phases.py C2 1024 > gpurun_out/ncu_${tag}.log 2>&1
tail -c 3000 gpurun_out/bench_${tag}.json gpurun_out/bench_ref_${tag}.json
