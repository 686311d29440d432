set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
SLOS_NO_PHASES=1 SLOS_SOLVES=5 python tests/gpu_phases.py C2 1024 2>&1 | tail -3
SLOS_NO_PHASES=1 SLOS_SOLVES=3 python tests/gpu_phases.py C4 64 2>&1 | tail -2
timeout 300 python bench.py --no-legs --no-cpu-baseline > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['kernel_ms_per_step'], d['roofline']['frac'])"
