timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in "SLOS_DP_BIG_COST=0" "X=1" "SLOS_DP_BIG_TSM=512"; do echo "== $v"; env $v SLOS_NO_PHASES=1 SLOS_SOLVES=3 python tests/gpu_phases.py C4 64 2>&1 | tail -2; done
SLOS_NO_PHASES=1 SLOS_SOLVES=3 python tests/gpu_phases.py C2 1024 2>&1 | tail -2
