run() { echo "== $*"; env "$@" SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2; }
run X=1
run SLOS_DP_TSM=256
run SLOS_DP_TSM=320
run SLOS_DP_TSM=384
run SLOS_DP_TSM=128
run SLOS_BUILD_SMEM_KB=20
run SLOS_BUILD_SMEM_KB=28
