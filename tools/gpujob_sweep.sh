# stage-time sweep over library variants and env knobs (C2 x 1024)
run() { echo "== $*"; env "$@" SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2; }
run X=1
run SLOS_SOLVE_PARTS=1
run SLOS_PRODUCT_LIB=exp/anc6/libslos_b200.so
run SLOS_PRODUCT_LIB=exp/t128/libslos_b200.so SLOS_DP_SMEM_KB=27
run SLOS_PRODUCT_LIB=exp/t128/libslos_b200.so SLOS_DP_SMEM_KB=27 SLOS_SOLVE_PARTS=1
run SLOS_PRODUCT_LIB=exp/t128/libslos_b200.so SLOS_DP_SMEM_KB=27 SLOS_DP_TSM=96
run SLOS_PRODUCT_LIB=exp/t128/libslos_b200.so SLOS_DP_SMEM_KB=27 SLOS_DP_TSM=96 SLOS_SOLVE_PARTS=1
