run() { echo "== $*"; env "$@" SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2; }
L=SLOS_PRODUCT_LIB=exp/split/libslos_b200.so
run $L
run $L SLOS_PART_SPLIT=0.35
run $L SLOS_PART_SPLIT=0.42
run $L SLOS_PART_SPLIT=0.58
run $L SLOS_PART_SPLIT=0.65
run $L SLOS_SOLVE_PARTS=3
run $L SLOS_SOLVE_PARTS=4
