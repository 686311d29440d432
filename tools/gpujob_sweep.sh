L=SLOS_PRODUCT_LIB=exp/prio/libslos_b200.so
for k in 1 2; do
echo "== base"; env $L SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2
echo "== rev"; env $L SLOS_PART_PRIO_REV=1 SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2
done
echo "== rev 3 parts"; env $L SLOS_PART_PRIO_REV=1 SLOS_SOLVE_PARTS=3 SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2
