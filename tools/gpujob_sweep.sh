for k in 1 2; do
echo "== base"; SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2
echo "== atom"; SLOS_PRODUCT_LIB=exp/atom/libslos_b200.so SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2
done
