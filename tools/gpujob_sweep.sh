L=SLOS_PRODUCT_LIB=exp/dp1024/libslos_b200.so
for v in X=1 $L; do echo "== $v"; env $v SLOS_NO_PHASES=1 SLOS_SOLVES=3 python tests/gpu_phases.py C4 64 2>&1 | tail -2; env $v python tests/gpu_p50.py C1 C2 C4; done
