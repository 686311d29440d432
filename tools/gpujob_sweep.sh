for k in 1 2; do for v in cur grp2 grp8; do echo "== $v"; SLOS_PRODUCT_LIB=exp/$v/libslos_b200.so SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -1; done; done
