run() { echo "== $*"; env "$@" SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2; }
run SLOS_PRODUCT_LIB=exp/bmb4/libslos_b200.so SLOS_BUILD_SMEM_KB=24
run SLOS_PRODUCT_LIB=exp/bmb4/libslos_b200.so SLOS_BUILD_SMEM_KB=16
run SLOS_PRODUCT_LIB=exp/bmb5/libslos_b200.so SLOS_BUILD_SMEM_KB=32
run SLOS_PRODUCT_LIB=exp/bmb5/libslos_b200.so SLOS_BUILD_SMEM_KB=24
run SLOS_PRODUCT_LIB=exp/bmb6/libslos_b200.so SLOS_BUILD_SMEM_KB=32
run SLOS_PRODUCT_LIB=exp/bmb6/libslos_b200.so SLOS_BUILD_SMEM_KB=24
run SLOS_BUILD_SMEM_KB=32
