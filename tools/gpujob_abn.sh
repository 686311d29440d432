# A/B/n of library builds on one box: bash tools/gpujob_abn.sh <family> <n> <dir>...
fam=$1; n=$2; shift 2
for k in 1 2 3; do
for v in "$@"; do echo "== $v"; SLOS_PRODUCT_LIB=exp/$v/libslos_b200.so SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py $fam $n 2>&1 | tail -1; done
done
