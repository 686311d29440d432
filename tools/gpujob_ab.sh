# A/B of two library builds on one box: bash tools/gpujob_ab.sh <dirA> <dirB> [family] [n]
fam=${3:-C2}; n=${4:-1024}
for k in 1 2 3; do
for v in $1 $2; do echo "== $v"; SLOS_PRODUCT_LIB=exp/$v/libslos_b200.so SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py $fam $n 2>&1 | tail -1; done
done
