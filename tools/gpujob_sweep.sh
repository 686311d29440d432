for k in 1 2; do
for v in oldhdr newhdr; do echo "== $v"; SLOS_PRODUCT_LIB=exp/$v/libslos_b200.so python tests/gpu_e2e_c5.py 2>&1 | tail -2; done
done
