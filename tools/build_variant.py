"""Build an experiment variant of the product library into exp/<name>/ with extra
nvcc defines; select it at run time with SLOS_PRODUCT_LIB=exp/<name>/libslos_b200.so.
usage: python tools/build_variant.py <name> -DFOO=1 ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_08784_b200 import _build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "exp", name, "libslos_b200.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
_build.build_product(force=True, defines=defs, out=out)
print(out)
