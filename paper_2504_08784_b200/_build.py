"""In-tree build of the native libraries (no JIT cache: the .so files travel to
the GPU box with the repo snapshot).

  libslos_b200.so      product: sm_100a kernels + C++ host shim (C-ABI)
  libslos_workload.so  synthetic instance generator (benchmark/test input)
Test infrastructure (oracle/Makefile): liboracle_slos.so, oracle/_ref/libslos_ref.so.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction (bit-exact fp64 vs the -O2 x86 reference)
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-ffp-contract=off", "-diag-suppress", "550"]


def _run(cmd, cwd=None):
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_product(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """The product library; `defines`/`out` build an experiment variant elsewhere
    (e.g. -DSLOS_DP_THREADS=128 into exp/, selected with SLOS_PRODUCT_LIB)."""
    out = out or os.path.join(PKG, "libslos_b200.so")
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", h) for h in ("slos_planner.h", "slos_plan_json.h", "slos_route.h", "slos_trace.h", "slos_fit.h")]
    if not force and not _stale(out, deps):
        return out
    bdir = os.path.join(PKG, "build") if not defines else os.path.join(os.path.dirname(out), "build")
    os.makedirs(bdir, exist_ok=True)
    ko = os.path.join(bdir, "slos_kernels.o")
    ho = os.path.join(bdir, "slos_host.o")
    k = _run([NVCC, *ARCH, *NVFLAGS, *defines, "-Xptxas", "-v", "-c", os.path.join(CSRC, "slos_kernels.cu"), "-o", ko])
    if verbose:
        sys.stderr.write(k.stderr)
    _run([NVCC, *ARCH, *NVFLAGS, *defines, "-x", "cu", "-c", os.path.join(CSRC, "slos_host.cpp"), "-o", ho])
    jo = os.path.join(bdir, "slos_json.o")  # host-only: plan_to_json serialisation
    _run(["g++", "-std=c++17", "-O2", "-fPIC", "-c", os.path.join(CSRC, "slos_json.cpp"), "-o", jo])
    ro = os.path.join(bdir, "slos_route.o")  # host-only: batched routing rounds over slos_plan_batch
    _run(["g++", "-std=c++17", "-O2", "-fPIC", "-c", os.path.join(CSRC, "slos_route.cpp"), "-o", ro])
    to = os.path.join(bdir, "slos_trace.o")  # host-only: batched trace generation (libstdc++ <random>)
    _run(["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-c", os.path.join(CSRC, "slos_trace.cpp"), "-o", to])
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-Xlinker", "-Bsymbolic", ko, ho, jo, ro, to, "-o", out,
          "-lpthread", "-ldl", "-lrt"])
    return out


def build_probe(force: bool = False) -> str:
    """libslos_probe.so: the shared-memory bandwidth probe bench.py measures the
    DP stage's roofline peak with (a measurement tool, not the planner ABI)."""
    out = os.path.join(PKG, "libslos_probe.so")
    src = os.path.join(CSRC, "slos_probe.cu")
    if force or _stale(out, [src]):
        _run([NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
              src, "-o", out])
    return out


def build_workload(force: bool = False) -> str:
    out = os.path.join(PKG, "libslos_workload.so")
    src = os.path.join(CSRC, "slos_workload.c")
    if force or _stale(out, [src]):
        _run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", out, src, "-lm"])
    return out


def build_oracle(force: bool = False) -> str:
    """Test-only checkers: the C restatement always, the compiled reference when
    /root/reference is present (on the GPU box the prebuilt copy is used)."""
    odir = os.path.join(ROOT, "oracle")
    _run(["make", "-s", "-C", odir, "oracle"])
    if os.path.isdir(os.environ.get("SLOS_REF", "/root/reference/proj")):
        _run(["make", "-s", "-j8", "-C", odir, "ref"])
    return os.path.join(odir, "liboracle_slos.so")


def build_integration(force: bool = False) -> None:
    """integration/_build/libslos_lockstep.so: the lockstep routing / sweep driver over
    the reference's simulator sources (compiled where they lie), when present."""
    if os.path.isdir(os.environ.get("SLOS_REF", "/root/reference/proj")):
        _run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "integration")])


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_workload(force)
    build_oracle(force)
    build_integration(force)
    build_product(force, verbose)
    build_probe(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
