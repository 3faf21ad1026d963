"""Build libfks.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# FKS_CHECKS=1: the checked build (bounds checks + traps in every kernel) as
# libfks_checked.so, objects in csrc/checked/ -- load it with FKS_LIB_VARIANT=checked.
# FKS_TIMING=1: the per-phase clock64 instrumentation of kernels3d.cu as libfks_timing.so.
CHECKED = bool(os.environ.get("FKS_CHECKS"))
TIMING = bool(os.environ.get("FKS_TIMING"))
# FKS_VARIANT=<tag> (with FKS_NVCC_EXTRA="-D...") builds a named development variant libfks_<tag>.so.
_TAG = "checked" if CHECKED else "timing" if TIMING else os.environ.get("FKS_VARIANT") or None
LIB = os.path.join(HERE, f"libfks_{_TAG}.so" if _TAG else "libfks.so")
OBJDIR = os.path.join(CSRC, _TAG) if _TAG else CSRC
SOURCES = ["fks_api.cu", "kernels2d.cu", "kernels2dp.cu", "kernels3d.cu", "kernels3d64.cu", "kernels_aux.cu",
           "kernels_bgk.cu", "kernels_small.cu"]
HEADERS = ["fft.cuh", "fftp.cuh", "common.cuh", "kernels.cuh", os.path.join("..", "..", "include", "fks.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = (["-DFKS_TIMING"] if os.environ.get("FKS_TIMING") else []) + (["-DFKS_CHECKS"] if CHECKED else []) + os.environ.get("FKS_NVCC_EXTRA", "").split() + ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]


# Per-file ptxas settings.  kernels3d.cu: --register-usage-level=6 (default 5) gives k_step3d a
# different register allocation, 17.88 vs 18.29 ms per C2 step (levels 6-10 produce the same SASS;
# profiles/r02_optimisation_log.md); applied to the other files it costs the 2D N = 64 kernel
# 20 % and the transport / BGK kernels 2-3 %, so it is not global.
FILE_FLAGS = {"kernels3d.cu": ["-Xptxas", "--register-usage-level=6"]}


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(s, verbose):
    src = os.path.join(CSRC, s)
    os.makedirs(OBJDIR, exist_ok=True)
    obj = os.path.join(OBJDIR, s.replace(".cu", ".o"))
    r = subprocess.run([NVCC, *FLAGS, *FILE_FLAGS.get(s, []), "-c", src, "-o", obj], capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {s}")
    with open(os.path.join(OBJDIR, s.replace(".cu", ".ptxas.txt")), "w") as fh:
        fh.write(r.stderr)
    return obj


def build(force=False, verbose=False):
    """Compile every .cu to an object (in parallel), link libfks.so; returns the library path."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", LIB, "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
