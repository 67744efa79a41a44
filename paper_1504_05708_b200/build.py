"""Builds the in-tree libduquad.so for sm_100a with nvcc (no JIT cache, no fallback)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libduquad.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    base = None
    if spec is not None and spec.submodule_search_locations:
        base = os.path.join(list(spec.submodule_search_locations)[0], "nccl")
    if base is None or not os.path.isdir(base):
        raise RuntimeError("NCCL headers/library (nvidia-nccl wheel) not found")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _cublas_libdir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    if spec is not None and spec.submodule_search_locations:
        d = os.path.join(list(spec.submodule_search_locations)[0], "cublas", "lib")
        if os.path.exists(os.path.join(d, "libcublas.so.12")):
            return d
    raise RuntimeError("cuBLAS (nvidia-cublas wheel) not found")


def build(verbose: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    inc, libdir = _nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "duquad.h")]
    extra = os.environ.get("DUQUAD_NVCC_EXTRA", "").split()   # e.g. instrumentation defines
    if not extra and os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(d) for d in deps):
        return OUT
    cmd = [nvcc, ARCH, *extra, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v" if verbose else "-O3",
           f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}", "-o", OUT + ".tmp", *srcs,
           f"-L{libdir}", "-l:libnccl.so.2", f"-Xlinker=-rpath,{libdir}",
           f"-L{_cublas_libdir()}", "-l:libcublas.so.12", f"-Xlinker=-rpath,{_cublas_libdir()}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if verbose:
        sys.stderr.write(r.stdout + r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
