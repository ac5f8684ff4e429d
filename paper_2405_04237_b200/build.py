"""Build libtsqr.so in-tree: nvcc for sm_100a, linked against the NCCL shipped with torch."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC_DIR = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(SRC_DIR, "tsqr.cu")]
DEPS = SOURCES + sorted(os.path.join(SRC_DIR, f) for f in os.listdir(SRC_DIR) if f.endswith(".cuh")) + [
    os.path.join(ROOT, "include", "tsqr.h")]
LIB = os.path.join(HERE, "libtsqr.so")


def nccl_dirs() -> tuple[str, str]:
    import nvidia.nccl
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc_cmd(out: str = LIB, extra: list[str] | None = None) -> list[str]:
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return [nvcc, "-shared", "-Xcompiler", "-fPIC", "-std=c++17", "-O3", "-lineinfo",
            "-gencode", "arch=compute_100a,code=sm_100a",
            "-I", os.path.join(ROOT, "include"), "-I", inc,
            "-o", out, *SOURCES,
            "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}", *(extra or [])]


def build(force: bool = False, verbose: bool = False) -> str:
    stale = not os.path.exists(LIB) or any(os.path.getmtime(LIB) < os.path.getmtime(d) for d in DEPS)
    if force or stale:
        cmd = nvcc_cmd(extra=["-Xptxas", "-v"] if verbose else None)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libtsqr.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


def build_profiling_variant(out: str = os.path.join(HERE, "libtsqr_prof.so")) -> str:
    """Development build with the cluster kernel's phase counters (-DTSQR_CL_PROF); load it with
    TSQR_LIB=<path>.  Never the product library."""
    r = subprocess.run(nvcc_cmd(out=out, extra=["-DTSQR_CL_PROF"]), capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building the profiling variant")
    return out


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
