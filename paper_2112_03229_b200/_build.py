"""Build of the product library libeossearch.so (nvcc, sm_100a, in-tree).

    python -m paper_2112_03229_b200._build [--force]

The library links the CUDA runtime statically (-cudart static) so it does not
depend on which libcudart torch happens to load; stream handles passed in from
torch are driver-level and interoperate.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libeossearch.so")
CHECKED_LIB = os.path.join(LIBDIR, "libeossearch_checked.so")  # -DEOS_DEVICE_CHECKS debug build
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def deps() -> list[str]:
    return sources() + glob.glob(os.path.join(CSRC, "*.h*")) + glob.glob(os.path.join(CSRC, "*.cuh")) \
        + [os.path.join(INCLUDE, "eossearch.h")]


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in deps())


def nvcc_cmd(out: str = LIB, extra: list[str] | None = None) -> list[str]:
    return [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
            "-Xcompiler", "-fvisibility=hidden", "-cudart", "static", "-I", INCLUDE, "-I", CSRC,
            "-Xptxas", "-v", *(extra or []), "-o", out, *sources()]


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib = CHECKED_LIB if checked else LIB
    if force or stale(lib):
        os.makedirs(LIBDIR, exist_ok=True)
        tmp = lib + ".tmp"
        r = subprocess.run(nvcc_cmd(tmp, ["-DEOS_DEVICE_CHECKS"] if checked else None),
                           capture_output=True, text=True)
        log = os.path.join(LIBDIR, "ptxas_checked.log" if checked else "ptxas.log")
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libeossearch.so")
        os.replace(tmp, lib)
        if verbose:
            print(f"built {lib}")
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv)
