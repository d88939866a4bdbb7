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
EXP_LIB = os.path.join(LIBDIR, "libeossearch_exp.so")  # A/B builds with extra -D flags (EOS_LIBRARY=exp)
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


COMMON = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler",
          "-fvisibility=hidden", "-I", INCLUDE, "-I", CSRC]


def nvcc_compile_cmd(src: str, obj: str, extra: list[str] | None = None) -> list[str]:
    return [NVCC, *COMMON, "-Xptxas", "-v", *(extra or []), "-c", "-o", obj, src]


def nvcc_link_cmd(out: str, objs: list[str]) -> list[str]:
    return [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs]


def build(force: bool = False, verbose: bool = False, checked: bool = False,
          exp_flags: list[str] | None = None) -> str:
    """Compile every source to an object in parallel (one nvcc per translation unit:
    the kernel instantiations are split over runtime.cu, search_api.cu and
    grid_api.cu), then link the shared library."""
    from concurrent.futures import ThreadPoolExecutor
    lib = EXP_LIB if exp_flags is not None else (CHECKED_LIB if checked else LIB)
    if not (force or exp_flags is not None or stale(lib)):
        return lib
    os.makedirs(LIBDIR, exist_ok=True)
    tag = "exp" if exp_flags is not None else ("checked" if checked else "product")
    objdir = os.path.join(LIBDIR, "obj_" + tag)
    os.makedirs(objdir, exist_ok=True)
    extra = exp_flags if exp_flags is not None else (["-DEOS_DEVICE_CHECKS"] if checked else None)
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        jobs.append((src, obj, nvcc_compile_cmd(src, obj, extra)))
    with ThreadPoolExecutor(len(jobs)) as ex:
        results = list(ex.map(lambda j: subprocess.run(j[2], capture_output=True, text=True), jobs))
    log = os.path.join(LIBDIR, {"exp": "ptxas_exp.log", "checked": "ptxas_checked.log"}.get(tag, "ptxas.log"))
    with open(log, "w") as f:
        for (src, _, _), r in zip(jobs, results):
            f.write(f"==== {os.path.basename(src)}\n" + r.stdout + r.stderr)
    bad = [(src, r) for (src, _, _), r in zip(jobs, results) if r.returncode != 0]
    if bad:
        for src, r in bad:
            sys.stderr.write(f"{src}:\n{r.stdout}{r.stderr}")
        raise RuntimeError("nvcc failed building libeossearch.so")
    tmp = lib + ".tmp"
    r = subprocess.run(nvcc_link_cmd(tmp, [j[1] for j in jobs]), capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libeossearch.so")
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}")
    return lib


if __name__ == "__main__":
    # --exp [-DNAME[=V] ...]: an A/B build of the same sources into libeossearch_exp.so, with
    # the experiment knobs compiled in (-DEOS_EXPERIMENTS; runtime.cu lists them)
    exp = (["-DEOS_EXPERIMENTS"] + [a for a in sys.argv[1:] if a.startswith("-D")]) \
        if "--exp" in sys.argv else None
    build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv, exp_flags=exp)
