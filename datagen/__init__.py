"""datagen -- seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the searched method (no lower-bound search,
no binning, no interpolation).  It only draws random numbers and applies the
value recipes of the synthetic workloads of BASELINE.json configs[0..4]
(DESIGN.md "Input recipe").  Targets are counter-based
(`gen_core.h`): element i of a stream is a pure function of (seed, stream, i),
so every rank of a sharded run and the host sampler see the same dataset.

Two native libraries:
  lib/libeosgen_host.so  (gcc)  -- host generators, used by tests/oracle side
  lib/libeosgen_dev.so   (nvcc) -- device generators (bench / GPU tests)
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBDIR = os.path.join(_HERE, "lib")
HOST_LIB = os.path.join(_LIBDIR, "libeosgen_host.so")
DEV_LIB = os.path.join(_LIBDIR, "libeosgen_dev.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_host(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, "gen_host.c"), os.path.join(_HERE, "gen_core.h")]
    if force or _stale(HOST_LIB, srcs):
        os.makedirs(_LIBDIR, exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-std=c11", "-o", HOST_LIB, srcs[0], "-lm"])
    return HOST_LIB


def build_device(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, "gen_device.cu"), os.path.join(_HERE, "gen_core.h")]
    if force or _stale(DEV_LIB, srcs):
        os.makedirs(_LIBDIR, exist_ok=True)
        subprocess.check_call([NVCC, *ARCH, "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
                               "-cudart", "static", "-fmad=false", "-o", DEV_LIB, srcs[0]])
    return DEV_LIB


def build(force: bool = False) -> None:
    build_host(force)
    build_device(force)


_host = None
_dev = None

_D = ctypes.c_double
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_P = ctypes.c_void_p


def host_lib():
    global _host
    if _host is None:
        lib = ctypes.CDLL(build_host())
        lib.gen_stream_key.argtypes = [_U64, _U64]
        lib.gen_stream_key.restype = _U64
        lib.gen_exp10_host.argtypes = [_D]
        lib.gen_exp10_host.restype = _D
        lib.gen_fill_loguniform.argtypes = [_U64, _U64, _I64, _I64, _D, _D, _P]
        lib.gen_sample_loguniform.argtypes = [_U64, _U64, _P, _I64, _D, _D, _P]
        lib.gen_fill_copies.argtypes = [_U64, _I64, _I64, _D, _D, _P, _I64, _U64, _P]
        lib.gen_sample_copies.argtypes = [_U64, _P, _I64, _D, _D, _P, _I64, _U64, _P]
        lib.gen_fill_walk.argtypes = [_U64, _I64, _I64, _D, _D, _D, _D, _P]
        lib.gen_sample_walk.argtypes = [_U64, _P, _I64, _D, _D, _D, _D, _P]
        lib.gen_walk_sum.argtypes = [_U64, _I64, _I64]
        lib.gen_walk_sum.restype = _U64
        lib.gen_fill_walk_from.argtypes = [_U64, _I64, _I64, _U64, _D, _D, _D, _D, _P]
        _host = lib
    return _host


def dev_lib():
    global _dev
    if _dev is None:
        lib = ctypes.CDLL(build_device())
        lib.gen_dev_fill_loguniform.argtypes = [_U64, _U64, _I64, _I64, _D, _D, _P, _P]
        lib.gen_dev_fill_copies.argtypes = [_U64, _I64, _I64, _D, _D, _P, _I64, _U64, _P, _P]
        lib.gen_dev_fill_walk.argtypes = [_U64, _I64, _I64, _D, _D, _D, _D, _P, _P]
        for f in (lib.gen_dev_fill_loguniform, lib.gen_dev_fill_copies, lib.gen_dev_fill_walk):
            f.restype = ctypes.c_int
        _dev = lib
    return _dev


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------------
# Tables (host, numpy; small).  Recipes: BASELINE.json configs, SURVEY.md §8(c)
# A15/A16/A19 and §8(d).
# --------------------------------------------------------------------------

def table_cfg1(seed: int = 0) -> np.ndarray:
    """n=64, 10^u, u ~ U[-4,4] with the endpoints pinned, strictly increasing."""
    rng = np.random.default_rng(seed)
    while True:
        u = np.concatenate([[-4.0, 4.0], rng.uniform(-4.0, 4.0, 62)])
        x = np.sort(10.0 ** u)
        if np.all(np.diff(x) > 0):
            return x


def table_cfg2(seed: int = 1) -> np.ndarray:
    """n=300 log-spaced over [1e-6, 1e3] with +-2% multiplicative jitter (kept sorted)."""
    rng = np.random.default_rng(seed)
    j = np.arange(300, dtype=np.float64)
    x = 10.0 ** (-6.0 + 9.0 * j / 299.0) * (1.0 + 0.02 * (2.0 * rng.random(300) - 1.0))
    x = np.sort(x)
    assert np.all(np.diff(x) > 0)
    return x


def table_cfg3(seed: int = 2) -> np.ndarray:
    """n=1000 log-spaced over [1e0, 1e8] (temperature-like)."""
    return 10.0 ** (8.0 * np.arange(1000, dtype=np.float64) / 999.0)


def grid_cfg4(seed: int = 3):
    """density axis 200 log-spaced [1e-6,1e3], temperature axis 100 log-spaced [1,1e8],
    P = rho*T^1.5*(1+0.01*sin(37*ln rho)), row-major [n_rho][n_T]."""
    rho = np.logspace(-6.0, 3.0, 200)
    T = np.logspace(0.0, 8.0, 100)
    P = rho[:, None] * T[None, :] ** 1.5 * (1.0 + 0.01 * np.sin(37.0 * np.log(rho)))[:, None]
    return rho, T, np.ascontiguousarray(P)


def grid_big2d(seed: int = 7):
    """A grid larger than shared memory (the EOSPAC 2-D analogue of `big`): density axis 1000
    log-spaced [1e-6, 1e3], temperature axis 800 log-spaced [1, 1e8], P as cfg4 -- 6.4 MB of P,
    kept in device memory (L2-resident).  Not a BASELINE.json config."""
    rho = np.logspace(-6.0, 3.0, 1000)
    T = np.logspace(0.0, 8.0, 800)
    P = rho[:, None] * T[None, :] ** 1.5 * (1.0 + 0.01 * np.sin(37.0 * np.log(rho)))[:, None]
    return rho, T, np.ascontiguousarray(P)


def table_cfg5(seed: int = 4) -> np.ndarray:
    """n=4096 clustered: 2867 entries log-uniform in [1e0,1e2], 1229 log-uniform over
    [1e-6,1e0) U [1e2,1e10).  Sorted, exact duplicates redrawn."""
    rng = np.random.default_rng(seed)
    n_in, n_out = 2867, 1229

    def draw_out(k):
        # the 14 outer decades: 6 below (-6..0) and 8 above (2..10)
        v = rng.uniform(0.0, 14.0, k)
        return np.where(v < 6.0, v - 6.0, v - 6.0 + 2.0)

    u = np.concatenate([rng.uniform(0.0, 2.0, n_in), draw_out(n_out)])
    x = np.sort(10.0 ** u)
    while True:
        dup = np.concatenate([[False], np.diff(x) == 0])
        if not dup.any():
            return x
        k = int(dup.sum())
        x[dup] = 10.0 ** rng.uniform(-6.0, 10.0, k)
        x = np.sort(x)


def table_paper_exemplar() -> np.ndarray:
    """The paper's exemplar shape: 110 log-spaced values over [3e-6, 5.4e4]."""
    return np.logspace(math.log10(3e-6), math.log10(5.4e4), 110)


def table_big(seed: int = 6, n: int = 1 << 20) -> np.ndarray:
    """A table far larger than shared memory (SURVEY §8(f) f4 "tables larger than smem"):
    n = 2^20 sorted values 10^u, u ~ U[-6, 10] (the cfg5 span, log-distributed like the
    paper's tables).  Not a BASELINE.json config; the f4 measurement workload."""
    rng = np.random.default_rng(seed)
    return np.sort(10.0 ** rng.uniform(-6.0, 10.0, n))


# --------------------------------------------------------------------------
# Target streams
# --------------------------------------------------------------------------

@dataclass
class TargetSpec:
    """How target i of a workload is drawn (all fields are plain data)."""
    kind: str                  # "loguniform" | "copies" | "walk"
    seed: int
    stream: int = 0
    a: float = 0.0             # log10 lower end
    w: float = 0.0             # log10 width
    copy_every: int = 0        # "copies": 1/copy_every positions are exact table entries
    x0: float = 0.0            # "walk": start (log10)
    c: float = 0.0             # "walk": log10 units per integer step unit
    lo: float = 0.0            # "walk": reflecting range (log10)
    hi: float = 0.0

    # ---------- host ----------
    def host_fill(self, offset: int, count: int, table: np.ndarray | None = None) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        if count == 0:
            return out
        L = host_lib()
        if self.kind == "loguniform":
            L.gen_fill_loguniform(self.seed, self.stream, offset, count, self.a, self.w, _ptr(out))
        elif self.kind == "copies":
            t = np.ascontiguousarray(table, dtype=np.float64)
            L.gen_fill_copies(self.seed, offset, count, self.a, self.w, _ptr(t), t.size,
                              self.copy_every, _ptr(out))
        elif self.kind == "walk":
            L.gen_fill_walk(self.seed, offset, count, self.x0, self.c, self.lo, self.hi, _ptr(out))
        else:
            raise ValueError(self.kind)
        return out

    def host_fill_parallel(self, offset: int, count: int, table: np.ndarray | None = None,
                           threads: int | None = None, walk_base: int | None = None,
                           out: np.ndarray | None = None):
        """host_fill over host threads (the ctypes calls release the GIL); the same bits
        as host_fill.  Returns (out, walk_end) where walk_end is the walk's step sum
        through offset+count-1 (pass it as walk_base of the next chunk to stream a walk
        in order without re-summing its prefix; None for the other kinds)."""
        from concurrent.futures import ThreadPoolExecutor
        threads = threads or len(os.sched_getaffinity(0))
        out = np.empty(count, dtype=np.float64) if out is None else out
        assert out.dtype == np.float64 and out.flags.c_contiguous and out.size >= count
        step = max(1, (count + threads - 1) // threads)
        parts = [(s, min(count, s + step)) for s in range(0, count, step)]
        L = host_lib()
        with ThreadPoolExecutor(max(1, len(parts))) as ex:
            if self.kind != "walk":
                def job(p):
                    s, e = p
                    out[s:e] = self.host_fill(offset + s, e - s, table)
                list(ex.map(job, parts))
                return out, None
            M = (1 << 64) - 1
            if walk_base is None:   # sum of the steps before offset, split over threads
                st = max(1, (offset + threads - 1) // threads)
                walk_base = sum(ex.map(lambda b: L.gen_walk_sum(self.seed, b, min(offset, b + st)),
                                       range(0, offset, st))) & M
            sums = list(ex.map(lambda p: L.gen_walk_sum(self.seed, offset + p[0], offset + p[1]),
                               parts))
            bases, acc = [], walk_base
            for v in sums:
                bases.append(acc)
                acc = (acc + v) & M

            def wjob(ip):
                (s, e), b = ip
                L.gen_fill_walk_from(self.seed, offset + s, e - s, b, self.x0, self.c, self.lo,
                                     self.hi, out[s:].ctypes.data)
            list(ex.map(wjob, zip(parts, bases)))
            return out, acc

    def host_sample(self, idx: np.ndarray, table: np.ndarray | None = None) -> np.ndarray:
        """Targets at the given global indices (walk: idx must be sorted)."""
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(idx.size, dtype=np.float64)
        if idx.size == 0:
            return out
        L = host_lib()
        if self.kind == "loguniform":
            L.gen_sample_loguniform(self.seed, self.stream, _ptr(idx), idx.size, self.a, self.w,
                                    _ptr(out))
        elif self.kind == "copies":
            t = np.ascontiguousarray(table, dtype=np.float64)
            L.gen_sample_copies(self.seed, _ptr(idx), idx.size, self.a, self.w, _ptr(t), t.size,
                                self.copy_every, _ptr(out))
        elif self.kind == "walk":
            if idx.size > 1 and np.any(np.diff(idx) < 0):
                raise ValueError("walk sampling needs sorted indices")
            L.gen_sample_walk(self.seed, _ptr(idx), idx.size, self.x0, self.c, self.lo, self.hi,
                              _ptr(out))
        else:
            raise ValueError(self.kind)
        return out

    # ---------- device (torch tensors; torch is plumbing only) ----------
    def device_fill(self, out, offset: int, table_dev=None, stream=None) -> None:
        import torch
        assert out.dtype == torch.float64 and out.is_cuda and out.is_contiguous()
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        L = dev_lib()
        count = out.numel()
        if self.kind == "loguniform":
            rc = L.gen_dev_fill_loguniform(self.seed, self.stream, offset, count, self.a, self.w,
                                           out.data_ptr(), st)
        elif self.kind == "copies":
            rc = L.gen_dev_fill_copies(self.seed, offset, count, self.a, self.w,
                                       table_dev.data_ptr(), table_dev.numel(), self.copy_every,
                                       out.data_ptr(), st)
        elif self.kind == "walk":
            rc = L.gen_dev_fill_walk(self.seed, offset, count, self.x0, self.c, self.lo, self.hi,
                                     out.data_ptr(), st)
        else:
            raise ValueError(self.kind)
        if rc != 0:
            raise RuntimeError(f"datagen device fill failed: cudaError {rc}")


def loguniform_over(table: np.ndarray, seed: int, stream: int = 0) -> TargetSpec:
    a = math.log10(float(table[0]))
    b = math.log10(float(table[-1]))
    return TargetSpec("loguniform", seed, stream, a=a, w=b - a)


@dataclass
class Workload:
    name: str
    count: int
    table: np.ndarray | None = None
    targets: TargetSpec | None = None
    # 2-D (cfg4)
    rho: np.ndarray | None = None
    T: np.ndarray | None = None
    P: np.ndarray | None = None
    rho_targets: TargetSpec | None = None
    T_targets: TargetSpec | None = None
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def is_2d(self) -> bool:
        return self.P is not None


def workload(name: str, count: int | None = None) -> Workload:
    """BASELINE.json configs[0..4] as cfg1..cfg5 (+ 'paper': the paper-shaped run,
    n=110 over [3e-6,5.4e4], m=5e6 log-uniform over 1e-10..1e10, P:224/P:243/P:290)."""
    if name == "cfg1":
        X = table_cfg1(0)
        spec = TargetSpec("copies", 0, a=-4.2, w=8.4, copy_every=100)
        return Workload(name, count or 100_000, X, spec,
                        note="n=64 table, 1e5 log-uniform targets over [1e-4.2,1e4.2] + 1% exact copies")
    if name == "cfg2":
        X = table_cfg2(1)
        return Workload(name, count or (1 << 27), X, loguniform_over(X, 1),
                        note="n=300 SESAME-density-like table, 2^27 log-uniform targets")
    if name == "cfg3":
        X = table_cfg3(2)
        x0 = float(np.random.default_rng(2).uniform(0.0, 8.0))
        sigma = 0.01  # decades per step
        c = sigma * math.sqrt(3.0) / 2.0 ** 32
        spec = TargetSpec("walk", 2, x0=x0, c=c, lo=0.0, hi=8.0)
        return Workload(name, count or (1 << 30), X, spec,
                        note="n=1000 table over [1,1e8], 2^30 reflected random-walk targets (log10 step sd 0.01)")
    if name == "cfg4":
        rho, T, P = grid_cfg4(3)
        return Workload(name, count or (1 << 28), rho=rho, T=T, P=P,
                        rho_targets=TargetSpec("loguniform", 3, 0, a=-6.0, w=9.0),
                        T_targets=TargetSpec("loguniform", 3, 1, a=0.0, w=8.0),
                        note="200x100 density x temperature grid, 2^28 log-uniform (rho,T) pairs")
    if name == "cfg5":
        X = table_cfg5(4)
        return Workload(name, count or (8 << 30), X, loguniform_over(X, 4),
                        note="n=4096 clustered table, 8*2^30 log-uniform targets")
    if name == "paper":
        X = table_paper_exemplar()
        return Workload(name, count or 5_000_000, X,
                        TargetSpec("loguniform", 5, a=-10.0, w=20.0),
                        note="paper-shaped: n=110 over [3e-6,5.4e4], 5e6 log-uniform over 1e-10..1e10")
    if name == "big2d":
        rho, T, P = grid_big2d(7)
        return Workload(name, count or (1 << 28), rho=rho, T=T, P=P,
                        rho_targets=TargetSpec("loguniform", 7, 0, a=-6.0, w=9.0),
                        T_targets=TargetSpec("loguniform", 7, 1, a=0.0, w=8.0),
                        note="1000x800 grid in device memory (larger than shared memory), "
                             "2^28 log-uniform (rho,T) pairs")
    if name == "big":
        X = table_big(6)
        return Workload(name, count or (1 << 27), X, loguniform_over(X, 6),
                        note="n=2^20 table (beyond shared memory: smem sample table + L2-resident packed nodes), "
                             "2^27 log-uniform targets")
    raise KeyError(name)


WORKLOADS = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "paper", "big", "big2d")
