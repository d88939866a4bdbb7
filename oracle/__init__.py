"""oracle -- the plain CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  The product path (paper_2112_03229_b200/) never
does, and this module never imports the product path.

The arithmetic lives in eos_oracle.c (plain C, fp64, each function citing the
PAPER.md passage it follows).  This wrapper only marshals numpy arrays and
splits a batch into contiguous chunks over host threads (ctypes releases the
GIL during the C call); the per-element computation is unchanged by that.

Pins: see the header of eos_oracle.c and tests/test_oracle.py.  No function
here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "lib", "liboracle.so")
_SRC = os.path.join(_HERE, "eos_oracle.c")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(_SRC) > os.path.getmtime(LIB):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-fno-fast-math",
                               "-ffp-contract=off", "-o", LIB, _SRC, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, I64 = ctypes.c_void_p, ctypes.c_int64
        L.oracle_lower_bound.argtypes = [P, I64, ctypes.c_double]
        L.oracle_lower_bound.restype = ctypes.c_int32
        L.oracle_search.argtypes = [P, I64, P, I64, P]
        L.oracle_interp2d.argtypes = [P, I64, P, I64, P, P, P, I64, P, P, P]
        L.oracle_counters.argtypes = [P, I64, P, P, I64, I64, P]
        L.oracle_interp2d_deriv.argtypes = [P, I64, P, I64, P, P, P, I64, P, P]
        L.oracle_interp2d_loglog.argtypes = [P, I64, P, I64, P, P, P, I64, P, P, P, P, P]
        L.oracle_mix64.argtypes = [ctypes.c_uint64]
        L.oracle_mix64.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _chunks(m: int, threads: int):
    threads = max(1, min(threads, (m + 65535) // 65536 or 1))
    step = (m + threads - 1) // threads
    return [(s, min(m, s + step)) for s in range(0, m, step)] if m else []


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def lower_bound(X, y: float) -> int:
    X = _f64(X)
    return int(lib().oracle_lower_bound(X.ctypes.data, X.size, float(y)))


def search(X, Y, threads: int | None = None) -> np.ndarray:
    """idx[i] = index of the last X entry <= Y[i]; 0 if none; n-1 above."""
    X, Y = _f64(X), _f64(Y)
    out = np.empty(Y.size, dtype=np.int32)
    L = lib()
    threads = threads or default_threads()

    def run(r):
        s, e = r
        L.oracle_search(X.ctypes.data, X.size, Y.ctypes.data + 8 * s, e - s, out.ctypes.data + 4 * s)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, _chunks(Y.size, threads)))
    return out


def interp2d(R, Tax, G, rho, T, threads: int | None = None):
    """(P, iR, iT): bilinear EOS interpolation on the bracket cells (eos_oracle.c)."""
    R, Tax, G, rho, T = _f64(R), _f64(Tax), _f64(G), _f64(rho), _f64(T)
    assert G.shape == (R.size, Tax.size) and rho.size == T.size
    m = rho.size
    P = np.empty(m, dtype=np.float64)
    iR = np.empty(m, dtype=np.int32)
    iT = np.empty(m, dtype=np.int32)
    L = lib()
    threads = threads or default_threads()

    def run(r):
        s, e = r
        L.oracle_interp2d(R.ctypes.data, R.size, Tax.ctypes.data, Tax.size, G.ctypes.data,
                          rho.ctypes.data + 8 * s, T.ctypes.data + 8 * s, e - s,
                          P.ctypes.data + 8 * s, iR.ctypes.data + 4 * s, iT.ctypes.data + 4 * s)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, _chunks(m, threads)))
    return P, iR, iT


def interp2d_deriv(R, Tax, G, rho, T, threads: int | None = None):
    """(dP/drho, dP/dT) of the bilinear interpolant (eos_oracle.c, reading R23)."""
    R, Tax, G, rho, T = _f64(R), _f64(Tax), _f64(G), _f64(rho), _f64(T)
    assert G.shape == (R.size, Tax.size) and rho.size == T.size
    m = rho.size
    dr = np.empty(m, dtype=np.float64)
    dt = np.empty(m, dtype=np.float64)
    L = lib()
    threads = threads or default_threads()

    def run(r):
        s, e = r
        L.oracle_interp2d_deriv(R.ctypes.data, R.size, Tax.ctypes.data, Tax.size, G.ctypes.data,
                                rho.ctypes.data + 8 * s, T.ctypes.data + 8 * s, e - s,
                                dr.ctypes.data + 8 * s, dt.ctypes.data + 8 * s)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, _chunks(m, threads)))
    return dr, dt


def interp2d_loglog(R, Tax, G, rho, T, threads: int | None = None):
    """(P, iR, iT, dP/drho, dP/dT): log-log bilinear interpolation (eos_oracle.c, R24)."""
    R, Tax, G, rho, T = _f64(R), _f64(Tax), _f64(G), _f64(rho), _f64(T)
    assert G.shape == (R.size, Tax.size) and rho.size == T.size
    m = rho.size
    P, dr, dt = (np.empty(m, dtype=np.float64) for _ in range(3))
    iR = np.empty(m, dtype=np.int32)
    iT = np.empty(m, dtype=np.int32)
    L = lib()
    threads = threads or default_threads()

    def run(r):
        s, e = r
        L.oracle_interp2d_loglog(R.ctypes.data, R.size, Tax.ctypes.data, Tax.size, G.ctypes.data,
                                 rho.ctypes.data + 8 * s, T.ctypes.data + 8 * s, e - s,
                                 P.ctypes.data + 8 * s, iR.ctypes.data + 4 * s,
                                 iT.ctypes.data + 4 * s, dr.ctypes.data + 8 * s,
                                 dt.ctypes.data + 8 * s)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, _chunks(m, threads)))
    return P, iR, iT, dr, dt


def mix64(z: int) -> int:
    """The splitmix64 finalizer of counter c2 (eos_oracle.c oracle_mix64)."""
    return int(lib().oracle_mix64(z & 0xFFFFFFFFFFFFFFFF))


def counters(X, Y, idx, global_offset: int = 0) -> np.ndarray:
    """uint64[8] validation counters of one shard (definitions in eos_oracle.c)."""
    X, Y = _f64(X), _f64(Y)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    c = np.zeros(8, dtype=np.uint64)
    lib().oracle_counters(X.ctypes.data, X.size, Y.ctypes.data, idx.ctypes.data, Y.size,
                          int(global_offset), c.ctypes.data)
    return c
