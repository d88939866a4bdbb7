"""measure -- roofline ceilings measured on the box (harness code for bench.py).

Not the product path and none of the method's arithmetic: trivial kernels that
move the same bytes as the search (probes.cu), timed with CUDA events on the
stream they are launched on.

  stream_ceiling_1d(Y, out)  best GB/s of a read-fp64 / write-int32 stream
                             (12 B per unit, the 1-D algorithmic mix)
  stream_ceiling_2d(...)     best GB/s of the 2-D mix (16 B in, 16 B out per pair)
  l2_gather_ceiling(bytes)   random 32-B sector gathers from an L2-resident
                             buffer with the tiered kernel's load instruction
  interp_mix_ceiling(...)    the shared-memory grid interpolation mix (2-D stream +
                             record and corner reads from shared memory)
  stream_gather_ceiling(Y, out, bytes)
                             the packed-table mix: the 1-D stream plus one
                             random 32-B sector gather per unit (same buffers)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "lib", "libeosmeasure.so")
SRC = os.path.join(_HERE, "probes.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_I = ctypes.c_int


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(SRC) > os.path.getmtime(LIB):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        subprocess.check_call([NVCC, *ARCH, "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
                               "-cudart", "static", "-o", LIB, SRC])
    return LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.probe_stream.argtypes = [_P, _P, _I64, _I, _P]
        L.probe_stream2d.argtypes = [_P, _P, _P, _P, _P, _I64, _P]
        L.probe_fill.argtypes = [_P, _U64, _P]
        L.probe_gather.argtypes = [_P, _U64, _I, _I, _P, _P]
        L.probe_gather_line.argtypes = [_P, _U64, _I, _I, _P, _P]
        L.probe_stream_gather.argtypes = [_P, _P, _I64, _P, _U64, _I, _P]
        L.probe_interp_mix.argtypes = [_P, _P, _P, _P, _P, _I64, _I, _I, _P]
        L.probe_interp_gg_mix.argtypes = [_P, _P, _P, _P, _P, _I64, _P, _I, _I, _I, _P]
        for f in (L.probe_stream, L.probe_stream2d, L.probe_fill, L.probe_gather, L.probe_gather_line,
                  L.probe_stream_variants, L.probe_sms, L.probe_stream_gather,
                  L.probe_stream_gather_variants, L.probe_interp_mix, L.probe_interp_gg_mix):
            f.restype = _I
        _lib = L
    return _lib


def _check(code: int, what: str):
    if code != 0:
        raise RuntimeError(f"{what}: cudaError {code}")


def _time(fn, reps: int, stream) -> float:
    """Mean ms per call of fn() over `reps` calls, CUDA events on `stream`."""
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def stream_ceiling_1d(Y, out, reps: int = 5) -> dict:
    """Best-of-shapes GB/s of the 1-D same-mix stream over the bench's own buffers
    (Y fp64[n] read, out int32[n] written; 12 B per unit)."""
    import torch
    L = lib()
    n = Y.numel() - (Y.numel() & 1)
    st = torch.cuda.current_stream()
    res = {}
    for v in range(L.probe_stream_variants()):
        ms = _time(lambda: _check(L.probe_stream(Y.data_ptr(), out.data_ptr(), n, v, st.cuda_stream),
                                  "probe_stream"), reps, st)
        res[v] = 12 * n / (ms * 1e-3) / 1e9
    best = max(res, key=res.get)
    return {"gbs": round(res[best], 1), "variant": best,
            "all_gbs": {str(k): round(v, 1) for k, v in res.items()},
            "what": "read fp64 + write int32 per unit (12 B), trivial kernel, best of "
                    f"{len(res)} launch shapes, {reps} launches each, same buffers as the bench"}


def stream_ceiling_2d(rho, T, P, iR, iT, reps: int = 5) -> dict:
    import torch
    L = lib()
    m = rho.numel() - (rho.numel() & 1)
    st = torch.cuda.current_stream()
    ms = _time(lambda: _check(L.probe_stream2d(rho.data_ptr(), T.data_ptr(), P.data_ptr(),
                                               iR.data_ptr(), iT.data_ptr(), m, st.cuda_stream),
                              "probe_stream2d"), reps, st)
    return {"gbs": round(32 * m / (ms * 1e-3) / 1e9, 1),
            "what": "read 2 fp64 + write fp64 + 2 int32 per pair (32 B), trivial kernel, "
                    f"{reps} launches, same buffers as the bench"}


def l2_gather_ceiling(buffer_bytes: int, rounds: int = 64, reps: int = 5) -> dict:
    """Random 32-B sector gathers (ld.global.nc.L1::no_allocate.v8.u32) from an
    L2-resident buffer of `buffer_bytes` (rounded down to a power of two of sectors),
    1024 threads x SMs, 1..8 independent chains per thread; best sectors/s."""
    import torch
    L = lib()
    sectors = 1
    while 2 * sectors * 32 <= buffer_bytes:
        sectors *= 2
    buf = torch.empty(8 * sectors, dtype=torch.int32, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    _check(L.probe_fill(buf.data_ptr(), 8 * sectors, st.cuda_stream), "probe_fill")
    nsm = L.probe_sms()
    res = {}
    for g in (1, 2, 4, 8):
        ms = _time(lambda: _check(L.probe_gather(buf.data_ptr(), sectors, g, rounds, sink.data_ptr(),
                                                 st.cuda_stream), "probe_gather"), reps, st)
        loads = nsm * 1024 * g * rounds
        res[g] = loads / (ms * 1e-3)
    best = max(res, key=res.get)
    return {"sectors_per_s": res[best], "gbs_sectors": round(32 * res[best] / 1e9, 1),
            "chains": best, "buffer_bytes": 32 * sectors,
            "all_gsectors_per_s": {str(k): round(v / 1e9, 2) for k, v in res.items()},
            "what": f"random 32-B sector gathers, {nsm} SMs x 1024 threads x chains, {rounds} "
                    "dependent rounds, ld.global.nc.L1::no_allocate.v8.u32"}


def l2_line_gather_ceiling(buffer_bytes: int, rounds: int = 64, reps: int = 5) -> dict:
    """Random 128-B line gathers where 4 lanes load the 4 sectors of one line with one
    instruction (measure/probes.cu k_gather_line); best lines/s over 1..8 chains."""
    import torch
    L = lib()
    lines = 1
    while 2 * lines * 128 <= buffer_bytes:
        lines *= 2
    buf = torch.empty(32 * lines, dtype=torch.int32, device="cuda")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    _check(L.probe_fill(buf.data_ptr(), 32 * lines, st.cuda_stream), "probe_fill")
    nsm = L.probe_sms()
    res = {}
    for g in (1, 2, 4, 8):
        ms = _time(lambda: _check(L.probe_gather_line(buf.data_ptr(), lines, g, rounds,
                                                      sink.data_ptr(), st.cuda_stream),
                                  "probe_gather_line"), reps, st)
        res[g] = nsm * 1024 // 4 * g * rounds / (ms * 1e-3)
    best = max(res, key=res.get)
    return {"lines_per_s": res[best], "chains": best, "buffer_bytes": 128 * lines,
            "all_glines_per_s": {str(k): round(v / 1e9, 2) for k, v in res.items()}}


def stream_gather_ceiling(Y, out, buffer_bytes: int, reps: int = 5) -> dict:
    """Best-of-shapes units/s of the packed-table same mix over the bench's own buffers:
    read fp64 Y, gather one random 32-B sector per unit from an L2-resident buffer of
    `buffer_bytes` (rounded down to a power of two of sectors), write int32 out."""
    import torch
    L = lib()
    sectors = 1
    while 2 * sectors * 32 <= buffer_bytes:
        sectors *= 2
    buf = torch.empty(8 * sectors, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    _check(L.probe_fill(buf.data_ptr(), 8 * sectors, st.cuda_stream), "probe_fill")
    n = Y.numel() - (Y.numel() & 1)
    res = {}
    for v in range(L.probe_stream_gather_variants()):
        ms = _time(lambda: _check(L.probe_stream_gather(Y.data_ptr(), out.data_ptr(), n, buf.data_ptr(),
                                                        sectors, v, st.cuda_stream),
                                  "probe_stream_gather"), reps, st)
        res[v] = n / (ms * 1e-3)
    best = max(res, key=res.get)
    return {"units_per_s": res[best], "variant": best, "buffer_bytes": 32 * sectors,
            "all_gunits_per_s": {str(k): round(v / 1e9, 2) for k, v in res.items()},
            "what": "read fp64 + one random 32-B sector gather (ld.global.nc.L1::no_allocate.v8.u32, "
                    "L2-resident buffer) + write int32 per unit, trivial kernel, best of "
                    f"{len(res)} launch shapes, {reps} launches each, same buffers as the bench"}


def interp_mix_ceiling(rho, T, P, iR, iT, nR: int, nT: int, reps: int = 5) -> dict:
    """Pairs/s of the shared-memory interpolation mix (measure/probes.cu k_interp_mix) on
    the bench's own buffers with an nR x nT grid: the ceiling of interp2d_kernel's
    L1TEX data-pipe traffic (its shared-memory reads plus the 2-D stream)."""
    import torch
    L = lib()
    m = rho.numel() - rho.numel() % 2048
    st = torch.cuda.current_stream()
    ms = _time(lambda: _check(L.probe_interp_mix(rho.data_ptr(), T.data_ptr(), P.data_ptr(), iR.data_ptr(),
                                                 iT.data_ptr(), m, nR, nT, st.cuda_stream),
                              "probe_interp_mix"), reps, st)
    return {"units_per_s": m / (ms * 1e-3), "grid": [nR, nT],
            "what": "2-D stream + per pair 2 bank-pinned 16-B record reads and 4 random 8-B corner "
                    "reads from an nR x nT fp64 grid in shared memory, no search and no "
                    f"interpolation arithmetic; interp2d_kernel's launch shape; {reps} launches"}


def interp_gg_mix_ceiling(rho, T, P, iR, iT, nR: int, nT: int, reps: int = 5) -> dict:
    """Pairs/s of the device-memory-grid interpolation mix (measure/probes.cu
    k_interp_gg_mix) on the bench's own buffers: the 2-D stream plus one 32-B cell-quad
    gather per pair from (nR-1) x (nT-1) quads in device memory (L2-resident) and the
    bank-pinned record reads (as many copies, up to 8, as fit in shared memory): the
    same-mix ceiling of interp2d_kernel with a grid in device memory."""
    import torch
    L = lib()
    m = rho.numel() - rho.numel() % 2048
    st = torch.cuda.current_stream()
    quads = torch.ones(4 * (nR - 1) * (nT - 1), dtype=torch.float64, device=rho.device)
    csh = 3
    while csh > 0 and 16 * ((nR + nT) << csh) > 200 * 1024:
        csh -= 1
    ms = _time(lambda: _check(L.probe_interp_gg_mix(rho.data_ptr(), T.data_ptr(), P.data_ptr(),
                                                    iR.data_ptr(), iT.data_ptr(), m, quads.data_ptr(),
                                                    nR, nT, csh, st.cuda_stream),
                              "probe_interp_gg_mix"), reps, st)
    del quads
    return {"units_per_s": m / (ms * 1e-3), "grid": [nR, nT], "record_copies": 1 << csh,
            "quad_bytes": 32 * (nR - 1) * (nT - 1),
            "what": "2-D stream + per pair one random 32-B cell-quad gather from device memory "
                    "(L2-resident) and 2 bank-pinned 16-B record reads from shared memory, no "
                    f"search and no interpolation arithmetic; interp2d_kernel's launch shape; "
                    f"{reps} launches"}
