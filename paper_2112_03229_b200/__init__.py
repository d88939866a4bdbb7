"""paper_2112_03229_b200 -- B200-native batched lower-bound search + EOS interpolation.

Thin Python binding (argument marshalling only) over the C ABI of
include/eossearch.h, implemented by lib/libeossearch.so (sm_100a kernels).
Every step of the hot path runs in that library; there is no Python or CPU
fallback: if the library is missing or cannot be loaded, importing the
binding's functions raises.

PyTorch is used only as the device-memory / stream provider: tensors are
passed as raw pointers with `torch.cuda.current_stream().cuda_stream`.

Paper: arXiv 2112.03229: lower-bound contract P:54, exponent hash
P:211-213, EOSPAC interpolation P:14/P:41.  Readings R<n>: DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import CHECKED_LIB as _CHECKED_LIB_PATH
from ._build import LIB as _LIB_PATH

__all__ = [
    "EosError", "Table", "Grid2D", "TableInfo", "plan_table", "load_library", "launch_count",
    "eos_search_create", "eos_search_create_ex", "eos_search", "eos_search_ex", "eos_search_host",
    "eos_search_destroy", "eos_table_info", "eos_plan_table", "eos_grid2d_create", "eos_interp2d",
    "eos_interp2d_host", "eos_grid2d_destroy", "eos_grid2d_info", "eos_status_str", "EOS_K_AUTO",
    "EOS_MAX_TABLE", "EOS_MAX_K", "EXPORTED_SYMBOLS", "EOS_HASH_AUTO", "EOS_HASH_EXPONENT",
    "EOS_HASH_LOG", "eos_plan_table_hash", "eos_search_create_hash", "eos_interp2d_ex",
    "eos_search_direct", "search_direct", "eos_grid2d_create_ex", "EOS_GRID_LINEAR",
    "EOS_GRID_LOGLOG", "EOS_MAX_TABLE_TIERED", "EOS_LEVELS_AUTO", "eos_search_create_levels",
    "eos_plan_table_levels", "plan_table_levels", "EOS_GRID_GLOBAL", "EOS_MAX_GRID_CELLS",
    "EOS_GRID_EXACT", "ABI_VERSION", "EOS_LEVELS_PACKED", "EOS_GRID_DIRECTORY",
    "EOS_LEVELS_PACKED_DEPTH",
]

EOS_MAX_TABLE = 16384
EOS_MAX_TABLE_TIERED = 1 << 29
EOS_LEVELS_AUTO = -1
EOS_LEVELS_PACKED = -2


def EOS_LEVELS_PACKED_DEPTH(d: int) -> int:
    """eos_search_create_levels: packed nodes with exactly d = 1..4 levels."""
    return -16 - d
EOS_MAX_K = 19
EOS_K_AUTO = -1
EOS_HASH_AUTO, EOS_HASH_EXPONENT, EOS_HASH_LOG = 0, 1, 2
EOS_GRID_LINEAR, EOS_GRID_LOGLOG, EOS_GRID_GLOBAL, EOS_GRID_EXACT, EOS_GRID_DIRECTORY = 0, 1, 2, 4, 8
ABI_VERSION = 5
EOS_MAX_GRID_CELLS = 1 << 28

STATUS = {
    0: "EOS_OK", 1: "EOS_ERR_NULL", 2: "EOS_ERR_SIZE", 3: "EOS_ERR_NONFINITE",
    4: "EOS_ERR_UNSORTED", 5: "EOS_ERR_DEVICE", 6: "EOS_ERR_CUDA", 7: "EOS_ERR_NOMEM",
    8: "EOS_ERR_UNSUPPORTED", 9: "EOS_ERR_ALIAS",
}

# every symbol include/eossearch.h declares
EXPORTED_SYMBOLS = (
    "eos_plan_table", "eos_search_create", "eos_search_create_ex", "eos_search", "eos_search_ex",
    "eos_search_host", "eos_table_info", "eos_search_destroy", "eos_grid2d_create",
    "eos_interp2d", "eos_interp2d_host", "eos_grid2d_info", "eos_grid2d_destroy",
    "eos_status_str", "eos_abi_version", "eos_launch_count", "eos_plan_table_hash",
    "eos_search_create_hash", "eos_interp2d_ex", "eos_search_direct", "eos_grid2d_create_ex",
    "eos_search_create_levels", "eos_plan_table_levels",
)


class EosError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        self.name = STATUS.get(code, f"status {code}")
        super().__init__(f"{where}: {self.name} ({eos_status_str(code)})")


class TableInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("key_mode", ctypes.c_int32), ("k", ctypes.c_int32),
                ("bins", ctypes.c_int32), ("max_occ", ctypes.c_int32), ("steps", ctypes.c_int32),
                ("base", ctypes.c_int32), ("image_bytes", ctypes.c_int64),
                ("device", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32),
                ("hash_kind", ctypes.c_int32), ("hash_mult", ctypes.c_uint32),
                ("levels", ctypes.c_int32), ("node_width", ctypes.c_int32), ("top_n", ctypes.c_int64),
                ("level_bytes", ctypes.c_int64), ("dir_entry_bytes", ctypes.c_int32),
                ("fast_steps", ctypes.c_int32), ("rare_steps", ctypes.c_int32),
                ("ring_stages", ctypes.c_int32), ("cell_map", ctypes.c_int32)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_ST = ctypes.c_int


def load_library():
    """Load lib/libeossearch.so (fails loudly: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    # EOS_LIBRARY=checked selects the bounds-checked debug build (tests only);
    # EOS_LIBRARY=exp an A/B tuning build (_build.py --exp -D...)
    which = os.environ.get("EOS_LIBRARY")
    path = _CHECKED_LIB_PATH if which == "checked" else (
        os.path.join(os.path.dirname(_LIB_PATH), f"libeossearch_{which}.so")  # exp, exp2, ...
        if which and which.startswith("exp") and which.isalnum() else _LIB_PATH)
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() "
                          "(python -m paper_2112_03229_b200._build); there is no CPU fallback")
    L = ctypes.CDLL(path)
    sig = {
        "eos_plan_table": [_P, _I64, _I32, _P, _P, _I64],
        "eos_plan_table_hash": [_P, _I64, _I32, _I64, _P, _P, _I64],
        "eos_search_create_hash": [_P, _I64, _I32, _I64, _P],
        "eos_search_create_levels": [_P, _I64, _I32, _I32, _I64, _P],
        "eos_plan_table_levels": [_P, _I64, _I32, _I32, _I64, _P],
        "eos_search_create": [_P, _I64, _P],
        "eos_search_create_ex": [_P, _I64, _I32, _P],
        "eos_search": [_P, _P, _I64, _P, _P],
        "eos_search_ex": [_P, _P, _I64, _P, _I64, _P, _P],
        "eos_search_host": [_P, _P, _I64, _P, _P],
        "eos_table_info": [_P, _P],
        "eos_search_destroy": [_P],
        "eos_grid2d_create": [_P, _I64, _P, _I64, _P, _P],
        "eos_grid2d_create_ex": [_P, _I64, _P, _I64, _P, _I32, _P],
        "eos_interp2d": [_P, _P, _P, _I64, _P, _P, _P, _P],
        "eos_interp2d_ex": [_P, _P, _P, _I64, _P, _P, _P, _P, _P, _P],
        "eos_search_direct": [_P, _I64, _P, _I64, _P, _P, _P],
        "eos_interp2d_host": [_P, _P, _P, _I64, _P, _P, _P, _P],
        "eos_grid2d_info": [_P, _P, _P],
        "eos_grid2d_destroy": [_P],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = _ST
    L.eos_status_str.argtypes = [_ST]
    L.eos_status_str.restype = ctypes.c_char_p
    L.eos_abi_version.restype = _I32
    L.eos_launch_count.restype = _I64
    if L.eos_abi_version() != ABI_VERSION:
        raise ImportError(f"{path}: ABI version {L.eos_abi_version()} != {ABI_VERSION} (stale build)")
    _lib = L
    return L


def _check(code: int, where: str):
    if code != 0:
        raise EosError(code, where)


def eos_status_str(code: int) -> str:
    return load_library().eos_status_str(code).decode()


def launch_count() -> int:
    """Kernel launches issued by libeossearch.so in this process."""
    return int(load_library().eos_launch_count())


def _f64_host(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _host(a, dtype, what: str, n: int | None = None):
    """A host buffer passed to the C ABI: a C-contiguous numpy array (or CPU tensor) of
    exactly `dtype`, with at least n elements.  Anything else raises: the library
    reads / writes n elements through the raw pointer."""
    import torch
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise TypeError(f"{what} must be a host array (got a CUDA tensor)")
        a = a.numpy()
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{what} must be a numpy array")
    if a.dtype != np.dtype(dtype):
        raise TypeError(f"{what} must be {np.dtype(dtype).name} (got {a.dtype.name})")
    if not a.flags.c_contiguous:
        raise ValueError(f"{what} must be C-contiguous")
    if n is not None and a.size < n:
        raise ValueError(f"{what} has {a.size} elements, needs {n}")
    return a


def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dev(t, dtype_name: str, what: str, n: int | None = None):
    """A device buffer passed to the C ABI: a contiguous CUDA tensor of exactly the
    dtype, with n elements if n is given (the kernels write exactly n)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA tensor")
    if t.dtype != getattr(torch, dtype_name):
        raise TypeError(f"{what} must be torch.{dtype_name}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    if n is not None and t.numel() != n:
        raise ValueError(f"{what} has {t.numel()} elements, needs {n}")
    return t


# ----------------------------------------------------------- raw C-ABI -----
def _hash_args(k, log_bins):
    if log_bins is not None:
        if k not in (None, EOS_K_AUTO):
            raise ValueError("give k (exponent hash) or log_bins (logarithm hash), not both")
        return EOS_HASH_LOG, int(log_bins)
    if k is None or k == EOS_K_AUTO:
        return EOS_HASH_AUTO, 0
    if k < 0:
        return EOS_HASH_EXPONENT, -1   # rejected by the library (EOS_ERR_UNSUPPORTED)
    return EOS_HASH_EXPONENT, int(k)


def eos_plan_table_hash(table, kind: int, param: int, with_directory: bool = True):
    """Host-only plan (no device): (TableInfo, directory u32[bins] | None)."""
    L = load_library()
    X = _f64_host(table)
    info = TableInfo()
    _check(L.eos_plan_table_hash(X.ctypes.data, X.size, kind, param, ctypes.byref(info), None, 0),
           "eos_plan_table")
    d = None
    if with_directory:
        d = np.empty(info.bins, dtype=np.uint32)
        _check(L.eos_plan_table_hash(X.ctypes.data, X.size, kind, param, ctypes.byref(info),
                                     d.ctypes.data, d.size), "eos_plan_table")
    return info, d


def eos_plan_table(table, k: int | None = EOS_K_AUTO, with_directory: bool = True,
                   log_bins: int | None = None):
    """Host-only plan: k = exponent-hash mantissa bits (None/-1 = automatic choice of
    any hash), or log_bins = |H| of the logarithm hash."""
    kind, param = _hash_args(k, log_bins)
    return eos_plan_table_hash(table, kind, param, with_directory)


plan_table = eos_plan_table


def eos_plan_table_levels(table, levels: int = EOS_LEVELS_AUTO, k: int | None = EOS_K_AUTO,
                          log_bins: int | None = None) -> TableInfo:
    """Host-only plan of a (possibly tiered) table: levels = D (-1 = automatic, -2 =
    packed)."""
    X = _f64_host(table)
    info = TableInfo()
    kind, param = _hash_args(k, log_bins)
    _check(load_library().eos_plan_table_levels(X.ctypes.data, X.size, levels, kind, param,
                                                ctypes.byref(info)), "eos_plan_table_levels")
    return info


plan_table_levels = eos_plan_table_levels


def eos_search_create(table) -> int:
    return eos_search_create_ex(table, EOS_K_AUTO)


def eos_search_create_ex(table, k: int = EOS_K_AUTO) -> int:
    L = load_library()
    X = _f64_host(table)
    h = ctypes.c_void_p()
    _check(L.eos_search_create_ex(X.ctypes.data, X.size, k, ctypes.byref(h)), "eos_search_create")
    return h.value


def eos_search_create_hash(table, kind: int, param: int) -> int:
    L = load_library()
    X = _f64_host(table)
    h = ctypes.c_void_p()
    _check(L.eos_search_create_hash(X.ctypes.data, X.size, kind, param, ctypes.byref(h)),
           "eos_search_create")
    return h.value


def eos_search_create_levels(table, levels: int, kind: int, param: int) -> int:
    L = load_library()
    X = _f64_host(table)
    h = ctypes.c_void_p()
    _check(L.eos_search_create_levels(X.ctypes.data, X.size, levels, kind, param, ctypes.byref(h)),
           "eos_search_create_levels")
    return h.value


def eos_search(handle: int, targets_ptr: int, count: int, idx_out_ptr: int, stream: int) -> None:
    _check(load_library().eos_search(handle, targets_ptr, count, idx_out_ptr, stream), "eos_search")


def eos_search_ex(handle, targets_ptr, count, idx_out_ptr, global_offset, counters_ptr, stream):
    _check(load_library().eos_search_ex(handle, targets_ptr, count, idx_out_ptr, global_offset,
                                        counters_ptr, stream), "eos_search_ex")


def eos_search_host(handle, targets_host_ptr, count, idx_out_host_ptr, stream):
    _check(load_library().eos_search_host(handle, targets_host_ptr, count, idx_out_host_ptr, stream),
           "eos_search_host")


def eos_search_direct(table_ptr, n, targets_ptr, count, idx_out_ptr, status_ptr, stream):
    _check(load_library().eos_search_direct(table_ptr, n, targets_ptr, count, idx_out_ptr,
                                            status_ptr, stream), "eos_search_direct")


def search_direct(table, targets, out=None, status=None, stream=None):
    """Zero-setup search: `table` is a CUDA float64 tensor (n <= 4096, sorted), no handle
    is created; the directory is built on the device by every CTA (f2)."""
    import torch
    _dev(table, "float64", "table")
    _dev(targets, "float64", "targets")
    if out is None:
        out = torch.empty(targets.numel(), dtype=torch.int32, device=targets.device)
    _dev(out, "int32", "out", targets.numel())
    sp = None
    if status is not None:
        _dev(status, "int32", "status", 1)
        sp = status.data_ptr()
    eos_search_direct(table.data_ptr(), table.numel(), targets.data_ptr(), targets.numel(),
                      out.data_ptr(), sp, _stream_ptr(stream))
    return out


def eos_table_info(handle) -> TableInfo:
    info = TableInfo()
    _check(load_library().eos_table_info(handle, ctypes.byref(info)), "eos_table_info")
    return info


def eos_search_destroy(handle) -> None:
    _check(load_library().eos_search_destroy(handle), "eos_search_destroy")


def eos_grid2d_create(rho, T, P, flags: int = EOS_GRID_LINEAR) -> int:
    L = load_library()
    r, t, p = _f64_host(rho), _f64_host(T), _f64_host(P)
    if p.size != r.size * t.size:
        raise ValueError("P must have n_rho * n_T values (row-major, T fastest)")
    h = ctypes.c_void_p()
    _check(L.eos_grid2d_create_ex(r.ctypes.data, r.size, t.ctypes.data, t.size, p.ctypes.data,
                                  flags, ctypes.byref(h)), "eos_grid2d_create")
    return h.value


eos_grid2d_create_ex = eos_grid2d_create


def eos_interp2d(handle, rho_ptr, T_ptr, count, P_ptr, iR_ptr, iT_ptr, stream):
    _check(load_library().eos_interp2d(handle, rho_ptr, T_ptr, count, P_ptr, iR_ptr, iT_ptr, stream),
           "eos_interp2d")


def eos_interp2d_ex(handle, rho_ptr, T_ptr, count, P_ptr, iR_ptr, iT_ptr, dPr_ptr, dPt_ptr, stream):
    _check(load_library().eos_interp2d_ex(handle, rho_ptr, T_ptr, count, P_ptr, iR_ptr, iT_ptr,
                                          dPr_ptr, dPt_ptr, stream), "eos_interp2d_ex")


def eos_interp2d_host(handle, rho_ptr, T_ptr, count, P_ptr, iR_ptr, iT_ptr, stream):
    _check(load_library().eos_interp2d_host(handle, rho_ptr, T_ptr, count, P_ptr, iR_ptr, iT_ptr,
                                            stream), "eos_interp2d_host")


def eos_grid2d_info(handle):
    a, b = TableInfo(), TableInfo()
    _check(load_library().eos_grid2d_info(handle, ctypes.byref(a), ctypes.byref(b)), "eos_grid2d_info")
    return a, b


def eos_grid2d_destroy(handle) -> None:
    _check(load_library().eos_grid2d_destroy(handle), "eos_grid2d_destroy")


# ------------------------------------------------------------ objects ------
class Table:
    """A search table bound to the current CUDA device (eos_search_create)."""

    def __init__(self, table, k: int | None = None, log_bins: int | None = None,
                 levels: int = EOS_LEVELS_AUTO):
        """k: exponent hash with k mantissa bits; log_bins: logarithm hash with |H| bins;
        neither: the automatic choice.  levels: D 8-ary global levels
        under a shared-memory sample table (tables above EOS_MAX_TABLE entries need
        D >= 1), EOS_LEVELS_PACKED (packed 16-bit residual nodes, the fewest levels that
        fit), EOS_LEVELS_PACKED_DEPTH(d) (exactly d levels of them) or
        EOS_LEVELS_AUTO.  Results never depend on any of them."""
        self.X = _f64_host(table)
        self._h = eos_search_create_levels(self.X, levels, *_hash_args(k, log_bins))
        self.info = eos_table_info(self._h)

    @property
    def handle(self) -> int:
        return self._h

    def search(self, targets, out=None, stream=None, counters=None, global_offset: int = 0):
        """int32 indices of the last table entry <= each target."""
        import torch
        _dev(targets, "float64", "targets")
        if out is None:
            out = torch.empty(targets.numel(), dtype=torch.int32, device=targets.device)
        _dev(out, "int32", "out", targets.numel())
        cptr = None
        if counters is not None:
            _dev(counters, "int64", "counters")
            if counters.numel() < 8:
                raise ValueError("counters needs 8 entries")
            cptr = counters.data_ptr()
        eos_search_ex(self._h, targets.data_ptr(), targets.numel(), out.data_ptr(), global_offset,
                      cptr, _stream_ptr(stream))
        return out

    def search_host(self, targets: np.ndarray, out: np.ndarray | None = None, stream=None,
                    sync: bool = True) -> np.ndarray:
        """End-to-end from host buffers (eos_search_host); pinned memory recommended."""
        import torch
        targets = _host(targets, np.float64, "targets")
        if out is None:
            out = np.empty(targets.size, dtype=np.int32)
        out_np = _host(out, np.int32, "out", targets.size)
        out_ptr = out_np.ctypes.data
        sp = _stream_ptr(stream)
        eos_search_host(self._h, targets.ctypes.data, targets.size, out_ptr, sp)
        if sync:
            torch.cuda.current_stream().synchronize() if stream is None else torch.cuda.synchronize()
        return out

    def close(self):
        if getattr(self, "_h", None):
            eos_search_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class Grid2D:
    """EOSPAC-style 2-D table (density x temperature) for eos_interp2d."""

    def __init__(self, rho, T, P, loglog: bool = False, global_grid: bool = False,
                 exact: bool = False, directory: bool = False):
        """loglog=True: interpolate ln P bilinearly in (ln rho, ln T) (EOS_GRID_LOGLOG, R24).
        global_grid=True: keep P in device memory even if it fits in shared memory
        (EOS_GRID_GLOBAL; grids too large for shared memory always are).
        exact=True: weights with the fp64 divide, in the formula's order (EOS_GRID_EXACT).
        directory=True: cells through the axis directories, not fitted cell maps
        (EOS_GRID_DIRECTORY; same results)."""
        self.rho, self.T = _f64_host(rho).copy(), _f64_host(T).copy()
        self.P = _f64_host(P).reshape(self.rho.size, self.T.size).copy()
        self.loglog = loglog
        flags = (EOS_GRID_LOGLOG if loglog else EOS_GRID_LINEAR) | (EOS_GRID_GLOBAL if global_grid else 0) \
            | (EOS_GRID_EXACT if exact else 0) | (EOS_GRID_DIRECTORY if directory else 0)
        self._h = eos_grid2d_create(self.rho, self.T, self.P, flags)
        self.rho_info, self.T_info = eos_grid2d_info(self._h)

    @property
    def handle(self) -> int:
        return self._h

    def interp(self, rho, T, P_out=None, irho_out=None, iT_out=None, brackets: bool = True,
               stream=None, derivatives: bool = False):
        """(P, irho, iT) -- or (P, irho, iT, dP/drho, dP/dT) with derivatives=True."""
        import torch
        _dev(rho, "float64", "rho")
        _dev(T, "float64", "T")
        m = rho.numel()
        if T.numel() != m:
            raise ValueError("rho and T must have the same length")
        if P_out is None:
            P_out = torch.empty(m, dtype=torch.float64, device=rho.device)
        if brackets and irho_out is None:
            irho_out = torch.empty(m, dtype=torch.int32, device=rho.device)
        if brackets and iT_out is None:
            iT_out = torch.empty(m, dtype=torch.int32, device=rho.device)
        _dev(P_out, "float64", "P_out", m)
        if irho_out is not None:
            _dev(irho_out, "int32", "irho_out", m)
        if iT_out is not None:
            _dev(iT_out, "int32", "iT_out", m)
        dr = dt = None
        if derivatives:
            dr = torch.empty(m, dtype=torch.float64, device=rho.device)
            dt = torch.empty(m, dtype=torch.float64, device=rho.device)
        eos_interp2d_ex(self._h, rho.data_ptr(), T.data_ptr(), m, P_out.data_ptr(),
                        irho_out.data_ptr() if irho_out is not None else None,
                        iT_out.data_ptr() if iT_out is not None else None,
                        dr.data_ptr() if dr is not None else None,
                        dt.data_ptr() if dt is not None else None, _stream_ptr(stream))
        if derivatives:
            return P_out, irho_out, iT_out, dr, dt
        return P_out, irho_out, iT_out

    def interp_host(self, rho: np.ndarray, T: np.ndarray, P_out=None, irho_out=None, iT_out=None,
                    stream=None, sync: bool = True):
        """End-to-end from host buffers (eos_interp2d_host): float64 rho, T of equal
        length; outputs float64 / int32 host arrays of at least that length."""
        import torch
        rho = _host(rho, np.float64, "rho")
        T = _host(T, np.float64, "T")
        m = rho.size
        if T.size != m:
            raise ValueError("rho and T must have the same length")
        P_out = np.empty(m, np.float64) if P_out is None else P_out
        irho_out = np.empty(m, np.int32) if irho_out is None else irho_out
        iT_out = np.empty(m, np.int32) if iT_out is None else iT_out
        P_np = _host(P_out, np.float64, "P_out", m)
        iR_np = _host(irho_out, np.int32, "irho_out", m)
        iT_np = _host(iT_out, np.int32, "iT_out", m)
        eos_interp2d_host(self._h, rho.ctypes.data, T.ctypes.data, m, P_np.ctypes.data,
                          iR_np.ctypes.data, iT_np.ctypes.data, _stream_ptr(stream))
        if sync:
            torch.cuda.synchronize()
        return P_out, irho_out, iT_out

    def close(self):
        if getattr(self, "_h", None):
            eos_grid2d_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
