"""Host-side logic of libeossearch.so, no GPU needed (-m "not gpu").

The library must load and export every symbol include/eossearch.h declares,
and eos_plan_table (validation, bin key, count directory, k choice) is
checked here against independent derivations (math.frexp exponents, brute
recounts, the oracle's answers, the paper's printed bin statistics).
"""
import math
import os
import re

import numpy as np
import pytest

import datagen
import oracle
import paper_2112_03229_b200 as eos
from paper_2112_03229_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    _build.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "eossearch.h")).read()
    return set(re.findall(r"^EOS_API\s+[\w\s\*]+?\b(eos_\w+)\(", src, flags=re.M))


def test_library_loads_and_exports_every_declared_symbol():
    L = eos.load_library()
    declared = header_symbols()
    assert len(declared) >= 16
    assert declared == set(eos.EXPORTED_SYMBOLS)
    for s in declared:
        assert hasattr(L, s), s
    assert L.eos_abi_version() == 5
    assert eos.eos_status_str(0) == "ok"
    assert "sorted" in eos.eos_status_str(4)


def test_table_info_struct_layout_matches_the_header(tmp_path):
    """The ctypes mirror of eos_table_info_t has the C struct's size and field offsets
    (gcc on include/eossearch.h), so eos_*_info never writes past a Python buffer."""
    import ctypes
    import subprocess
    fields = [f for f, _ in eos.TableInfo._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "eossearch.h"\n'
                   "int main(void) {\n"
                   '  printf("%zu\\n", sizeof(eos_table_info_t));\n'
                   + "".join(f'  printf("%zu\\n", offsetof(eos_table_info_t, {f}));\n' for f in fields)
                   + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(_build.ROOT, "include"), "-o", str(exe),
                    str(src)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(eos.TableInfo)
    assert got[1:] == [getattr(eos.TableInfo, f).offset for f in fields]


def test_sm100a_cubin_embedded():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


# ---------------------------------------------------------------- plan -----
def fine_index_frexp(x: float, k: int) -> int:
    """Independent bin index of a positive normal x: e*2^k + floor((m-1)*2^k), x = m*2^e."""
    f, E = math.frexp(x)
    m, e = 2.0 * f, E - 1
    return e * (1 << k) + int(math.floor((m - 1.0) * (1 << k)))


def unpack(d):
    return (d & 0xFFFF).astype(np.int64), (d >> 16).astype(np.int64)


def random_positive_tables(rng, count):
    for t in range(count):
        n = int(rng.integers(1, 400))
        if t % 3 == 0:
            X = 10.0 ** rng.uniform(-8, 8, n)
        elif t % 3 == 1:
            X = 2.0 ** rng.integers(-30, 30, n).astype(np.float64)
        else:
            X = np.round(10.0 ** rng.uniform(0, 1, n), 2)
        yield np.sort(X)


def test_directory_invariants_and_recount():
    rng = np.random.default_rng(0)
    for X in random_positive_tables(rng, 60):
        for k in range(0, 11):
            fi = np.array([fine_index_frexp(x, k) for x in X])
            try:
                info, d = eos.plan_table(X, k)
            except eos.EosError as e:   # directory would not fit in shared memory
                assert e.code == 8 and 8 * X.size + 4 * (fi[-1] - fi[0] + 1) > 200 * 1024
                continue
            lo, occ = unpack(d)
            assert info.bins == d.size and info.k == k and info.key_mode == 0
            assert lo[0] == 0 and lo[-1] + occ[-1] == X.size
            assert np.all(lo[1:] == lo[:-1] + occ[:-1])
            assert info.max_occ == occ.max()
            assert info.steps == math.ceil(math.log2(info.max_occ + 1))
            # recount with the frexp-derived fine index
            assert info.bins == fi[-1] - fi[0] + 1
            cnt = np.bincount(fi - fi[0], minlength=info.bins)
            assert np.array_equal(cnt, occ)


def test_k0_is_the_paper_exponent_hash():
    """k = 0: bins are the binary exponents spanned; bin id = floor(log2 x) - e_min."""
    X = np.sort(10.0 ** np.random.default_rng(1).uniform(-6, 6, 500))
    info, d = eos.plan_table(X, 0)
    e = np.array([math.frexp(x)[1] - 1 for x in X])
    assert np.array_equal(e, np.floor(np.log2(X)).astype(int))
    assert info.bins == e.max() - e.min() + 1
    assert np.array_equal(unpack(d)[1], np.bincount(e - e.min(), minlength=info.bins))


def test_paper_exemplar_bin_statistics():
    """a log-distributed table over 3e-6..5.4e4 spans 'about 34 powers of 2', giving
    '110/34 = 3.235' entries per bin.  The exponent hash (k=0) gives 35 bins here."""
    import datagen
    X = datagen.table_paper_exemplar()
    info, d = eos.plan_table(X, 0)
    assert info.bins in (34, 35)
    assert 3.0 <= X.size / info.bins <= 3.5
    assert info.bins == 35 and abs(X.size / info.bins - 3.14) < 0.01


def _bin_of(y, info, X):
    """bin of target y under mode 0 (test-side restatement, for the bracketing check)."""
    hi = (np.array([y]).view(np.uint64)[0] >> np.uint64(32)) & np.uint64(0x7FFFFFFF)
    kb = int(hi) >> (20 - info.k)
    xlo = X[X > 0][0] if np.any(X > 0) else X[-1]
    base = (int(np.array([xlo]).view(np.uint64)[0] >> np.uint64(32)) & 0x7FFFFFFF) >> (20 - info.k)
    return min(max(kb, base), base + info.bins - 1) - base


def test_directory_brackets_the_oracle_answer():
    """For every in-range target the oracle's count lies inside the target's bin range
    [lo_b, lo_b + occ_b] (SPEC 'Bracketing' property), at every k."""
    import datagen
    for name in ("cfg1", "cfg2", "cfg3", "cfg5"):
        w = datagen.workload(name, count=3000)
        X = w.table
        Y = w.targets.host_fill(0, w.count, X)
        Y = np.concatenate([Y, X, np.nextafter(X, 0), np.nextafter(X, np.inf)])
        ref = oracle.search(X, Y)
        for k in (0, 2, 5, 9):
            info, d = eos.plan_table(X, k)
            lo, occ = unpack(d)
            for y, r in zip(Y, ref):
                if not (y >= X[0]):
                    continue
                b = _bin_of(y, info, X)
                assert lo[b] <= r + 1 <= lo[b] + occ[b], (name, k, y)


def test_auto_k_reaches_short_searches_on_configs():
    import datagen
    chosen = {}
    for name in ("cfg1", "cfg2", "cfg3", "cfg5", "paper"):
        X = datagen.workload(name, count=1).table
        info, _ = eos.plan_table(X)
        chosen[name] = (info.k, info.bins, info.steps, info.image_bytes)
        assert info.image_bytes <= 200 * 1024 or info.k == 0
    assert chosen["cfg2"][2] == 1 and chosen["cfg3"][2] == 1
    assert chosen["cfg5"][2] <= 3
    rho, T, _ = datagen.grid_cfg4()
    for ax in (rho, T):
        assert eos.plan_table(ax)[0].steps == 1


def test_validation_status_codes():
    def code(X, k=eos.EOS_K_AUTO):
        try:
            eos.plan_table(np.asarray(X, dtype=np.float64), k)
            return 0
        except eos.EosError as e:
            return e.code
    assert code([]) == 2
    assert code(np.arange(eos.EOS_MAX_TABLE + 1, dtype=float)) == 2
    assert code(np.arange(eos.EOS_MAX_TABLE, dtype=float)) == 0
    assert code([1.0, np.nan]) == 3
    assert code([1.0, np.inf]) == 3
    assert code([2.0, 1.0]) == 4
    assert code([1.0, 1.0, 1.0]) == 0            # duplicates allowed
    assert code([1.0, 2.0], k=21) == 8
    assert code([1.0, 2.0], k=-2) == 8
    assert code([7.0]) == 0                       # n = 1
    with pytest.raises(eos.EosError) as ei:
        L = eos.load_library()
        X = np.array([1.0, 2.0, 4.0])
        info = eos.TableInfo()
        d = np.zeros(1, np.uint32)
        r = L.eos_plan_table(X.ctypes.data, 3, 0, __import__("ctypes").byref(info), d.ctypes.data, 1)
        eos._check(r, "cap")
    assert ei.value.code == 2


def test_key_modes_and_degenerate_tables():
    info, d = eos.plan_table([-2.0, -0.5, 0.0, 0.5])
    assert info.key_mode == 1
    info, d = eos.plan_table([-0.0, 1.0, 2.0])     # -0.0 canonicalised -> mode 0
    assert info.key_mode == 0
    info, d = eos.plan_table([0.0, 0.0])           # all zeros: one bin
    assert info.bins == 1 and info.max_occ == 2
    info, d = eos.plan_table([0.0, 5e-324, 1e-310, 2.2250738585072014e-308, 1.0], 0)
    lo, occ = unpack(d)
    assert lo[0] == 0 and occ.sum() == 5
    # a table of 16384 equal values: one bin holding everything (16-bit occ field)
    info, d = eos.plan_table(np.full(eos.EOS_MAX_TABLE, 3.0))
    assert info.max_occ == eos.EOS_MAX_TABLE and info.steps == 15


def test_mode1_directory_monotone_over_mixed_signs():
    rng = np.random.default_rng(5)
    for _ in range(30):
        X = np.sort(rng.normal(0, 100, int(rng.integers(2, 300))))
        for k in (0, 3, 8):
            try:
                info, d = eos.plan_table(X, k)
            except eos.EosError as e:   # a sign-crossing key spans ~2046 exponents per 2^k
                assert e.code == 8 and k > 0
                continue
            lo, occ = unpack(d)
            assert info.key_mode == 1
            assert lo[0] == 0 and lo[-1] + occ[-1] == X.size
            assert np.all(lo[1:] == lo[:-1] + occ[:-1])


# ------------------------------------------------------ logarithm hash (f1) --
def _keys(X):
    return ((np.asarray(X, dtype=np.float64).view(np.uint64) >> np.uint64(32)) &
            np.uint64(0x7FFFFFFF)).astype(np.int64)


@pytest.mark.parametrize("H", [1, 2, 7, 34, 110, 1000, 20000])
def test_log_hash_directory_and_eq1_range(H):
    """'any value we search for that is within [Xmin, Xmax] must satisfy
    0 <= hash(x) < |H|' -- and the directory is the exact count over those bins."""
    rng = np.random.default_rng(H)
    for _ in range(20):
        X = np.sort(10.0 ** rng.uniform(-6, 6, int(rng.integers(1, 500))))
        info, d = eos.plan_table(X, log_bins=H)
        lo, occ = unpack(d)
        assert info.hash_kind == eos.EOS_HASH_LOG and info.k == -1
        assert 1 <= info.bins <= H
        assert lo[0] == 0 and lo[-1] + occ[-1] == X.size
        assert np.all(lo[1:] == lo[:-1] + occ[:-1])
        # recount: bin = floor((key - key(X0)) * M / 2^32), the fixed-point log2 scaled
        kx = _keys(X)
        b = ((kx - kx[0]) * int(info.hash_mult)) >> 32
        assert b.max() == info.bins - 1 < H
        assert np.array_equal(np.bincount(b, minlength=info.bins), occ)
        # monotone in the value, equal-width in log2 up to the bit-pattern approximation
        assert np.all(np.diff(b) >= 0)


def test_log_hash_bins_have_equal_log_width():
    """Eq. 1: bins of equal width in log_b; with the fixed-point log2 of the
    IEEE bits the width is constant in key units, and within 0.09 log2 of the true log."""
    X = datagen_table()
    info, _ = eos.plan_table(X, log_bins=34)
    kx = _keys(X)
    approx_log2 = kx / 2.0 ** 20 - 1023
    assert np.max(np.abs(approx_log2 - np.log2(X))) < 0.0861
    width_log2 = 2.0 ** 32 / info.hash_mult / 2 ** 20
    assert abs(width_log2 * 34 - (approx_log2[-1] - approx_log2[0])) < 2 * width_log2


def datagen_table():
    import datagen
    return datagen.table_paper_exemplar()


def test_log_hash_brackets_oracle_answer():
    import datagen
    for name in ("cfg1", "cfg2", "cfg5"):
        w = datagen.workload(name, count=2000)
        X = w.table
        Y = np.concatenate([w.targets.host_fill(0, w.count, X), X, np.nextafter(X, 0)])
        ref = oracle.search(X, Y)
        kx = _keys(X)
        for H in (5, 64, 999):
            info, d = eos.plan_table(X, log_bins=H)
            lo, occ = unpack(d)
            ky = _keys(Y)
            b = np.minimum(((np.maximum(ky, info.base) - info.base) * int(info.hash_mult)) >> 32,
                           info.bins - 1)
            inr = Y >= X[0]
            assert np.all(lo[b][inr] <= ref[inr] + 1)
            assert np.all(ref[inr] + 1 <= lo[b][inr] + occ[b][inr])


def test_auto_choice_never_worse_in_steps_than_any_exponent_k():
    import datagen
    X = datagen.table_cfg1()
    auto, _ = eos.plan_table(X)
    for k in range(0, 12):
        try:
            e, _ = eos.plan_table(X, k)
        except eos.EosError:
            continue
        assert auto.steps <= e.steps or e.image_bytes > 144 * 1024
    assert auto.steps == 1 and auto.image_bytes <= 32 * 1024   # 4 CTAs x 256 per SM


# ------------------------------------------------- tiered tables (f4) ------
def test_tiered_plan_levels_and_sizes():
    """eos_plan_table_levels (eossearch.h): D = 0 up to EOS_MAX_TABLE, then the
    smallest D with n1 = ceil(n/8^D) <= 32768; levels hold n1 8^(D-d) entries each
    (d = 0..D-1), 8 B fp64 + 4 B key; the smem image holds the sample table
    X[::8^D] as 32-bit keys plus its directory."""
    rng = np.random.default_rng(7)
    pad16 = lambda b: (b + 15) // 16 * 16  # noqa: E731
    for n, D in [(1, 0), (16384, 0), (16385, 1), (262144, 1), (262145, -1), (1 << 20, -1),
                 (1 << 21, -2), ((1 << 21) + 1, -2)]:
        X = np.sort(10.0 ** rng.uniform(-6, 10, n))
        info = eos.plan_table_levels(X)
        if D < 0:  # 8-ary levels would need D >= 2: packed nodes, -D levels (their own test)
            assert info.levels == -D and info.node_width == 15, n
            continue
        assert info.levels == D and info.n == n, (n, info.levels)
        assert info.node_width == (8 if D else 0)
        n1 = -(-n // 8 ** D)
        assert info.top_n == n1 <= (eos.EOS_MAX_TABLE if D == 0 else 32768)
        assert info.level_bytes == 12 * sum(n1 * 8 ** (D - d) for d in range(D))
        if D == 0:   # the single-level plan
            top, _ = eos.plan_table(X, with_directory=False)
            for f in ("bins", "max_occ", "steps", "k", "hash_kind", "hash_mult", "image_bytes"):
                assert getattr(info, f) == getattr(top, f), (n, f)
        else:        # keys of the sample table X[::8^D] under the tiered image budget
            budget = min(176 * 1024, 4 * n1 + max(48 * 1024, 8 * n1))
            assert info.image_bytes == pad16(4 * n1) + pad16(4 * info.bins) <= budget
            assert info.steps == int(np.ceil(np.log2(info.max_occ + 1)))
            if info.hash_kind == eos.EOS_HASH_EXPONENT:
                ref, _ = eos.plan_table(X[::8 ** D], k=info.k, with_directory=False)
                assert (ref.bins, ref.max_occ, ref.steps) == (info.bins, info.max_occ, info.steps)
    # explicit D on small tables (testing the tiered path at any size)
    X = np.sort(rng.uniform(1, 2, 1000))
    for D in range(0, 6):
        info = eos.plan_table_levels(X, levels=D)
        assert info.levels == D and info.top_n == -(-1000 // 8 ** D)


def _keys_mode0(v):
    return (np.ascontiguousarray(v).view(np.uint64) >> np.uint64(32)).astype(np.int64) & 0x7FFFFFFF


@pytest.mark.parametrize("n,depth", [(300_001, 1), (1 << 20, 1), (1_500_000, 1), (16_385, 1),
                                     (1000, 1), (4_000_000, 2), (1000, 2), (300_001, 3),
                                     (40_000, 4)])
def test_packed_plan_fields_and_sample_hash(n, depth):
    """eos_plan_table_levels(EOS_LEVELS_PACKED[_DEPTH(D)]) (eos_internal.h PackedPlan):
    levels d = D-1..0 of ceil(n/15^(d+1)) nodes of 32 B after the 32-B padded fp64 table;
    the sample table X[::15^D] as u16 residuals, one u32 directory entry per bin pair and
    the 32-B level table within 224 KB; the bins are the key's bits above sh = 20 - k (hb
    aligned), recounted here, and S is the fewest lifting steps over every residual width
    that fits (bins of <= 63 entries).  EOS_LEVELS_PACKED takes the fewest levels."""
    rng = np.random.default_rng(n)
    X = np.sort(10.0 ** rng.uniform(-6, 10, n))
    info = eos.plan_table_levels(X, levels=eos.EOS_LEVELS_PACKED_DEPTH(depth))
    if n in (4_000_000, 1_500_000, 1 << 20):  # the fewest levels that fit
        auto = eos.plan_table_levels(X, levels=eos.EOS_LEVELS_PACKED)
        assert auto.levels == depth and auto.as_dict() == info.as_dict()
    pad16 = lambda b: (b + 15) // 16 * 16  # noqa: E731
    n1 = -(-n // 15 ** depth)
    assert (info.levels, info.node_width, info.top_n, info.n) == (depth, 15, n1, n)
    nodes = sum(-(-n // 15 ** (d + 1)) for d in range(depth))
    assert info.level_bytes == (8 * n + 31) // 32 * 32 + 32 * nodes
    assert info.hash_kind == eos.EOS_HASH_EXPONENT and 4 <= info.k <= 19
    assert info.dir_entry_bytes == 2
    budget = 224 * 1024
    assert info.image_bytes == pad16(2 * n1) + pad16(4 * ((info.bins + 1) // 2)) + 32 <= budget

    K = _keys_mode0(X[::15 ** depth])

    def plan(sh):
        hb = int(K[0]) & ~((1 << sh) - 1)
        bins = ((int(K[-1]) - hb) >> sh) + 1
        occ = np.bincount((K - hb) >> sh, minlength=bins)
        return hb, bins, int(occ.max())
    sh = 20 - info.k
    hb, bins, mo = plan(sh)
    assert (info.base, info.bins, info.max_occ) == (hb, bins, mo)
    assert info.steps == int(np.ceil(np.log2(mo + 1))) <= 6
    for other in range(1, 17):
        _, b2, m2 = plan(other)
        if pad16(2 * n1) + pad16(4 * ((b2 + 1) // 2)) + 32 <= budget and m2 <= 63:
            assert int(np.ceil(np.log2(m2 + 1))) >= info.steps, other


def test_packed_plan_auto_choice_and_errors():
    rng = np.random.default_rng(9)
    X = np.sort(10.0 ** rng.uniform(-6, 10, 400_000))
    assert eos.plan_table_levels(X).node_width == 15                 # AUTO, n > 8 x 32768
    assert eos.plan_table_levels(X, k=8).node_width == 8             # explicit hash: 8-ary
    assert eos.plan_table_levels(X[:200_000]).node_width == 8        # one 8-ary level
    assert eos.plan_table_levels(X, levels=2).node_width == 8
    for bad, code in [(np.full(300_000, 2.5), "EOS_ERR_UNSUPPORTED"),   # one bin of 20000
                      (np.sort(10.0 ** rng.uniform(-6, 10, 4_000_000)), "EOS_ERR_UNSUPPORTED"),
                      (np.empty(0), "EOS_ERR_SIZE")]:
        with pytest.raises(eos.EosError) as e:
            eos.plan_table_levels(bad, levels=eos.EOS_LEVELS_PACKED_DEPTH(1))
        assert e.value.name == code
    # more levels fit: one bin of 89 entries at D = 3, of 6 at D = 4
    assert eos.plan_table_levels(np.full(300_000, 2.5), levels=eos.EOS_LEVELS_PACKED).levels == 4
    for lv in (eos.EOS_LEVELS_PACKED_DEPTH(0), eos.EOS_LEVELS_PACKED_DEPTH(5), -3):
        with pytest.raises(eos.EosError) as e:
            eos.plan_table_levels(X, levels=lv)
        assert e.value.name == "EOS_ERR_UNSUPPORTED"
    # AUTO falls back to 8-ary levels when packed does not fit
    assert eos.plan_table_levels(np.full(300_000, 2.5)).node_width == 8
    bad = X.copy()
    bad[1000] = np.nan
    with pytest.raises(eos.EosError) as e:
        eos.plan_table_levels(bad, levels=eos.EOS_LEVELS_PACKED)
    assert e.value.name == "EOS_ERR_NONFINITE"
    bad = X.copy()
    bad[1000], bad[1001] = bad[1001], bad[1000]
    with pytest.raises(eos.EosError) as e:
        eos.plan_table_levels(bad)
    assert e.value.name == "EOS_ERR_UNSORTED"


def test_tiered_plan_errors():
    X = np.arange(1.0, 20001.0)
    with pytest.raises(eos.EosError) as e:
        eos.plan_table_levels(X, levels=0)          # n1 = n > EOS_MAX_TABLE
    assert e.value.name == "EOS_ERR_SIZE"
    with pytest.raises(eos.EosError) as e:
        eos.plan_table_levels(X, levels=6)
    assert e.value.name == "EOS_ERR_UNSUPPORTED"
    with pytest.raises(eos.EosError) as e:
        eos.plan_table_levels(np.empty(0))
    assert e.value.name == "EOS_ERR_SIZE"
    bad = X.copy()
    bad[17_000] = np.nan
    with pytest.raises(eos.EosError) as e:
        eos.plan_table_levels(bad)
    assert e.value.name == "EOS_ERR_NONFINITE"
    bad = X.copy()
    bad[17_000], bad[17_001] = bad[17_001], bad[17_000]
    with pytest.raises(eos.EosError) as e:
        eos.plan_table_levels(bad)
    assert e.value.name == "EOS_ERR_UNSORTED"
    # duplicates and a -0.0 head are valid (P:54-56 non-decreasing; R6)
    dup = np.concatenate([[-0.0], np.repeat(np.arange(1.0, 9000.0), 3)])
    info = eos.plan_table_levels(dup)
    assert info.levels == 1 and info.key_mode == 0


def test_grid_cell_limit_checked_before_any_work():
    """eos_grid2d_create_ex rejects n_rho n_T > EOS_MAX_GRID_CELLS (EOS_ERR_SIZE) before
    reading P or touching a device, and unknown flags (EOS_ERR_UNSUPPORTED)."""
    import ctypes
    L = eos.load_library()
    L.eos_grid2d_create_ex.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                       ctypes.c_void_p]
    R = np.arange(1.0, 2.0 ** 15 + 1)
    T = np.arange(1.0, 2.0 ** 14 + 1)
    P = np.ones(4)
    h = ctypes.c_void_p()
    rc = L.eos_grid2d_create_ex(R.ctypes.data, R.size, T.ctypes.data, T.size, P.ctypes.data, 0,
                                ctypes.byref(h))
    assert rc == 2
    rc = L.eos_grid2d_create_ex(R.ctypes.data, 4, T.ctypes.data, 4, P.ctypes.data, 16,
                                ctypes.byref(h))
    assert rc == 8


def test_header_is_plain_c_and_the_example_links(tmp_path):
    """include/eossearch.h compiles as C11 and examples/c_abi_example.c links against the
    library with gcc (the boundary needs no C++ or torch types)."""
    import subprocess
    lib = os.path.join(ROOT, "paper_2112_03229_b200", "lib")
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-O1", "-I",
                        os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                        os.path.join(ROOT, "examples", "c_abi_example.c"), "-L", lib,
                        "-leossearch", "-L", "/usr/local/cuda/lib64", "-lcudart",
                        "-o", str(tmp_path / "ex")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def _product_lines(text: str):
    """Source lines compiled into the product library: everything outside
    `#ifdef EOS_EXPERIMENTS` blocks (their `#else` branches are product code)."""
    out, stack = [], []
    for line in text.splitlines():
        t = line.strip()
        if t.startswith("#if"):
            stack.append("EOS_EXPERIMENTS" in t and t.startswith("#ifdef"))
            continue
        if t.startswith("#else") and stack:
            stack[-1] = False
            continue
        if t.startswith("#endif") and stack:
            stack.pop()
            continue
        if not any(stack):
            out.append(line)
    return out


def test_product_library_reads_no_environment():
    """The product library's launch shapes and layouts follow from the plan alone: every
    getenv in csrc/ sits inside an `#ifdef EOS_EXPERIMENTS` block (the A/B build,
    _build.py --exp), and each experiment knob is listed in runtime.cu's header."""
    import glob
    import re
    csrc = os.path.join(ROOT, "paper_2112_03229_b200", "csrc")
    knobs = set()
    for f in sorted(glob.glob(os.path.join(csrc, "*"))):
        text = open(f).read()
        prod = "\n".join(_product_lines(text))
        assert "getenv" not in prod, f"{f}: getenv outside #ifdef EOS_EXPERIMENTS"
        for call in re.findall(r"getenv\(([^;]*?)\)", text):
            knobs |= set(re.findall(r'"(EOS_[A-Z0-9_]+)"', call))
    header = open(os.path.join(csrc, "runtime.cu")).read().split("\n\n")[0]
    assert {"EOS_SEARCH_VARIANT", "EOS_LAYOUT", "EOS_SMALL_TILES"} <= knobs
    assert not [k for k in knobs if k not in header]


def _lifting_probes_brute(o, S):
    """Executed probes of S-step predicated binary lifting in a bin of o entries, averaged
    over the o+1 target gaps, by direct simulation (kernels.cuh lookup)."""
    total = 0
    for cf in range(o + 1):
        c, s = 0, (1 << (S - 1)) if S > 0 else 0
        while s > 0:
            if c + s <= o:
                total += 1
                if c + s <= cf:
                    c += s
            s >>= 1
    return total / (o + 1)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5", "paper"])
def test_automatic_plan_is_the_argmin_of_the_cost_model(name):
    """The automatic hash choice (table_build.cpp plan_auto, which evaluates candidates from
    runs of the sorted keys) equals the argmin of the DESIGN.md §6.3 cost model recomputed
    here from every candidate's full directory, over every lifting layout (16/32-bit
    directory entries, SF fixed steps, rare branch): 3.5 + 6.1 E[probes] + issue + shape
    penalty, issue = S + [S > 3], SF = min(S, 3), 16-bit entries whenever they fit;
    ties to the smaller image, then the exponent hash, image budget 200 KB."""
    X = datagen.workload(name, count=10).table
    n = X.size
    pad16 = lambda b: (b + 15) & ~15  # noqa: E731
    budget = 200 * 1024

    def shape(img):
        return (0.0 if img <= 32768 else 1.0 if img <= 73728 else 1.5 if img <= 102400
                else 3.0 if img <= 147456 else 4.5)

    def cost(info, d):
        occ = (d >> 16).astype(np.int64)
        S = info.steps
        vals, counts = np.unique(occ, return_counts=True)
        probes = sum(int(c) * _lifting_probes_brute(int(o), S) for o, c in zip(vals, counts))
        probes /= info.bins
        sf = min(S, 3)
        big = S > sf
        issue = S + (1.0 if big else 0.0)
        img32 = pad16(8 * n) + pad16(4 * info.bins)
        best_l = (3.5 + 6.1 * probes + issue + shape(img32), img32, 0, sf, big)
        if n <= 8192 and occ.max() <= 7:
            img16 = pad16(8 * n) + pad16(2 * info.bins)
            c16 = 3.5 + 6.1 * probes + issue + shape(img16)
            if c16 < best_l[0] + 1e-9:
                best_l = (c16, img16, 1, sf, big)
        return best_l

    best = None
    cands = [(eos.EOS_HASH_EXPONENT, k) for k in range(eos.EOS_MAX_K + 1)]
    H, max_bins = 1.0, (budget - pad16(8 * n)) // (2 if n <= 4096 else 4)
    while H <= max_bins:
        cands.append((eos.EOS_HASH_LOG, int(H)))
        H *= 2 ** 0.125
    for kind, param in cands:
        try:
            info, d = eos.eos_plan_table_hash(X, kind, param)
        except eos.EosError:   # image beyond what shared memory holds
            continue
        c, img, d16, sf, big = cost(info, d)
        assert (info.dir_entry_bytes, info.fast_steps, info.rare_steps) == (2 if d16 else 4, sf, int(big))
        if best is not None and img > budget:
            continue
        if best is None or c < best[0] - 1e-9 or (c < best[0] + 1e-9 and img < best[1]):
            best = (c, img, info.bins, info.hash_kind, info.steps)
    auto, _ = eos.eos_plan_table(X, eos.EOS_K_AUTO, with_directory=False)
    assert (auto.bins, auto.hash_kind, auto.steps) == best[2:], (auto.bins, best)


# ------------------------------------------- binding argument checks (CPU) --
def _unbound(cls):
    """An object of the binding class with a dummy handle: the argument checks run before
    any C call, so a rejected call never reaches the library (no device needed)."""
    o = cls.__new__(cls)
    o._h = 0xDEAD
    return o


@pytest.mark.parametrize("bad", ["f32", "short", "strided", "i64_out"])
def test_search_host_rejects_bad_host_buffers(bad):
    t = _unbound(eos.Table)
    y = np.linspace(1.0, 2.0, 1000)
    out = np.empty(1000, np.int32)
    if bad == "f32":
        y = y.astype(np.float32)
    elif bad == "short":
        out = np.empty(999, np.int32)
    elif bad == "strided":
        y = np.linspace(1.0, 2.0, 2000)[::2]
    else:
        out = np.empty(1000, np.int64)
    with pytest.raises((TypeError, ValueError)):
        t.search_host(y, out=out, sync=False)
    t._h = None


@pytest.mark.parametrize("bad", ["f32_rho", "len_T", "short_P", "i64_bracket", "f32_out",
                                 "strided_T"])
def test_interp_host_rejects_bad_host_buffers(bad):
    g = _unbound(eos.Grid2D)
    m = 500
    rho, T = np.linspace(1, 2, m), np.linspace(3, 4, m)
    P, iR, iT = np.empty(m), np.empty(m, np.int32), np.empty(m, np.int32)
    if bad == "f32_rho":
        rho = rho.astype(np.float32)
    elif bad == "len_T":
        T = T[:-1]
    elif bad == "short_P":
        P = P[:-1]
    elif bad == "i64_bracket":
        iR = np.empty(m, np.int64)
    elif bad == "f32_out":
        P = np.empty(m, np.float32)
    else:
        T = np.linspace(3, 4, 2 * m)[::2]
    with pytest.raises((TypeError, ValueError)):
        g.interp_host(rho, T, P, iR, iT, sync=False)
    g._h = None


@pytest.mark.parametrize("kw", [{"k": 0}, {"k": 3}, {"log_bins": 4096}, {}])
def test_tiered_explicit_hash_fits_its_key_image(kw):
    """A tiered table's sample table is staged as 32-bit keys: an explicit hash is accepted
    when the KEY image fits shared memory (the fp64 image of a 31250-entry sample table
    would not), as the automatic choice is."""
    X = np.sort(10.0 ** np.random.default_rng(5).uniform(-6, 10, 250_000))
    info = eos.eos_plan_table_levels(X, eos.EOS_LEVELS_AUTO, **kw)
    assert info.levels == 1 and info.top_n == 31250
    assert info.image_bytes <= 200 * 1024
