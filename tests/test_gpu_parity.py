"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle (-m gpu).

Indices must be bit-identical to the oracle; interpolated values within
1e-12 relative (BASELINE.json north_star).  Oracle inputs always come from
the host generators (datagen host side), never from the device; the device
generators are proven bit-identical to the host ones first.
"""
import math

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2112_03229_b200 as eos  # noqa: E402
from tests._golden import interp_cases, lower_bound_cases  # noqa: E402

DEV = torch.device("cuda:0")
REL_TOL = 1e-12  # north_star: "within 1e-12 relative for fp64 interpolated values"


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def gpu_search(X, Y, k=None, log_bins=None, **kw):
    t = eos.Table(X, k=k, log_bins=log_bins)
    out = t.search(to_dev(Y), **kw)
    torch.cuda.synchronize()
    r = out.cpu().numpy()
    t.close()
    return r


def assert_same(got, ref, Y=None):
    bad = np.flatnonzero(got != ref)
    if bad.size:
        i = bad[:8]
        raise AssertionError(f"{bad.size} mismatches; first at {i}: gpu {got[i]} oracle {ref[i]}"
                             + (f" y {Y[i]}" if Y is not None else ""))


def feasible_ks(X, ks):
    out = []
    for k in ks:
        try:
            eos.plan_table(X, eos.EOS_K_AUTO if k is None else k, with_directory=False)
            out.append(k)
        except eos.EosError:
            pass
    return out


# --------------------------------------------------------------- smoke -----
def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


# ----------------------------------------------------------- generators ----
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5", "paper"])
def test_device_generators_bit_identical_to_host(name):
    w = datagen.workload(name, count=300_001)
    for off in (0, 12_345):
        n = w.count - off
        d = torch.empty(n, dtype=torch.float64, device=DEV)
        tab = to_dev(w.table)
        w.targets.device_fill(d, off, table_dev=tab)
        h = w.targets.host_fill(off, n, w.table)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy().view(np.uint64), h.view(np.uint64))


def test_device_generators_cfg4():
    w = datagen.workload("cfg4", count=100_000)
    for spec in (w.rho_targets, w.T_targets):
        d = torch.empty(w.count, dtype=torch.float64, device=DEV)
        spec.device_fill(d, 0)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), spec.host_fill(0, w.count))


# ------------------------------------------------------------ 1-D parity ---
@pytest.mark.parametrize("name", sorted(lower_bound_cases().keys()))
def test_golden_cases_every_k(name):
    X, cases = lower_bound_cases()[name]
    ys = np.array([c[0] for c in cases] * 37)  # repeated: crosses the vector body and tail
    exp = np.array([c[1] for c in cases] * 37, dtype=np.int32)
    for k in feasible_ks(X, [None, 0, 1, 2, 4, 8, 12, 19]):
        assert_same(gpu_search(X, ys, k=k), exp, ys)
    for H in (1, 2, 3, 17, 1000):   # the logarithm hash, any |H|
        assert_same(gpu_search(X, ys, log_bins=H), exp, ys)


def _edge_tables(rng, count):
    for t in range(count):
        n = int(rng.integers(1, 14))
        kind = t % 7
        if kind == 0:
            X = 10.0 ** rng.uniform(-8, 8, n)
        elif kind == 1:
            X = 2.0 ** rng.integers(-20, 20, n).astype(np.float64)
        elif kind == 2:
            X = np.concatenate([[0.0], rng.uniform(0, 1, n) * 1e-310, 10.0 ** rng.uniform(-5, 5, n)])
        elif kind == 3:
            X = np.round(rng.uniform(1.0, 1.01, n), 3)
        elif kind == 4:
            X = np.concatenate([rng.normal(0, 10, n), [0.0, -0.0]])
        elif kind == 5:
            X = rng.choice([1.0, 2.0, 3.0], n)
        else:
            X = -(10.0 ** rng.uniform(-3, 3, n))
        yield np.sort(X)


def _probes(X):
    p = [0.0, -0.0, math.inf, -math.inf, math.nan, 5e-324, 2.2250738585072014e-308, 1e-300,
         1e300, -1.0, 1.0, 2.0, 0.5, -1e-310]
    for x in X:
        p += [x, math.nextafter(x, math.inf), math.nextafter(x, -math.inf)]
        if x != 0:
            e = math.floor(math.log2(abs(x)))
            p += [math.copysign(2.0 ** e, x), math.nextafter(math.copysign(2.0 ** e, x), 0.0)]
    for a, b in zip(X[:-1], X[1:]):
        p.append(0.5 * (a + b))
    return np.array(p)


def test_edge_tables_exhaustive_probes_every_k():
    rng = np.random.default_rng(2024)
    checked = 0
    for X in _edge_tables(rng, 140):
        P = _probes(X)
        P = np.concatenate([P, rng.permutation(np.repeat(P, 5))])
        ref = oracle.search(X, P)
        for k in feasible_ks(X, [None, 0, 1, 3, 6, 10]):
            assert_same(gpu_search(X, P, k=k), ref, P)
            checked += P.size
        for H in (1, 5, 300):
            assert_same(gpu_search(X, P, log_bins=H), ref, P)
    assert checked > 100_000


def test_cfg1_full_every_k():
    w = datagen.workload("cfg1")
    Y = w.targets.host_fill(0, w.count, w.table)
    ref = oracle.search(w.table, Y)
    for k in feasible_ks(w.table, [None] + list(range(0, 16))):
        assert_same(gpu_search(w.table, Y, k=k), ref, Y)
    for H in (1, 10, 64, 500, 1722, 5000, 40000):
        assert_same(gpu_search(w.table, Y, log_bins=H), ref, Y)


@pytest.mark.parametrize("count", [0, 1, 2, 3, 5, 511, 2047, 2048, 2049, 4097, 65_537, 1_000_003])
@pytest.mark.parametrize("y_off,o_off", [(0, 0), (1, 0), (0, 1), (1, 1), (3, 2)])
def test_ragged_and_misaligned(count, y_off, o_off):
    w = datagen.workload("cfg2", count=count + 8)
    Yall = w.targets.host_fill(0, count + 8, w.table)
    yd = to_dev(Yall)[y_off:y_off + count]
    od_all = torch.full((count + 8,), -7, dtype=torch.int32, device=DEV)
    od = od_all[o_off:o_off + count]
    t = eos.Table(w.table)
    t.search(yd, out=od)
    torch.cuda.synchronize()
    got = od_all.cpu().numpy()
    assert_same(got[o_off:o_off + count], oracle.search(w.table, Yall[y_off:y_off + count]))
    assert np.all(got[:o_off] == -7) and np.all(got[o_off + count:] == -7)  # no stray writes
    t.close()


@pytest.mark.parametrize("count", [2_350_077, 2_350_078, 4_000_001, 9_999_999])
@pytest.mark.parametrize("y_off,o_off", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("table,kw", [("cfg2", {}), ("cfg5", {}), ("cfg5", {"k": 0})])
def test_ring_launches_ragged_and_misaligned(count, y_off, o_off, table, kw):
    """Launches large enough for the shared-memory ring kernel (>= 4 stages of 3968 targets
    per SM): odd and even lengths, an unaligned first target (scalar head), an odd last
    one (scalar tail), and outputs that are not 8-byte aligned (the register kernels
    take those); bit-exact, no stray writes.  (k = 0 on cfg5: S = 9, the rare-branch
    layout.)"""
    w = datagen.workload(table, count=count + 8)
    Yall = w.targets.host_fill(0, count + 8, w.table)
    Yall[y_off] = np.nan
    Yall[y_off + count - 1] = w.table[-1]
    yd = to_dev(Yall)[y_off:y_off + count]
    od_all = torch.full((count + 8,), -7, dtype=torch.int32, device=DEV)
    od = od_all[o_off:o_off + count]
    t = eos.Table(w.table, **kw)
    t.search(yd, out=od)
    torch.cuda.synchronize()
    got = od_all.cpu().numpy()
    assert_same(got[o_off:o_off + count], oracle.search(w.table, Yall[y_off:y_off + count]))
    assert np.all(got[:o_off] == -7) and np.all(got[o_off + count:] == -7)  # no stray writes
    t.close()


@pytest.mark.parametrize("case", ["mode1_s2", "mode1_deep", "dups_s3", "zero_head_s3", "s2_d16",
                                  "n8192_s3", "k0_deep", "d32_deep"])
def test_ring_kernel_layouts(case):
    """Ring-kernel launches (>= 4 stages per SM) over every layout it can get: key modes 0
    and 1, S = 2 and 3 (16-bit entries), deep tables with the stride branch (S >= 4, 32-bit
    entries), a 0.0 head with subnormals, duplicate runs, the largest 16-bit table; bit-exact
    against the oracle."""
    rng = np.random.default_rng(sum(map(ord, case)))
    kw = {}
    if case == "mode1_s2":       # key mode 1 (all negative), S = 2
        X = np.sort(rng.uniform(-5, -1, 1000))
    elif case == "mode1_deep":   # key mode 1 (both signs), S = 6
        X = np.sort(rng.uniform(-50, 50, 1000))
    elif case == "dups_s3":
        X = np.sort(np.repeat(10 ** rng.uniform(-2, 4, 500), 3))
    elif case == "zero_head_s3":
        X = np.concatenate([np.zeros(3), np.sort(10 ** rng.uniform(-300, 2, 2000))])
        kw = {"log_bins": 1500}
    elif case == "s2_d16":
        X = np.sort(10 ** rng.uniform(-3, 5, 2000))
        kw = {"log_bins": 16000}
    elif case == "n8192_s3":     # the largest table with 16-bit entries, a 101 KB image
        X = np.sort(10 ** rng.uniform(-6, 10, 8192))
    elif case == "k0_deep":      # the paper's exponent hash on cfg5: S = 9
        X = datagen.table_cfg5(4)
        kw = {"k": 0}
    else:                        # S = 4, 32-bit entries
        X = np.sort(10 ** rng.uniform(-3, 5, 6000))
        kw = {"log_bins": 3000}
    t = eos.Table(X, **kw)
    assert t.info.steps >= 2, t.info.as_dict()
    m = 5_000_003
    lo, hi = float(X[0]), float(X[-1])
    if lo > 0:
        Y = 10 ** rng.uniform(np.log10(lo) - 0.3, np.log10(hi) + 0.3, m)
    else:
        Y = rng.uniform(lo - 1, hi + 1, m)
    Y[:X.size] = X
    Y[X.size:X.size + 6] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 5e-324]
    got = t.search(to_dev(Y)).cpu().numpy()
    assert t.info.ring_stages >= 2, t.info.as_dict()
    assert_same(got, oracle.search(X, Y), Y)
    t.close()


@pytest.mark.parametrize("table,kw", [("cfg1", {}), ("cfg2", {"log_bins": 12000}),
                                      ("cfg5", {}), ("cfg5", {"log_bins": 5000}),
                                      ("cfg2", {"k": 0})])
def test_small_launch_tiles_match_default_tiles_and_oracle(table, kw):
    """Launches whose default tiling leaves most SMs idle run the small-tile shape
    (search_api.cu launch_search): every shape family (image <= 32 KB / <= 72 KB / larger,
    fixed steps / rare branch), counts on both sides of the switch, ragged heads and tails;
    bit-exact against the oracle, and each slice equal to the same targets inside one
    400,003-target launch (default tiles)."""
    w = datagen.workload(table, count=400_003)
    Yall = w.targets.host_fill(0, w.count, w.table)
    Yall[:4] = [np.nan, -np.inf, np.inf, 0.0]
    t = eos.Table(w.table, **kw)
    whole = t.search(to_dev(Yall)).cpu().numpy()
    assert_same(whole, oracle.search(w.table, Yall), Yall)
    for count, off in ((1, 0), (7, 1), (1000, 3), (50_001, 1), (151_553, 0), (151_552, 2),
                       (300_001, 1), (400_000, 3)):
        Y = Yall[off:off + count]
        a = t.search(to_dev(Yall)[off:off + count])
        torch.cuda.synchronize()
        assert_same(a.cpu().numpy(), oracle.search(w.table, Y), Y)
        assert np.array_equal(a.cpu().numpy(), whole[off:off + count])
    t.close()


@pytest.mark.parametrize("loglog,global_grid", [(False, False), (True, False), (False, True),
                                                (True, True)])
def test_small_launch_tiles_2d_match_default_tiles_and_oracle(loglog, global_grid):
    """2-D launches with fewer default tiles than half the SMs run the small-tile kernel
    (grid_api.cu launch_interp: the image without G, corners from cell quads in device
    memory): brackets and P bit-identical to the same pairs inside one 160,003-pair launch
    (default tiles), brackets equal to the oracle's, P within the bar, on both sides of the
    switch (74 tiles = 151,552 pairs)."""
    w = datagen.workload("cfg4", count=160_003)
    rho = w.rho_targets.host_fill(0, w.count)
    T = w.T_targets.host_fill(0, w.count)
    rho[:3] = [np.nan, w.rho[0] / 3, w.rho[-1] * 3]
    rho[3:3 + w.rho.size] = w.rho
    g = eos.Grid2D(w.rho, w.T, w.P, loglog=loglog, global_grid=global_grid)
    whole = [x.cpu().numpy() for x in g.interp(to_dev(rho), to_dev(T))]
    whole_d = [x.cpu().numpy() for x in g.interp(to_dev(rho), to_dev(T), derivatives=True)]
    ref_all = (oracle.interp2d_loglog if loglog else oracle.interp2d)(w.rho, w.T, w.P, rho, T)
    for count, off in ((1, 0), (7, 1), (1000, 0), (20_001, 1), (151_551, 0), (151_553, 1),
                       (160_000, 2)):
        rd, td = to_dev(rho)[off:off + count], to_dev(T)[off:off + count]
        a = g.interp(rd, td)
        ad = g.interp(rd, td, derivatives=True)  # the derivative kernels switch too
        torch.cuda.synchronize()
        for x, y in list(zip(a, whole)) + list(zip(ad, whole_d)):
            assert np.array_equal(x.cpu().numpy(), y[off:off + count], equal_nan=True)
        assert np.array_equal(a[1].cpu().numpy(), ref_all[1][off:off + count])
        assert np.array_equal(a[2].cpu().numpy(), ref_all[2][off:off + count])
        check_interp(a[0].cpu().numpy(), ref_all[0][off:off + count])
    g.close()


@pytest.mark.parametrize("kind", ["loguniform", "mixed_sign"])
def test_tiered_small_launch_tiles_match_default_tiles_and_oracle(kind):
    """Tiered tables: launches whose default tiles would leave most SMs idle use 512 x 1
    tiles; bit-exact against the oracle and against the same targets inside one large
    launch (default tiles), on both sides of the switch."""
    rng = np.random.default_rng(11)
    X = np.sort(10.0 ** rng.uniform(-6, 10, 200_003))
    if kind == "mixed_sign":
        X = np.sort(np.concatenate([-X[:50_000], X[50_000:]]))
    Yall = np.concatenate([10.0 ** rng.uniform(-7, 11, 320_000) * rng.choice([-1.0, 1.0], 320_000),
                           X[::7], [np.nan, np.inf, -np.inf, 0.0]])
    t = eos.Table(X, levels=1)
    whole = t.search(to_dev(Yall)).cpu().numpy()
    assert_same(whole, oracle.search(X, Yall), Yall)
    for count, off in ((1, 0), (999, 3), (100_003, 1), (303_103, 0), (320_000, 5)):
        Y = Yall[off:off + count]
        a = t.search(to_dev(Yall)[off:off + count])
        torch.cuda.synchronize()
        assert_same(a.cpu().numpy(), oracle.search(X, Y), Y)
        assert np.array_equal(a.cpu().numpy(), whole[off:off + count])
    t.close()


def test_counters_match_oracle():
    w = datagen.workload("cfg1", count=777_777)
    Y = w.targets.host_fill(0, w.count, w.table)
    Y[::1001] = np.nan
    Y[3::5003] = np.inf
    off = 5_000_000_000
    ref_idx = oracle.search(w.table, Y)
    ref = oracle.counters(w.table, Y, ref_idx, off)
    t = eos.Table(w.table)
    c = torch.zeros(8, dtype=torch.int64, device=DEV)
    idx = t.search(to_dev(Y), counters=c, global_offset=off)
    torch.cuda.synchronize()
    assert_same(idx.cpu().numpy(), ref_idx)
    assert np.array_equal(c.cpu().numpy().view(np.uint64), ref)
    # accumulation over two shards == whole
    c2 = torch.zeros(8, dtype=torch.int64, device=DEV)
    yd = to_dev(Y)
    h = 300_001
    t.search(yd[:h], counters=c2, global_offset=off)
    t.search(yd[h:], counters=c2, global_offset=off + h)
    torch.cuda.synchronize()
    assert np.array_equal(c2.cpu().numpy().view(np.uint64), ref)
    t.close()


def test_errors_are_reported():
    t = eos.Table([1.0, 2.0, 3.0])
    y = torch.ones(16, dtype=torch.float64, device=DEV)
    with pytest.raises(eos.EosError) as e:   # output aliasing the input
        eos.eos_search(t.handle, y.data_ptr(), 16, y.data_ptr() + 8, 0)
    assert e.value.code == 9
    with pytest.raises(eos.EosError) as e:
        eos.eos_search(t.handle, 0, 16, y.data_ptr(), 0)
    assert e.value.code == 1
    with pytest.raises(eos.EosError) as e:
        eos.eos_search(t.handle, y.data_ptr(), -1, y.data_ptr(), 0)
    assert e.value.code == 2
    eos.eos_search(t.handle, 0, 0, 0, 0)  # count == 0: no-op
    with pytest.raises(eos.EosError):
        eos.Table([2.0, 1.0])
    n0 = eos.launch_count()
    t.search(y)
    assert eos.launch_count() == n0 + 1
    t.close()


# -------------------------------------------------------- full configs -----
def invariant_on_device(Xd, Yd, Id, chunk=1 << 26):
    """P:54 bracketing on every output: X[i] <= y < X[i+1] (or i = n-1); y < X[0] / NaN -> 0."""
    n = Xd.numel()
    for s in range(0, Yd.numel(), chunk):
        y = Yd[s:s + chunk]
        i = Id[s:s + chunk].long()
        assert int(i.min()) >= 0 and int(i.max()) <= n - 1
        inr = y >= Xd[0]
        assert bool((i[~inr] == 0).all())
        yi, ii = y[inr], i[inr]
        assert bool((Xd[ii] <= yi).all())
        assert bool(((ii == n - 1) | (yi < Xd[torch.clamp(ii + 1, max=n - 1)])).all())


def test_cfg2_full_bit_exact():
    w = datagen.workload("cfg2")
    Yh = w.targets.host_fill(0, w.count, w.table)
    ref = oracle.search(w.table, Yh)
    Yd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.targets.device_fill(Yd, 0)
    t = eos.Table(w.table)
    out = t.search(Yd)
    torch.cuda.synchronize()
    assert_same(out.cpu().numpy(), ref)
    t.close()


def _sampled_check(w, Yd, out, nsample=1 << 20, seed=0):
    idx = np.sort(np.random.default_rng(seed).integers(0, w.count, nsample))
    idx[:2] = [0, w.count - 1]
    idx = np.sort(idx)
    Ys = w.targets.host_sample(idx, w.table)
    ref = oracle.search(w.table, Ys)
    got = out[torch.from_numpy(idx).to(DEV)].cpu().numpy()
    assert_same(got, ref, Ys)
    # the device stream really is the host stream at those positions
    assert np.array_equal(Yd[torch.from_numpy(idx).to(DEV)].cpu().numpy(), Ys)


def test_cfg3_full_sampled_and_invariant():
    w = datagen.workload("cfg3")
    Yd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.targets.device_fill(Yd, 0)
    t = eos.Table(w.table)
    out = t.search(Yd)
    torch.cuda.synchronize()
    _sampled_check(w, Yd, out)
    invariant_on_device(to_dev(w.table), Yd, out)
    # k-invariance on a 2^27 slice: the paper's pure exponent hash (k=0) gives the same indices
    t0 = eos.Table(w.table, k=0)
    s = Yd[:1 << 27]
    assert torch.equal(t0.search(s), out[:1 << 27])
    t.close()
    t0.close()


def test_cfg5_full_sampled_invariant_counters():
    w = datagen.workload("cfg5")
    Yd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.targets.device_fill(Yd, 0)
    t = eos.Table(w.table)
    out = torch.empty(w.count, dtype=torch.int32, device=DEV)
    t.search(Yd, out=out)
    torch.cuda.synchronize()
    _sampled_check(w, Yd, out, nsample=1 << 21, seed=5)
    Xd = to_dev(w.table)
    invariant_on_device(Xd, Yd, out)
    # counters of a validation launch over a 2^26 shard in the middle == oracle counters there
    off = 5 << 30
    m = 1 << 26
    c = torch.zeros(8, dtype=torch.int64, device=DEV)
    t.search(Yd[off:off + m], out=torch.empty(m, dtype=torch.int32, device=DEV), counters=c,
             global_offset=off)
    Yh = w.targets.host_fill(off, m, w.table)
    ref = oracle.counters(w.table, Yh, oracle.search(w.table, Yh), off)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy().view(np.uint64), ref)
    for kw in ({"k": 0}, {"k": 7}, {"k": 9}, {"log_bins": 5000}):
        tk = eos.Table(w.table, **kw)
        assert torch.equal(tk.search(Yd[off:off + m]), out[off:off + m])
        tk.close()
    t.close()
    del Yd, out


# ------------------------------------------------------------------ 2-D ----
def check_interp(Pg, Pr):
    nan_g, nan_r = np.isnan(Pg), np.isnan(Pr)
    assert np.array_equal(nan_g, nan_r)
    ok = ~nan_r
    err = np.abs(Pg[ok] - Pr[ok])
    tol = REL_TOL * np.abs(Pr[ok])
    assert np.all(err <= tol), float(np.max(err / np.maximum(np.abs(Pr[ok]), 1e-300)))
    return float(np.max(err / np.maximum(np.abs(Pr[ok]), 1e-300))) if ok.any() else 0.0


def test_interp_golden():
    R, T, G, cases = interp_cases()
    rho = np.array([c[0] for c in cases] * 300)
    tt = np.array([c[1] for c in cases] * 300)
    g = eos.Grid2D(R, T, G)
    P, iR, iT = g.interp(to_dev(rho), to_dev(tt))
    torch.cuda.synchronize()
    assert np.array_equal(P.cpu().numpy(), np.array([c[2] for c in cases] * 300))
    assert np.array_equal(iR.cpu().numpy(), np.array([c[3] for c in cases] * 300))
    assert np.array_equal(iT.cpu().numpy(), np.array([c[4] for c in cases] * 300))
    g.close()


def test_interp_random_grids_edges():
    rng = np.random.default_rng(11)
    for t in range(25):
        nr, nt = int(rng.integers(2, 60)), int(rng.integers(2, 60))
        R = np.unique(10.0 ** rng.uniform(-6, 3, nr))
        T = np.unique(10.0 ** rng.uniform(0, 8, nt))
        if R.size < 2 or T.size < 2:
            continue
        G = rng.uniform(-5, 5, (R.size, T.size)) if t % 2 else rng.uniform(0.5, 5, (R.size, T.size))
        m = 20_011
        rho = 10.0 ** rng.uniform(-7, 4, m)
        tt = 10.0 ** rng.uniform(-1, 9, m)
        rho[:R.size] = R
        tt[:T.size] = T
        rho[-5:] = [np.nan, np.inf, -np.inf, 0.0, -1.0]
        g = eos.Grid2D(R, T, G)
        P, iR, iT = g.interp(to_dev(rho), to_dev(tt))
        torch.cuda.synchronize()
        Pr, iRr, iTr = oracle.interp2d(R, T, G, rho, tt)
        assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
        Pg = P.cpu().numpy()
        if t % 2:   # signed grid: cancellation -> the bound relative to the corner terms
            ok = ~np.isnan(Pr)
            assert np.array_equal(np.isnan(Pg), ~ok)
            sc = interp_scale(R, T, G, rho, tt, iRr, iTr)
            assert np.all(np.abs(Pg[ok] - Pr[ok]) <= REL_TOL * sc[ok])
        else:
            check_interp(Pg, Pr)
        g.close()


def test_interp_cfg4_sampled_full_and_prefix_exact():
    w = datagen.workload("cfg4")
    rd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    td = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.rho_targets.device_fill(rd, 0)
    w.T_targets.device_fill(td, 0)
    g = eos.Grid2D(w.rho, w.T, w.P)
    P, iR, iT = g.interp(rd, td)
    torch.cuda.synchronize()
    # full 2^22 prefix against the oracle
    m = 1 << 22
    rh = w.rho_targets.host_fill(0, m)
    th = w.T_targets.host_fill(0, m)
    Pr, iRr, iTr = oracle.interp2d(w.rho, w.T, w.P, rh, th)
    assert np.array_equal(iR[:m].cpu().numpy(), iRr) and np.array_equal(iT[:m].cpu().numpy(), iTr)
    check_interp(P[:m].cpu().numpy(), Pr)
    # sampled over the whole 2^28 stream
    idx = np.sort(np.random.default_rng(3).integers(0, w.count, 1 << 20))
    rs, ts = w.rho_targets.host_sample(idx), w.T_targets.host_sample(idx)
    Pr, iRr, iTr = oracle.interp2d(w.rho, w.T, w.P, rs, ts)
    di = torch.from_numpy(idx).to(DEV)
    assert np.array_equal(iR[di].cpu().numpy(), iRr) and np.array_equal(iT[di].cpu().numpy(), iTr)
    check_interp(P[di].cpu().numpy(), Pr)
    g.close()


# ------------------------------------------------------- host end-to-end ---
def test_search_host_pipeline_matches():
    w = datagen.workload("cfg2", count=(1 << 25) + 12345)
    Y = torch.from_numpy(w.targets.host_fill(0, w.count, w.table)).pin_memory()
    out = torch.empty(w.count, dtype=torch.int32).pin_memory()
    t = eos.Table(w.table)
    t.search_host(Y.numpy(), out)
    assert_same(out.numpy(), oracle.search(w.table, Y.numpy()))
    # pageable buffers work too
    small = w.targets.host_fill(0, 100_003, w.table)
    assert_same(t.search_host(small), oracle.search(w.table, small))
    t.close()


@pytest.mark.parametrize("global_grid", [False, True])
def test_interp_host_pipeline_matches(global_grid):
    w = datagen.workload("cfg4", count=(1 << 23) + 3)
    rh = w.rho_targets.host_fill(0, w.count)
    th = w.T_targets.host_fill(0, w.count)
    g = eos.Grid2D(w.rho, w.T, w.P, global_grid=global_grid)
    P, iR, iT = g.interp_host(rh, th)
    Pr, iRr, iTr = oracle.interp2d(w.rho, w.T, w.P, rh, th)
    assert np.array_equal(iR, iRr) and np.array_equal(iT, iTr)
    check_interp(P, Pr)
    g.close()


# ------------------------------------------------- f4: derivatives, mode 1 --
def _check_deriv(got, ref, cond):
    """Derivatives within 1e-12 of their condition scale `cond` (deriv_cond, DESIGN.md
    §4 "Comparison bounds"): the sum of the absolute values of the terms the derivative
    is computed from.  A difference of cell values cancels, so the error of a few-ulp
    perturbation of the weight is bounded relative to those terms, not to |ref|
    (|ref| <= cond always).  NaN must match NaN."""
    nan_g, nan_r = np.isnan(got), np.isnan(ref)
    assert np.array_equal(nan_g, nan_r)
    ok = ~nan_r
    bar = REL_TOL * np.nan_to_num(cond[ok], nan=np.inf, posinf=np.inf)
    err = np.abs(got[ok] - ref[ok])
    assert np.all(err <= bar), float(np.max(err / np.maximum(bar, 1e-300)) * REL_TOL)


def deriv_cond(R, T, G, rho, tt, iR, iT, P=None, loglog=False):
    """Condition scales of dP/drho and dP/dT on each bracket cell (R23 / R24), used only
    as the tolerance scale of _check_deriv -- not expected values.  For dP/drho:
      (|(1-ty)(g10-g00)| + |ty(g11-g01)| + |g11-g01-g10+g00|) / width
    (the terms of the numerator, plus its sensitivity to the weight ty); for log-log
    grids g = ln G, width = ln R[c+1] - ln R[c], times |P / rho|, plus |dP/drho| times
    (1 + sum |ln G| of the corners) for the relative error of P itself."""
    R, T, G = np.asarray(R), np.asarray(T), np.asarray(G)
    ci = np.minimum(iR, R.size - 2)
    cj = np.minimum(iT, T.size - 2)
    xr, xt, ax, at, g = (np.log(rho), np.log(tt), np.log(R), np.log(T), np.log(G)) if loglog \
        else (rho, tt, R, T, G)
    with np.errstate(all="ignore"):
        tx = np.clip((xr - ax[ci]) / (ax[ci + 1] - ax[ci]), 0, 1)
        ty = np.clip((xt - at[cj]) / (at[cj + 1] - at[cj]), 0, 1)
        g00, g01, g10, g11 = g[ci, cj], g[ci, cj + 1], g[ci + 1, cj], g[ci + 1, cj + 1]
        cross = np.abs(g11 - g01 - g10 + g00)
        kr = (np.abs((1 - ty) * (g10 - g00)) + np.abs(ty * (g11 - g01)) + cross) / (ax[ci + 1] - ax[ci])
        kt = (np.abs((1 - tx) * (g01 - g00)) + np.abs(tx * (g11 - g10)) + cross) / (at[cj + 1] - at[cj])
        if loglog:
            sl = 1 + np.abs(g00) + np.abs(g01) + np.abs(g10) + np.abs(g11)
            sr = ((1 - ty) * (g10 - g00) + ty * (g11 - g01)) / (ax[ci + 1] - ax[ci])
            st = ((1 - tx) * (g01 - g00) + tx * (g11 - g10)) / (at[cj + 1] - at[cj])
            kr = np.abs(P / rho) * (kr + np.abs(sr) * sl)
            kt = np.abs(P / tt) * (kt + np.abs(st) * sl)
    return kr, kt


def interp_scale(R, T, G, rho, tt, iR, iT):
    """Condition scale of P (linear grids): |(1-tx)(1-ty) g00| + |(1-tx) ty g01| + |tx (1-ty)
    g10| + |tx ty g11| -- equal to |P| where the corners share a sign, larger where the
    bilinear form cancels (eossearch.h: the default layout's bound is 1e-12 of this)."""
    R, T, G = np.asarray(R), np.asarray(T), np.asarray(G)
    ci = np.minimum(iR, R.size - 2)
    cj = np.minimum(iT, T.size - 2)
    with np.errstate(all="ignore"):
        tx = np.clip((rho - R[ci]) / (R[ci + 1] - R[ci]), 0, 1)
        ty = np.clip((tt - T[cj]) / (T[cj + 1] - T[cj]), 0, 1)
        return (np.abs((1 - tx) * (1 - ty) * G[ci, cj]) + np.abs((1 - tx) * ty * G[ci, cj + 1])
                + np.abs(tx * (1 - ty) * G[ci + 1, cj]) + np.abs(tx * ty * G[ci + 1, cj + 1]))


def test_interp_derivatives_match_oracle():
    w = datagen.workload("cfg4", count=(1 << 20) + 3)
    rho = w.rho_targets.host_fill(0, w.count)
    T = w.T_targets.host_fill(0, w.count)
    rho[:4] = [np.nan, w.rho[0] / 10, w.rho[-1] * 10, w.rho[5]]
    T[4:8] = [np.nan, w.T[0] / 10, w.T[-1] * 10, w.T[7]]
    g = eos.Grid2D(w.rho, w.T, w.P)
    P, iR, iT, dR, dT = g.interp(to_dev(rho), to_dev(T), derivatives=True)
    torch.cuda.synchronize()
    Pr, iRr, iTr = oracle.interp2d(w.rho, w.T, w.P, rho, T)
    dRr, dTr = oracle.interp2d_deriv(w.rho, w.T, w.P, rho, T)
    assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
    check_interp(P.cpu().numpy(), Pr)
    kr, kt = deriv_cond(w.rho, w.T, w.P, rho, T, iRr, iTr)
    _check_deriv(dR.cpu().numpy(), dRr, kr)
    _check_deriv(dT.cpu().numpy(), dTr, kt)
    # without derivatives the values are unchanged
    P2, _, _ = g.interp(to_dev(rho), to_dev(T))
    torch.cuda.synchronize()
    assert np.array_equal(P2.cpu().numpy(), P.cpu().numpy(), equal_nan=True)
    g.close()


def test_interp_negative_axes_mode1_and_odd_sizes():
    rng = np.random.default_rng(31)
    for t in range(12):
        R = np.unique(rng.normal(0, 50, int(rng.integers(2, 80))))
        T = np.unique(rng.uniform(-5, 5, int(rng.integers(2, 40))))
        if R.size < 2 or T.size < 2:
            continue
        G = rng.uniform(0.5, 5.0, (R.size, T.size))
        m = 10_007
        rho = rng.uniform(R[0] - 10, R[-1] + 10, m)
        tt = rng.uniform(T[0] - 1, T[-1] + 1, m)
        rho[:R.size] = R
        tt[-T.size:] = T
        rho[R.size:R.size + 2] = [-0.0, 0.0]
        g = eos.Grid2D(R, T, G, global_grid=bool(t % 2))  # odd draws: P in device memory
        assert g.rho_info.key_mode == 1
        P, iR, iT, dR, dT = g.interp(to_dev(rho), to_dev(tt), derivatives=True)
        torch.cuda.synchronize()
        Pr, iRr, iTr = oracle.interp2d(R, T, G, rho, tt)
        dRr, dTr = oracle.interp2d_deriv(R, T, G, rho, tt)
        assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
        check_interp(P.cpu().numpy(), Pr)
        kr, kt = deriv_cond(R, T, G, rho, tt, iRr, iTr)
        _check_deriv(dR.cpu().numpy(), dRr, kr)
        _check_deriv(dT.cpu().numpy(), dTr, kt)
        g.close()


# ---------------------------------------------------- f2: zero-setup search --
def direct(X, Y, **kw):
    out = eos.search_direct(to_dev(X), to_dev(Y), **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("name", sorted(lower_bound_cases().keys()))
def test_direct_golden(name):
    X, cases = lower_bound_cases()[name]
    ys = np.array([c[0] for c in cases] * 101)
    exp = np.array([c[1] for c in cases] * 101, dtype=np.int32)
    assert_same(direct(X, ys), exp, ys)


def test_direct_edge_tables_and_configs():
    rng = np.random.default_rng(77)
    for X in _edge_tables(rng, 80):
        P = _probes(X)
        P = np.concatenate([P, rng.permutation(np.repeat(P, 3))])
        assert_same(direct(X, P), oracle.search(X, P), P)
    for name in ("cfg1", "cfg2", "cfg3", "cfg5", "paper"):
        w = datagen.workload(name, count=(1 << 21) + 5)
        Y = w.targets.host_fill(0, w.count, w.table)
        assert_same(direct(w.table, Y), oracle.search(w.table, Y), Y)
        yd = to_dev(Y)[1:]   # misaligned view
        out = eos.search_direct(to_dev(w.table), yd)
        torch.cuda.synchronize()
        assert_same(out.cpu().numpy(), oracle.search(w.table, Y[1:]))


@pytest.mark.parametrize("run", [1, 2, 3, 4, 7, 8, 15, 16, 31, 100])
def test_direct_every_block_step_count(run):
    """The zero-setup kernel learns S (in-bin steps) only after building the directory and
    dispatches per CTA to a fixed-S body (S <= 4) or the runtime-S body: tables whose largest
    bin holds `run` equal entries (S = ceil(log2(run + 1))), mixed signs for mode 1, with
    probes at, between and around every entry, bit-exact against the oracle."""
    rng = np.random.default_rng(run)
    for neg in (False, True):
        base = np.sort(10.0 ** rng.uniform(-5, 5, 300))
        X = np.sort(np.concatenate([base, np.full(run - 1, base[137])]))
        if neg:
            X = np.sort(np.concatenate([-X[:40], X[40:]]))
        P = _probes(X)
        P = np.concatenate([P, rng.permutation(np.repeat(P, 5)),
                            10.0 ** rng.uniform(-6, 6, 50_001) * rng.choice([-1.0, 1.0], 50_001)])
        assert_same(direct(X, P), oracle.search(X, P), P)


def test_direct_reports_invalid_tables_and_limits():
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    y = torch.linspace(0, 10, 5000, dtype=torch.float64, device=DEV)
    eos.search_direct(torch.tensor([1.0, 3.0, 2.0], dtype=torch.float64, device=DEV), y, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 4          # EOS_ERR_UNSORTED
    st.zero_()
    eos.search_direct(torch.tensor([1.0, float("nan"), 2.0], dtype=torch.float64, device=DEV), y,
                      status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 3          # EOS_ERR_NONFINITE
    st.zero_()
    eos.search_direct(torch.tensor([1.0, 2.0, 2.0, 5.0], dtype=torch.float64, device=DEV), y,
                      status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    with pytest.raises(eos.EosError) as e:
        eos.search_direct(torch.ones(4097, dtype=torch.float64, device=DEV), y)
    assert e.value.code == 2
    assert_same(direct(np.array([7.0]), np.array([1.0, 7.0, 9.0, np.nan])), np.zeros(4, np.int32))


def test_handles_sharing_a_kernel_do_not_interfere():
    """A big-image table created first, then a small-image one using the same kernel
    instantiation: the first must still launch (the smem limit is per kernel, not per table)."""
    rng = np.random.default_rng(3)
    Xb = np.logspace(-3, 3, 1000)
    Xs = np.logspace(-3, 3, 100)
    big = eos.Table(Xb, log_bins=30000)   # S=1, 16-bit directory, ~68 KB image: 2 x 512 shape
    small = eos.Table(Xs, log_bins=30000)  # S=1, 16-bit directory, ~61 KB: same kernel instantiation
    assert big.info.steps == small.info.steps == 1
    assert big.info.dir_entry_bytes == small.info.dir_entry_bytes == 2
    assert 32 * 1024 < small.info.image_bytes < big.info.image_bytes <= 72 * 1024
    Y = 10.0 ** rng.uniform(-4, 4, 100_003)
    yd = to_dev(Y)
    for t, X in ((big, Xb), (small, Xs), (big, Xb)):
        out = t.search(yd)
        torch.cuda.synchronize()
        assert_same(out.cpu().numpy(), oracle.search(X, Y))
    big.close()
    small.close()


# ------------------------------------------------------ f4: log-log grids ---
def test_loglog_grid_matches_oracle():
    w = datagen.workload("cfg4", count=(1 << 20) + 1)
    rho = w.rho_targets.host_fill(0, w.count)
    T = w.T_targets.host_fill(0, w.count)
    rho[:5] = [np.nan, w.rho[0] / 10, w.rho[-1] * 10, w.rho[5], -1.0]
    T[5:8] = [np.nan, w.T[0] / 10, w.T[-1] * 10]
    g = eos.Grid2D(w.rho, w.T, w.P, loglog=True)
    P, iR, iT, dR, dT = g.interp(to_dev(rho), to_dev(T), derivatives=True)
    P0, _, _ = g.interp(to_dev(rho), to_dev(T))
    torch.cuda.synchronize()
    Pr, iRr, iTr, dRr, dTr = oracle.interp2d_loglog(w.rho, w.T, w.P, rho, T)
    assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
    err = check_interp(P.cpu().numpy(), Pr)
    assert err < 1e-13   # device vs libm log1p/exp: a few ulp
    assert np.array_equal(P0.cpu().numpy(), P.cpu().numpy(), equal_nan=True)
    kr, kt = deriv_cond(w.rho, w.T, w.P, rho, T, iRr, iTr, Pr, True)
    _check_deriv(dR.cpu().numpy(), dRr, kr)
    _check_deriv(dT.cpu().numpy(), dTr, kt)
    g.close()
    with pytest.raises(eos.EosError) as e:
        bad = w.P.copy()
        bad[3, 4] = -1.0
        eos.Grid2D(w.rho, w.T, bad, loglog=True)
    assert e.value.code == 8


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("global_grid", [False, True])
@pytest.mark.parametrize("max_ln_width", [1.0, 0.4, 0.2])
def test_loglog_rough_surfaces_narrow_cells(seed, global_grid, max_ln_width):
    """Log-log grids with no smoothness: every ln G node independent over +-10, axes with
    cells from 1e-4 to `max_ln_width` wide in ln (so |ln G| jumps of ~20 across a 1e-4
    cell).  P within 1e-12 relative of the oracle at every point (R24's log1p form keeps
    both sides well-conditioned), brackets exact, derivatives within their condition
    scale.  max_ln_width 0.2 (every cell ratio <= e^0.2 < 1.25) takes the kernel's
    8-term log1p series (log1p_cell<8>), 0.4 (every ratio <= 1.5) the 12-term one, 1.0
    the general log1p."""
    rng = np.random.default_rng(500 + seed)
    def axis(a, n):
        return np.exp(a + np.cumsum(np.concatenate(
            [[0.0], 10 ** rng.uniform(-4, np.log10(max_ln_width), n - 1)])))
    nR, nT = (int(rng.integers(20, 200)), int(rng.integers(20, 120)))
    R, T = axis(-8.0, nR), axis(2.0, nT)
    G = np.exp(rng.uniform(-10, 10, (nR, nT)))
    m = 1 << 18
    rho = np.exp(rng.uniform(np.log(R[0]) - 0.5, np.log(R[-1]) + 0.5, m))
    tt = np.exp(rng.uniform(np.log(T[0]) - 0.5, np.log(T[-1]) + 0.5, m))
    # targets inside the narrowest cells, at nodes and next to them
    narrow = np.argsort(np.diff(np.log(R)))[:8]
    rho[:800] = np.repeat(R[narrow], 100) * np.exp(rng.uniform(0, 1, 800) * np.repeat(
        np.log(R[narrow + 1] / R[narrow]), 100))
    rho[800:800 + nR], rho[800 + nR:800 + 2 * nR] = R, np.nextafter(R, np.inf)
    tt[-nT:] = T
    rho[-4:] = [np.nan, 0.0, np.inf, -2.0]
    g = eos.Grid2D(R, T, G, loglog=True, global_grid=global_grid)
    P, iR, iT, dR, dT = g.interp(to_dev(rho), to_dev(tt), derivatives=True)
    torch.cuda.synchronize()
    Pr, iRr, iTr, dRr, dTr = oracle.interp2d_loglog(R, T, G, rho, tt)
    assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
    check_interp(P.cpu().numpy(), Pr)
    kr, kt = deriv_cond(R, T, G, rho, tt, iRr, iTr, Pr, True)
    _check_deriv(dR.cpu().numpy(), dRr, kr)
    _check_deriv(dT.cpu().numpy(), dTr, kt)
    g.close()


def test_loglog_host_pipeline():
    w = datagen.workload("cfg4", count=300_007)
    rho = w.rho_targets.host_fill(0, w.count)
    T = w.T_targets.host_fill(0, w.count)
    g = eos.Grid2D(w.rho, w.T, w.P, loglog=True)
    P, iR, iT = g.interp_host(rho, T)
    Pr, iRr, iTr, _, _ = oracle.interp2d_loglog(w.rho, w.T, w.P, rho, T)
    assert np.array_equal(iR, iRr) and np.array_equal(iT, iTr)
    check_interp(P, Pr)
    g.close()


# ------------------------------------- tiered tables -----
# Tables larger than shared memory: smem sample table T1 = X[::8^D] plus D
# 8-ary levels in global memory (eossearch.h eos_search_create_levels).  The
# answer is the same P:54 lower bound for every D; the oracle is unchanged.
def tiered_search(X, Y, levels, k=None, log_bins=None, **kw):
    t = eos.Table(X, k=k, log_bins=log_bins, levels=levels)
    assert t.info.levels == (levels if levels >= 0 else t.info.levels)
    out = t.search(to_dev(Y), **kw)
    torch.cuda.synchronize()
    r = out.cpu().numpy()
    t.close()
    return r


@pytest.mark.parametrize("name", sorted(lower_bound_cases().keys()))
def test_tiered_golden_every_depth(name):
    X, cases = lower_bound_cases()[name]
    ys = np.array([c[0] for c in cases] * 37)
    exp = np.array([c[1] for c in cases] * 37, dtype=np.int32)
    for D in (1, 2, 3, 5):
        assert_same(tiered_search(X, ys, D), exp, ys)


def test_tiered_edge_tables_exhaustive_probes():
    rng = np.random.default_rng(77)
    checked = 0
    for X in _edge_tables(rng, 140):
        P = _probes(X)
        P = np.concatenate([P, rng.permutation(np.repeat(P, 3))])
        ref = oracle.search(X, P)
        for D in (1, 2, 4):
            assert_same(tiered_search(X, P, D), ref, P)
            checked += P.size
    assert checked > 50_000


def _big_table(rng, n, kind):
    if kind == "loguniform":
        return np.sort(10.0 ** rng.uniform(-6, 10, n))
    if kind == "dups":      # runs of equal entries straddling level blocks
        return np.sort(np.repeat(10.0 ** rng.uniform(-3, 3, n // 7 + 1), 7)[:n])
    if kind == "mixed":     # negatives (key mode 1), +-0 and subnormals
        X = np.concatenate([rng.normal(0, 1e3, n - 4), [0.0, -0.0, 5e-324, -5e-324]])
        return np.sort(X)
    if kind == "dense":     # every entry shares its key (upper word) with its neighbours:
        return np.sort(1.0 + rng.uniform(0, 1e-7, n))  # the fp64 tie path at every level
    if kind == "zerohead":  # a 0.0 head, subnormals, then normals (mode 0)
        X = np.concatenate([np.zeros(5), rng.uniform(0, 1e-308, n // 3),
                            10.0 ** rng.uniform(-300, 300, n - 5 - n // 3)])
        return np.sort(X)
    raise KeyError(kind)


def _big_probes(rng, X, m):
    lo, hi = X[0], X[-1]
    j = rng.integers(0, X.size, m // 4)
    pos = X[X > 0]
    a, b = (math.log10(pos[0]), math.log10(pos[-1])) if pos.size else (-300.0, 300.0)
    Y = np.concatenate([
        X[j], np.nextafter(X[j], np.inf), np.nextafter(X[j], -np.inf),
        np.sign(rng.uniform(-1, 1, m // 8)) * 10.0 ** rng.uniform(a - 1, b + 1, m // 8),
        rng.uniform(lo, hi, m // 8) if np.isfinite(hi - lo) else X[j[: m // 8]],
        [np.nan, np.inf, -np.inf, 0.0, -0.0, lo, hi, 5e-324, -5e-324],
    ])
    return rng.permutation(Y)


@pytest.mark.parametrize("n,kind", [(16385, "loguniform"), ((1 << 17) + 3, "dups"),
                                    ((1 << 20), "loguniform"), (300_001, "mixed"),
                                    (70_001, "zerohead"), ((1 << 22) + 12345, "loguniform"),
                                    (200_001, "dense")])
def test_tiered_large_tables_full(n, kind):
    rng = np.random.default_rng(n)
    X = _big_table(rng, n, kind)
    Y = _big_probes(rng, X, 1 << 20)
    ref = oracle.search(X, Y)
    t = eos.Table(X)
    assert t.info.levels >= 1 and t.info.n == n
    out = t.search(to_dev(Y))
    torch.cuda.synchronize()
    assert_same(out.cpu().numpy(), ref, Y)
    # the same answers at a deeper structure and with another hash of T1
    t2 = eos.Table(X, levels=t.info.levels + 1, log_bins=97)
    out2 = t2.search(to_dev(Y))
    torch.cuda.synchronize()
    assert_same(out2.cpu().numpy(), ref, Y)
    t.close()
    t2.close()


def test_tiered_big_workload_full_sampled_and_counters():
    """The bench's `big` workload (n = 2^20, 2^27 targets) in the bench's launch
    configuration (the automatic structure: packed nodes): 2^20 sampled outputs vs the
    oracle, the bracketing invariant on every output, and the counters of the whole
    stream vs the oracle's."""
    w = datagen.workload("big")
    t = eos.Table(w.table)
    assert t.info.levels == 1 and t.info.node_width == 15
    Yd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.targets.device_fill(Yd, 0)
    out = t.search(Yd)
    torch.cuda.synchronize()
    _sampled_check(w, Yd, out)
    invariant_on_device(to_dev(w.table), Yd, out)
    c = torch.zeros(8, dtype=torch.int64, device=DEV)
    out2 = t.search(Yd[: 1 << 24], counters=c)
    torch.cuda.synchronize()
    assert torch.equal(out2, out[: 1 << 24])
    Yh = w.targets.host_fill(0, 1 << 24)
    ref = oracle.counters(w.table, Yh, oracle.search(w.table, Yh), 0)
    assert np.array_equal(c.cpu().numpy().view(np.uint64), ref)
    t.close()


@pytest.mark.parametrize("count", [1, 3, 2049, 65_537])
@pytest.mark.parametrize("y_off,o_off", [(0, 0), (1, 1), (3, 2)])
def test_tiered_ragged_and_misaligned(count, y_off, o_off):
    rng = np.random.default_rng(count)
    X = _big_table(rng, 50_000, "dups")
    Yall = _big_probes(rng, X, count + 64)[: count + 8]
    yd = to_dev(Yall)[y_off:y_off + count]
    od_all = torch.full((count + 8,), -7, dtype=torch.int32, device=DEV)
    od = od_all[o_off:o_off + count]
    t = eos.Table(X)
    t.search(yd, out=od)
    torch.cuda.synchronize()
    got = od_all.cpu().numpy()
    assert_same(got[o_off:o_off + count], oracle.search(X, Yall[y_off:y_off + count]))
    assert np.all(got[:o_off] == -7) and np.all(got[o_off + count:] == -7)
    t.close()


def test_tiered_host_pipeline_and_counters():
    rng = np.random.default_rng(5)
    X = _big_table(rng, 100_000, "loguniform")
    Y = _big_probes(rng, X, 1 << 21)
    ref = oracle.search(X, Y)
    t = eos.Table(X)
    got = t.search_host(np.ascontiguousarray(Y))
    assert_same(got, ref, Y)
    off = 123_456_789
    c = torch.zeros(8, dtype=torch.int64, device=DEV)
    t.search(to_dev(Y), counters=c, global_offset=off)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy().view(np.uint64), oracle.counters(X, Y, ref, off))
    t.close()


# ------------------------------ packed tables (EOS_LEVELS_PACKED, §6.5) -----
# D levels of 15-entry nodes of 16-bit residual keys (one 32-B sector each) under
# a sample table of 16-bit residuals: the same P:54 lower bound, settled exactly
# from the fp64 values wherever residuals tie.
PACKED = eos.EOS_LEVELS_PACKED


def _packed(X, depth=1):
    """depth: exactly that many levels (EOS_LEVELS_PACKED_DEPTH), or None: the fewest
    that fit (EOS_LEVELS_PACKED)."""
    t = eos.Table(X, levels=PACKED if depth is None else eos.EOS_LEVELS_PACKED_DEPTH(depth))
    D = t.info.levels
    assert t.info.node_width == 15 and (depth is None or D == depth)
    assert t.info.top_n == -(-X.size // 15 ** D)
    return t


@pytest.mark.parametrize("depth", [1, 2, 3])
@pytest.mark.parametrize("name", sorted(lower_bound_cases().keys()))
def test_packed_golden(name, depth):
    X, cases = lower_bound_cases()[name]
    ys = np.array([c[0] for c in cases] * 37)
    exp = np.array([c[1] for c in cases] * 37, dtype=np.int32)
    t = _packed(X, depth)
    assert_same(t.search(to_dev(ys)).cpu().numpy(), exp, ys)
    t.close()


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_packed_edge_tables_exhaustive_probes(depth):
    rng = np.random.default_rng(78 + depth)
    checked = 0
    for X in _edge_tables(rng, 140):
        P = _probes(X)
        P = np.concatenate([P, rng.permutation(np.repeat(P, 3))])
        t = _packed(X, depth)
        assert_same(t.search(to_dev(P)).cpu().numpy(), oracle.search(X, P), P)
        t.close()
        checked += P.size
    assert checked > 20_000


def _clustered(rng, n):
    """Tight clusters at log-spread centres: nodes straddle the gaps, so their key
    spans need shifts s_j > 0 and truncated residuals tie often."""
    c = 10.0 ** rng.uniform(-30, 30, n // 40 + 1)
    X = np.repeat(c, 40)[:n] * (1.0 + rng.uniform(0, 1e-9, n))
    X = np.sort(X)
    X[:n // 50] = np.sort(rng.uniform(1e-300, 1e-290, n // 50))
    return np.sort(X)


@pytest.mark.parametrize("n,kind,depth", [((1 << 20), "loguniform", 1), (300_001, "zerohead", 1),
                                          (500_003, "dups", 1), (1_500_001, "loguniform", 1),
                                          (333_337, "clustered", 1), (16_385, "loguniform", 1),
                                          (400_001, "mixed", 1), ((1 << 20), "loguniform", 2),
                                          (4_000_037, "loguniform", None), (500_003, "dups", 3),
                                          (333_337, "clustered", 2), (300_001, "zerohead", 4),
                                          (400_001, "dense", None)])
def test_packed_large_tables_full(n, kind, depth):
    rng = np.random.default_rng(n + 1)
    X = _clustered(rng, n) if kind == "clustered" else _big_table(rng, n, kind)
    Y = _big_probes(rng, X, 1 << 20)
    ref = oracle.search(X, Y)
    try:
        t = _packed(X, depth)
    except eos.EosError as e:  # the sample table does not fit at this depth: AUTO's choice
        assert "UNSUPPORTED" in str(e) and kind in ("mixed", "zerohead"), e
        t = eos.Table(X)
        assert t.info.node_width == 8 or t.info.levels > depth
    out = t.search(to_dev(Y))
    torch.cuda.synchronize()
    assert_same(out.cpu().numpy(), ref, Y)
    c = torch.zeros(8, dtype=torch.int64, device=DEV)
    t.search(to_dev(Y[: 1 << 18]), counters=c, global_offset=12345)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy().view(np.uint64),
                          oracle.counters(X, Y[: 1 << 18], ref[: 1 << 18], 12345))
    t.close()


@pytest.mark.parametrize("count", [1, 3, 2049, 65_537, 300_001])
@pytest.mark.parametrize("y_off,o_off,depth", [(0, 0, 1), (1, 1, 1), (3, 2, 1), (1, 1, 2)])
def test_packed_ragged_misaligned_and_small_launches(count, y_off, o_off, depth):
    rng = np.random.default_rng(count + 3)
    X = _big_table(rng, 400_000, "loguniform")
    Yall = _big_probes(rng, X, count + 64)[: count + 8]
    yd = to_dev(Yall)[y_off:y_off + count]
    od_all = torch.full((count + 8,), -7, dtype=torch.int32, device=DEV)
    od = od_all[o_off:o_off + count]
    t = _packed(X, depth)
    t.search(yd, out=od)
    torch.cuda.synchronize()
    got = od_all.cpu().numpy()
    assert_same(got[o_off:o_off + count], oracle.search(X, Yall[y_off:y_off + count]))
    assert np.all(got[:o_off] == -7) and np.all(got[o_off + count:] == -7)
    t.close()


def test_packed_host_pipeline():
    rng = np.random.default_rng(6)
    X = _big_table(rng, 700_001, "loguniform")
    Y = _big_probes(rng, X, 1 << 21)
    t = _packed(X)
    assert_same(t.search_host(np.ascontiguousarray(Y)), oracle.search(X, Y), Y)
    t.close()


# ------------------------------------ maximum sizes and deep bins (S > 8) ---
@pytest.mark.parametrize("kind", ["all_equal", "three_values", "max_random", "dup_runs"])
def test_max_table_and_runtime_steps(kind):
    """n = EOS_MAX_TABLE (16384) tables, including bins deeper than the
    template steps (S > 8: the runtime-S instantiation, kernels.cuh lookup<0>)."""
    rng = np.random.default_rng(len(kind))
    n = eos.EOS_MAX_TABLE
    if kind == "all_equal":
        X = np.full(n, 3.0)
    elif kind == "three_values":
        X = np.sort(rng.choice([0.5, 2.0, 1e3], n))
    elif kind == "max_random":
        X = np.sort(10.0 ** rng.uniform(-8, 8, n))
    else:
        X = np.sort(np.repeat(10.0 ** rng.uniform(-2, 2, n // 300 + 1), 300)[:n])
    Y = _big_probes(rng, X, 1 << 19)
    ref = oracle.search(X, Y)
    for k in feasible_ks(X, [None, 0, 3]):
        t = eos.Table(X, k=k)
        if kind in ("all_equal", "three_values", "dup_runs"):
            assert t.info.steps > 8
        out = t.search(to_dev(Y))
        torch.cuda.synchronize()
        assert_same(out.cpu().numpy(), ref, Y)
        c = torch.zeros(8, dtype=torch.int64, device=DEV)
        t.search(to_dev(Y), counters=c, global_offset=7)
        torch.cuda.synchronize()
        assert np.array_equal(c.cpu().numpy().view(np.uint64), oracle.counters(X, Y, ref, 7))
        t.close()
    # the same tables tiered (the sample table inherits the deep bins)
    assert_same(tiered_search(X, Y, 2), ref, Y)


# ------------------------------ 2-D regular axes, node and near-node targets --
@pytest.mark.parametrize("axes", ["logspace", "linspace", "mixed", "perturbed"])
@pytest.mark.parametrize("loglog", [False, True])
def test_interp_regular_axes_node_targets(axes, loglog):
    """Logspace / linspace axes (the EOSPAC table shapes) with targets at, just below
    and just above every node, out of range and special values: brackets equal the
    oracle's, values within the 1e-12 bar, derivative and plain kernels agree."""
    rng = np.random.default_rng(sum(map(ord, axes)))
    if axes == "logspace":
        R, T = np.logspace(-6, 3, 200), np.logspace(0, 8, 100)
    elif axes == "linspace":
        R, T = np.linspace(0.5, 50.0, 150), np.linspace(1.0, 2.0, 77)
    elif axes == "mixed":
        R, T = np.logspace(-3, 3, 120), np.linspace(10.0, 1e4, 90)
    else:  # nodes moved by up to 0.1%
        R = np.logspace(-2, 2, 64) * (1 + 0.001 * rng.uniform(-1, 1, 64))
        T = np.logspace(1, 5, 50)
    G = np.exp(rng.uniform(0.0, 3.0, (R.size, T.size)))
    m = 1 << 18
    rho = 10 ** rng.uniform(np.log10(R[0]) - 0.5, np.log10(R[-1]) + 0.5, m)
    tt = 10 ** rng.uniform(np.log10(T[0]) - 0.5, np.log10(T[-1]) + 0.5, m)
    k = R.size
    rho[:k], rho[k:2 * k], rho[2 * k:3 * k] = R, np.nextafter(R, 0), np.nextafter(R, np.inf)
    kt = T.size
    tt[-kt:], tt[-2 * kt:-kt], tt[-3 * kt:-2 * kt] = T, np.nextafter(T, 0), np.nextafter(T, np.inf)
    rho[3 * k:3 * k + 6] = [np.nan, np.inf, -np.inf, 0.0, -0.0, -1.0]
    tt[3 * k + 6:3 * k + 12] = [np.nan, np.inf, -np.inf, 0.0, -0.0, -1.0]
    g = eos.Grid2D(R, T, G, loglog=loglog)
    # regular axes take fitted cell maps (1: log, 2: linear), both axes or neither
    assert (g.rho_info.cell_map, g.T_info.cell_map) == {
        "logspace": (1, 1), "linspace": (2, 2), "mixed": (1, 2), "perturbed": (1, 1)}[axes]
    P, iR, iT, dR, dT = g.interp(to_dev(rho), to_dev(tt), derivatives=True)
    P0, iR0, iT0 = g.interp(to_dev(rho), to_dev(tt))
    torch.cuda.synchronize()
    assert np.array_equal(P.cpu().numpy(), P0.cpu().numpy(), equal_nan=True)
    assert torch.equal(iR, iR0) and torch.equal(iT, iT0)
    if loglog:
        Pr, iRr, iTr, dRr, dTr = oracle.interp2d_loglog(R, T, G, rho, tt)
    else:
        Pr, iRr, iTr = oracle.interp2d(R, T, G, rho, tt)
        dRr, dTr = oracle.interp2d_deriv(R, T, G, rho, tt)
    assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
    check_interp(P.cpu().numpy(), Pr)
    kr, kt = deriv_cond(R, T, G, rho, tt, iRr, iTr, Pr, loglog)
    _check_deriv(dR.cpu().numpy(), dRr, kr)
    _check_deriv(dT.cpu().numpy(), dTr, kt)
    g.close()


def _near_node_targets(rng, X, m):
    """m targets: random in range and beyond, every node, its neighbours one ulp away,
    and points within 1e-7 relative below each node (where a fitted map is near the top
    of its unit)."""
    n = X.size
    lo, hi = (np.log(X[0]), np.log(X[-1])) if X[0] > 0 else (None, None)
    y = (np.exp(rng.uniform(lo - 0.3, hi + 0.3, m)) if lo is not None
         else rng.uniform(X[0] - 0.1 * (X[-1] - X[0]), X[-1] + 0.1 * (X[-1] - X[0]), m))
    k = 0
    for part in (X, np.nextafter(X, -np.inf), np.nextafter(X, np.inf),
                 X - np.abs(X) * rng.uniform(0, 1e-7, n)):
        y[k:k + n] = part
        k += n
    return y


@pytest.mark.parametrize("loglog,global_grid", [(False, False), (True, False), (False, True),
                                                (True, True)])
def test_cell_map_equals_directory_lookup_cfg4(loglog, global_grid):
    """cfg4's log-spaced axes take the fitted log map; the mapped kernels give results
    bit-identical to the directory kernels (EOS_GRID_DIRECTORY) -- P, brackets and both
    derivatives -- on random, node, near-node and special targets, and the brackets
    equal the oracle's."""
    w = datagen.workload("cfg4", count=1 << 20)
    rng = np.random.default_rng(44)
    rho = np.concatenate([w.rho_targets.host_fill(0, w.count), _near_node_targets(rng, w.rho, 4096)])
    tt = np.concatenate([w.T_targets.host_fill(0, w.count), _near_node_targets(rng, w.T, 4096)])
    tt[-4096:] = tt[-4096:][rng.permutation(4096)]
    rho[:8] = [np.nan, np.inf, -np.inf, 0.0, -0.0, -1.0, 5e-324, 1e308]
    tt[8:16] = [np.nan, np.inf, -np.inf, 0.0, -0.0, -1.0, 5e-324, 1e308]
    gm = eos.Grid2D(w.rho, w.T, w.P, loglog=loglog, global_grid=global_grid)
    gd = eos.Grid2D(w.rho, w.T, w.P, loglog=loglog, global_grid=global_grid, directory=True)
    assert (gm.rho_info.cell_map, gm.T_info.cell_map) == (1, 1)
    assert (gd.rho_info.cell_map, gd.T_info.cell_map) == (0, 0)
    outs = []
    for g in (gm, gd):
        outs.append([t.cpu().numpy() for t in g.interp(to_dev(rho), to_dev(tt), derivatives=True)])
        outs.append([t.cpu().numpy() for t in g.interp(to_dev(rho), to_dev(tt))])
    for a, b in zip(outs[0] + outs[1], outs[2] + outs[3]):
        assert np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                              b.view(np.uint64) if b.dtype == np.float64 else b)
    iRr, iTr = oracle.search(w.rho, rho), oracle.search(w.T, tt)
    assert np.array_equal(outs[0][1], iRr) and np.array_equal(outs[0][2], iTr)
    gm.close()
    gd.close()


@pytest.mark.parametrize("dev", [0.2, 0.45, 0.49, 0.7])
@pytest.mark.parametrize("kind", ["log", "linear"])
def test_cell_map_near_its_acceptance_bound(dev, kind):
    """Axes whose nodes drift off a regular grid by up to 2 dev cells (0 at the ends,
    the most in the middle, plus an alternating +-dev/4 jitter): the fitted map is
    accepted while the nodes' spread leaves room for the device error bound (dev <=
    0.49) and refused above (0.7); either way brackets equal the oracle's and P is
    within the bar, including targets at the nodes, one ulp around them and within
    1e-7 below them."""
    rng = np.random.default_rng(int(dev * 100) + (kind == "log"))
    def axis(n, a, b):
        j = np.arange(n)
        wob = np.sin(np.pi * j / (n - 1))
        u = j + (2 * dev - dev / 2) * wob + dev / 4 * np.where(j % 2 == 0, -1.0, 1.0) * wob
        u[0], u[-1] = 0.0, n - 1.0
        return np.exp(a + (b - a) * u / (n - 1)) if kind == "log" else a + (b - a) * u / (n - 1)
    R, T = axis(150, -5.0, 4.0), axis(90, 0.5, 9.0)
    G = rng.uniform(1.0, 2.0, (R.size, T.size))
    m = 1 << 18
    rho, tt = _near_node_targets(rng, R, m), _near_node_targets(rng, T, m)
    tt = tt[rng.permutation(m)]
    g = eos.Grid2D(R, T, G)
    want = (1 if kind == "log" else 2) if dev < 0.5 else 0
    assert (g.rho_info.cell_map, g.T_info.cell_map) == (want, want)
    P, iR, iT = g.interp(to_dev(rho), to_dev(tt))
    torch.cuda.synchronize()
    Pr, iRr, iTr = oracle.interp2d(R, T, G, rho, tt)
    assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
    check_interp(P.cpu().numpy(), Pr)
    g.close()


# --------------------------------------- streams, host threads, CUDA graphs --
def test_concurrent_streams_and_host_threads_share_handles():
    """Handles are immutable (eossearch.h): concurrent calls on one table / grid
    from several host threads, each on its own stream, give the oracle's answers."""
    import threading
    w = datagen.workload("cfg2", count=1 << 20)
    g4 = datagen.workload("cfg4", count=1 << 18)
    tab = eos.Table(w.table)
    big = eos.Table(datagen.table_big(6))
    grid = eos.Grid2D(g4.rho, g4.T, g4.P)
    jobs, errors = [], []
    for j in range(6):
        Y = w.targets.host_fill(j * w.count, w.count, w.table)
        rho = g4.rho_targets.host_fill(j * g4.count, g4.count)
        T = g4.T_targets.host_fill(j * g4.count, g4.count)
        jobs.append((Y, rho, T))

    def run(j):
        try:
            Y, rho, T = jobs[j]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                yd, rd, td = to_dev(Y), to_dev(rho), to_dev(T)
                outs = []
                for _ in range(3):
                    outs.append((tab.search(yd, stream=s), big.search(yd, stream=s),
                                 grid.interp(rd, td, stream=s)))
            s.synchronize()
            ref = oracle.search(w.table, Y)
            refb = oracle.search(big.X, Y)
            Pr, iRr, iTr = oracle.interp2d(g4.rho, g4.T, g4.P, rho, T)
            for a, b, (P, iR, iT) in outs:
                assert_same(a.cpu().numpy(), ref, Y)
                assert_same(b.cpu().numpy(), refb, Y)
                assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
                check_interp(P.cpu().numpy(), Pr)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=run, args=(j,)) for j in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[0]
    tab.close()
    big.close()
    grid.close()


def test_cuda_graph_capture_and_replay():
    """eos_search / eos_interp2d launches (programmatic dependent launch included)
    captured into a CUDA graph and replayed over changing inputs."""
    w = datagen.workload("cfg5", count=(1 << 20) + 3)
    g4 = datagen.workload("cfg4", count=(1 << 18) + 1)
    tab = eos.Table(w.table)
    big = eos.Table(datagen.table_big(6))
    grid = eos.Grid2D(g4.rho, g4.T, g4.P)
    Yd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    Rd = torch.empty(g4.count, dtype=torch.float64, device=DEV)
    Td = torch.empty(g4.count, dtype=torch.float64, device=DEV)
    o1 = torch.empty(w.count, dtype=torch.int32, device=DEV)
    o2 = torch.empty(w.count, dtype=torch.int32, device=DEV)
    P = torch.empty(g4.count, dtype=torch.float64, device=DEV)
    iR = torch.empty(g4.count, dtype=torch.int32, device=DEV)
    iT = torch.empty(g4.count, dtype=torch.int32, device=DEV)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(2):
            tab.search(Yd, out=o1, stream=s)
            big.search(Yd, out=o2, stream=s)
            grid.interp(Rd, Td, P_out=P, irho_out=iR, iT_out=iT, stream=s)
    for rep in range(3):
        Y = w.targets.host_fill(rep * w.count, w.count, w.table)
        rho = g4.rho_targets.host_fill(rep * g4.count, g4.count)
        T = g4.T_targets.host_fill(rep * g4.count, g4.count)
        Yd.copy_(torch.from_numpy(Y))
        Rd.copy_(torch.from_numpy(rho))
        Td.copy_(torch.from_numpy(T))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert_same(o1.cpu().numpy(), oracle.search(w.table, Y), Y)
        assert_same(o2.cpu().numpy(), oracle.search(big.X, Y), Y)
        Pr, iRr, iTr = oracle.interp2d(g4.rho, g4.T, g4.P, rho, T)
        assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
        check_interp(P.cpu().numpy(), Pr)
    tab.close()
    big.close()
    grid.close()


# ------------------------- 2-D grids in device memory (EOS_GRID_GLOBAL) -----
@pytest.mark.parametrize("loglog", [False, True])
def test_global_grid_cfg4_matches_shared_and_oracle(loglog):
    """The cfg4 grid forced into device memory (cell quads) gives the shared-memory
    kernel's brackets and values (same arithmetic), hence the oracle's."""
    w = datagen.workload("cfg4", count=(1 << 20) + 7)
    rho = w.rho_targets.host_fill(0, w.count)
    T = w.T_targets.host_fill(0, w.count)
    rho[:3] = [np.nan, w.rho[0] / 3, w.rho[-1] * 3]
    T[3:6] = [np.nan, w.T[0] / 3, w.T[-1] * 3]
    rho[6:6 + w.rho.size] = w.rho
    gs = eos.Grid2D(w.rho, w.T, w.P, loglog=loglog)
    gg = eos.Grid2D(w.rho, w.T, w.P, loglog=loglog, global_grid=True)
    a = gs.interp(to_dev(rho), to_dev(T), derivatives=True)
    b = gg.interp(to_dev(rho), to_dev(T), derivatives=True)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert np.array_equal(x.cpu().numpy(), y.cpu().numpy(), equal_nan=True)
    ref = (oracle.interp2d_loglog if loglog else oracle.interp2d)(w.rho, w.T, w.P, rho, T)
    assert np.array_equal(b[1].cpu().numpy(), ref[1]) and np.array_equal(b[2].cpu().numpy(), ref[2])
    check_interp(b[0].cpu().numpy(), ref[0])
    gs.close()
    gg.close()


@pytest.mark.parametrize("shape,loglog", [
    ((600, 500), False), ((600, 500), True), ((1000, 800), False),
    ((3000, 7), False), ((2, 16000), False), ((8000, 3), True)])
def test_large_grids_in_device_memory(shape, loglog):
    """Grids larger than shared memory (P in device memory as cell quads; axes in smem
    with as many record copies as fit): brackets bit-exact, P and derivatives within the
    bar."""
    rng = np.random.default_rng(shape[0] + shape[1])
    nR, nT = shape
    R = np.sort(np.unique(10 ** rng.uniform(-4, 4, nR)))
    T = np.sort(np.unique(10 ** rng.uniform(0, 6, nT)))
    while R.size < nR or T.size < nT:   # redraw on (unlikely) duplicates
        R = np.sort(np.unique(10 ** rng.uniform(-4, 4, nR)))
        T = np.sort(np.unique(10 ** rng.uniform(0, 6, nT)))
    # a rough surface: every node independent over 4 decades (also for log-log grids)
    G = np.exp(rng.uniform(-5, 5, (nR, nT)))
    m = 1 << 19
    rho = 10 ** rng.uniform(-4.3, 4.3, m)
    tt = 10 ** rng.uniform(-0.3, 6.3, m)
    rho[:nR // 4] = R[: nR // 4]
    tt[-(nT // 4 or 1):] = T[-(nT // 4 or 1):]
    rho[nR:nR + 4] = [np.nan, np.inf, 0.0, -1.0]
    g = eos.Grid2D(R, T, G, loglog=loglog)
    P, iR, iT, dR, dT = g.interp(to_dev(rho), to_dev(tt), derivatives=True)
    P0, _, _ = g.interp(to_dev(rho), to_dev(tt))
    torch.cuda.synchronize()
    if loglog:
        Pr, iRr, iTr, dRr, dTr = oracle.interp2d_loglog(R, T, G, rho, tt)
    else:
        Pr, iRr, iTr = oracle.interp2d(R, T, G, rho, tt)
        dRr, dTr = oracle.interp2d_deriv(R, T, G, rho, tt)
    assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
    check_interp(P.cpu().numpy(), Pr)
    assert np.array_equal(P0.cpu().numpy(), P.cpu().numpy(), equal_nan=True)
    kr, kt = deriv_cond(R, T, G, rho, tt, iRr, iTr, Pr, loglog)
    _check_deriv(dR.cpu().numpy(), dRr, kr)
    _check_deriv(dT.cpu().numpy(), dTr, kt)
    g.close()


# ------------------------------------------------ the ABI from plain C -------
def test_plain_c_program_uses_the_abi(tmp_path):
    """examples/c_abi_example.c (gcc, libcudart, no Python on the call path) creates a
    table, searches a device batch and the host-buffer path, and interpolates a grid."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2112_03229_b200", "lib")
    exe = tmp_path / "c_abi_example"
    subprocess.run(["gcc", "-std=c11", "-O2", "-I", os.path.join(root, "include"),
                    "-I", "/usr/local/cuda/include", os.path.join(root, "examples", "c_abi_example.c"),
                    "-L", lib, "-leossearch", "-L", "/usr/local/cuda/lib64", "-lcudart",
                    "-o", str(exe)], check=True)
    env = dict(os.environ, LD_LIBRARY_PATH=lib + ":/usr/local/cuda/lib64:"
               + os.environ.get("LD_LIBRARY_PATH", ""))
    for X in (datagen.table_cfg2(1), datagen.table_big(6)):   # single-level and tiered
        w = datagen.loguniform_over(X, 11)
        Y = w.host_fill(0, (1 << 20) + 5)
        Y[:6] = [np.nan, np.inf, -np.inf, -0.0, X[0], X[-1]]
        (tmp_path / "t.f64").write_bytes(X.tobytes())
        (tmp_path / "y.f64").write_bytes(Y.tobytes())
        r = subprocess.run([str(exe), str(tmp_path / "t.f64"), str(tmp_path / "y.f64"),
                            str(tmp_path / "i.i32"), str(tmp_path / "h.i32")],
                           env=env, capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        ref = oracle.search(X, Y)
        assert_same(np.frombuffer((tmp_path / "i.i32").read_bytes(), dtype=np.int32), ref, Y)
        assert_same(np.frombuffer((tmp_path / "h.i32").read_bytes(), dtype=np.int32), ref, Y)


def test_paper_shaped_run_full_bit_exact():
    """The paper-shaped run (R17): n = 110 log-spaced over [3e-6, 5.4e4],
    5e6 targets log-uniform over 1e-10..1e10 (about half out of range), in full."""
    w = datagen.workload("paper")
    Yd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.targets.device_fill(Yd, 0)
    t = eos.Table(w.table)
    out = t.search(Yd)
    torch.cuda.synchronize()
    Y = w.targets.host_fill(0, w.count)
    assert np.array_equal(Yd.cpu().numpy(), Y)
    ref = oracle.search(w.table, Y)
    assert_same(out.cpu().numpy(), ref, Y)
    inside = np.mean((Y >= w.table[0]) & (Y <= w.table[-1]))
    assert 0.45 < inside < 0.55
    t.close()
