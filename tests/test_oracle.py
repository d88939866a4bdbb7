"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: the paper's definition worked
by hand (golden files), brute force on tiny inputs, a library routine
(numpy / bisect / scipy), closed forms, or invariants.
"""
import bisect
import math

import numpy as np
import pytest

import oracle
from tests._golden import interp_cases, lower_bound_cases

SPECIALS = [0.0, -0.0, math.inf, -math.inf, math.nan, 5e-324, 2.2250738585072014e-308,
            math.nextafter(2.2250738585072014e-308, 0.0), 1e-300, 1e300, -1.0, 1.0, 2.0, 0.5]


def brute_force(X, y):
    """Linear count straight from P:54: last element <= y, 0 if none."""
    c = 0
    for x in X:
        if x <= y:
            c += 1
    return max(c - 1, 0)


def probes_for(X):
    p = list(SPECIALS)
    for x in X:
        p += [x, math.nextafter(x, math.inf), math.nextafter(x, -math.inf)]
        if x > 0:
            e = math.floor(math.log2(x))
            p += [2.0 ** e, math.nextafter(2.0 ** e, 0.0), 2.0 ** (e + 1)]
    for a, b in zip(X[:-1], X[1:]):
        p.append(0.5 * (a + b))
    return np.array(p, dtype=np.float64)


# ---------------------------------------------------------------- golden ----
@pytest.mark.parametrize("name", sorted(lower_bound_cases().keys()))
def test_golden_lower_bound(name):
    X, cases = lower_bound_cases()[name]
    ys = np.array([c[0] for c in cases])
    exp = np.array([c[1] for c in cases], dtype=np.int32)
    got = oracle.search(X, ys)
    assert got.tolist() == exp.tolist(), list(zip(ys.tolist(), got.tolist(), exp.tolist()))
    for y, e in cases:
        assert oracle.lower_bound(X, y) == e


# ------------------------------------------------------------ brute force ---
def _random_tables(rng, count):
    for t in range(count):
        n = int(rng.integers(1, 13))
        kind = t % 6
        if kind == 0:      # log-uniform
            X = 10.0 ** rng.uniform(-8, 8, n)
        elif kind == 1:    # exact powers of two
            X = 2.0 ** rng.integers(-20, 20, n).astype(np.float64)
        elif kind == 2:    # zero head + subnormals
            X = np.concatenate([[0.0], rng.uniform(0, 1, n) * 1e-310, 10.0 ** rng.uniform(-5, 5, n)])
        elif kind == 3:    # dense cluster with duplicates
            X = np.round(rng.uniform(1.0, 1.01, n), 3)
        elif kind == 4:    # mixed sign with zeros
            X = np.concatenate([rng.normal(0, 10, n), [0.0, -0.0]])
        else:              # heavy duplicates
            X = rng.choice([1.0, 2.0, 3.0], n)
        yield np.sort(X)


def test_brute_force_exhaustive_tiny_tables():
    rng = np.random.default_rng(12345)
    total = 0
    for X in _random_tables(rng, 600):
        P = probes_for(X)
        got = oracle.search(X, P, threads=1)
        exp = [brute_force(X, y) for y in P]
        assert got.tolist() == exp, X
        total += P.size
    assert total > 20000


def test_every_probe_of_every_prefix_table():
    """Exhaustive over all prefixes of a fixed table containing every hazard."""
    base = [0.0, 5e-324, 1e-310, 2.2250738585072014e-308, 0.25, 0.5, 0.5, 1.0, 1.5, 2.0, 3.0,
            3.0, 3.0, 8.0, 1e300]
    for n in range(1, len(base) + 1):
        X = np.array(base[:n])
        P = probes_for(X)
        assert oracle.search(X, P, threads=1).tolist() == [brute_force(X, y) for y in P]


# --------------------------------------------------------- library routine --
def test_numpy_searchsorted_and_bisect_nan_masked():
    import datagen
    w = datagen.workload("cfg1")
    X = w.table
    Y = w.targets.host_fill(0, w.count, X)
    Y[::997] = np.nan
    got = oracle.search(X, Y)
    ref = np.clip(np.searchsorted(X, Y, side="right") - 1, 0, None)
    nan = np.isnan(Y)
    assert np.array_equal(got[~nan], ref[~nan])
    assert np.all(got[nan] == 0)          # reading R4 (numpy would say n-1)
    for y in Y[:2000]:
        if not math.isnan(y):
            assert oracle.lower_bound(X, y) == max(bisect.bisect_right(list(X), y) - 1, 0)


def test_bracketing_invariant_all_outputs():
    import datagen
    for name in ("cfg1", "paper"):
        w = datagen.workload(name, count=200_000)
        X = w.table
        Y = w.targets.host_fill(0, w.count, X)
        idx = oracle.search(X, Y).astype(np.int64)
        n = X.size
        inr = Y >= X[0]
        assert np.all(idx[~inr] == 0)
        i = idx[inr]
        y = Y[inr]
        assert np.all(X[i] <= y)
        assert np.all((i == n - 1) | (y < X[np.minimum(i + 1, n - 1)]))


def test_permutation_invariance():
    rng = np.random.default_rng(7)
    X = np.sort(10.0 ** rng.uniform(-6, 3, 300))
    Y = 10.0 ** rng.uniform(-7, 4, 50_000)
    perm = rng.permutation(Y.size)
    assert np.array_equal(oracle.search(X, Y)[perm], oracle.search(X, Y[perm]))


def test_threads_do_not_change_result():
    rng = np.random.default_rng(8)
    X = np.sort(rng.uniform(0, 1, 1000))
    Y = rng.uniform(-0.1, 1.1, 300_001)
    assert np.array_equal(oracle.search(X, Y, threads=1), oracle.search(X, Y, threads=7))


# ---------------------------------------------------------- interpolation ---
def test_golden_interp2d():
    R, T, G, cases = interp_cases()
    rho = np.array([c[0] for c in cases])
    t = np.array([c[1] for c in cases])
    P, iR, iT = oracle.interp2d(R, T, G, rho, t)
    for k, (r, tt, p, i, j) in enumerate(cases):
        assert P[k] == p, (r, tt, P[k], p)
        assert (iR[k], iT[k]) == (i, j)


def _axes(rng, nr=37, nt=23):
    R = np.sort(10.0 ** rng.uniform(-6, 3, nr))
    T = np.sort(10.0 ** rng.uniform(0, 8, nt))
    assert np.all(np.diff(R) > 0) and np.all(np.diff(T) > 0)
    return R, T


def test_interp_reproduces_bilinear_closed_form():
    rng = np.random.default_rng(1)
    R, T = _axes(rng)
    a, b, c, d = 3.0, 0.7, 1.3e-4, 2.1e-7
    G = a + b * R[:, None] + c * T[None, :] + d * R[:, None] * T[None, :]
    rho = 10.0 ** rng.uniform(np.log10(R[0]), np.log10(R[-1]), 20000)
    tt = 10.0 ** rng.uniform(np.log10(T[0]), np.log10(T[-1]), 20000)
    rho = np.clip(rho, R[0], R[-1])
    tt = np.clip(tt, T[0], T[-1])
    P, _, _ = oracle.interp2d(R, T, G, rho, tt)
    exact = a + b * rho + c * tt + d * rho * tt
    assert np.max(np.abs(P - exact) / np.abs(exact)) < 1e-12


def test_interp_nodes_exact_and_1d_reduction():
    rng = np.random.default_rng(2)
    R, T = _axes(rng)
    G = rng.uniform(1.0, 5.0, (R.size, T.size))
    rr, tt = np.meshgrid(R, T, indexing="ij")
    P, iR, iT = oracle.interp2d(R, T, G, rr.ravel(), tt.ravel())
    assert np.array_equal(P, G.ravel())
    assert np.array_equal(iR, np.repeat(np.arange(R.size), T.size))
    # G depending on rho only -> 1-D linear interpolation (np.interp clamps the same way)
    g1 = rng.uniform(1.0, 5.0, R.size)
    G1 = np.repeat(g1[:, None], T.size, axis=1)
    rho = 10.0 ** rng.uniform(-7, 4, 30000)
    t = 10.0 ** rng.uniform(-1, 9, 30000)
    P1, _, _ = oracle.interp2d(R, T, G1, rho, t)
    assert np.max(np.abs(P1 - np.interp(rho, R, g1)) / np.abs(P1)) < 1e-13


def test_interp_scipy_and_convex_hull():
    from scipy.interpolate import RegularGridInterpolator
    import datagen
    w = datagen.workload("cfg4", count=100_000)
    rho = w.rho_targets.host_fill(0, w.count)
    t = w.T_targets.host_fill(0, w.count)
    rho = np.clip(rho, w.rho[0], w.rho[-1])
    t = np.clip(t, w.T[0], w.T[-1])
    P, iR, iT = oracle.interp2d(w.rho, w.T, w.P, rho, t)
    ref = RegularGridInterpolator((w.rho, w.T), w.P, method="linear")(np.stack([rho, t], 1))
    assert np.max(np.abs(P - ref) / np.abs(ref)) < 1e-12
    ci = np.minimum(iR, w.rho.size - 2)
    cj = np.minimum(iT, w.T.size - 2)
    corners = np.stack([w.P[ci, cj], w.P[ci, cj + 1], w.P[ci + 1, cj], w.P[ci + 1, cj + 1]])
    lo, hi = corners.min(0), corners.max(0)
    assert np.all(P >= lo * (1 - 1e-15)) and np.all(P <= hi * (1 + 1e-15))


def test_interp_nan_propagates_bracket_zero():
    R, T, G, _ = interp_cases()
    P, iR, iT = oracle.interp2d(R, T, G, np.array([np.nan, 1.5]), np.array([15.0, np.nan]))
    assert np.isnan(P).all()
    assert iR.tolist() == [0, 0] and iT.tolist() == [0, 0]


# --------------------------------------------------------------- counters ---
def _mix64_np(z):
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def test_mix64_published_splitmix64_vectors():
    """oracle_mix64 reproduces the published splitmix64 streams (tests/golden/
    splitmix64_vectors.txt): output k of seed s = mix64(s + k * golden gamma)."""
    import os
    gamma = 0x9E3779B97F4A7C15
    n = 0
    with open(os.path.join(os.path.dirname(__file__), "golden", "splitmix64_vectors.txt")) as f:
        for raw in f:
            tok = raw.split("#", 1)[0].split()
            if not tok:
                continue
            assert tok[0] == "seed"
            s = int(tok[1], 0)
            for k, want in enumerate(tok[2:], start=1):
                assert oracle.mix64((s + k * gamma) & 0xFFFFFFFFFFFFFFFF) == int(want, 0)
                n += 1
    assert n == 8


def test_counter_c2_distinguishes_position_and_index_at_large_n():
    """R25: c2's term mix64(mix64(pos) ^ idx) differs for different indices at the same
    position, also past 2^20 entries and positions (the round-1 packing (pos << 20) | idx
    aliased there)."""
    X = np.arange((1 << 21) + 2, dtype=np.float64)   # indices up to 2^21 are valid
    pos = (1 << 33) + 5
    y = np.array([1.5])
    a = oracle.counters(X, y, np.array([1 << 21], np.int32), pos)[2]
    b = oracle.counters(X, y, np.array([0], np.int32), pos)[2]
    c = oracle.counters(X, y, np.array([0], np.int32), pos + (1 << 1))[2]
    assert len({int(a), int(b), int(c)}) == 3
    assert int(b) == oracle.mix64(oracle.mix64(pos) ^ 0)


def test_counters_match_definitions():
    rng = np.random.default_rng(3)
    X = np.sort(10.0 ** rng.uniform(-3, 3, 100))
    Y = 10.0 ** rng.uniform(-4, 4, 10000)
    Y[::50] = np.nan
    Y[1::77] = X[rng.integers(0, X.size, Y[1::77].size)]
    idx = oracle.search(X, Y)
    off = 123456789
    c = oracle.counters(X, Y, idx, off)
    pos = np.arange(Y.size, dtype=np.uint64) + np.uint64(off)
    with np.errstate(over="ignore"):
        c2 = np.sum(_mix64_np(_mix64_np(pos) ^ idx.astype(np.uint64)), dtype=np.uint64)
    assert c[0] == Y.size
    assert c[1] == idx.astype(np.uint64).sum()
    assert c[2] == c2
    assert c[3] == np.sum(~(Y >= X[0]))
    assert c[4] == np.sum(Y > X[-1])
    assert c[5] == np.sum(np.isnan(Y))
    assert c[6] == np.sum(Y == X[idx])
    assert c[7] == 0
    # shard additivity (what the NCCL all_reduce relies on)
    h = 4321
    c_a = oracle.counters(X, Y[:h], idx[:h], off)
    c_b = oracle.counters(X, Y[h:], idx[h:], off + h)
    with np.errstate(over="ignore"):
        assert np.array_equal(c_a + c_b, c)


# ----------------------------------------------------- interp derivatives ---
def test_interp_derivatives_closed_form_and_outside():
    """For G = a + b*rho + c*T + d*rho*T the bilinear interpolant is exact, so its
    derivatives are b + d*T and c + d*rho inside the grid; outside an axis range the
    clamped interpolant is constant along it (derivative 0); NaN propagates (R23)."""
    rng = np.random.default_rng(4)
    # well-conditioned axes: a difference quotient loses ~log10(|G| / |dG|) digits
    R = np.unique(rng.uniform(1.0, 10.0, 37))
    T = np.unique(rng.uniform(1.0, 10.0, 23))
    a, b, c, d = 3.0, 0.7, -1.3, 0.21
    G = a + b * R[:, None] + c * T[None, :] + d * R[:, None] * T[None, :]
    rho = rng.uniform(R[0], R[-1], 20000)
    t = rng.uniform(T[0], T[-1], 20000)
    dr, dt = oracle.interp2d_deriv(R, T, G, rho, t)
    assert np.max(np.abs(dr - (b + d * t))) < 1e-12
    assert np.max(np.abs(dt - (c + d * rho))) < 1e-12
    out = np.array([R[0] / 2, R[-1] * 2, np.nan, R[1]])
    tt = np.array([T[3], T[3], T[3], T[-1] * 3])
    dr, dt = oracle.interp2d_deriv(R, T, G, out, tt)
    assert dr[0] == 0.0 and dr[1] == 0.0 and np.isnan(dr[2]) and dr[3] != 0.0
    assert dt[3] == 0.0 and dt[0] != 0.0


def test_interp_derivatives_match_finite_differences():
    """Central differences of the oracle's own P inside a cell (the interpolant is
    bilinear there, so the difference quotient is exact up to rounding)."""
    rng = np.random.default_rng(5)
    R, T = _axes(rng)
    G = rng.uniform(1.0, 5.0, (R.size, T.size))
    i = rng.integers(0, R.size - 1, 500)
    j = rng.integers(0, T.size - 1, 500)
    fr, ft = rng.uniform(0.2, 0.8, 500), rng.uniform(0.2, 0.8, 500)
    rho = R[i] + fr * (R[i + 1] - R[i])
    t = T[j] + ft * (T[j + 1] - T[j])
    hr = 1e-4 * (R[i + 1] - R[i])
    ht = 1e-4 * (T[j + 1] - T[j])
    dr, dt = oracle.interp2d_deriv(R, T, G, rho, t)
    pp, _, _ = oracle.interp2d(R, T, G, rho + hr, t)
    pm, _, _ = oracle.interp2d(R, T, G, rho - hr, t)
    assert np.allclose((pp - pm) / (2 * hr), dr, rtol=1e-6, atol=1e-9 * np.abs(dr).max())
    pp, _, _ = oracle.interp2d(R, T, G, rho, t + ht)
    pm, _, _ = oracle.interp2d(R, T, G, rho, t - ht)
    assert np.allclose((pp - pm) / (2 * ht), dt, rtol=1e-6, atol=1e-9 * np.abs(dt).max())


# ------------------------------------------------------- log-log bilinear ---
def test_loglog_is_exact_for_power_laws():
    """R24: interpolating ln P bilinearly in (ln rho, ln T) reproduces G = C rho^a T^b
    exactly (up to rounding) inside the grid, with dP/drho = a P / rho, dP/dT = b P / T."""
    rng = np.random.default_rng(9)
    R, T = _axes(rng)
    C, a, b = 2.5, 1.0, 1.5
    G = C * R[:, None] ** a * T[None, :] ** b
    rho = 10.0 ** rng.uniform(np.log10(R[0]), np.log10(R[-1]), 20000)
    t = 10.0 ** rng.uniform(np.log10(T[0]), np.log10(T[-1]), 20000)
    rho = np.clip(rho, R[0], R[-1])
    t = np.clip(t, T[0], T[-1])
    P, iR, iT, dr, dt = oracle.interp2d_loglog(R, T, G, rho, t)
    exact = C * rho ** a * t ** b
    assert np.max(np.abs(P / exact - 1)) < 1e-12
    assert np.max(np.abs(dr / (a * exact / rho) - 1)) < 1e-9
    assert np.max(np.abs(dt / (b * exact / t) - 1)) < 1e-9
    assert np.array_equal(iR, oracle.search(R, rho)) and np.array_equal(iT, oracle.search(T, t))


def test_loglog_nodes_outside_and_nan():
    rng = np.random.default_rng(10)
    R, T = _axes(rng)
    G = rng.uniform(1.0, 50.0, (R.size, T.size))
    rr, tt = np.meshgrid(R, T, indexing="ij")
    P, _, _, _, _ = oracle.interp2d_loglog(R, T, G, rr.ravel(), tt.ravel())
    assert np.max(np.abs(P / G.ravel() - 1)) < 1e-14            # nodes (exp(log g) round trip)
    rho = np.array([R[0] / 10, R[-1] * 10, np.nan, R[2], -1.0])
    t = np.array([T[1], T[1], T[1], np.nan, T[1]])
    P, _, _, dr, dt = oracle.interp2d_loglog(R, T, G, rho, t)
    assert abs(P[0] / G[0, 1] - 1) < 1e-14 and abs(P[1] / G[-1, 1] - 1) < 1e-14   # clamped
    assert dr[0] == 0.0 and dr[1] == 0.0
    assert np.isnan(P[2]) and np.isnan(dr[2]) and np.isnan(P[3]) and np.isnan(dt[3])
    assert np.isnan(P[4])                                         # ln of a negative density


def _loglog_decimal(R, T, G, rho, t, digits=40):
    """R24 evaluated with 40-digit decimal logarithms and exponentials (Python's decimal
    module: ln/exp correctly rounded at the context precision), brackets from bisect.
    Returns P and dP/drho as Python floats."""
    import bisect
    from decimal import Decimal, localcontext
    out_p, out_d = [], []
    with localcontext() as ctx:
        ctx.prec = digits
        D = Decimal
        for x, y in zip(rho, t):
            i = max(bisect.bisect_right(list(R), x) - 1, 0)
            j = max(bisect.bisect_right(list(T), y) - 1, 0)
            ci, cj = min(i, len(R) - 2), min(j, len(T) - 2)
            lr0, lr1 = D(R[ci]).ln(), D(R[ci + 1]).ln()
            lt0, lt1 = D(T[cj]).ln(), D(T[cj + 1]).ln()
            tx = min(max((D(x).ln() - lr0) / (lr1 - lr0), D(0)), D(1))
            ty = min(max((D(y).ln() - lt0) / (lt1 - lt0), D(0)), D(1))
            l00, l01 = D(G[ci][cj]).ln(), D(G[ci][cj + 1]).ln()
            l10, l11 = D(G[ci + 1][cj]).ln(), D(G[ci + 1][cj + 1]).ln()
            lp = (1 - tx) * ((1 - ty) * l00 + ty * l01) + tx * ((1 - ty) * l10 + ty * l11)
            p = lp.exp()
            sr = ((1 - ty) * (l10 - l00) + ty * (l11 - l01)) / (lr1 - lr0)
            out_p.append(float(p))
            out_d.append(float(p * sr / D(x)))
    return np.array(out_p), np.array(out_d)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_loglog_matches_40_digit_evaluation_on_narrow_cells_rough_surfaces(seed):
    """R24 pinned against the formula evaluated with 40-digit logarithms: random rough
    surfaces (ln G uniform over [-10, 10] per node, no smoothness) on axes with cells
    1e-4 .. 1e-2 wide in ln.  The oracle's log1p form keeps P within 1e-13 relative;
    the literal fp64 ln(rho) - ln(R) form loses ~|ln rho| / 1e-4 ulps of the weight
    there, i.e. > 1e-12 of P (checked below, so the pin tells the two apart)."""
    rng = np.random.default_rng(40 + seed)
    def axis(a, n):
        return np.exp(a + np.cumsum(np.concatenate([[0.0], 10 ** rng.uniform(-4, -2, n - 1)])))
    R, T = axis(-12.0, 40), axis(14.0, 30)
    G = np.exp(rng.uniform(-10, 10, (R.size, T.size)))
    m = 400
    rho = np.exp(rng.uniform(np.log(R[0]), np.log(R[-1]), m))
    t = np.exp(rng.uniform(np.log(T[0]), np.log(T[-1]), m))
    P, iR, iT, dr, dt = oracle.interp2d_loglog(R, T, G, rho, t)
    Pd, drd = _loglog_decimal(R, T, G, rho, t)
    assert np.max(np.abs(P / Pd - 1)) < 1e-13
    assert np.max(np.abs(dr - drd) / np.abs(drd)) < 1e-11
    # the literal difference-of-logs form in fp64, for contrast
    ci = np.minimum(iR, R.size - 2)
    cj = np.minimum(iT, T.size - 2)
    tx = np.clip((np.log(rho) - np.log(R[ci])) / (np.log(R[ci + 1]) - np.log(R[ci])), 0, 1)
    ty = np.clip((np.log(t) - np.log(T[cj])) / (np.log(T[cj + 1]) - np.log(T[cj])), 0, 1)
    L = np.log(G)
    lp = (1 - tx) * ((1 - ty) * L[ci, cj] + ty * L[ci, cj + 1]) + tx * ((1 - ty) * L[ci + 1, cj]
                                                                     + ty * L[ci + 1, cj + 1])
    assert np.max(np.abs(np.exp(lp) / Pd - 1)) > 1e-12
