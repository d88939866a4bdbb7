"""Full-stream parity at BASELINE.json's full sizes, every element (PAPER.md P:54 defines
the result element by element).

cfg3 (2^30 random-walk targets), cfg4 (2^28 pairs) and cfg5 (8*2^30 targets) run ONE
launch each over the whole device-resident stream, with the automatic plan -- the launch
configuration bench.py times -- and every output is compared with the CPU oracle on the
same targets generated on the host (datagen's host generator; the device generator's
equality with it is checked on every chunk).  Indices must be bit-exact; interpolated P
within the 1e-12 relative bar (BASELINE.json north star).  Runs ~1-2 minutes on a B200
box (the oracle over all host cores is the long pole).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402

DEV = torch.device("cuda", 0)
CHUNK = 1 << 27
THREADS = len(os.sched_getaffinity(0))
REL_TOL = 1e-12


def _host_fill(spec, table, offset, count, walk_base=None):
    """Host targets [offset, offset + count) over host threads (datagen's parallel host
    fill: the same bits as the serial generator; for the walk, walk_base chains chunks)."""
    return spec.host_fill_parallel(offset, count, table, threads=THREADS, walk_base=walk_base)


def _counters(X, Y, idx, off):
    """oracle.counters over host threads (sub-range sums add modulo 2^64)."""
    step = (Y.size + THREADS - 1) // THREADS
    with ThreadPoolExecutor(THREADS) as ex:
        parts = list(ex.map(lambda s: oracle.counters(X, Y[s:s + step], idx[s:s + step], off + s),
                            range(0, Y.size, step)))
    return np.sum(parts, axis=0, dtype=np.uint64)


def _check_chunk_targets(dev_vals, host_vals, rng):
    """The device-generated stream equals the host stream the oracle saw (64 K samples
    per chunk, plus both ends)."""
    n = host_vals.size
    idx = np.unique(np.concatenate([rng.integers(0, n, 1 << 16), [0, n - 1]]))
    got = dev_vals[torch.from_numpy(idx).to(DEV)].cpu().numpy()
    assert np.array_equal(got.view(np.uint64), host_vals[idx].view(np.uint64))


def _compare_indices(got, ref, Y, where):
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, (f"{where}: {bad.size} mismatches, first at {bad[:5]}: "
                           f"y={Y[bad[:5]]} gpu={got[bad[:5]]} oracle={ref[bad[:5]]}")


def test_cfg5_every_lookup_bit_exact():
    """cfg5: n = 4096 clustered table, all 8 * 2^30 targets of one launch vs the oracle."""
    w = datagen.workload("cfg5")
    Yd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.targets.device_fill(Yd, 0)
    out = torch.empty(w.count, dtype=torch.int32, device=DEV)
    t = eos.Table(w.table)
    t.search(Yd, out=out)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    cref = np.zeros(8, dtype=np.uint64)
    for off in range(0, w.count, CHUNK):
        n = min(CHUNK, w.count - off)
        Y, _ = _host_fill(w.targets, w.table, off, n)
        _check_chunk_targets(Yd[off:off + n], Y, rng)
        ref = oracle.search(w.table, Y, threads=THREADS)
        _compare_indices(out[off:off + n].cpu().numpy(), ref, Y, f"cfg5 chunk at {off}")
        # validation counters (a11) of the whole stream: chunk sums add modulo 2^64
        cref += _counters(w.table, Y, ref, off)
    c = torch.zeros(8, dtype=torch.int64, device=DEV)
    t.search(Yd, out=out, counters=c)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy().view(np.uint64), cref)
    assert int(cref[0]) == w.count
    t.close()


def test_cfg3_every_lookup_bit_exact():
    """cfg3: n = 1000 table, all 2^30 random-walk targets of one launch vs the oracle."""
    w = datagen.workload("cfg3")
    Yd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.targets.device_fill(Yd, 0)
    out = torch.empty(w.count, dtype=torch.int32, device=DEV)
    t = eos.Table(w.table)
    t.search(Yd, out=out)
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    base = 0   # walk position before the chunk (the step sum through off - 1)
    for off in range(0, w.count, CHUNK):
        n = min(CHUNK, w.count - off)
        Y, base = _host_fill(w.targets, None, off, n, walk_base=base)
        _check_chunk_targets(Yd[off:off + n], Y, rng)
        ref = oracle.search(w.table, Y, threads=THREADS)
        _compare_indices(out[off:off + n].cpu().numpy(), ref, Y, f"cfg3 chunk at {off}")
    t.close()


def test_cfg4_every_pair():
    """cfg4: 200 x 100 grid, all 2^28 (rho, T) pairs of one launch: both brackets bit-exact,
    P within 1e-12 relative of the oracle."""
    w = datagen.workload("cfg4")
    rd = torch.empty(w.count, dtype=torch.float64, device=DEV)
    td = torch.empty(w.count, dtype=torch.float64, device=DEV)
    w.rho_targets.device_fill(rd, 0)
    w.T_targets.device_fill(td, 0)
    g = eos.Grid2D(w.rho, w.T, w.P)
    P, iR, iT = g.interp(rd, td)
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    worst = 0.0
    for off in range(0, w.count, CHUNK):
        n = min(CHUNK, w.count - off)
        rho, _ = _host_fill(w.rho_targets, None, off, n)
        T, _ = _host_fill(w.T_targets, None, off, n)
        _check_chunk_targets(rd[off:off + n], rho, rng)
        _check_chunk_targets(td[off:off + n], T, rng)
        Pr, iRr, iTr = oracle.interp2d(w.rho, w.T, w.P, rho, T, threads=THREADS)
        _compare_indices(iR[off:off + n].cpu().numpy(), iRr, rho, f"cfg4 rho brackets at {off}")
        _compare_indices(iT[off:off + n].cpu().numpy(), iTr, T, f"cfg4 T brackets at {off}")
        Pg = P[off:off + n].cpu().numpy()
        assert not np.isnan(Pg).any() and not np.isnan(Pr).any()
        rel = np.abs(Pg - Pr) / np.abs(Pr)
        assert rel.max() <= REL_TOL, (off, float(rel.max()), int(np.argmax(rel)))
        worst = max(worst, float(rel.max()))
    g.close()
    print(f"cfg4: 2^28 pairs, brackets exact, max rel |dP| {worst:.3e}")


def test_cfg4_exact_layout_every_pair_bit_identical():
    """EOS_GRID_EXACT: the weights divide as the formula does, in the formula's order, so P
    is bit-identical to the oracle's fp64 evaluation (R14) -- on the first 2^26 pairs of
    cfg4 plus the grid nodes, the points just inside / outside the range, and NaN."""
    w = datagen.workload("cfg4")
    m = 1 << 26
    rho, _ = _host_fill(w.rho_targets, None, 0, m)
    T, _ = _host_fill(w.T_targets, None, 0, m)
    nodes = np.repeat(w.rho, w.T.size)
    rho[:nodes.size] = nodes
    T[:nodes.size] = np.tile(w.T, w.rho.size)
    rho[nodes.size:nodes.size + 6] = [np.nan, w.rho[0] / 2, w.rho[-1] * 2, 0.0, np.inf, -1.0]
    g = eos.Grid2D(w.rho, w.T, w.P, exact=True)
    P, iR, iT = g.interp(torch.from_numpy(rho).to(DEV), torch.from_numpy(T).to(DEV))
    torch.cuda.synchronize()
    Pr, iRr, iTr = oracle.interp2d(w.rho, w.T, w.P, rho, T, threads=THREADS)
    assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
    assert np.array_equal(P.cpu().numpy().view(np.uint64), Pr.view(np.uint64))
    g.close()


@pytest.mark.parametrize("seed", range(6))
def test_exact_layout_random_signed_grids_bit_identical(seed):
    """EOS_GRID_EXACT on random grids with signed values (cancellation inside cells, where
    the default layout's few-ulp weights only meet the corner-scaled bound): bit-identical
    P, brackets exact, with and without derivatives (the derivative formula R23 divides
    too, so it matches bit for bit as well)."""
    rng = np.random.default_rng(100 + seed)
    nR, nT = int(rng.integers(2, 300)), int(rng.integers(2, 200))
    R = np.sort(rng.choice(rng.uniform(-50, 50, 4 * nR), nR, replace=False))
    T = np.sort(rng.choice(10 ** rng.uniform(-3, 3, 4 * nT), nT, replace=False))
    G = rng.normal(0, 1, (nR, nT)) * 10 ** rng.uniform(-3, 3, (nR, nT))
    m = 1 << 18
    rho = rng.uniform(R[0] - 5, R[-1] + 5, m)
    tt = 10 ** rng.uniform(np.log10(T[0]) - 0.2, np.log10(T[-1]) + 0.2, m)
    rho[:nR] = R
    tt[m - nT:] = T
    g = eos.Grid2D(R, T, G, exact=True)
    P, iR, iT, dR, dT = g.interp(torch.from_numpy(rho).to(DEV), torch.from_numpy(tt).to(DEV),
                                 derivatives=True)
    torch.cuda.synchronize()
    Pr, iRr, iTr = oracle.interp2d(R, T, G, rho, tt)
    dRr, dTr = oracle.interp2d_deriv(R, T, G, rho, tt)
    assert np.array_equal(iR.cpu().numpy(), iRr) and np.array_equal(iT.cpu().numpy(), iTr)
    assert np.array_equal(P.cpu().numpy(), Pr)
    assert np.array_equal(dR.cpu().numpy(), dRr, equal_nan=True)
    assert np.array_equal(dT.cpu().numpy(), dTr, equal_nan=True)
    g.close()
