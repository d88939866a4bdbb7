#!/usr/bin/env python
"""Randomised parity soak (GPU): random tables, plans and targets against the CPU oracle for a
fixed wall-clock budget.

    python scripts/fuzz.py [--minutes 5] [--seed 0]

1-D: table sizes 1 .. 300000 of several shapes (tables up to 4096 entries also through the
zero-setup eos_search_direct) (log-uniform, exact powers of two, duplicate
runs, mixed signs with +-0, zero heads with subnormals, dense keys), every plan kind
(automatic, exponent k, log |H|, forced tiered depth D, packed nodes), targets drawn around the entries
(+-1 ulp, midpoints) plus log-uniform, out-of-range and special values.  Indices must be
bit-exact.  2-D: random grids (logspace with jitter / random axes, mode 0 and 1, shared or
device memory, linear or log-log, with derivatives); brackets bit-exact, P within 1e-12.
Prints one JSON summary line; exits 1 on any mismatch.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402


def rand_table(rng):
    kind = rng.integers(0, 6)
    n = int(np.exp(rng.uniform(0, np.log(300_000))))
    if kind == 0:
        X = 10.0 ** rng.uniform(-8, 8, n)
    elif kind == 1:
        X = 2.0 ** rng.integers(-30, 30, n).astype(np.float64)
    elif kind == 2:
        X = np.repeat(10.0 ** rng.uniform(-3, 3, max(1, n // 7)), 7)[:n]
    elif kind == 3:
        X = np.concatenate([rng.normal(0, 100, max(n - 2, 1)), [0.0, -0.0]])
    elif kind == 4:
        X = np.concatenate([[0.0, 0.0], rng.uniform(0, 1e-308, n // 3 + 1),
                            10.0 ** rng.uniform(-300, 300, n)])[:n]
    else:
        X = 1.0 + rng.uniform(0, 1e-9, n)
    return np.sort(X), int(kind)


def targets_for(rng, X, m):
    j = rng.integers(0, X.size, m // 2)
    pos = X[X > 0]
    a, b = (math.log10(pos[0]), math.log10(pos[-1])) if pos.size else (-10.0, 10.0)
    Y = np.concatenate([
        X[j], np.nextafter(X[j], np.inf)[: m // 8], np.nextafter(X[j], -np.inf)[: m // 8],
        np.sign(rng.uniform(-1, 1, m // 4)) * 10.0 ** rng.uniform(a - 1, b + 1, m // 4),
        [np.nan, np.inf, -np.inf, 0.0, -0.0, 5e-324, -5e-324, X[0], X[-1]],
    ])
    return rng.permutation(Y)


def fuzz_1d(rng, dev, stats):
    X, kind = rand_table(rng)
    n = X.size
    plan = rng.integers(0, 5)
    kw = {}
    if plan == 1:
        kw["k"] = int(rng.integers(0, 12))
    elif plan == 2:
        kw["log_bins"] = int(np.exp(rng.uniform(0, np.log(40000))))
    elif plan == 3:
        kw["levels"] = int(rng.integers(1, 6))
    elif plan == 4:  # packed nodes: the fewest levels, or 1..4 levels
        d = int(rng.integers(0, 5))
        kw["levels"] = eos.EOS_LEVELS_PACKED if d == 0 else eos.EOS_LEVELS_PACKED_DEPTH(d)
    try:
        t = eos.Table(X, **kw)
    except eos.EosError as e:
        stats["rejected_plans"] += 1   # e.g. k too fine for the image budget, D too shallow
        if e.name not in ("EOS_ERR_UNSUPPORTED", "EOS_ERR_SIZE"):
            raise
        return
    # mostly small launches (the small-tile shape); one in four large enough for the default
    # tiles (>= half the SMs' worth of tiles); one in sixteen large enough for the ring
    # kernel of deep tables (>= 4 stages of 7936 targets per SM)
    u = int(rng.integers(0, 16))
    m = int(rng.integers(1, 1 << 16)) if u >= 4 else (
        int(rng.integers(1 << 18, 1 << 19)) if u >= 1 else int(rng.integers(4_700_000, 6_000_000)))
    Y = targets_for(rng, X, m)
    got = t.search(torch.from_numpy(Y).to(dev)).cpu().numpy()
    ref = oracle.search(X, Y)
    bad = np.flatnonzero(got != ref)
    stats["tables"] += 1
    stats["lookups"] += Y.size
    stats["max_n"] = max(stats["max_n"], n)
    stats["tiered"] += int(t.info.levels > 0)
    stats["packed"] += int(t.info.node_width == 15)
    if bad.size:
        stats["mismatches"].append({"n": n, "kind": kind, "plan": kw, "levels": t.info.levels,
                                    "first": [float(Y[bad[0]]), int(got[bad[0]]), int(ref[bad[0]])]})
    t.close()
    if n <= 4096 and plan == 0:  # the zero-setup path on the same table and targets
        gd = eos.search_direct(torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev)).cpu().numpy()
        stats["direct_tables"] += 1
        bad = np.flatnonzero(gd != ref)
        if bad.size:
            stats["mismatches"].append({"n": n, "kind": kind, "direct": True,
                                        "first": [float(Y[bad[0]]), int(gd[bad[0]]), int(ref[bad[0]])]})


def fuzz_2d(rng, dev, stats):
    nR, nT = int(rng.integers(2, 700)), int(rng.integers(2, 400))
    loglog = bool(rng.integers(0, 2))
    mode1 = (not loglog) and bool(rng.integers(0, 3) == 0)

    def axis(n, lo, hi):
        # logspace with a jitter of up to +-0.55 cells: fitted cell maps are accepted
        # below a spread of ~1 cell and refused above (kernels.cuh axis_cell_rec)
        amp = rng.uniform(0.0, 0.55)
        u = np.linspace(lo, hi, n) + (hi - lo) / max(n - 1, 1) * rng.uniform(-amp, amp, n)
        v = 10.0 ** np.sort(u)
        return np.unique(v) if not mode1 else np.unique(np.sort(rng.normal(0, 50, n)))

    R, T = axis(nR, -4, 4), axis(nT, 0, 6)
    if R.size < 2 or T.size < 2:
        return
    if loglog:  # rough surfaces (R24's log1p form needs no smoothness)
        G = np.exp(rng.uniform(-10, 10, (R.size, T.size)))
    else:
        G = rng.uniform(-5, 5, (R.size, T.size))
    gl = bool(rng.integers(0, 2))
    g = eos.Grid2D(R, T, G, loglog=loglog, global_grid=gl)
    m = int(rng.integers(1, 1 << 15))
    lo_r, hi_r = (R[0] - 1, R[-1] + 1) if mode1 else (R[0] / 3, R[-1] * 3)
    rho = rng.uniform(lo_r, hi_r, m) if mode1 else 10 ** rng.uniform(np.log10(lo_r), np.log10(hi_r), m)
    tt = 10 ** rng.uniform(np.log10(T[0] / 3), np.log10(T[-1] * 3), m) if T[0] > 0 else \
        rng.uniform(T[0] - 1, T[-1] + 1, m)
    k = min(m, R.size)
    rho[:k] = R[:k]
    if m > 3 * k:  # next to the nodes: one ulp below, and within 1e-7 below
        rho[k:2 * k] = np.nextafter(R[:k], -np.inf)
        rho[2 * k:3 * k] = R[:k] - np.abs(R[:k]) * rng.uniform(0, 1e-7, k)
    stats["mapped_grids"] += int(g.rho_info.cell_map != 0)
    P, iR, iT = g.interp(torch.from_numpy(rho).to(dev), torch.from_numpy(tt).to(dev))
    if loglog:
        Pr, iRr, iTr = oracle.interp2d_loglog(R, T, G, rho, tt)[:3]
    else:
        Pr, iRr, iTr = oracle.interp2d(R, T, G, rho, tt)
    P, iR, iT = P.cpu().numpy(), iR.cpu().numpy(), iT.cpu().numpy()
    stats["grids"] += 1
    stats["pairs"] += m
    ok = np.array_equal(iR, iRr) and np.array_equal(iT, iTr)
    nan_ok = np.array_equal(np.isnan(P), np.isnan(Pr))
    fin = ~np.isnan(Pr)
    scale = np.abs(Pr[fin]) if loglog else np.maximum(np.abs(Pr[fin]), np.abs(G).max())
    val_ok = bool(np.all(np.abs(P[fin] - Pr[fin]) <= 1e-12 * scale)) if fin.any() else True
    if not (ok and nan_ok and val_ok):
        stats["mismatches"].append({"grid": [int(R.size), int(T.size)], "loglog": loglog,
                                    "global": gl, "mode1": mode1, "brackets_ok": ok,
                                    "nan_ok": nan_ok, "values_ok": val_ok})
    g.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=5.0)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(a.seed)
    stats = {"tables": 0, "lookups": 0, "tiered": 0, "packed": 0, "direct_tables": 0, "max_n": 0, "rejected_plans": 0,
             "grids": 0, "mapped_grids": 0, "pairs": 0, "mismatches": []}
    t_end = time.time() + 60 * a.minutes
    it = 0
    while time.time() < t_end:
        (fuzz_2d if it % 4 == 3 else fuzz_1d)(rng, dev, stats)
        it += 1
    stats["seconds"] = round(60 * a.minutes)
    stats["ok"] = not stats["mismatches"]
    print(json.dumps(stats))
    sys.exit(0 if stats["ok"] else 1)


if __name__ == "__main__":
    main()
