#!/usr/bin/env python
"""Small end-to-end run of every kernel path for compute-sanitizer (memcheck/racecheck/
synccheck/initcheck) and the bounds-checked build (EOS_LIBRARY=checked): 1-D search (modes
0/1, every schedule, counters, ragged + misaligned, host pipeline), tiered tables, the
zero-setup search, and 2-D interpolation (shared-memory and device-memory grids, derivatives,
log-log), on small sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for name in ("cfg1", "cfg2", "cfg5"):
        w = datagen.workload(name, count=50_001)
        Y = torch.from_numpy(w.targets.host_fill(0, w.count, w.table)).to(dev)
        for k in (None, 0, 3):
            t = eos.Table(w.table, k=k)
            for off in (0, 1):
                y = Y[off:]
                o = torch.empty(y.numel() + 1, dtype=torch.int32, device=dev)[1 - off:][: y.numel()]
                t.search(y, out=o)
                c = torch.zeros(8, dtype=torch.int64, device=dev)
                t.search(y, out=o, counters=c)
            t.search_host(w.targets.host_fill(0, 20_000, w.table))
            t.close()
    t = eos.Table(np.array([-3.0, -1.0, 0.0, 2.0, 2.0, 8.0]))
    t.search(torch.linspace(-5, 10, 9999, dtype=torch.float64, device=dev))
    t.close()
    # tiered tables (D = 1, 2 and a deep forced D = 4) with counters, ragged views
    for n, D in ((40_000, -1), (300_000, -1), (5_000, 4)):
        X = np.sort(10.0 ** np.random.default_rng(n).uniform(-6, 10, n))
        t = eos.Table(X, levels=D)
        Y = torch.from_numpy(10.0 ** np.random.default_rng(1).uniform(-7, 11, 30_001)).to(dev)
        t.search(Y)
        t.search(Y[1:], counters=torch.zeros(8, dtype=torch.int64, device=dev))
        t.close()
    # zero-setup search
    Xd = torch.from_numpy(datagen.table_cfg5(4)).to(dev)
    eos.search_direct(Xd, torch.from_numpy(10.0 ** np.random.default_rng(2).uniform(-7, 11, 20_001)).to(dev))
    g = datagen.workload("cfg4", count=30_001)
    r = torch.from_numpy(g.rho_targets.host_fill(0, g.count)).to(dev)
    tt = torch.from_numpy(g.T_targets.host_fill(0, g.count)).to(dev)
    for loglog in (False, True):
        for global_grid in (False, True):
            grid = eos.Grid2D(g.rho, g.T, g.P, loglog=loglog, global_grid=global_grid)
            grid.interp(r, tt)
            grid.interp(r[1:], tt[1:], brackets=False)
            grid.interp(r, tt, derivatives=True)
            grid.interp_host(g.rho_targets.host_fill(0, 1000), g.T_targets.host_fill(0, 1000))
            grid.close()
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
