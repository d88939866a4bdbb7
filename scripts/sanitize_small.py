#!/usr/bin/env python
"""Small end-to-end run of every kernel path for compute-sanitizer (memcheck/racecheck/
synccheck/initcheck): 1-D search (modes 0/1, every schedule, counters, ragged + misaligned,
host pipeline) and 2-D interpolation, on small sizes."""
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
    g = datagen.workload("cfg4", count=30_001)
    grid = eos.Grid2D(g.rho, g.T, g.P)
    r = torch.from_numpy(g.rho_targets.host_fill(0, g.count)).to(dev)
    tt = torch.from_numpy(g.T_targets.host_fill(0, g.count)).to(dev)
    grid.interp(r, tt)
    grid.interp(r[1:], tt[1:], brackets=False)
    grid.interp_host(g.rho_targets.host_fill(0, 1000), g.T_targets.host_fill(0, 1000))
    grid.close()
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
