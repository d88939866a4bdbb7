#!/usr/bin/env python
"""Tuning experiment (not product): interp2d launch-shape variants on cfg4 (EOS_INTERP_VARIANT)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402
from exp_search import time_fn  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    dev = torch.device("cuda:0")
    w = datagen.workload("cfg4")
    n = w.count
    rd = torch.empty(n, dtype=torch.float64, device=dev)
    td = torch.empty(n, dtype=torch.float64, device=dev)
    w.rho_targets.device_fill(rd, 0)
    w.T_targets.device_fill(td, 0)
    P = torch.empty(n, dtype=torch.float64, device=dev)
    iR = torch.empty(n, dtype=torch.int32, device=dev)
    iT = torch.empty(n, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    res = {"count": n}
    ref = None
    for v in ["0", "1", "2", "3", "4", "5", "6", "0"]:
        os.environ["EOS_INTERP_VARIANT"] = v
        g = eos.Grid2D(w.rho, w.T, w.P)
        r = time_fn(lambda: eos.eos_interp2d(g.handle, rd.data_ptr(), td.data_ptr(), n, P.data_ptr(),
                                             iR.data_ptr(), iT.data_ptr(), st), steps)
        r["GBps_median"] = 32 * n / r["median_ms"] / 1e6
        if ref is None:
            ref = (P.clone(), iR.clone(), iT.clone())
        else:
            r["same_idx"] = bool(torch.equal(iR, ref[1]) and torch.equal(iT, ref[2]))
            r["max_rel"] = float(((P - ref[0]).abs() / ref[0].abs()).max())
        res[f"v{v}" + ("_2" if f"v{v}" in res else "")] = r
        g.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
