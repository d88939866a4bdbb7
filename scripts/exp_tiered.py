#!/usr/bin/env python
"""Table-size sweep of the search: n = 2^8 .. 2^26 log-uniform tables,
the same 2^27 log-uniform targets, automatic plan (shared-memory table up to 16384
entries, tiered above).  Reports Glookups/s, the depth D and where the levels live
(L2-resident below ~7e6 entries).  Spot-checks 2^16 outputs against the oracle.

    python scripts/exp_tiered.py [--count 134217728]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1 << 27)
    ap.add_argument("--logn", default="8,10,12,14,15,16,17,18,20,22,24,26")
    ap.add_argument("--log-bins", default="auto",
                    help="comma list: 'auto' or |H| of the shared-memory table's log hash")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    spec = datagen.TargetSpec("loguniform", 9, 0, a=-6.0, w=16.0)
    Y = torch.empty(a.count, dtype=torch.float64, device=dev)
    spec.device_fill(Y, 0)
    out = torch.empty(a.count, dtype=torch.int32, device=dev)
    idx = np.sort(np.random.default_rng(0).integers(0, a.count, 1 << 16))
    Ys = spec.host_sample(idx)
    rows = []
    s = torch.cuda.Stream()
    for ln, hb in ((int(x), h) for x in a.logn.split(",") for h in a.log_bins.split(",")):
        n = 1 << ln
        X = np.sort(10.0 ** np.random.default_rng(ln).uniform(-6.0, 10.0, n))
        try:
            t = eos.Table(X, log_bins=None if hb == "auto" else int(hb))
        except eos.EosError as e:
            print(json.dumps({"log2_n": ln, "log_bins": hb, "error": str(e)}), file=sys.stderr)
            continue
        info = t.info
        with torch.cuda.stream(s):
            for _ in range(3):
                t.search(Y, out=out, stream=s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record(s)
        for _ in range(reps):
            eos.eos_search(t.handle, Y.data_ptr(), a.count, out.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        got = out[torch.from_numpy(idx).to(dev)].cpu().numpy()
        ok = bool(np.array_equal(got, oracle.search(X, Ys)))
        rows.append({"log2_n": ln, "n": n, "log_bins": hb, "bins": info.bins,
                     "levels": info.levels, "top_n": info.top_n,
                     "steps": info.steps, "image_bytes": info.image_bytes,
                     "level_bytes": info.level_bytes, "ms": round(ms, 4),
                     "Glookups_s": round(a.count / ms / 1e6, 2),
                     "hbm_frac": round(12 * a.count / (ms * 1e-3) / 6544e9, 4),
                     "sample_matches_oracle": ok})
        r = rows[-1]
        print(f"n=2^{ln} H={hb} bins={r['bins']} D={r['levels']} S={r['steps']} "
              f"image={r['image_bytes']} {r['Glookups_s']} Glookups/s ok={r['sample_matches_oracle']}",
              file=sys.stderr, flush=True)
        t.close()
    print(json.dumps({"count": a.count, "targets": "log-uniform 1e-6..1e10", "rows": rows}))


if __name__ == "__main__":
    main()
