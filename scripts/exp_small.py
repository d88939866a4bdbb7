#!/usr/bin/env python
"""Small-batch regime sweep: time create + search over m = 10^2 .. 10^8
for several k on a table, per launch (CUDA graph of 20 launches) and eager.

    python scripts/exp_small.py [--workload cfg1] [--ks auto,0,2,5,9]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg1")
    ap.add_argument("--ks", default="auto,0,2,5,9")
    ap.add_argument("--counts", default="100,1000,10000,100000,1000000,10000000,100000000")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    counts = [int(c) for c in a.counts.split(",")]
    w = datagen.workload(a.workload, count=max(counts))
    Y = torch.empty(max(counts), dtype=torch.float64, device=dev)
    w.targets.device_fill(Y, 0, table_dev=torch.from_numpy(w.table).to(dev))
    out = torch.empty(max(counts), dtype=torch.int32, device=dev)
    res = {"workload": a.workload, "rows": []}
    s = torch.cuda.Stream()
    for kk in a.ks.split(","):
        k = None if kk == "auto" else int(kk)
        try:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            t = eos.Table(w.table, k=k)
            torch.cuda.synchronize()
            create_us = (time.perf_counter() - t0) * 1e6
        except eos.EosError as e:
            res["rows"].append({"k": kk, "error": str(e)})
            continue
        for m in counts:
            with torch.cuda.stream(s):
                for _ in range(3):
                    eos.eos_search(t.handle, Y.data_ptr(), m, out.data_ptr(), s.cuda_stream)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    eos.eos_search(t.handle, Y.data_ptr(), m, out.data_ptr(), s.cuda_stream)
            with torch.cuda.stream(s):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(reps):
                    g.replay()
                e1.record(s)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (20 * reps)
            res["rows"].append({"k": t.info.k, "S": t.info.steps, "image_bytes": t.info.image_bytes,
                                "m": m, "us_per_launch": round(us, 3),
                                "Glookups_s": round(m / us / 1e3, 3), "create_us": round(create_us, 1)})
            del g
        t.close()
    # zero-setup path (f2): no create at all
    Xd = torch.from_numpy(w.table).to(dev)
    for m in counts:
        with torch.cuda.stream(s):
            for _ in range(3):
                eos.eos_search_direct(Xd.data_ptr(), Xd.numel(), Y.data_ptr(), m, out.data_ptr(), None,
                                      s.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                eos.eos_search_direct(Xd.data_ptr(), Xd.numel(), Y.data_ptr(), m, out.data_ptr(),
                                      None, s.cuda_stream)
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(5):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 100
        res["rows"].append({"k": "direct", "m": m, "us_per_launch": round(us, 3),
                            "Glookups_s": round(m / us / 1e3, 3), "create_us": 0.0})
        del g
    # host cost of create (plan + upload + configure), warm
    t0 = time.perf_counter()
    for _ in range(20):
        eos.Table(w.table).close()
    res["create_us_warm"] = round((time.perf_counter() - t0) / 20 * 1e6, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
