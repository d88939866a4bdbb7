#!/usr/bin/env python
"""Tuning experiment (not part of the product): time search1d launch-shape
variants (EOS_SEARCH_VARIANT) and k choices on a workload, next to plain
streaming references (torch copy kernels), with CUDA events.

    python scripts/exp_search.py [--workload cfg2] [--steps 200] [--count N]
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
import paper_2112_03229_b200 as eos  # noqa: E402

VARIANTS = ["static256u4", "static512u4", "clc256u4", "clc256u8", "clc256u2", "clc512u4", "clc512u2",
            "clc1024u4", "clc1024u2", "clc128u8"]


def time_fn(fn, steps, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    s = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s)
    for a, b in ev:
        a.record(s)
        fn()
        b.record(s)
    t1.record(s)
    torch.cuda.synchronize()
    per = np.array([a.elapsed_time(b) for a, b in ev])
    return {"mean_ms": float(per.mean()), "median_ms": float(np.median(per)), "min_ms": float(per.min()),
            "max_ms": float(per.max()), "step_ms": t0.elapsed_time(t1) / steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--count", type=int, default=None)
    ap.add_argument("--ks", default="")
    ap.add_argument("--logbins", default="")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--variants", default=",".join(VARIANTS))
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    w = datagen.workload(a.workload, count=a.count)
    n = w.count
    Y = torch.empty(n, dtype=torch.float64, device=dev)
    w.targets.device_fill(Y, 0, table_dev=torch.from_numpy(w.table).to(dev))
    out = torch.empty(n, dtype=torch.int32, device=dev)
    algo = 12 * n
    res = {"workload": a.workload, "count": n}
    st = torch.cuda.current_stream().cuda_stream

    # streaming references
    y64 = torch.empty(n, dtype=torch.float64, device=dev)
    r = time_fn(lambda: y64.copy_(Y), a.steps)
    r["GBps"] = 16 * n / r["median_ms"] / 1e6
    res["ref_copy_fp64"] = r
    yi = Y.view(torch.int32)[::2]
    r = time_fn(lambda: out.copy_(yi), a.steps)
    r["GBps"] = algo / r["median_ms"] / 1e6
    res["ref_strided_read8_write4"] = r

    ref_out = None
    for v in a.variants.split(",") + ["default"] + a.variants.split(","):
        os.environ["EOS_SEARCH_VARIANT"] = v
        t = eos.Table(w.table)
        key = "v_" + v + ("_2" if ("v_" + v) in res else "")
        r = time_fn(lambda: eos.eos_search(t.handle, Y.data_ptr(), n, out.data_ptr(), st), a.steps)
        r["GBps_median"] = algo / r["median_ms"] / 1e6
        r["GBps_mean"] = algo / r["mean_ms"] / 1e6
        r["info"] = t.info.as_dict()
        if ref_out is None:
            ref_out = out.clone()
        else:
            r["same_as_first"] = bool(torch.equal(out, ref_out))
        res[key] = r
        t.close()
    os.environ.pop("EOS_SEARCH_VARIANT", None)
    plans = [("k%d" % int(x), {"k": int(x)}) for x in a.ks.split(",") if x]
    plans += [("H%d" % int(x), {"log_bins": int(x)}) for x in a.logbins.split(",") if x]
    plans = plans * a.repeat
    for name, kw in plans:
        try:
            t = eos.Table(w.table, **kw)
        except eos.EosError as e:
            res[name] = str(e)
            continue
        k = name + ("_2" if name in res else "")
        r = time_fn(lambda: eos.eos_search(t.handle, Y.data_ptr(), n, out.data_ptr(), st), a.steps)
        r["GBps_median"] = algo / r["median_ms"] / 1e6
        r["info"] = t.info.as_dict()
        r["same_as_first"] = bool(torch.equal(out, ref_out)) if ref_out is not None else None
        res[k] = r
        t.close()

    # CUDA graph of 20 launches (default variant)
    t = eos.Table(w.table)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            eos.eos_search(t.handle, Y.data_ptr(), n, out.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            eos.eos_search(t.handle, Y.data_ptr(), n, out.data_ptr(), s.cuda_stream)
    r = time_fn(g.replay, max(3, a.steps // 20))
    r["per_launch_ms"] = r["median_ms"] / 20
    r["GBps"] = algo / r["per_launch_ms"] / 1e6
    res["graph20"] = r
    t.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
