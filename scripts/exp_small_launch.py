#!/usr/bin/env python
"""Small launches, GPU box: default tiles against the small-tile shapes
(EOS_SMALL_TILES=0/1) for 1-D single-level tables, tiered tables and 2-D grids, graph-timed
per launch through bench.py.  Prints one JSON object (profiles/r01_exp_small_launch.json)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("cfg2", []), ("cfg5", []), ("big", []), ("cfg4", []), ("cfg4", ["--loglog"]),
         ("cfg4", ["--derivatives"]), ("big2d", [])]
COUNTS = [10_007, 50_021, 100_003, 200_003]


def run(w, extra, count, small):
    env = dict(os.environ, EOS_SMALL_TILES=str(small))
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", w, *extra, "--count",
           str(count), "--steps", "1000", "--warmup", "20", "--no-e2e", "--no-cpu"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600).stdout
    d = json.loads(out.strip().splitlines()[-1])
    return round(d["ms_per_step"] * 1e3, 3)


def main():
    rows = []
    for w, extra in CASES:
        for c in COUNTS:
            rows.append({"workload": w, "args": extra, "count": c,
                         "us_default_tiles": run(w, extra, c, 0),
                         "us_small_tiles": run(w, extra, c, 1)})
            print(json.dumps(rows[-1]), file=sys.stderr)
    print(json.dumps({"what": "us per launch (CUDA graph of 1000 launches), EOS_SMALL_TILES=0 "
                      "(default tiles) vs 1 (small-tile shapes where they apply)", "rows": rows}))


if __name__ == "__main__":
    main()
