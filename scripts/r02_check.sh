#!/bin/bash
# quick A/B of the current product library on the 1-D configs (20-step runs, same box)
cd "$(dirname "$0")/.."
run() {
  tag=$1; shift
  timeout 300 python bench.py --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu "$@" > gpurun_out/r02_chk_$tag.json 2> gpurun_out/r02_chk_$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r02_chk_{tag}.json").read().strip().splitlines()[-1])
    p = d["plan"]["launch"]
    print(f"{tag:16s} {d['value']:8.1f} {d['unit']} frac {d['roofline']['frac']:.3f} vs_stream "
          f"{d['roofline']['frac_vs_stream']:.3f} clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']} {p}", flush=True)
except Exception as e:
    print(tag, "FAILED", e)
PY
}
run cfg5
run cfg2 --workload cfg2
run cfg3 --workload cfg3
