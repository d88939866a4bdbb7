#!/bin/bash
# shared helper of the r02 A/B scripts: run <tag> [ENV=V ...] with BENCH_ARGS / STEPS
run() {  # tag, env...   (bench args in $BENCH_ARGS)
  tag=$1; shift
  env "$@" EOS_LIBRARY=exp timeout 300 python bench.py --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu \
    $BENCH_ARGS > gpurun_out/r02_exp_$tag.json 2> gpurun_out/r02_exp_$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r02_exp_{tag}.json").read().strip().splitlines()[-1])
    p = d["plan"]["launch"]
    print(f"{tag:30s} {d['value']:8.1f} G/s frac {d['roofline']['frac']:.3f} vs_stream "
          f"{d['roofline']['frac_vs_stream']:.3f} clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']} "
          f"bins {p.get('bins')} S {p.get('steps')} d{p.get('dir_entry_bytes')} sf {p.get('fast_steps')} "
          f"rare {p.get('rare_steps')}", flush=True)
except Exception as e:
    print(tag, "FAILED", e, open(f"gpurun_out/r02_exp_{tag}.err").read()[-400:])
PY
}
