#!/bin/bash
# cfg5 lifting-layout / launch-shape A/B on one box (experiment build: EOS_LIBRARY=exp,
# EOS_LAYOUT=d16,sf,big, EOS_SEARCH_VARIANT=<shape>).  One bench JSON line per variant in
# gpurun_out/r02_exp_<tag>.json and a summary line on stdout.
cd "$(dirname "$0")/.."
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
for v in ${VARIANTS:-cfg5}; do :; done
BENCH_ARGS="" run cfg5_auto
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_sf3 EOS_LAYOUT=1,3,0
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d32_sf3 EOS_LAYOUT=0,3,0
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_sf3_s512u4 EOS_LAYOUT=1,3,0 EOS_SEARCH_VARIANT=static512u4
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_sf3_s512u8 EOS_LAYOUT=1,3,0 EOS_SEARCH_VARIANT=static512u8
BENCH_ARGS="" run cfg5_auto_s1024u2 EOS_SEARCH_VARIANT=static1024u2
BENCH_ARGS="" run cfg5_auto_clc1024u4 EOS_SEARCH_VARIANT=clc1024u4
BENCH_ARGS="--log-bins 13777" run cfg5_h13k_d16_sf3big EOS_LAYOUT=1,3,1 EOS_SEARCH_VARIANT=static512u4
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_sf2big EOS_LAYOUT=1,2,1
BENCH_ARGS="--workload cfg2" STEPS=200 run cfg2_auto
BENCH_ARGS="--workload cfg3" STEPS=50 run cfg3_auto
