#!/bin/bash
# cfg5 lifting-layout A/B on one box (experiment build: EOS_LIBRARY=exp, EOS_LAYOUT=d16,sf,big).
# Output: one bench JSON line per variant in gpurun_out/r02_exp_cfg5_<tag>.json
cd "$(dirname "$0")/.."
run() {  # tag, env..., -- bench args
  tag=$1; shift
  env "$@" EOS_LIBRARY=exp timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu \
    $BENCH_ARGS > gpurun_out/r02_exp_cfg5_$tag.json 2> gpurun_out/r02_exp_cfg5_$tag.err
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r02_exp_cfg5_{tag}.json").read().strip().splitlines()[-1])
    p = d["plan"]["launch"]
    print(f"{tag:28s} {d['value']:8.1f} G/s frac {d['roofline']['frac']:.3f} vs_stream "
          f"{d['roofline']['frac_vs_stream']:.3f} clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']} "
          f"bins {p['bins']} S {p['steps']} d{p['dir_entry_bytes']} sf {p['fast_steps']} rare {p['rare_steps']}")
except Exception as e:
    print(tag, "FAILED", e)
PY
}
BENCH_ARGS="" run auto
BENCH_ARGS="--log-bins 27554" run h27k_d16_sf2 EOS_LAYOUT=1,2,1
BENCH_ARGS="--log-bins 27554" run h27k_d16_sf1 EOS_LAYOUT=1,1,1
BENCH_ARGS="--log-bins 27554" run h27k_d32_sf3 EOS_LAYOUT=0,3,0
BENCH_ARGS="--log-bins 27554" run h27k_d32_sf2 EOS_LAYOUT=0,2,1
BENCH_ARGS="--log-bins 55108" run h55k_d16_sf1 EOS_LAYOUT=1,1,1
BENCH_ARGS="--log-bins 55108" run h55k_d16_sf2 EOS_LAYOUT=1,2,1
BENCH_ARGS="--log-bins 13777" run h13k_d16_sf2 EOS_LAYOUT=1,2,1
BENCH_ARGS="--log-bins 27554" run h27k_d16_sf2_s1024u2 EOS_LAYOUT=1,2,1 EOS_SEARCH_VARIANT=static1024u2
BENCH_ARGS="--log-bins 27554" run h27k_d16_sf2_clc1024 EOS_LAYOUT=1,2,1 EOS_SEARCH_VARIANT=clc1024u4
BENCH_ARGS="--log-bins 13777" run h13k_d16_sf2_s512u4 EOS_LAYOUT=1,2,1 EOS_SEARCH_VARIANT=static512u4
