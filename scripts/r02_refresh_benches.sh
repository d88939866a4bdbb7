#!/bin/bash
# Every bench line kept under profiles/ for round 2 (GPU box): gpurun_out/r02b_<name>.json.
OUT=gpurun_out
run() {  # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > $OUT/r02b_$name.json 2> $OUT/r02b_$name.err; echo "bench $name rc=$?"
  python -c "import json;d=json.load(open('$OUT/r02b_$name.json'));r=d.get('roofline',{});print('  ', d['value'], d['unit'], r.get('frac'), r.get('frac_vs_stream'), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', (d.get('e2e') or {}).get('value'))" 2>/dev/null || tail -n 3 $OUT/r02b_$name.err
}
run cfg5
run cfg5_k20 --steps 20 --warmup 3
run cfg2 --workload cfg2 --steps 1000 --warmup 10
run cfg3 --workload cfg3 --steps 100 --warmup 5
run cfg4 --workload cfg4 --steps 100 --warmup 5
run cfg1 --workload cfg1 --steps 1000 --warmup 10
run paper --workload paper --steps 200 --warmup 5
run big --workload big --steps 200 --warmup 5
run big2d --workload big2d --steps 200 --warmup 5
run cfg2_direct --workload cfg2 --direct --steps 200 --warmup 5
run cfg4_loglog --workload cfg4 --loglog --steps 100 --warmup 5
run cfg4_derivatives --workload cfg4 --derivatives --steps 100 --warmup 5
run cfg4_loglog_derivatives --workload cfg4 --loglog --derivatives --steps 100 --warmup 5
python bench.py --impl reference --steps 5 --warmup 1 > $OUT/r02b_reference_cfg5.json 2>&1; echo "reference rc=$?"; tail -c 400 $OUT/r02b_reference_cfg5.json
