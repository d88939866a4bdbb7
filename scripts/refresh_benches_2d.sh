#!/bin/bash
# The 2-D bench lines kept under profiles/ (GPU box): writes gpurun_out/rb_<name>.json.
OUT=gpurun_out
run() {  # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > $OUT/rb_$name.json 2> $OUT/rb_$name.err; echo "bench $name rc=$?"
  python -c "import json;d=json.load(open('$OUT/rb_$name.json'));print('  ', d['value'], d['unit'], d.get('roofline',{}).get('frac'), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', (d.get('e2e') or {}).get('value'))" 2>/dev/null || tail -n 3 $OUT/rb_$name.err
}
run cfg4 --workload cfg4 --steps 100 --warmup 5
run big2d --workload big2d --steps 200 --warmup 5
run cfg4_loglog --workload cfg4 --loglog --steps 200 --warmup 5
run cfg4_derivatives --workload cfg4 --derivatives --steps 200 --warmup 5
run cfg4_loglog_derivatives --workload cfg4 --loglog --derivatives --steps 200 --warmup 5
