#!/bin/bash
# packed tables: parity (product + bounds-checked build), then big: packed vs 8-ary
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or tiered" > gpurun_out/r02_packed_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/r02_packed_tests.log
EOS_LIBRARY=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed" > gpurun_out/r02_packed_tests_checked.log 2>&1
echo "checked rc=$?"; tail -3 gpurun_out/r02_packed_tests_checked.log
for rep in 1 2; do
  for lv in -1 2; do
    timeout 300 python bench.py --workload big --levels $lv --steps 20 --warmup 3 --no-e2e --no-cpu \
      > gpurun_out/r02_packed_big_L${lv}_$rep.json 2> gpurun_out/r02_packed_big_L${lv}_$rep.err
    python -c "import json;d=json.loads(open('gpurun_out/r02_packed_big_L${lv}_$rep.json').read().strip().splitlines()[-1]);print('levels $lv', d['value'], d['roofline'].get('frac'), d['clocks']['sm_mhz'], d.get('plan',{}).get('launch',{}))" || tail -5 gpurun_out/r02_packed_big_L${lv}_$rep.err
  done
done
