#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for lib in product exp; do
  EOS_LIBRARY=$lib timeout 300 python bench.py --workload big2d --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/pf_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/pf_b.json').read().strip().splitlines()[-1]);print('$lib big2d', d['value'], d['clocks']['sm_mhz'])"
  EOS_LIBRARY=$lib timeout 300 python bench.py --workload cfg4 --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/pf_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/pf_b.json').read().strip().splitlines()[-1]);print('$lib cfg4', d['value'], d['clocks']['sm_mhz'])"
done; done
