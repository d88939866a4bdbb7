#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python bench.py --workload cfg4 --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/c4_b.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/c4_b.json').read().strip().splitlines()[-1]);print('cfg4', d['value'], d['clocks']['sm_mhz'])"
B="python bench.py --workload cfg4 --steps 3 --warmup 3 --no-e2e --no-cpu --eager --count 67108864"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp2d -s 3 -c 1 -o gpurun_out/r02_cfg4_${TAG:-a} $B > gpurun_out/c4_ncu.log 2>&1; echo ncu=$?
