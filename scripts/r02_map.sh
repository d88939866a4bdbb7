#!/bin/bash
# fitted cell maps: 2-D parity tests, then cfg4 benches (mapped vs directory)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "loglog or interp or grid or cell_map" > gpurun_out/map_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/map_tests.log
for a in "" "--derivatives" "--loglog" "--loglog --derivatives"; do
  timeout 300 python bench.py --workload cfg4 $a --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/map_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/map_b.json').read().strip().splitlines()[-1]);print('cfg4 $a', d['value'], d['clocks']['sm_mhz'], d['roofline']['frac'])" || tail -3 gpurun_out/map_b.json
done
timeout 300 python bench.py --workload big2d --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/map_b.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/map_b.json').read().strip().splitlines()[-1]);print('big2d', d['value'], d['clocks']['sm_mhz'])"
TAG=map bash scripts/r02_cfg4_ncu.sh
