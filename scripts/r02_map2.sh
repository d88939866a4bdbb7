#!/bin/bash
# fitted cell maps + L2 prefetch of the tile after next: 2-D tests (product and
# bounds-checked builds), then cfg4 A/B (product vs exp = no L2 prefetch)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "loglog or interp or grid or cell_map" > gpurun_out/map_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/map_tests.log
EOS_LIBRARY=checked timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "cell_map or regular_axes" > gpurun_out/map_tests_checked.log 2>&1; echo "checked rc=$?"; tail -1 gpurun_out/map_tests_checked.log
for rep in 1 2; do
for lib in product exp; do
for a in "" "--loglog" "--derivatives"; do
  EOS_LIBRARY=$lib timeout 300 python bench.py --workload cfg4 $a --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/map_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/map_b.json').read().strip().splitlines()[-1]);print('$lib cfg4 $a', d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/map_b.json
done; done; done
EOS_LIBRARY=product timeout 300 python bench.py --workload big2d --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/map_b.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/map_b.json').read().strip().splitlines()[-1]);print('big2d', d['value'], d['clocks']['sm_mhz'])"
TAG=pf bash scripts/r02_cfg4_ncu.sh
