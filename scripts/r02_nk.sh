#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "deriv or loglog or interp or grid or cell_map" > gpurun_out/nk_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/nk_tests.log
for rep in 1 2; do
for a in "--workload cfg4 --loglog" "--workload cfg4 --loglog --derivatives"; do
  timeout 300 python bench.py $a --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/nk_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/nk_b.json').read().strip().splitlines()[-1]);print('$a', d['value'], d['clocks']['sm_mhz'])" || tail -2 gpurun_out/nk_b.json
done; done
TAG=nk bash scripts/r02_ll_ncu.sh
