#!/bin/bash
# log-log: parity tests, bench, ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "loglog or interp or grid" > gpurun_out/ll_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ll_tests.log
for a in "--loglog" "--loglog --derivatives" "--loglog" ; do
  timeout 300 python bench.py --workload cfg4 $a --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/ll_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ll_b.json').read().strip().splitlines()[-1]);print('$a', d['value'], d['clocks']['sm_mhz'])"
done
TAG=${TAG:-c} bash scripts/r02_ll_ncu.sh
