#!/bin/bash
# derivative kernels: launch shape A/B (product 512 threads vs exp)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
EOS_LIBRARY=exp timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "deriv or loglog or regular_axes or cell_map" > gpurun_out/deriv_tests.log 2>&1; echo "tests(exp) rc=$?"; tail -1 gpurun_out/deriv_tests.log
for rep in 1 2; do
for lib in product exp; do
  for a in "--workload cfg4 --derivatives" "--workload cfg4 --loglog --derivatives" "--workload big2d --derivatives"; do
  EOS_LIBRARY=$lib timeout 300 python bench.py $a --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/deriv_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/deriv_b.json').read().strip().splitlines()[-1]);print('$lib $a', d['value'], d['clocks']['sm_mhz'])" || tail -2 gpurun_out/deriv_b.json
  done
done; done
