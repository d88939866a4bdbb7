#!/bin/bash
# 1-D static schedule: the next tile's loads before this tile's lookups (exp build) vs product
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
EOS_LIBRARY=exp timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "packed or tiered or big or maximum" > gpurun_out/early_tests.log 2>&1; echo "tests(exp) rc=$?"; tail -1 gpurun_out/early_tests.log
for rep in 1 2; do
for lib in product exp; do
  for a in "--workload big" "--workload big --levels 2"; do
  EOS_LIBRARY=$lib timeout 300 python bench.py $a --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/early_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/early_b.json').read().strip().splitlines()[-1]);print('$lib $a', d['value'], d['clocks']['sm_mhz'])" || tail -2 gpurun_out/early_b.json
  done
done; done
for lib in product exp; do EOS_LIBRARY=$lib timeout 600 python scripts/exp_tiered.py --logn 12,14,16,18,22 > gpurun_out/early_tiered_$lib.json 2>&1; echo "$lib"; python -c "
import json; d=json.loads(open('gpurun_out/early_tiered_$lib.json').read().strip().splitlines()[-1])
print([(r['log2_n'], r['Glookups_s'], r['sample_matches_oracle']) for r in d['rows']])" || tail -c 300 gpurun_out/early_tiered_$lib.json; done
