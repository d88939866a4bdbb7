#!/bin/bash
# L2 prefetch in the static 1-D schedule: A/B product vs exp (no prefetch), and parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "packed or tiered or big or maximum" > gpurun_out/pf1_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pf1_tests.log
for rep in 1 2; do
for lib in product exp; do
  for a in "--workload big" "--workload big --levels 2" "--workload cfg5 --count 2147483648"; do
  EOS_LIBRARY=$lib timeout 300 python bench.py $a --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/pf_b.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/pf_b.json').read().strip().splitlines()[-1]);print('$lib $a', d['value'], d['clocks']['sm_mhz'])" || tail -2 gpurun_out/pf_b.json
  done
done; done
for lib in product exp; do EOS_LIBRARY=$lib timeout 600 python scripts/exp_tiered.py --logn 14,16,18 > gpurun_out/pf_tiered_$lib.json 2>&1; echo "$lib"; tail -c 600 gpurun_out/pf_tiered_$lib.json; echo; done
