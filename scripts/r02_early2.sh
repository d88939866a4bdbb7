#!/bin/bash
# early next-tile loads (product): parity + big + table-size sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/early2_suite.log 2>&1; echo "suite rc=$?"; tail -1 gpurun_out/early2_suite.log
for rep in 1 2; do
  timeout 300 python bench.py --workload big --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/early2_big.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/early2_big.json').read().strip().splitlines()[-1]);l=d['roofline']['l2'];print('big', d['value'], d['clocks']['sm_mhz'], l['frac'], l.get('frac_vs_stream_gather'))"
done
timeout 900 python scripts/exp_tiered.py > gpurun_out/early2_tiered.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/early2_tiered.json').read().strip().splitlines()[-1])
print([(r['log2_n'], r['levels'], r['Glookups_s'], r['sample_matches_oracle']) for r in d['rows']])"
B="python bench.py --workload big --steps 3 --warmup 3 --no-e2e --no-cpu --eager"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02_big_early $B > /dev/null 2>&1; echo ncu=$?
