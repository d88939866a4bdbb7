#!/bin/bash
# multi-level packed tables: parity (product + checked), table-size sweep, big, fuzz
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "packed or tiered or big" > gpurun_out/pkd_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pkd_tests.log
EOS_LIBRARY=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "packed" > gpurun_out/pkd_tests_checked.log 2>&1; echo "checked rc=$?"; tail -1 gpurun_out/pkd_tests_checked.log
timeout 300 python bench.py --workload big --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/pkd_big.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/pkd_big.json').read().strip().splitlines()[-1]);l=d['roofline']['l2'];print('big', d['value'], d['clocks']['sm_mhz'], l['frac'], l.get('frac_vs_stream_gather'))"
timeout 1200 python scripts/exp_tiered.py > gpurun_out/pkd_tiered.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/pkd_tiered.json').read().strip().splitlines()[-1])
print([(r['log2_n'], r['levels'], r['Glookups_s'], r['sample_matches_oracle']) for r in d['rows']])" || tail -5 gpurun_out/pkd_tiered.json
timeout 600 python scripts/fuzz.py --minutes 5 --seed 321 > gpurun_out/pkd_fuzz.json 2> gpurun_out/pkd_fuzz.err; echo "fuzz rc=$?"; tail -c 300 gpurun_out/pkd_fuzz.json
