#!/bin/bash
# packed tables with 64-bit key residuals: parity (product + checked), then big
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "packed or tiered or big" > gpurun_out/pk64_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pk64_tests.log
EOS_LIBRARY=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "packed" > gpurun_out/pk64_tests_checked.log 2>&1; echo "checked rc=$?"; tail -1 gpurun_out/pk64_tests_checked.log
for rep in 1 2; do
timeout 300 python bench.py --workload big --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/pk64_b.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/pk64_b.json').read().strip().splitlines()[-1]);l=d['roofline']['l2'];print('big', d['value'], d['clocks']['sm_mhz'], l['frac'], l.get('frac_vs_stream_gather'))" || tail -3 gpurun_out/pk64_b.json
done
B="python bench.py --workload big --steps 3 --warmup 3 --no-e2e --no-cpu --eager"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02_big_pk64 $B > /dev/null 2>&1; echo ncu=$?
