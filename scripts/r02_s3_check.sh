#!/bin/bash
# Restored-container check: full GPU suite (incl. the full-stream parity tests), smoke,
# the driver's default bench line (cfg5), and the cfg5 launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s3_smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_full_streams.py -q -x -s -m gpu --durations=0 > gpurun_out/s3_full.log 2>&1
echo "full rc=$?"; tail -n 15 gpurun_out/s3_full.log
timeout 1800 python -m pytest tests -q -x -m gpu --ignore=tests/test_gpu_full_streams.py > gpurun_out/s3_suite.log 2>&1
echo "suite rc=$?"; tail -2 gpurun_out/s3_suite.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s3_smoke.log
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/s3_bench.json'));r=d['roofline'];print(d['value'],d['unit'],r['frac'],r.get('frac_vs_stream'),d['clocks'])"
