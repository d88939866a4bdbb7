#!/bin/bash
# packed tables: parity again (product + checked), then an ncu --set full capture of big
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or tiered" > gpurun_out/r02_packed_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02_packed_tests.log
EOS_LIBRARY=checked timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed" > gpurun_out/r02_packed_tests_checked.log 2>&1
echo "checked rc=$?"; tail -2 gpurun_out/r02_packed_tests_checked.log
B="python bench.py --workload big --steps 3 --warmup 3 --no-e2e --no-cpu --eager"
$B > gpurun_out/r02_pk_n.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02_big_packed $B > gpurun_out/r02_pk_ncu.log 2>&1; echo ncu=$?
