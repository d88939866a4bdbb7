#!/bin/bash
# full GPU suite, a fuzz soak, and an ncu --set full capture of the packed `big` kernel
cd "$(dirname "$0")/.."
timeout 2400 python -m pytest tests -q -x -m gpu > gpurun_out/r02_gpu_suite.log 2>&1
echo "suite rc=$?"; tail -2 gpurun_out/r02_gpu_suite.log
timeout 900 python scripts/fuzz.py --minutes ${FUZZ_MIN:-6} --seed ${FUZZ_SEED:-301} > gpurun_out/r02_fuzz.json 2> gpurun_out/r02_fuzz.err
echo "fuzz rc=$?"; tail -c 600 gpurun_out/r02_fuzz.json
B="python bench.py --workload big --steps 3 --warmup 3 --no-e2e --no-cpu --eager"
$B > gpurun_out/r02_pk_n.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02_big_packed $B > gpurun_out/r02_pk_ncu.log 2>&1; echo ncu=$?
