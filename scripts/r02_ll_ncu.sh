#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --workload cfg4 --loglog --steps 3 --warmup 3 --no-e2e --no-cpu --eager --count 67108864"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp2d -s 3 -c 1 -o gpurun_out/r02_cfg4_loglog_${TAG:-b} $B > gpurun_out/ll_ncu.log 2>&1; echo ncu=$?
