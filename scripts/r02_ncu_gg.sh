#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --eager --count 67108864"
$B --workload big2d > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp2d -s 3 -c 1 -o gpurun_out/r02_big2d $B --workload big2d > /dev/null 2>&1; echo ncu1=$?
$B --workload cfg4 --derivatives > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp2d -s 3 -c 1 -o gpurun_out/r02_cfg4_deriv $B --workload cfg4 --derivatives > /dev/null 2>&1; echo ncu2=$?
