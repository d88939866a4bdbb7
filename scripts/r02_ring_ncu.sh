#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --eager --count 268435456"
$B > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02_cfg5_ring $B > /dev/null 2>&1; echo ncu=$?
