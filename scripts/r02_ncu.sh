#!/bin/bash
# ncu evidence for round 2 (each command first runs clean without ncu):
#  - cfg5 full-size launch: DRAM bytes per launch (the bench's roofline.traffic)
#  - cfg5 at 2^27 targets: --set full capture of the ring kernel
#  - cfg2 at full size: --set full capture of the register kernel
#  - cfg5 default bench (10 steps): launch list (kernel share of the step)
cd "$(dirname "$0")/.."
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --eager"
$B > gpurun_out/r02_n1.json 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:search1d -s 3 -c 1 --csv $B > gpurun_out/r02_ncu_traffic_cfg5.csv 2> gpurun_out/r02_ncu1.err; echo ncu1=$?
$B --count 134217728 > gpurun_out/r02_n2.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02_cfg5_final $B --count 134217728 > gpurun_out/r02_ncu2.log 2>&1; echo ncu2=$?
$B --workload cfg2 > gpurun_out/r02_n3.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02_cfg2_final $B --workload cfg2 > gpurun_out/r02_ncu3.log 2>&1; echo ncu3=$?
$B --workload cfg2 > /dev/null 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:search1d -s 3 -c 1 --csv $B --workload cfg2 > gpurun_out/r02_ncu_traffic_cfg2.csv 2> /dev/null; echo ncu4=$?
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02_n5.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_cfg5_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02_ncu5.log 2>&1; echo ncu5=$?
