#!/bin/bash
# Final round-2 bench lines on the final library (every workload), DRAM traffic of the
# bench's exact launches (cfg4, big), --set full captures (cfg4, log-log, big), launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/r02_refresh_benches.sh
run() {  # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/r02b_$name.json 2> gpurun_out/r02b_$name.err; echo "bench $name rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/r02b_$name.json'));r=d.get('roofline',{});print('  ', d['value'], d['unit'], r.get('frac'), r.get('frac_vs_stream'), d['clocks']['sm_mhz'])" 2>/dev/null || tail -n 3 gpurun_out/r02b_$name.err
}
run big2d_derivatives --workload big2d --derivatives --steps 100 --warmup 5
run big_levels2 --workload big --levels 2 --steps 200 --warmup 5
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --eager"
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -s 3 -c 1 --csv"
for w in cfg5 cfg2 cfg4 big; do
  k=$([ $w = cfg4 ] && echo interp2d || echo search1d)
  $B --workload $w > gpurun_out/r02e_n_$w.json 2>&1 && ncu $M -k regex:$k $B --workload $w > gpurun_out/r02_ncu_traffic_$w.csv 2> gpurun_out/r02e_ncu_$w.err; echo "traffic $w=$?"
done
$B --workload cfg4 --count 67108864 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:interp2d -s 3 -c 1 -o gpurun_out/r02e_cfg4 $B --workload cfg4 --count 67108864 > /dev/null 2>&1; echo full_cfg4=$?
$B --workload cfg4 --loglog --count 67108864 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:interp2d -s 3 -c 1 -o gpurun_out/r02e_cfg4_loglog $B --workload cfg4 --loglog --count 67108864 > /dev/null 2>&1; echo full_ll=$?
$B --workload big > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02e_big $B --workload big > /dev/null 2>&1; echo full_big=$?
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02e_n5.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_cfg5_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02e_ncu5.log 2>&1; echo launches=$?
