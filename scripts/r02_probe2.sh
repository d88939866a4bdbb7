#!/bin/bash
# big with the stream+gather ceiling; ncu --set full of the cfg4 log-log kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python bench.py --workload big --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/p2_big.json 2> gpurun_out/p2_big.err; echo "big rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/p2_big.json').read().strip().splitlines()[-1]);l=d['roofline']['l2'];print(d['value'], l['frac'], l.get('frac_vs_stream_gather'), l.get('stream_gather_ceiling',{}).get('all_gunits_per_s'))" || tail -5 gpurun_out/p2_big.err
timeout 300 python bench.py --workload cfg4 --loglog --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/p2_ll.json 2>&1; echo "ll rc=$?"; head -c 300 gpurun_out/p2_ll.json; echo
B="python bench.py --workload cfg4 --loglog --steps 3 --warmup 3 --no-e2e --no-cpu --eager --count 67108864"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp2d -s 3 -c 1 -o gpurun_out/r02_cfg4_loglog $B > gpurun_out/p2_ll_ncu.log 2>&1; echo ncu=$?
