#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for a in "--workload cfg4" "--workload cfg4 --loglog" "--workload big2d"; do
timeout 300 python bench.py $a --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/l1p.json 2> gpurun_out/l1p.err
python -c "import json;d=json.loads(open('gpurun_out/l1p.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$a', d['value'], d['clocks']['sm_mhz'], r.get('frac_vs_stream'), r.get('l1'))" || tail -3 gpurun_out/l1p.err
done
