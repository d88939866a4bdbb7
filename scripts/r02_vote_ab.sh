#!/bin/bash
# same-box A/B: product (warp vote on S = 3 batches) vs exp build with -DEOS_NO_VOTE
cd "$(dirname "$0")/.."
for rep in 1 2; do
for lib in product exp; do
  for arg in "" "--log-bins 27554"; do
    tag=${lib}_$(echo $arg | tr -d ' -')_$rep
    if [ $lib = exp ]; then export EOS_LIBRARY=exp; else unset EOS_LIBRARY; fi
    timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu $arg > gpurun_out/r02_vab_$tag.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/r02_vab_$tag.json'));print('$tag', d['value'], d['roofline']['frac_vs_stream'], d['clocks']['sm_mhz'])"
  done
done
done
