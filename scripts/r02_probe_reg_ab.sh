#!/bin/bash
# same-box A/B: product (probe register defined once per lookup) vs exp build of the
# previous kernels (a CS2R per lifting step)
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
for lib in product exp; do
  tag=${lib}_$rep
  if [ $lib = exp ]; then export EOS_LIBRARY=exp; else unset EOS_LIBRARY; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02_pab_$tag.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r02_pab_$tag.json'));print('$tag', d['value'], d['roofline']['frac_vs_stream'], d['clocks']['sm_mhz'])"
done
done
unset EOS_LIBRARY
