#!/bin/bash
# Zero-setup search: directory size A/B (product vs libeossearch_exp.so), GPU box.
one() {
  local lib=$1; shift
  EOS_LIBRARY=$lib timeout 600 python bench.py --direct "$@" --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$*', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
}
for r in 1 2; do for lib in product exp; do
  one $lib --workload cfg2 --steps 200 --warmup 5
  one $lib --workload cfg5 --count 2147483648 --steps 40 --warmup 3
  one $lib --workload cfg3 --count 268435456 --steps 100 --warmup 5
done; done
for lib in product exp; do EOS_LIBRARY=$lib python scripts/exp_small.py --workload cfg5 --ks auto --counts 100000,10000000 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', [(r['m'], r['us_per_launch']) for r in d['rows'] if r['k']=='direct'])"; done
