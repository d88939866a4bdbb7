#!/bin/bash
# A/B of the product library against libeossearch_exp.so (EOS_LIBRARY=exp), same box,
# alternating: bash scripts/exp_ab_lib.sh [workload args ...]
one() {  # lib, args
  local lib=$1; shift
  EOS_LIBRARY=$lib timeout 600 python bench.py "$@" --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$*', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
}
for r in 1 2; do
  for lib in product exp; do
    one $lib --workload cfg2 --steps 500 --warmup 5
    one $lib --workload cfg3 --count 268435456 --steps 200 --warmup 5
    one $lib --workload cfg5 --count 2147483648 --steps 40 --warmup 3
    one $lib --workload cfg4 --steps 100 --warmup 5
  done
done
