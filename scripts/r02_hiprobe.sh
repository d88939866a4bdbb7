#!/bin/bash
# A/B: mode-0 lifting on the entries' upper words (exp build, -DEOS_EXP_HIPROBE) vs the product
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
EOS_LIBRARY=exp timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "not interp and not loglog and not grid and not cfg4 and not cell_map" > gpurun_out/hp_tests.log 2>&1; echo "tests(exp) rc=$?"; tail -1 gpurun_out/hp_tests.log
one() {  # tag lib args...
  local tag=$1 lib=$2; shift 2
  env EOS_LIBRARY=$lib timeout 300 python bench.py "$@" --no-e2e --no-cpu > gpurun_out/hp_$tag.json 2> gpurun_out/hp_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/hp_$tag.json').read().strip().splitlines()[-1]);print('$tag', d['value'], d['roofline']['frac_vs_stream'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/hp_$tag.err
}
for r in 1 2 3; do
  one prod_$r product --steps 60 --warmup 5
  one hi_$r exp --steps 60 --warmup 5
done
for r in 1 2; do
  one prod_n16k_$r product --workload cfg5 --count 2147483648 --steps 100 --warmup 5
  one hi_n16k_$r exp --workload cfg5 --count 2147483648 --steps 100 --warmup 5
done
EOS_LIBRARY=exp timeout 600 python scripts/fuzz.py --minutes 3 --seed 611 > gpurun_out/hp_fuzz.json 2> gpurun_out/hp_fuzz.err; echo "fuzz(exp) rc=$?"; tail -c 300 gpurun_out/hp_fuzz.json
