#!/bin/bash
# log-log launch shape A/B: product (1024 x 1) vs expa (512 x 2), expb (512 x 1), expc (768 x 1)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
one() {  # tag lib args...
  local tag=$1 lib=$2; shift 2
  env EOS_LIBRARY=$lib timeout 300 python bench.py --workload cfg4 "$@" --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/s3ls_$tag.json 2> gpurun_out/s3ls_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/s3ls_$tag.json').read().strip().splitlines()[-1]);print('$tag', d['value'], d['roofline']['frac_vs_stream'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/s3ls_$tag.err
}
for r in 1 2; do
  one prod_$r product --loglog
  one a_$r expa --loglog
  one b_$r expb --loglog
  one c_$r expc --loglog
done
EOS_LIBRARY=expa timeout 600 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "loglog" > gpurun_out/s3ls_tests_a.log 2>&1; echo "tests expa rc=$?"; tail -1 gpurun_out/s3ls_tests_a.log
