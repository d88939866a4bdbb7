#!/bin/bash
# log-log: both-records mapped axes (product) vs the branch form (exp, -DEOS_EXP_LL_ONE);
# big2d with the device-memory-grid same-mix ceiling
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "loglog or interp or grid" > gpurun_out/s3ll_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/s3ll_tests.log
one() {  # tag libenv args...
  local tag=$1 lib=$2; shift 2
  env EOS_LIBRARY=$lib timeout 300 python bench.py --workload cfg4 "$@" --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/s3ll_$tag.json 2> gpurun_out/s3ll_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/s3ll_$tag.json').read().strip().splitlines()[-1]);print('$tag', d['value'], d['roofline']['frac_vs_stream'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/s3ll_$tag.err
}
for r in 1 2 3; do
  one ll_both_$r product --loglog
  one ll_one_$r exp --loglog
done
for r in 1 2; do
  one lld_both_$r product --loglog --derivatives
  one lld_one_$r exp --loglog --derivatives
done
timeout 300 python bench.py --workload big2d --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/s3_big2d.json 2> gpurun_out/s3_big2d.err
python -c "import json;d=json.load(open('gpurun_out/s3_big2d.json'));print('big2d', d['value'], d['roofline'].get('l2'))" || tail -3 gpurun_out/s3_big2d.err
timeout 600 python scripts/fuzz.py --minutes 3 --seed 401 > gpurun_out/s3_fuzz.json 2> gpurun_out/s3_fuzz.err; echo "fuzz rc=$?"; tail -c 400 gpurun_out/s3_fuzz.json
