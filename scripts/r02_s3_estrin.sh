#!/bin/bash
# log-log: Estrin polynomials (product) vs Horner (exp, -DEOS_EXP_LL_HORNER); parity tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "loglog or interp or grid or smoke" > gpurun_out/s3e_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/s3e_tests.log
one() {  # tag lib args...
  local tag=$1 lib=$2; shift 2
  env EOS_LIBRARY=$lib timeout 300 python bench.py --workload cfg4 "$@" --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/s3e_$tag.json 2> gpurun_out/s3e_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/s3e_$tag.json').read().strip().splitlines()[-1]);print('$tag', d['value'], d['roofline']['frac_vs_stream'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/s3e_$tag.err
}
for r in 1 2 3; do
  one est_$r product --loglog
  one hor_$r exp --loglog
done
for r in 1 2; do
  one estd_$r product --loglog --derivatives
  one hord_$r exp --loglog --derivatives
done
timeout 600 python scripts/fuzz.py --minutes 2 --seed 411 > gpurun_out/s3e_fuzz.json 2> gpurun_out/s3e_fuzz.err; echo "fuzz rc=$?"; tail -c 300 gpurun_out/s3e_fuzz.json
