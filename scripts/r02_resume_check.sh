#!/bin/bash
# resume check after a lost session: smoke, full GPU suite, short fuzz, default bench, packed `big` ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/rc_smoke.log
timeout 2400 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/rc_gpu_suite.log 2>&1
echo "suite rc=$?"; tail -3 gpurun_out/rc_gpu_suite.log
timeout 900 python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err; echo "bench rc=$?"; head -c 1500 gpurun_out/rc_bench.json
timeout 300 python bench.py --workload big --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/rc_big.json 2>&1; echo "big rc=$?"; head -c 600 gpurun_out/rc_big.json
timeout 600 python scripts/fuzz.py --minutes ${FUZZ_MIN:-5} --seed ${FUZZ_SEED:-301} > gpurun_out/rc_fuzz.json 2> gpurun_out/rc_fuzz.err
echo "fuzz rc=$?"; tail -c 600 gpurun_out/rc_fuzz.json
B="python bench.py --workload big --steps 3 --warmup 3 --no-e2e --no-cpu --eager"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search1d -s 3 -c 1 -o gpurun_out/r02_big_packed $B > gpurun_out/rc_pk_ncu.log 2>&1; echo ncu=$?
