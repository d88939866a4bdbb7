#!/bin/bash
# full GPU suite, smoke, fuzz soak
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/full_smoke.log
timeout 2400 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/full_gpu_suite.log 2>&1; echo "suite rc=$?"; tail -2 gpurun_out/full_gpu_suite.log
timeout 900 python scripts/fuzz.py --minutes ${FUZZ_MIN:-8} --seed ${FUZZ_SEED:-311} > gpurun_out/full_fuzz.json 2> gpurun_out/full_fuzz.err; echo "fuzz rc=$?"; tail -c 400 gpurun_out/full_fuzz.json
