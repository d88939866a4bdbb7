#!/bin/bash
# final soak: GPU suite on the bounds-checked build, fuzz on the checked and product builds
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
EOS_LIBRARY=checked timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/fs_suite_checked.log 2>&1; echo "suite(checked) rc=$?"; tail -2 gpurun_out/fs_suite_checked.log
EOS_LIBRARY=checked timeout 1200 python scripts/fuzz.py --minutes ${FUZZ_MIN:-8} --seed 511 > gpurun_out/fs_fuzz_checked_511.json 2> gpurun_out/fs_fuzz_checked.err; echo "fuzz(checked) rc=$?"; tail -c 500 gpurun_out/fs_fuzz_checked_511.json
timeout 1200 python scripts/fuzz.py --minutes ${FUZZ_MIN:-8} --seed 521 > gpurun_out/fs_fuzz_521.json 2> gpurun_out/fs_fuzz.err; echo "fuzz rc=$?"; tail -c 500 gpurun_out/fs_fuzz_521.json
