#!/bin/bash
cd "$(dirname "$0")/.."
source scripts/r02_exp_lib.sh
BENCH_ARGS="" run cfg5_auto_ring8
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_ring8
BENCH_ARGS="" run cfg5_auto_noring EOS_RING=0
