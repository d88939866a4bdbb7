#!/bin/bash
# ring kernel after the mbarrier suspend hint, vs the register kernel
cd "$(dirname "$0")/.."
source scripts/r02_exp_lib.sh
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_ring_susp EOS_LAYOUT=1,3,0 EOS_RING=6
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_noring_susp EOS_LAYOUT=1,3,0
BENCH_ARGS="" run cfg5_auto_susp
BENCH_ARGS="--workload cfg2" STEPS=200 run cfg2_ring_susp EOS_RING=6
