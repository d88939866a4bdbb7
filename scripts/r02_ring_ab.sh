#!/bin/bash
# ring kernel vs register-prefetch kernels (experiment build: EOS_RING=0 disables the ring)
cd "$(dirname "$0")/.."
source scripts/r02_exp_lib.sh
BENCH_ARGS="" run cfg5_ring
BENCH_ARGS="" run cfg5_noring EOS_RING=0
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_ring EOS_LAYOUT=1,3,0
BENCH_ARGS="--workload cfg2" STEPS=200 run cfg2_ring
BENCH_ARGS="--workload cfg2" STEPS=200 run cfg2_noring EOS_RING=0
BENCH_ARGS="--workload cfg3" STEPS=50 run cfg3_ring
BENCH_ARGS="--workload cfg3" STEPS=50 run cfg3_noring EOS_RING=0
