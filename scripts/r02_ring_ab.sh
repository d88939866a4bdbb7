#!/bin/bash
# ring kernel vs register-prefetch kernels (experiment build: EOS_RING=0 disables the ring,
# EOS_RING=n caps its stages)
cd "$(dirname "$0")/.."
source scripts/r02_exp_lib.sh
BENCH_ARGS="" run cfg5_ring
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_ring
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_ring3 EOS_RING=3
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_noring EOS_RING=0
BENCH_ARGS="--log-bins 13777" run cfg5_h13k_ring
BENCH_ARGS="--workload cfg2" STEPS=200 run cfg2_ring
BENCH_ARGS="--workload cfg2" STEPS=200 run cfg2_ring4 EOS_RING=4
BENCH_ARGS="--workload cfg3" STEPS=50 run cfg3_ring
