#!/bin/bash
# ring kernel with enough stages on cfg5 (16-bit directory, 86 KB image -> 4 stages)
cd "$(dirname "$0")/.."
source scripts/r02_exp_lib.sh
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_ring EOS_LAYOUT=1,3,0 EOS_RING=6
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_noring EOS_LAYOUT=1,3,0
BENCH_ARGS="--log-bins 20000" run cfg5_h20k_d16_ring EOS_LAYOUT=1,3,0 EOS_RING=6
BENCH_ARGS="--log-bins 13777" run cfg5_h13k_d16_ring EOS_LAYOUT=1,3,1 EOS_RING=6
BENCH_ARGS="--log-bins 27554" STEPS=60 run cfg5_h27k_d16_ring_long EOS_LAYOUT=1,3,0 EOS_RING=6
BENCH_ARGS="" STEPS=60 run cfg5_auto_long
