#!/bin/bash
# ring kernel without per-stage divisions; 4 or 8 targets per lane per stage
cd "$(dirname "$0")/.."
source scripts/r02_exp_lib.sh
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_ring4 EOS_LAYOUT=1,3,0 EOS_RING=6
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_ring8 EOS_LAYOUT=1,3,0 EOS_RING=6 EOS_RING_PL=8
BENCH_ARGS="--log-bins 13777" run cfg5_h13k_d16_ring8 EOS_LAYOUT=1,3,1 EOS_RING=6 EOS_RING_PL=8
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_d16_noring EOS_LAYOUT=1,3,0
BENCH_ARGS="--workload cfg2" STEPS=200 run cfg2_ring4 EOS_RING=6
BENCH_ARGS="--workload cfg2" STEPS=200 run cfg2_ring8 EOS_RING=6 EOS_RING_PL=8
