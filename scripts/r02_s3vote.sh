#!/bin/bash
cd "$(dirname "$0")/.."
source scripts/r02_exp_lib.sh
BENCH_ARGS="" run cfg5_vote
BENCH_ARGS="--log-bins 27554" run cfg5_h27k_vote
BENCH_ARGS="" STEPS=100 run cfg5_vote_k100
