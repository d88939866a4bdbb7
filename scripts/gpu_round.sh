#!/bin/bash
# One gpurun call: build check, GPU tests, bench, ncu launch list + full capture.
# usage (on the GPU box): bash scripts/gpu_round.sh [stages...]  (default: all)
set -u
OUT=gpurun_out
mkdir -p $OUT
STAGES="${*:-smi smoke tests bench ncu}"
has() { [[ " $STAGES " == *" $1 "* ]]; }
if has smi; then
  nvidia-smi > $OUT/smi.txt 2>&1
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv >> $OUT/smi.txt 2>&1
  nproc >> $OUT/smi.txt; free -g >> $OUT/smi.txt
fi
if has build; then
  timeout 900 python __graft_entry__.py > $OUT/build.log 2>&1; echo "build rc=$?"
fi
if has smoke; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
  tail -3 $OUT/smoke.log
fi
if has tests; then
  timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
  tail -15 $OUT/pytest_gpu.log
fi
if has checked; then
  EOS_LIBRARY=checked timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu_checked.log 2>&1; echo "pytest gpu (checked build) rc=$?"
  tail -n 2 $OUT/pytest_gpu_checked.log
  for rp in 0; do
    EOS_INTERP_REP=$rp EOS_LIBRARY=checked timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "interp or loglog" > $OUT/pytest_checked_rep$rp.log 2>&1; echo "pytest interp checked rep=$rp rc=$?"
  done
  tail -n 4 $OUT/pytest_gpu_checked.log
  EOS_LIBRARY=checked timeout 600 python scripts/sanitize_small.py > $OUT/checked_small.log 2>&1; echo "checked small rc=$?"; tail -n 2 $OUT/checked_small.log
fi
if has bench; then
  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
  cat $OUT/bench.json; tail -5 $OUT/bench.err
fi
if has bencheager; then
  timeout 900 python bench.py --eager --no-cpu > $OUT/bench_eager.json 2> $OUT/bench_eager.err; echo "bench eager rc=$?"
  cat $OUT/bench_eager.json
fi
if has bench5; then
  timeout 900 python bench.py --workload cfg5 --steps 60 --warmup 5 --no-cpu --no-e2e > $OUT/bench_cfg5.json 2> $OUT/bench_cfg5.err; echo "bench cfg5 rc=$?"
  cat $OUT/bench_cfg5.json | head -c 600; echo
fi
if has pdlab; then
  for wl in cfg2 cfg3 cfg4; do
    for pdl in 0 1 0 1; do
      EOS_PDL=$pdl timeout 600 python bench.py --workload $wl --steps 300 --warmup 5 --no-cpu --no-e2e > $OUT/pdl_${wl}_$pdl.json 2>/dev/null
      python -c "import json;d=json.load(open('$OUT/pdl_${wl}_$pdl.json'));print('$wl pdl=$pdl', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
    done
  done
fi
if has bench4; then
  for flags in "" "--loglog" "--derivatives" "--loglog --derivatives"; do
    timeout 600 python bench.py --workload cfg4 $flags --steps 100 --warmup 5 --no-cpu --no-e2e > $OUT/b4.json 2>/dev/null
    python -c "import json;d=json.load(open('$OUT/b4.json'));print('cfg4 [$flags]', d['value'], d['unit'], d['roofline']['frac'], d['ms_per_step'])"
  done
fi
if has benchall; then
  for wl in cfg1 cfg3 cfg4 cfg5 paper; do
    timeout 900 python bench.py --workload $wl --steps 100 --warmup 5 --no-cpu > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err; echo "bench $wl rc=$?"
    cat $OUT/bench_$wl.json; tail -3 $OUT/bench_$wl.err
  done
fi
if has tiered; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tiered or smoke or golden" > $OUT/pytest_tiered.log 2>&1; echo "pytest tiered rc=$?"
  tail -n 5 $OUT/pytest_tiered.log
  for v in default static512u4 static1024u2 clc1024u2 static1024u1; do
    EOS_TIERED_VARIANT=$v timeout 600 python bench.py --workload big --steps 200 --warmup 5 --no-cpu --no-e2e > $OUT/big_$v.json 2> $OUT/big_$v.err
    python -c "import json;d=json.load(open('$OUT/big_$v.json'));r=d['roofline'];print('big $v', d['value'], r['frac'], r['l2'], d['clocks']['sm_mhz'])" || tail -n 3 $OUT/big_$v.err
  done
  for D in 3 4; do
    timeout 600 python bench.py --workload big --levels $D --steps 200 --warmup 5 --no-cpu --no-e2e > $OUT/big_D$D.json 2> $OUT/big_D$D.err
    python -c "import json;d=json.load(open('$OUT/big_D$D.json'));r=d['roofline'];print('big D=$D', d['value'], r['frac'], r['l2']['frac'])" || tail -n 3 $OUT/big_D$D.err
  done
fi
if has ncubig; then
  CMD="python bench.py --workload big --steps 6 --warmup 2 --no-e2e --no-cpu --eager"
  $CMD > $OUT/ncubig_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:search1d_tiered -s 2 -c 1 \
      -o $OUT/prof_big -f $CMD > $OUT/ncubig_full.log 2>&1; echo "ncu big rc=$?"
  python scripts/ncu_summary.py $OUT/prof_big.ncu-rep > $OUT/ncu_summary_big.json
  ncu -i $OUT/prof_big.ncu-rep --page raw --csv > $OUT/ncu_raw_big.csv 2>/dev/null
  ncu -i $OUT/prof_big.ncu-rep --page details --csv > $OUT/ncu_details_big.csv 2>/dev/null
  rm -f $OUT/prof_big.ncu-rep
fi
if has ncuw; then  # generic: NCU_W=<workload> NCU_K=<kernel regex> NCU_TAG=<name> [NCU_ARGS=...]
  CMD="python bench.py --workload $NCU_W ${NCU_ARGS:-} --steps 6 --warmup 2 --no-e2e --no-cpu --eager"
  $CMD > $OUT/ncuw_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$NCU_K -s 2 -c 1 \
      -o $OUT/prof_$NCU_TAG -f $CMD > $OUT/ncuw_full.log 2>&1; echo "ncu $NCU_TAG rc=$?"
  python scripts/ncu_summary.py $OUT/prof_$NCU_TAG.ncu-rep > $OUT/ncu_summary_$NCU_TAG.json
  ncu -i $OUT/prof_$NCU_TAG.ncu-rep --page details --csv > $OUT/ncu_details_$NCU_TAG.csv 2>/dev/null
  rm -f $OUT/prof_$NCU_TAG.ncu-rep
fi
if has benchw; then  # BENCH_W=<workload> BENCH_TAG=<name> [BENCH_ARGS=...]
  timeout 900 python bench.py --workload $BENCH_W ${BENCH_ARGS:-} > $OUT/bench_$BENCH_TAG.json 2> $OUT/bench_$BENCH_TAG.err; echo "bench $BENCH_TAG rc=$?"
  head -c 600 $OUT/bench_$BENCH_TAG.json; echo
fi
if has benchbig; then
  timeout 900 python bench.py --workload big --steps 200 --warmup 5 > $OUT/bench_big.json 2> $OUT/bench_big.err; echo "bench big rc=$?"
  cat $OUT/bench_big.json | head -c 1500; echo; tail -n 3 $OUT/bench_big.err
fi
if has interpv; then
  EOS_INTERP_VARIANT=7 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "interp or smoke" > $OUT/pytest_interp_v7.log 2>&1; echo "pytest interp v7 rc=$?"; tail -n 2 $OUT/pytest_interp_v7.log
  for v in 0 7 8 0 7 8; do
    EOS_INTERP_VARIANT=$v timeout 600 python bench.py --workload cfg4 --steps 200 --warmup 5 --no-cpu --no-e2e > $OUT/b4v.json 2>/dev/null
    python -c "import json;d=json.load(open('$OUT/b4v.json'));print('cfg4 v$v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
fi
if has lift; then
  for r in 1 2; do
    for v in default clc256u4_lift1 clc256u4_lift2; do
      EOS_SEARCH_VARIANT=$v timeout 600 python bench.py --workload cfg2 --steps 500 --warmup 5 --no-cpu --no-e2e > $OUT/lift.json 2>/dev/null
      python -c "import json;d=json.load(open('$OUT/lift.json'));print('cfg2 $v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
    done
    for v in default static1024u4_lift1 static1024u4_lift2; do
      EOS_SEARCH_VARIANT=$v timeout 600 python bench.py --workload cfg5 --count 2147483648 --steps 20 --warmup 3 --no-cpu --no-e2e > $OUT/lift.json 2>/dev/null
      python -c "import json;d=json.load(open('$OUT/lift.json'));print('cfg5 $v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
    done
  done
fi
if has guess; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "interp or smoke or loglog" > $OUT/pytest_guess.log 2>&1; echo "pytest interp rc=$?"; tail -n 3 $OUT/pytest_guess.log
  for r in 1 2; do
    for gs in 1 0; do
      for fl in "" "--derivatives" "--loglog"; do
        EOS_INTERP_GUESS=$gs timeout 600 python bench.py --workload cfg4 $fl --steps 200 --warmup 5 --no-cpu --no-e2e > $OUT/g4.json 2>/dev/null
        python -c "import json;d=json.load(open('$OUT/g4.json'));print('cfg4 guess=$gs [$fl]', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['config']['table']['rho'].get('cell_map'))"
      done
    done
  done
fi
if has hostpipe; then
  for r in 1 2; do
    for cfg in "2 23" "3 22" "4 22" "3 23" "4 21" "2 22"; do
      set -- $cfg
      EOS_HOST_SLOTS=$1 EOS_HOST_CHUNK_LOG2=$2 timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-steps 20 > $OUT/hp.json 2>/dev/null
      python -c "import json;d=json.load(open('$OUT/hp.json'));print('slots=$1 chunk=2^$2 e2e', d['e2e']['value'], d['e2e']['ms_per_step'])"
    done
  done
fi
if has roll; then
  for r in 1 2; do
    for v in default static1024u4_roll1 static1024u4_roll2; do
      EOS_SEARCH_VARIANT=$v timeout 600 python bench.py --workload cfg5 --steps 30 --warmup 3 --no-cpu --no-e2e > $OUT/roll.json 2>/dev/null
      python -c "import json;d=json.load(open('$OUT/roll.json'));print('cfg5 $v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
    done
    for v in default static256u4 static256u4_roll1 static512u4_roll1; do
      EOS_SEARCH_VARIANT=$v timeout 600 python bench.py --workload cfg2 --steps 500 --warmup 5 --no-cpu --no-e2e > $OUT/roll.json 2>/dev/null
      python -c "import json;d=json.load(open('$OUT/roll.json'));print('cfg2 $v', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
    done
  done
fi
if has rep; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "interp or smoke or loglog or graph or concurrent" > $OUT/pytest_rep.log 2>&1; echo "pytest interp (rep) rc=$?"; tail -n 3 $OUT/pytest_rep.log
  EOS_INTERP_REP=0 timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "interp" > $OUT/pytest_norep.log 2>&1; echo "pytest interp (no rep) rc=$?"; tail -n 2 $OUT/pytest_norep.log
  for r in 1 2; do
    for rp in 2 0; do
      for fl in "" "--derivatives"; do
        EOS_INTERP_REP=$rp timeout 600 python bench.py --workload cfg4 $fl --steps 200 --warmup 5 --no-cpu --no-e2e > $OUT/r4.json 2>/dev/null
        python -c "import json;d=json.load(open('$OUT/r4.json'));print('cfg4 rep=$rp [$fl]', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
      done
    done
  done
  CMD="python bench.py --workload cfg4 --count 268435456 --steps 5 --warmup 2 --no-e2e --no-cpu --eager"
  $CMD > $OUT/ncu_plain_rep.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp2d -s 2 -c 1 \
      -o $OUT/prof_rep -f $CMD > $OUT/ncu_full_rep.log 2>&1; echo "ncu rep rc=$?"
  python scripts/ncu_summary.py $OUT/prof_rep.ncu-rep > $OUT/ncu_summary_rep.json
  ncu -i $OUT/prof_rep.ncu-rep --page details --csv > $OUT/ncu_details_rep.csv 2>/dev/null
  ncu -i $OUT/prof_rep.ncu-rep --page source --csv > $OUT/ncu_source_rep.csv 2>/dev/null
  rm -f $OUT/prof_rep.ncu-rep
fi
if has exp; then
  timeout 900 python scripts/exp_search.py --workload cfg2 --ks 2,3,4,5,6,7,8 > $OUT/exp_cfg2.json 2> $OUT/exp_cfg2.err; echo "exp cfg2 rc=$?"
  timeout 900 python scripts/exp_search.py --workload cfg3 --steps 50 --ks 3,4,5,6,7,8 > $OUT/exp_cfg3.json 2> $OUT/exp_cfg3.err; echo "exp cfg3 rc=$?"
  timeout 900 python scripts/exp_search.py --workload cfg5 --count 1073741824 --steps 50 --ks 4,5,6,7,8,9 > $OUT/exp_cfg5.json 2> $OUT/exp_cfg5.err; echo "exp cfg5 rc=$?"
  for f in $OUT/exp_cfg*.err; do tail -n 2 $f; done
fi
if has expi; then
  timeout 900 python scripts/exp_interp.py > $OUT/exp_interp.json 2> $OUT/exp_interp.err; echo "exp interp rc=$?"; tail -n 3 $OUT/exp_interp.err
fi
if has exps; then
  timeout 900 python scripts/exp_small.py > $OUT/exp_small_cfg1.json 2> $OUT/exp_small.err; echo "exp small rc=$?"; tail -n 3 $OUT/exp_small.err
  timeout 900 python scripts/exp_small.py --workload cfg5 --ks auto,5,7,9 > $OUT/exp_small_cfg5.json 2>> $OUT/exp_small.err; echo "exp small5 rc=$?"
fi
for tool in memcheck racecheck synccheck initcheck; do
  if has san_$tool; then
    python scripts/sanitize_small.py > $OUT/san_plain.log 2>&1 && \
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_small.py > $OUT/san_$tool.log 2>&1
    echo "sanitizer $tool rc=$?"; tail -n 5 $OUT/san_$tool.log
  fi
done
if has torchrun1; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 200 --warmup 5 --no-cpu > $OUT/bench_torchrun1.json 2> $OUT/bench_torchrun1.err; echo "torchrun1 rc=$?"
  cat $OUT/bench_torchrun1.json; tail -n 3 $OUT/bench_torchrun1.err
fi
if has exph; then
  timeout 900 python scripts/exp_search.py --workload cfg2 --variants default --ks 5 --logbins 5000 --repeat 2 > $OUT/exph_cfg2.json 2> $OUT/exph.err; echo "exph cfg2 rc=$?"
  timeout 900 python scripts/exp_search.py --workload cfg5 --count 1073741824 --steps 40 --variants default --ks 9 --logbins 24000 --repeat 2 > $OUT/exph_cfg5.json 2>> $OUT/exph.err; echo "exph cfg5 rc=$?"
  timeout 900 python scripts/exp_search.py --workload cfg3 --steps 40 --variants default --ks 6 --logbins 4000 --repeat 2 > $OUT/exph_cfg3.json 2>> $OUT/exph.err; echo "exph cfg3 rc=$?"
  tail -n 3 $OUT/exph.err
fi
if has ncu2; then
  for wl in cfg4 cfg5; do
    CMD="python bench.py --workload $wl --count 268435456 --steps 5 --warmup 2 --no-e2e --no-cpu --eager"
    $CMD > $OUT/ncu_plain_$wl.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:'search1d|interp2d' -s 2 -c 1 \
        -o $OUT/prof_$wl -f $CMD > $OUT/ncu_full_$wl.log 2>&1; echo "ncu $wl rc=$?"
    python scripts/ncu_summary.py $OUT/prof_$wl.ncu-rep > $OUT/ncu_summary_$wl.json
    ncu -i $OUT/prof_$wl.ncu-rep --page details --csv > $OUT/ncu_details_$wl.csv 2>/dev/null
    ncu -i $OUT/prof_$wl.ncu-rep --page source --csv > $OUT/ncu_source_$wl.csv 2>/dev/null
    rm -f $OUT/prof_$wl.ncu-rep
  done
fi
if has ncufinal; then
  CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu"
  $CMD > $OUT/ncuf_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file $OUT/launches_final.csv $CMD > $OUT/ncuf_launches.log 2>&1; echo "ncu launches rc=$?"
  for wl in cfg2 cfg3 cfg5; do
    CMD="python bench.py --workload $wl --count 134217728 --steps 6 --warmup 2 --no-e2e --no-cpu --eager"
    $CMD > $OUT/ncuf_plain_$wl.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:search1d -s 2 -c 1 \
        -o $OUT/prof_final_$wl -f $CMD > $OUT/ncuf_full_$wl.log 2>&1; echo "ncu full $wl rc=$?"
    python scripts/ncu_summary.py $OUT/prof_final_$wl.ncu-rep > $OUT/ncu_summary_$wl.json
    ncu -i $OUT/prof_final_$wl.ncu-rep --page details --csv > $OUT/ncu_details_$wl.csv 2>/dev/null
    ncu -i $OUT/prof_final_$wl.ncu-rep --page raw --csv > $OUT/ncu_raw_$wl.csv 2>/dev/null
    rm -f $OUT/prof_final_$wl.ncu-rep
  done
fi
if has ncu; then
  CMD="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --eager"
  $CMD > $OUT/ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  $CMD > $OUT/ncu_plain2.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:search1d -s 5 -c 1 \
      -o $OUT/prof_search1d -f $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
  tail -3 $OUT/ncu_full.log
fi
