#!/bin/bash
# Device-memory grids: cell quads (default) against row pairs (EOS_GG_QUAD_MB=0), GPU box.
python -m pytest tests -m gpu -x -q -k "grid or interp or global or big2d" 2>&1 | tail -2
run() { python bench.py --workload big2d "$@" --steps 200 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])'; }
for a in "" "--derivatives"; do
echo -n "quad $a "; run $a
echo -n "quad L1 $a "; EOS_GG_QUAD_L1=1 run $a
for kb in 64 128 200; do echo -n "quad smem$kb $a "; EOS_GG_SMEM_KB=$kb run $a; done
done
