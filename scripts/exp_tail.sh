#!/bin/bash
# 1-D launches of awkward sizes (ragged last tile), graph-timed, GPU box.
for w in cfg2 cfg5; do
for c in 100000 150000 200000 250000 300000 350000 400000 500000 1000001 4000037; do
echo -n "$w $c "; python bench.py --workload $w --count $c --steps 2000 --warmup 20 --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], round(d["ms_per_step"]*1e3, 2), "us")'
done; done
