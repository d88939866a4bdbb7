#!/bin/bash
# 2-D small-launch sweep: default tiles against the small-tile kernels (EOS_SMALL_TILES), GPU box.
for w in "cfg4" "cfg4 --loglog" "big2d" "cfg4 --derivatives" "cfg4 --loglog --derivatives"; do
for c in 10000 50000 100000 150000 250000; do
for e in 0 1; do
echo -n "$w $c small=$e "; EOS_SMALL_TILES=$e python bench.py --workload $w --count $c --steps 2000 --warmup 20 --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], round(d["ms_per_step"]*1e3, 2), "us")'
done; done; done
