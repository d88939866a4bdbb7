#!/bin/bash
# Small-launch sweep: default tiles against the small-tile shape (EOS_SMALL_TILES), GPU box.
for c in 150000 200000 250000 300000 350000 400000 500000; do
for e in 0 1; do
echo -n "$c small=$e "; EOS_SMALL_TILES=$e python bench.py --workload cfg1 --count $c --steps 3000 --warmup 20 --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'
done; done
for w in cfg2 cfg5; do for c in 100000 300000; do for e in 0 1; do
echo -n "$w $c small=$e "; EOS_SMALL_TILES=$e python bench.py --workload $w --count $c --steps 3000 --warmup 20 --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])'
done; done; done
