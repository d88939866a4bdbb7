#!/bin/bash
# Tiered tables, small launches: default tiles against the 512 x 1 small shape (EOS_SMALL_TILES).
for c in 10003 50001 100003 200003 250007 300007; do for e in 0 1; do
echo -n "big $c small=$e "; EOS_SMALL_TILES=$e python bench.py --workload big --count $c --steps 1000 --warmup 20 --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], round(d["ms_per_step"]*1e3, 2), "us")'
done; done
