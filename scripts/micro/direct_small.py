#!/usr/bin/env python
"""One zero-setup search launch at a small batch (for ncu): cfg5 table (n=4096), m targets."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
name = sys.argv[2] if len(sys.argv) > 2 else "cfg5"
w = datagen.workload(name, count=m)
X = torch.from_numpy(w.table).cuda()
Y = torch.from_numpy(w.targets.host_fill(0, m, w.table)).cuda()
for _ in range(3):
    eos.search_direct(X, Y)
torch.cuda.synchronize()
print("ok")
