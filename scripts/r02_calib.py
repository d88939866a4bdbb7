"""Calibration on the box: same-mix stream ceilings (1-D at cfg2 and cfg5 sizes, 2-D at cfg4
size) and the L2 random-sector gather ceiling (measure/)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import measure

out = {}
for name, n in (("cfg2", 1 << 27), ("cfg5", 8 << 30)):
    Y = torch.empty(n, dtype=torch.float64, device="cuda")
    Y.uniform_(1.0, 2.0)
    o = torch.empty(n, dtype=torch.int32, device="cuda")
    out["stream1d_" + name] = measure.stream_ceiling_1d(Y, o, reps=5 if n < 1 << 30 else 3)
    del Y, o
    torch.cuda.empty_cache()
m = 1 << 28
a = torch.rand(m, dtype=torch.float64, device="cuda"); b = torch.rand(m, dtype=torch.float64, device="cuda")
P = torch.empty(m, dtype=torch.float64, device="cuda")
i1 = torch.empty(m, dtype=torch.int32, device="cuda"); i2 = torch.empty(m, dtype=torch.int32, device="cuda")
out["stream2d_cfg4"] = measure.stream_ceiling_2d(a, b, P, i1, i2)
del a, b, P, i1, i2
torch.cuda.empty_cache()
for mb in (4, 16, 64):
    out[f"l2_gather_{mb}MB"] = measure.l2_gather_ceiling(mb << 20)
print(json.dumps(out, indent=1))
