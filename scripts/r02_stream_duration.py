"""Same-mix stream probe (measure/probes.cu variant 1, the best shape) at cfg5 size, timed
over short and long runs with NVML clocks: does the ceiling hold under the power cap that
long cfg5 runs reach?"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import measure
from bench import ClockSampler

n = 8 << 30
Y = torch.empty(n, dtype=torch.float64, device="cuda")
Y.uniform_(1.0, 2.0)
o = torch.empty(n, dtype=torch.int32, device="cuda")
L = measure.lib()
st = torch.cuda.current_stream()
f = lambda: measure._check(L.probe_stream(Y.data_ptr(), o.data_ptr(), n, 1, st.cuda_stream), "p")
f(); torch.cuda.synchronize()
for reps in (5, 50, 200):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record(st)
        for _ in range(reps):
            f()
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"reps": reps, "gbs": round(12 * n / (ms * 1e-3) / 1e9, 1), "clock": clk.summary()}), flush=True)
