"""Same-mix stream probes (measure/probes.cu) at cfg5 size, every launch shape, with the SM
clock sampled during each (NVML): which memory pattern reaches the ceiling in a persistent
kernel."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import measure
from bench import ClockSampler

n = int(sys.argv[1]) if len(sys.argv) > 1 else (8 << 30)
only = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else None
Y = torch.empty(n, dtype=torch.float64, device="cuda")
Y.uniform_(1.0, 2.0)
o = torch.empty(n, dtype=torch.int32, device="cuda")
L = measure.lib()
st = torch.cuda.current_stream()
res = {}
for v in range(L.probe_stream_variants()):
    if only is not None and v not in only:
        continue
    f = lambda: measure._check(L.probe_stream(Y.data_ptr(), o.data_ptr(), n, v, st.cuda_stream), "p")
    f(); torch.cuda.synchronize()
    reps = 5 if n >= (1 << 30) else 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record(st)
        for _ in range(reps):
            f()
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # correctness of the probe: out = lo ^ hi of every target
    idx = torch.randint(0, n, (1 << 16,), device="cuda")
    bits = Y[idx].view(torch.int64)
    want = ((bits & 0xFFFFFFFF) ^ (bits >> 32)).to(torch.int32)
    ok = bool(torch.equal(o[idx], want))
    res[v] = {"gbs": round(12 * n / (ms * 1e-3) / 1e9, 1), "clock": clk.summary(), "ok": ok}
    print(v, res[v], flush=True)
print(json.dumps(res))
