#!/usr/bin/env python
"""Host-buffer entry point at small and medium counts (GPU box): eos_search_host against the
bare pinned copies it contains (torch H2D + D2H of the same bytes), per call."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2112_03229_b200 as eos  # noqa: E402


def timed(fn, reps=50):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    w = datagen.workload("cfg2", count=1 << 24)
    t = eos.Table(w.table)
    s = torch.cuda.current_stream()
    for m in (10_000, 100_000, 1_000_000, 5_000_000, 16_000_000):
        Yh = torch.from_numpy(w.targets.host_fill(0, m, w.table)).pin_memory()
        Ih = torch.empty(m, dtype=torch.int32).pin_memory()
        Yd = torch.empty(m, dtype=torch.float64, device="cuda")
        Id = torch.empty(m, dtype=torch.int32, device="cuda")
        us_api = timed(lambda: eos.eos_search_host(t.handle, Yh.data_ptr(), m, Ih.data_ptr(), s.cuda_stream))
        us_h2d = timed(lambda: Yd.copy_(Yh, non_blocking=True))
        us_d2h = timed(lambda: Ih.copy_(Id, non_blocking=True))
        us_all = timed(lambda: (Yd.copy_(Yh, non_blocking=True), t.search(Yd, out=Id), Ih.copy_(Id, non_blocking=True)))
        print(f"m={m:>9} api {us_api:9.1f} us ({m / us_api / 1e3:6.2f} G/s)  torch h2d {us_h2d:8.1f}  d2h {us_d2h:8.1f}  "
              f"h2d+search+d2h {us_all:9.1f}")


if __name__ == "__main__":
    main()
