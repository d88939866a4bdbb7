#!/usr/bin/env python
"""bench.py -- throughput of the hot path on B200 (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (127.0.0.1, a free port); under torchrun the world
size must equal N.

A step = one pass of the hot path (stage table, stream targets, bin
lookup, in-bin search, fix-up, store indices) over one batch of synthetic input resident
in HBM: ONE kernel launch of eos_search (cfg4: of eos_interp2d).  Default workload:
BASELINE.json configs[4] (cfg5: n=4096 clustered table, 8*2^30 fp64 targets sharded
evenly over the ranks -- the configuration the metric "Glookups/s per GPU and box
(1/2/4/8 B200)" is quoted on; 103 GB, it fits one B200).  Other configs are parity cases
(tests/); --workload selects them for diagnostics.

Prints ONE JSON line on rank 0.  `value` = lookups (pairs for cfg4) of all ranks /
max-over-ranks device time, in G/s.  `e2e` = the same metric through the C-ABI
host-buffer entry point (eos_search_host: pinned H2D + search + D2H inside the timed
region).  `roofline` = the kernel's algorithmic bytes / its CUDA-event launch time vs the
measured HBM copy peak, and vs the same-mix stream ceiling measured in this run
(measure/probes.cu).  `cpu_baseline` = the CPU oracle (oracle/, test infrastructure)
timed on this host on a bounded sample, all cores and one core.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Glookups/s per GPU and box (1/2/4/8 B200); achieved HBM GB/s vs peak"
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (6.65 TB/s), used only without MEASURED_PEAKS.json


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg5",
                    choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "paper", "big", "big2d"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--k", type=int, default=None, help="override the directory k (default: auto)")
    ap.add_argument("--log-bins", type=int, default=None,
                    help="override: logarithm hash with this |H| (default: automatic choice)")
    ap.add_argument("--levels", type=int, default=-1,
                    help="tiered table depth D (default: auto; `big` needs D >= 3)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--count", type=int, default=None, help="override targets per GPU (testing)")
    ap.add_argument("--loglog", action="store_true", help="cfg4: log-log grid (EOS_GRID_LOGLOG)")
    ap.add_argument("--derivatives", action="store_true", help="cfg4: also write dP/drho, dP/dT")
    ap.add_argument("--global-grid", action="store_true",
                    help="2-D: keep the grid in device memory (EOS_GRID_GLOBAL)")
    ap.add_argument("--direct", action="store_true",
                    help="1-D: time the zero-setup eos_search_direct (f2; n <= 4096)")
    ap.add_argument("--eager", action="store_true",
                    help="launch each step from Python with per-launch events instead of a CUDA graph")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """NVML samples of SM clock + clock-event reasons during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.ok = False
        self.samples, self.reasons = [], set()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _reasons(self):
        nv = self.nv
        f = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        return f(self.h)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self._reasons()
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# --------------------------------------------------------- distributed -----
from paper_2112_03229_b200.dist import Dist, counters_to_u64, shard  # noqa: E402


# ------------------------------------------------------------ our arm ------
def run_ours(a, d: Dist):
    import torch
    import datagen
    import paper_2112_03229_b200 as eos

    torch.cuda.set_device(d.local)
    dev = torch.device("cuda", d.local)
    w = datagen.workload(a.workload)
    strong = a.workload == "cfg5"
    per_gpu = a.count or w.count
    if strong:
        total = a.count or w.count
        offset, count = shard(total, d.world, d.rank)
    else:
        total = per_gpu * d.world
        offset, count = per_gpu * d.rank, per_gpu
    is2d = w.is_2d
    bytes_per = 32 if is2d else 12
    stream = torch.cuda.current_stream()

    # inputs resident in HBM, generated in place (rank-invariant counter RNG)
    if is2d:
        rho = torch.empty(count, dtype=torch.float64, device=dev)
        T = torch.empty(count, dtype=torch.float64, device=dev)
        w.rho_targets.device_fill(rho, offset)
        w.T_targets.device_fill(T, offset)
        P = torch.empty(count, dtype=torch.float64, device=dev)
        iR = torch.empty(count, dtype=torch.int32, device=dev)
        iT = torch.empty(count, dtype=torch.int32, device=dev)
        obj = eos.Grid2D(w.rho, w.T, w.P, loglog=a.loglog, global_grid=a.global_grid)
        info = {"rho": obj.rho_info.as_dict(), "T": obj.T_info.as_dict(),
                "grid": "loglog" if a.loglog else "linear", "derivatives": a.derivatives,
                "grid_cells": int(w.P.size),
                "grid_in": "device memory" if (a.global_grid or 8 * w.P.size > 200 * 1024)
                           else "shared memory"}
        dPr = torch.empty(count, dtype=torch.float64, device=dev) if a.derivatives else None
        dPt = torch.empty(count, dtype=torch.float64, device=dev) if a.derivatives else None
        if a.derivatives:
            bytes_per = 48

        def step(sp=None):
            eos.eos_interp2d_ex(obj.handle, rho.data_ptr(), T.data_ptr(), count, P.data_ptr(),
                                iR.data_ptr(), iT.data_ptr(),
                                dPr.data_ptr() if dPr is not None else None,
                                dPt.data_ptr() if dPt is not None else None,
                                sp or stream.cuda_stream)
    else:
        Y = torch.empty(count, dtype=torch.float64, device=dev)
        w.targets.device_fill(Y, offset, table_dev=torch.from_numpy(w.table).to(dev))
        out = torch.empty(count, dtype=torch.int32, device=dev)
        obj = eos.Table(w.table, k=a.k, log_bins=a.log_bins, levels=a.levels)
        info = obj.info.as_dict()
        if a.direct:  # zero setup: the directory is built on the device by every CTA (f2)
            Xd = torch.from_numpy(w.table).to(dev)
            info = {"n": int(w.table.size), "api": "eos_search_direct (no handle)"}

            def step(sp=None):
                eos.eos_search_direct(Xd.data_ptr(), Xd.numel(), Y.data_ptr(), count, out.data_ptr(),
                                      None, sp or stream.cuda_stream)
        else:
            def step(sp=None):
                eos.eos_search(obj.handle, Y.data_ptr(), count, out.data_ptr(),
                               sp or stream.cuda_stream)
    torch.cuda.synchronize()

    for _ in range(max(a.warmup, 0)):
        step()
    torch.cuda.synchronize()
    launches0 = eos.launch_count()
    if a.eager:
        # K launches from Python with an event pair around each (diagnostic mode)
        ts = stream
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(a.steps)]

        def timed():
            for i in range(a.steps):
                ev[i][0].record(ts)
                step()
                ev[i][1].record(ts)
    else:
        # the K steps captured once into a CUDA graph and replayed (no host launch gaps)
        ts = torch.cuda.Stream(device=dev)
        ts.wait_stream(stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=ts):
            for _ in range(a.steps):
                step(ts.cuda_stream)
        torch.cuda.synchronize()
        with torch.cuda.stream(ts):
            g.replay()  # one untimed replay (graph upload)
        torch.cuda.synchronize()

        def timed():
            with torch.cuda.stream(ts):  # CUDAGraph.replay() launches on the current stream
                g.replay()
    launches_captured = eos.launch_count() - launches0
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d.barrier()
    torch.cuda.synchronize()
    with ClockSampler(d.local) as clk:
        t0.record(ts)
        timed()
        t1.record(ts)
        torch.cuda.synchronize()
    d.barrier()
    launches = a.steps if not a.eager else eos.launch_count() - launches0
    ms_total = t0.elapsed_time(t1)
    # one kernel per step: its average launch duration over the timed region
    kern_ms = float(np.mean([x.elapsed_time(y) for x, y in ev])) if a.eager else ms_total / a.steps
    tm = torch.tensor([ms_total, kern_ms], dtype=torch.float64, device=dev)
    d.allreduce(tm, "max")
    ms_total, kern_ms_max = float(tm[0]), float(tm[1])
    ms_step = ms_total / a.steps
    value = total / (ms_step * 1e-3) / 1e9  # G units / s, whole job

    # SURVEY §8(d) protocol: 20 individually event-timed launches (median / min), after the
    # timed region; reported beside `value`, which stays the graph-timed mean
    trial_ms = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        trial_ms.append(e0.elapsed_time(e1))
    tt = torch.tensor([float(np.median(trial_ms)), float(np.min(trial_ms))], dtype=torch.float64,
                      device=dev)
    d.allreduce(tt, "max")
    trials = {"n": 20, "median_ms": round(float(tt[0]), 5), "min_ms": round(float(tt[1]), 5),
              "value_at_median": round(total / (float(tt[0]) * 1e-3) / 1e9, 3),
              "value_at_min": round(total / (float(tt[1]) * 1e-3) / 1e9, 3),
              "note": "eager launches with an event pair each, max over ranks"}

    # validation counters over this shard (untimed), reduced with one NCCL all_reduce
    counters = None
    if not is2d:
        c = torch.zeros(8, dtype=torch.int64, device=dev)
        obj.search(Y, out=out, counters=c, global_offset=offset)
        d.reduce_counters(c)
        counters = counters_to_u64(c.cpu().tolist())

    # ---- e2e through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(a, d, w, obj, offset, count, total, is2d, dev)

    # same-mix stream ceiling, measured now on this rank's own buffers (trivial kernels of
    # measure/probes.cu moving the same bytes per unit); the search output is rewritten
    # afterwards only by the probe, so it runs after the counters
    import measure
    if is2d:
        ceiling = measure.stream_ceiling_2d(rho, T, P, iR, iT)
    else:
        ceiling = measure.stream_ceiling_1d(Y, out)
    cg = torch.tensor([ceiling["gbs"]], dtype=torch.float64, device=dev)
    d.allreduce(cg, "min")

    hbm_peak, peak_src = peaks()
    achieved = bytes_per * count / (kern_ms * 1e-3) / 1e9
    plan = plan_signature(a, obj, is2d)
    res = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "Gpairs/s" if is2d else "Glookups/s",
        "n_gpus": d.world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": round(ms_step, 5),
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded counter-based generators, generated in HBM; DESIGN.md input recipe)",
        "config": bench_config(a, w, d.world),
        "plan": {"table": info, "launch": plan},
        "gpu_launches": int(launches),
        "timing": ("eager: K launches, CUDA events per launch" if a.eager else
                   f"CUDA graph of the K={a.steps} search launches ({launches_captured} captured), "
                   "events on the replay stream around one replay"),
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": hbm_peak,
            "unit": "GB/s",
            "frac": round(achieved / hbm_peak, 4),
            "traffic": ncu_traffic(a.workload, count, plan),
            "kernel": "interp2d_kernel" if is2d else (
                "search1d_direct_kernel" if a.direct else
                "search1d_packed_kernel" if obj.info.node_width == 15 else
                "search1d_tiered_kernel" if obj.info.levels > 0 else "search1d_kernel"),
            "kernel_ms_avg": round(kern_ms, 5),
            "kernel_ms_avg_max_rank": round(kern_ms_max, 5),
            "algorithmic_bytes_per_launch": bytes_per * count,
            "peak_source": peak_src,
            "stream_ceiling": {**ceiling, "gbs_min_over_ranks": float(cg[0])},
            "frac_vs_stream": round(achieved / float(cg[0]), 4),
            "note": ("peak = 1:1 copy bandwidth; this stream reads:writes "
                     + ("1:1 (16 B in, 16 B out per pair)" if is2d and not a.derivatives else
                        "1:2 (16 B in, 32 B out per pair)" if is2d else
                        "2:1 (8 B in, 4 B out per lookup)")
                     + ", so frac can exceed 1; frac_vs_stream divides by a trivial kernel "
                       "moving the same bytes per unit on the same buffers in this run"),
        },
        "clocks": clk.summary(),
        "e2e": e2e,
        "trials": trials,
    }
    if is2d and not a.global_grid and not a.derivatives and 8 * len(w.rho) * len(w.T) <= 200 * 1024:
        # shared-memory grids: L1TEX data-pipe bound; the same mix of
        # shared-memory reads and stream as a trivial kernel, measured now
        im = measure.interp_mix_ceiling(rho, T, P, iR, iT, len(w.rho), len(w.T))
        res["roofline"]["l1"] = {
            "bound": "l1tex data pipe (shared-memory gathers + stream)",
            "achieved_gunits_s": round(count / (kern_ms * 1e-3) / 1e9, 2),
            "ceiling_gunits_s": round(im["units_per_s"] / 1e9, 2),
            "frac": round(count / (kern_ms * 1e-3) / im["units_per_s"], 4), "peak_source": "measured",
            "probe": im}
    elif is2d and not a.derivatives and not a.loglog:
        # grid in device memory: one 32-B cell-quad gather per pair from
        # L2 beside the 2-D stream; the same mix as a trivial kernel, measured now
        im = measure.interp_gg_mix_ceiling(rho, T, P, iR, iT, len(w.rho), len(w.T))
        res["roofline"]["l2"] = {
            "bound": "l2 sector gathers + hbm stream (one cell quad per pair)",
            "achieved_gunits_s": round(count / (kern_ms * 1e-3) / 1e9, 2),
            "ceiling_gunits_s": round(im["units_per_s"] / 1e9, 2),
            "frac": round(count / (kern_ms * 1e-3) / im["units_per_s"], 4), "peak_source": "measured",
            "probe": im}
    if not is2d and obj.info.levels > 0:
        # tiered table: each level reads one 32-B sector from L2 (packed
        # tables: one level of nodes); random sector gathers, not HBM, bound it.  Ceiling
        # measured now (measure/probes.cu: the same 256-bit load, an L2-resident buffer of
        # the gathered levels' size).
        gathered = (32 * obj.info.top_n if obj.info.node_width == 15 else obj.info.level_bytes)
        gl = measure.l2_gather_ceiling(max(int(gathered), 1 << 20))
        levels = obj.info.levels
        ach = levels * count / (kern_ms * 1e-3)
        res["roofline"]["l2"] = {
            "bound": "l1tex/l2 sector gathers", "sectors_per_lookup": levels,
            "achieved_gsectors_s": round(ach / 1e9, 2),
            "peak_gsectors_s": round(gl["sectors_per_s"] / 1e9, 2),
            "frac": round(ach / gl["sectors_per_s"], 4), "peak_source": "measured",
            "probe": gl}
        if obj.info.node_width == 15:
            # one sector per lookup: the same mix (stream + one gather per unit) as a
            # trivial kernel is the kernel's own ceiling, measured on the same buffers
            sg = measure.stream_gather_ceiling(Y, out, max(int(gathered), 1 << 20))
            res["roofline"]["l2"]["stream_gather_ceiling"] = sg
            res["roofline"]["l2"]["frac_vs_stream_gather"] = round(count / (kern_ms * 1e-3) / sg["units_per_s"], 4)
    if counters is not None:
        res["validation"] = {"counters_u64": counters}
    if d.world == 1 and d.rank == 0 and not a.no_cpu:
        res["cpu_baseline"] = cpu_baseline(w, is2d, loglog=a.loglog, deriv=a.derivatives)
    return res


def bench_config(a, w, world):
    """The workload this line measures (identical in both arms)."""
    strong = a.workload == "cfg5"
    per_gpu = (a.count or w.count) // (world if strong else 1)
    total = (a.count or w.count) if strong else per_gpu * world
    bytes_per = (48 if a.derivatives else 32) if w.is_2d else 12
    cfg = {"workload": a.workload, "desc": w.note, "units_total": total,
           "units_per_gpu": per_gpu, "bytes_per_unit": bytes_per,
           "parallelism": f"dp{world} (target-stream sharding, no data-path collective)",
           "l2": (f"inputs larger than L2: {bytes_per * per_gpu / 1e9:.2f} GB streamed per step per "
                  "GPU (126 MB L2), no flush needed") if bytes_per * per_gpu > 4 * 126e6 else
                 "inputs L2-resident (launch-bound parity config)"}
    for k in ("loglog", "derivatives", "global_grid", "direct"):
        if getattr(a, k, False):
            cfg[k] = True
    return cfg


def plan_signature(a, obj, is2d):
    if is2d:
        return {"kind": "interp2d", "loglog": a.loglog, "global_grid": a.global_grid,
                "derivatives": a.derivatives}
    i = obj.info
    return {"kind": "tiered" if i.levels > 0 else ("direct" if a.direct else "search"),
            "hash_kind": i.hash_kind, "bins": i.bins, "steps": i.steps,
            "dir_entry_bytes": i.dir_entry_bytes, "fast_steps": i.fast_steps,
            "rare_steps": i.rare_steps, "levels": i.levels, "node_width": i.node_width,
            "ring_stages": i.ring_stages}


def run_e2e(a, d, w, obj, offset, count, total, is2d, dev):
    import torch
    import paper_2112_03229_b200 as eos
    steps = a.e2e_steps or max(3, min(20, a.steps // 50))
    stream = torch.cuda.current_stream()
    # bounded host footprint: at most 2^28 units per rank per e2e step (cfg5 would need 96 GiB pinned)
    count = min(count, 1 << 28)
    total = count * d.world
    if is2d:
        rh = torch.empty(count, dtype=torch.float64).pin_memory()
        th = torch.empty(count, dtype=torch.float64).pin_memory()
        rh.numpy()[:] = w.rho_targets.host_fill(offset, count)
        th.numpy()[:] = w.T_targets.host_fill(offset, count)
        Ph = torch.empty(count, dtype=torch.float64).pin_memory()
        iRh = torch.empty(count, dtype=torch.int32).pin_memory()
        iTh = torch.empty(count, dtype=torch.int32).pin_memory()
        h2d, d2h = 16 * count, 16 * count

        def step():
            eos.eos_interp2d_host(obj.handle, rh.data_ptr(), th.data_ptr(), count, Ph.data_ptr(),
                                  iRh.data_ptr(), iTh.data_ptr(), stream.cuda_stream)
    else:
        Yh = torch.empty(count, dtype=torch.float64).pin_memory()
        fill_host_parallel(w, offset, count, Yh.numpy())
        Ih = torch.empty(count, dtype=torch.int32).pin_memory()
        h2d, d2h = 8 * count, 4 * count

        def step():
            eos.eos_search_host(obj.handle, Yh.data_ptr(), count, Ih.data_ptr(), stream.cuda_stream)
    for _ in range(3):  # warm-up
        step()
    torch.cuda.synchronize()
    if not a.e2e_steps:  # >= ~50 ms of timed calls (small launches are noisy), 3 .. 2000 steps
        import time
        t_probe = time.perf_counter()
        step()
        torch.cuda.synchronize()
        probe_ms = (time.perf_counter() - t_probe) * 1e3
        steps = int(min(2000, max(steps, 50.0 / max(probe_ms, 1e-3))))
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d.barrier()
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    d.barrier()
    tm = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
    d.allreduce(tm, "max")
    ms = float(tm[0]) / steps
    return {"value": round(total / (ms * 1e-3) / 1e9, 4), "unit": "Gpairs/s" if is2d else "Glookups/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "ms_per_step": round(ms, 3), "api": "eos_interp2d_host" if is2d else "eos_search_host",
            "units_per_step": total, "host_buffers": "pinned"}


def fill_host_parallel(w, offset, count, out, threads=None):
    from concurrent.futures import ThreadPoolExecutor
    threads = threads or host_cores()
    if w.targets.kind == "walk":
        out[:] = w.targets.host_fill(offset, count)
        return
    step = (count + threads - 1) // threads

    def job(s):
        e = min(count, s + step)
        out[s:e] = w.targets.host_fill(offset + s, e - s, w.table)
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(0, count, step)))


def ncu_traffic(workload, count, plan):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from an
    `ncu --set full` capture of exactly this launch -- same workload, same units per GPU,
    same plan -- kept under profiles/ (scripts/ncu_traffic.py); else null."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        v = d.get(workload)
        if isinstance(v, dict) and v.get("captured_units") == count and v.get("plan") == plan:
            return v.get("dram_bytes_per_launch")
    return None


# -------------------------------------------------------- CPU oracle -------
def oracle_run(w, is2d, sample: int, threads: int, loglog: bool = False, deriv: bool = False):
    """Time the oracle (as it stands) on the first `sample` units of the workload -- the
    oracle function of the same variant (log-log / derivatives) as the GPU arm."""
    import oracle
    if is2d:
        rho = w.rho_targets.host_fill(0, sample)
        T = w.T_targets.host_fill(0, sample)
        t = time.perf_counter()
        if loglog:   # P, brackets and both derivatives in one call
            oracle.interp2d_loglog(w.rho, w.T, w.P, rho, T, threads=threads)
        else:
            oracle.interp2d(w.rho, w.T, w.P, rho, T, threads=threads)
            if deriv:
                oracle.interp2d_deriv(w.rho, w.T, w.P, rho, T, threads=threads)
        return time.perf_counter() - t
    Y = np.empty(sample, dtype=np.float64)
    fill_host_parallel(w, 0, sample, Y)
    t = time.perf_counter()
    oracle.search(w.table, Y, threads=threads)
    return time.perf_counter() - t


def cpu_sample_size(w, is2d):
    return min(w.count, (1 << 25) if is2d else (1 << 27))


def cpu_baseline(w, is2d, min_cpu_s: float = 12.0, max_passes: int = 20, loglog: bool = False,
                 deriv: bool = False):
    """The oracle as it stands, on the first `sample` units of the workload, repeated
    until about `min_cpu_s` seconds of CPU work (threads x wall) are done, over all host
    cores; plus the paper's single-core protocol ("All the tests were run on a
    single core"): ns per unit on a fixed 2^24-unit prefix (2^22 pairs in 2-D), 1 thread."""
    threads = host_cores()
    sample = cpu_sample_size(w, is2d)
    times = []
    while not times or (sum(times) * threads < min_cpu_s and len(times) < max_passes):
        times.append(oracle_run(w, is2d, sample, threads, loglog, deriv))
    dt = float(np.sum(times))
    one = min(w.count, (1 << 22) if is2d else (1 << 24))
    t1 = oracle_run(w, is2d, one, 1, loglog, deriv)
    return {"value": round(len(times) * sample / dt / 1e9, 5),
            "unit": "Gpairs/s" if is2d else "Glookups/s", "cores": threads, "kind": "oracle",
            "sample": f"first {sample} units of {w.name} (host-generated, same recipe) x "
                      f"{len(times)} passes, oracle/eos_oracle.c over {threads} threads; "
                      f"{dt:.2f} s wall ({dt * threads:.1f} CPU-s); cpu: {cpu_model()}",
            "single_core": {"ns_per_unit": round(t1 / one * 1e9, 2), "units": one, "threads": 1,
                            "value": round(one / t1 / 1e9, 6),
                            "protocol": "P:222 single core; first 2^24 units (2^22 pairs)"}}


# ------------------------------------------------------ reference arm ------
def run_reference(a, d: Dist):
    """The oracle as the reference arm, on rank 0 only: exactly W warm-up and K timed steps
    of the same workload and config as our arm, each step a bounded sample of it (the
    first `sample` units, sized from the warm-up rate so that the K steps take about a
    minute of wall time)."""
    import datagen
    w = datagen.workload(a.workload)
    is2d = w.is_2d
    threads = host_cores()
    probe = min(w.count, 1 << 16)
    t = oracle_run(w, is2d, probe, threads, a.loglog, a.derivatives)
    rate = probe / max(t, 1e-6)
    cap = min(w.count, (1 << 23) if is2d else (1 << 25))
    sample = int(min(cap, max(probe, rate * 60.0 / max(a.steps, 1))))
    for _ in range(a.warmup):
        oracle_run(w, is2d, sample, threads, a.loglog, a.derivatives)
    times = [oracle_run(w, is2d, sample, threads, a.loglog, a.derivatives) for _ in range(a.steps)]
    s = float(np.mean(times)) if times else t
    value = sample / s / 1e9
    unit = "Gpairs/s" if is2d else "Glookups/s"
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": unit,
        "n_gpus": d.world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(s * 1e3, 3),
        "higher_is_better": True, "scaling": "strong" if a.workload == "cfg5" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same recipe, host-generated)",
        "config": bench_config(a, w, d.world),
        "cpu_baseline": {"value": round(value, 6), "unit": unit, "cores": threads, "kind": "oracle",
                         "sample": f"each step: the first {sample} units of {w.name}, oracle/"
                                   f"eos_oracle.c over {threads} threads; cpu: {cpu_model()}"},
        "e2e": {"value": round(value, 6), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference arm = the CPU oracle (no reference implementation exists; PAPER.md "
                "only); one step = the oracle over a bounded sample of the workload",
    }


def self_launch(a) -> int:
    """--gpus N outside a torchrun environment: re-run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1, a free port)."""
    import socket
    import subprocess
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(a))
    d = Dist()
    if d.world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={d.world}")
    if a.impl == "reference":
        if d.rank == 0:
            print(json.dumps(run_reference(a, d)), flush=True)
        return
    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(d.local)
    d.init("nccl")
    try:
        res = run_ours(a, d)
        if d.rank == 0:
            print(json.dumps(res), flush=True)
    finally:
        d.close()


if __name__ == "__main__":
    main()
