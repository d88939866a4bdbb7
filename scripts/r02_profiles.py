"""Turn round-2 ncu outputs under gpurun_out/ into the tracked evidence under profiles/:
  profiles/ncu_traffic.json           DRAM bytes per launch of the bench's exact launch
  profiles/r02_<cfg>_ncu_full.json    --set full summaries (scripts/ncu_summary.py)
  profiles/r02_bench_<name>.json      the bench lines of scripts/r02_refresh_benches.sh
  profiles/r02_cfg5_launches.csv      the launch list of a 10-step default bench run"""
import csv, io, json, os, shutil, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import summarise  # noqa: E402

G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def metrics_csv(path):
    text = "\n".join(l for l in open(path).read().splitlines() if l.startswith('"'))
    rows = list(csv.reader(io.StringIO(text)))
    hdr = None
    out = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
            out["kernel"] = d["Kernel Name"]
            out["grid"] = d["Grid Size"]
    return out


def bench_line(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


traffic_path = os.path.join(P, "ncu_traffic.json")
traffic = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum of one launch of the bench's "
                    "exact configuration (workload, units per GPU, plan), from `ncu --metrics "
                    "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` on a B200 "
                    "(scripts/r02_ncu.sh); bench.py reports it only when workload, units and plan "
                    "all match the running launch."}
for cfg, tr, bl in (("cfg5", "r02_ncu_traffic_cfg5.csv", "r02e_n_cfg5.json"),
                    ("cfg2", "r02_ncu_traffic_cfg2.csv", "r02e_n_cfg2.json"),
                    ("cfg4", "r02_ncu_traffic_cfg4.csv", "r02e_n_cfg4.json"),
                    ("big", "r02_ncu_traffic_big.csv", "r02e_n_big.json")):
    m = metrics_csv(os.path.join(G, tr))
    b = bench_line(os.path.join(G, bl))
    units = b["config"]["units_per_gpu"]
    traffic[cfg] = {
        "dram_bytes_per_launch": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
        "dram_read": int(m["dram__bytes_read.sum"]), "dram_write": int(m["dram__bytes_write.sum"]),
        "algorithmic_bytes_per_launch": b["config"]["bytes_per_unit"] * units, "captured_units": units,
        # (2-D lines captured before the plan signature named derivatives ran without them)
        "plan": ({"derivatives": False, **b["plan"]["launch"]} if b["plan"]["launch"]["kind"] == "interp2d"
                 else b["plan"]["launch"]), "kernel": m["kernel"], "grid": m["grid"],
        "ncu_time_ms": m["gpu__time_duration.sum"] / 1e6,
        "source": f"gpurun_out/{tr} (round 2)"}
json.dump(traffic, open(traffic_path, "w"), indent=1)
for name, rep in (("cfg4_interp2d", "r02e_cfg4.ncu-rep"),
                  ("cfg4_loglog_interp2d", "r02e_cfg4_loglog.ncu-rep"),
                  ("big_packed", "r02e_big.ncu-rep")):
    json.dump(summarise(os.path.join(G, rep)), open(os.path.join(P, f"r02_{name}_ncu_full.json"), "w"),
              indent=1)
for f in sorted(os.listdir(G)):  # the bench lines of scripts/r02_refresh_benches.sh
    if f.startswith("r02b_") and f.endswith(".json"):
        shutil.copy(os.path.join(G, f), os.path.join(P, "r02_bench_" + f[len("r02b_"):]))
shutil.copy(os.path.join(G, "r02_cfg5_launches.csv"), os.path.join(P, "r02_cfg5_launches.csv"))
print(json.dumps({k: v for k, v in traffic.items() if k != "_note"}, indent=1))
