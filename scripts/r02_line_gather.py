"""Random sector vs cooperative 128-B line gathers from L2-resident buffers (measure/):
does a whole line requested by 4 lanes of one instruction cost the t-stage one pass?"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import measure
out = {}
for mb in (4, 16, 64):
    out[f"sector_{mb}MB"] = measure.l2_gather_ceiling(mb << 20)
    out[f"line_{mb}MB"] = measure.l2_line_gather_ceiling(mb << 20)
    print(mb, "sectors/s", round(out[f"sector_{mb}MB"]["sectors_per_s"] / 1e9, 1),
          "lines/s", round(out[f"line_{mb}MB"]["lines_per_s"] / 1e9, 1), flush=True)
print(json.dumps(out))
