#!/usr/bin/env python
"""Per-opcode executed thread-instructions per unit from an ncu report's SASS source page.
usage: ncu_mix.py REPORT UNITS"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, units = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc = h.index("Thread Instructions Executed"), h.index("Source")
c = Counter()
for r in rows[2:]:
    if not r[ia].isdigit():
        continue
    toks = r[isrc].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    c[op.split(".")[0]] += int(r[ia])
tot = sum(c.values())
print(f"total {tot / units:.1f} thread-instructions per unit")
for k, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{k:12s} {v / units:7.1f}")
