#!/usr/bin/env python
"""Top stalled SASS instructions of one kernel in an ncu report."""
import csv
import io
import subprocess
import sys

path, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", kname,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[start]
si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ei, ti = h.index("Instructions Executed"), h.index("Avg. Threads Executed")
data = []
for idx, r in enumerate(rows[start + 1:]):
    if len(r) <= max(wi, ei, ti):
        continue
    try:
        w = float(r[wi] or 0)
    except ValueError:
        continue
    data.append((w, idx, r[si][:75], r[ei], r[ti]))
tot = sum(d[0] for d in data) or 1
print("samples", tot, "instructions", len(data))
for w, idx, s, e, t in sorted(data, reverse=True)[:top]:
    print(f"{100 * w / tot:5.1f}% {idx:5d} {s:75s} exec={e} thr={t}")
