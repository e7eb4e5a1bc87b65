#!/usr/bin/env python
"""Per-kernel averages from an ncu launch list (CSV of `--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum`), and the DRAM bytes per K4 (= K4a + K4b) launch
that bench.py reports as `roofline.traffic`.

    python tools/launch_traffic.py profiles/r01b_launches.csv profiles/r01b_traffic.json
"""
import ast
import csv
import json
import sys
from collections import defaultdict

K4A = ("k_lookup_fast", "k_lookup_items")
K4B = ("k_accumulate",)


def short(name):
    return name.split("(")[0].replace("void ", "").strip()


def main(src, dst, corr=19900200, bytes_per_corr=84):
    rows = []
    with open(src) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    # keep full-batch launches only (the staged host-output path launches per factor range)
    gmax = defaultdict(int)
    for r in rows:
        g = ast.literal_eval(r["Grid Size"])
        gmax[short(r["Kernel Name"])] = max(gmax[short(r["Kernel Name"])], g[0] * g[1] * g[2])
    rows = [r for r in rows if (lambda g: g[0] * g[1] * g[2])(ast.literal_eval(r["Grid Size"]))
            == gmax[short(r["Kernel Name"])]]
    per = defaultdict(lambda: defaultdict(list))
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        per[short(r["Kernel Name"])][r["Metric Name"]].append(v)
    kern = {k: {m: sum(v) / len(v) for m, v in ms.items()} for k, ms in per.items()}
    counts = {k: len(ms.get("gpu__time_duration.sum", [])) for k, ms in per.items()}
    k4 = 0.0
    names = []
    for k, ms in kern.items():
        if k.startswith(K4A) or k.startswith(K4B):
            k4 += ms.get("dram__bytes_read.sum", 0.0) + ms.get("dram__bytes_write.sum", 0.0)
            names.append(k)
    total_t = sum(ms.get("gpu__time_duration.sum", 0.0) * counts[k] for k, ms in kern.items())
    out = {
        "kernel": "K4 = " + " + ".join(sorted(names)) + " (one launch each per step)",
        "dram_bytes_per_launch": k4,
        "algorithmic_bytes_per_launch": corr * bytes_per_corr,
        "per_kernel": kern,
        "launches": counts,
        "time_share": {k: ms.get("gpu__time_duration.sum", 0.0) * counts[k] / total_t
                       for k, ms in kern.items()},
        "source": f"ncu launch list {src}",
    }
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: round(v, 3) for k, v in out["time_share"].items()}))
    print("K4 DRAM bytes per launch", k4)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
