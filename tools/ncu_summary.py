#!/usr/bin/env python
"""Summarise an ncu report: per kernel key throughput / occupancy / stall metrics."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def main(path, json_out=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    summary = {}
    for r in rows[2:]:
        d0 = dict(zip(hdr, r))
        name = d0.get("Kernel Name", "").split("(")[0].replace("void ", "").strip()
        summary.setdefault(name, {
            "time_us": d0.get("gpu__time_duration.sum"),
            "l2_hit_rate_pct": d0.get("lts__t_sector_hit_rate.pct"),
            "l1_hit_rate_pct": d0.get("l1tex__t_sector_hit_rate.pct"),
            "l1_throughput_pct": d0.get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": d0.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": d0.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "dram_read_mb": d0.get("dram__bytes_read.sum"),
            "dram_write_mb": d0.get("dram__bytes_write.sum"),
            "registers": d0.get("launch__registers_per_thread")})
        d = dict(zip(hdr, r))
        print("==", d.get("Kernel Name", "")[:90])
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]}")
        st = {k[len(STALLS):]: float(v or 0) for k, v in d.items()
              if k.startswith(STALLS) and not k.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:7]
        print("   stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
    if json_out:
        import json

        with open(json_out, "w") as f:
            json.dump({k: {m: float(v) if v not in (None, "") else None for m, v in d.items()}
                       for k, d in summary.items()}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
