#!/usr/bin/env python
"""K4 time on config 5 under different factor orders (the batch's items follow the target
maps' order of appearance): the workload's (submap-index order of targets), targets along a
Morton curve of the submap positions, and a random target order.  Each on a fresh batch;
CUDA events, L2 flushed before each launch, median of --reps."""
import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_00242_b200 import _lib, workloads  # noqa: E402


def morton_rank(pos):
    lo, hi = pos.min(0), pos.max(0)
    q = np.clip(((pos - lo) / np.maximum(hi - lo, 1e-12) * 1023).astype(np.int64), 0, 1023)
    code = np.zeros(len(pos), np.int64)
    for bit in range(10):
        for ax in range(3):
            code |= ((q[:, ax] >> bit) & 1) << (3 * bit + ax)
    rank = np.empty(len(pos), np.int64)
    rank[np.argsort(code, kind="stable")] = np.arange(len(pos))
    return rank


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    ctx = _lib.context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    wl = workloads.global_mapping()
    poses = torch.from_numpy(wl.pose_table).cuda()
    out = torch.zeros((len(wl.pairs), 92), dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    i, j = wl.pairs[:, 0], wl.pairs[:, 1]
    mr = morton_rank(wl.pose_table[:, 4:7])
    rng = np.random.default_rng(0)
    perm_t = rng.permutation(wl.n_submaps)
    orders = {"workload": np.arange(len(i)),
              "morton_targets": np.lexsort((i, mr[j])),
              "morton_targets_sources": np.lexsort((mr[i], mr[j])),
              "random_targets": np.lexsort((i, perm_t[j]))}
    res = {}
    for name, order in orders.items():
        b = wl.batch(order, ctx=ctx)
        ctx.set_stream(st.cuda_stream)
        b.compose_device(poses.data_ptr(), poses.shape[0])
        for mode, tag in ((0, "linearize"), (1, "cost")):
            ts = []
            for k in range(a.reps + 3):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                b.accumulate_device(mode)
                e1.record()
                torch.cuda.synchronize()
                if k >= 3:
                    ts.append(e0.elapsed_time(e1))
            res[f"{name}_k4_{tag}_ms"] = round(statistics.median(ts), 4)
        ts = []
        for k in range(a.reps + 3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.linearize_poses_device(poses.data_ptr(), poses.shape[0], 0, out.data_ptr())
            e1.record()
            torch.cuda.synchronize()
            if k >= 3:
                ts.append(e0.elapsed_time(e1))
        res[f"{name}_step_ms"] = round(statistics.median(ts), 4)
        del b
    print(json.dumps(res))


if __name__ == "__main__":
    main()
