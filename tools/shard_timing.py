#!/usr/bin/env python
"""Single-GPU model of the N-rank global-mapping step (bench.py --gpus N): the device work
of the slowest rank's pair-disjoint shard — K-compose, K4a, K4b, K5 and K6 writing its blocks
into the global layout (exchange "reduce", bench.py's default) — timed with CUDA events on one
B200 (L2 flushed between steps), and the sum-reduction to the solver rank priced from its
bytes at the measured NVLink peer bandwidth (B200_PROFILING.md: 770 GB/s per direction) plus
a fixed collective latency.  The collective is not executed here (one GPU); prints one JSON
object per N."""
import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_00242_b200 import _lib, sharding, workloads  # noqa: E402

NVLINK_GBS = 770.0
COLLECTIVE_LATENCY_US = 12.0  # small-message NCCL all-gather latency on 8 GPUs (assumed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--sharding", choices=["target", "pair"], default="target")
    a = ap.parse_args()
    ctx = _lib.context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    wl = workloads.global_mapping()
    F, V = len(wl.pairs), wl.pose_table.shape[0]
    w = np.array([len(wl.source_index[i]) for i in wl.pairs[:, 0]])
    poses = torch.from_numpy(wl.pose_table).cuda()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    base = None
    for n in [int(x) for x in a.ranks.split(",")]:
        if n == 1:
            shards = [np.arange(F)]
        elif a.sharding == "target":
            shards = sharding.target_shards(wl.pairs[:, 1], w, n, wl.pose_table[:, 4:7])
        else:
            shards = sharding.pair_shards(wl.pairs[:, 0], wl.pairs[:, 1], w, n)
        ex = sharding.PairExchange(wl.pairs[:, 0], wl.pairs[:, 1], np.zeros(F, bool), V, shards)
        r = int(np.argmax([w[s].sum() for s in shards]))  # the slowest rank
        b = wl.batch(shards[r], ctx=ctx)
        ctx.set_stream(st.cuda_stream)
        b.assemble_setup_mapped(V, ex.rank_pairs[r], ex.gidx[r], len(ex.pairs))
        rec = torch.zeros((len(shards[r]), 92), dtype=torch.float64, device="cuda")
        ne = torch.zeros(ex.size, dtype=torch.float64, device="cuda")

        def timeit(fn):
            ts = []
            for k in range(a.reps + 3):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                if k >= 3:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            return statistics.median(ts)

        lin = timeit(lambda: b.linearize_poses_device(poses.data_ptr(), V, 0, rec.data_ptr()))
        parts = {
            "compose_us": timeit(lambda: b.compose_device(poses.data_ptr(), V)),
            "k4a_us": timeit(lambda: b.accumulate_device(_lib.MODE_INLIERS)),
            "k4_us": timeit(lambda: b.accumulate_device(_lib.MODE_LINEARIZE)),
            "k5_us": timeit(lambda: b.finalize_device(_lib.MODE_LINEARIZE, rec.data_ptr())),
            "k6_us": timeit(lambda: b.assemble_records_device(rec.data_ptr(), ne.data_ptr())),
            "zero_us": timeit(lambda: ne.zero_()),
        }
        full = timeit(lambda: (ne.zero_(),
                               b.linearize_poses_device(poses.data_ptr(), V, 0, rec.data_ptr()),
                               b.assemble_records_device(rec.data_ptr(), ne.data_ptr())))
        b.capture_assemble_graph(poses.data_ptr(), V, rec.data_ptr(), ne.data_ptr(), True)
        graph_full = timeit(lambda: b.launch_graph())
        b.capture_graph(poses.data_ptr(), V, 0, rec.data_ptr())
        graph_lin = timeit(lambda: b.launch_graph())
        parts["graph_zero_linearize_k6_us"] = graph_full
        parts["graph_linearize_us"] = graph_lin
        if n > 1:
            full = min(full, graph_full)
        else:
            lin = min(lin, graph_lin)
        xbytes = ex.size * 8
        xus = (xbytes / (NVLINK_GBS * 1e9) * 1e6 + COLLECTIVE_LATENCY_US) if n > 1 else 0.0
        step_us = (full if n > 1 else lin) + xus
        if base is None:
            base = step_us
        print(json.dumps({
            "ranks": n, "sharding": a.sharding, "slowest_rank_factors": len(shards[r]),
            "slowest_rank_points": int(w[shards[r]].sum()), "items": b.num_items,
            "linearize_us": round(lin, 1), "zero_linearize_k6_us": round(full, 1),
            "reduce_bytes": xbytes, **{k: round(v, 1) for k, v in parts.items()},
            "exchange_model_us": round(xus, 1), "step_model_us": round(step_us, 1),
            "speedup_vs_1": round(base / step_us, 2)}), flush=True)


if __name__ == "__main__":
    main()
