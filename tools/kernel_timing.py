#!/usr/bin/env python
"""Per-kernel timing of the batched path on the config-5 workload (CUDA events, same stream).

Times K4 in each mode (linearize / cost / inliers-only) with and without an L2 flush between
launches, plus K-compose and K5.  Used to attribute K4 time to the lookup phase vs the fp64
compute phase.  Prints one JSON object.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_00242_b200 import _lib, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--submaps", type=int, default=1000)
    ap.add_argument("--neighbors", type=int, default=50)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    ctx = _lib.context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx.set_stream(s.cuda_stream)
    wl = workloads.global_mapping(a.submaps, a.neighbors)
    b = wl.batch(ctx=ctx)
    poses = torch.from_numpy(wl.pose_table).cuda()
    out = torch.zeros((len(wl.pairs), 92), dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    b.compose_device(poses.data_ptr(), poses.shape[0])
    res = {"corr": wl.num_points, "factors": len(wl.pairs), "items": b.num_items}

    def timeit(fn, flush_l2):
        ts = []
        for k in range(a.reps + 3):
            if flush_l2:
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if k >= 3:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    for name, mode in (("linearize", 0), ("cost", 1), ("inliers", 3)):
        for fl in (False, True):
            res[f"k4_{name}_{'flush' if fl else 'warm'}_ms"] = timeit(
                lambda: b.accumulate_device(mode), fl)
    res["compose_ms"] = timeit(lambda: b.compose_device(poses.data_ptr(), poses.shape[0]), False)
    b.accumulate_device(0)
    res["finalize_ms"] = timeit(lambda: b.finalize_device(0, out.data_ptr()), False)
    b.finalize_device(3, out.data_ptr())
    torch.cuda.synchronize()
    # normal-equation assembly (K6 + cost): full assemble step minus the linearize step
    b.assemble_setup(poses.shape[0])
    ne = torch.empty(b.asm_size, dtype=torch.float64, device="cuda")
    res["step_linearize_ms"] = timeit(
        lambda: b.linearize_poses_device(poses.data_ptr(), poses.shape[0], 0, out.data_ptr()), True)
    res["step_assemble_ms"] = timeit(
        lambda: b.assemble_poses_device(poses.data_ptr(), poses.shape[0], ne.data_ptr()), True)
    res["assemble_only_ms"] = res["step_assemble_ms"] - res["step_linearize_ms"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
