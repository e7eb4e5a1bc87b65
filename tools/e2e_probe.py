#!/usr/bin/env python
"""e2e probe (config 5): the host-buffer batch API with pinned outputs, fp32 and fp64 records,
median of N calls; the staging knobs (VGICP_STAGES, VGICP_STAGE_STREAMS, VGICP_STAGE_RATIO)
are read from the environment at batch creation.  Prints one JSON object."""
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_00242_b200 import _lib, workloads  # noqa: E402


def main(reps=30):
    wl = workloads.global_mapping()
    b = wl.batch()
    poses = torch.from_numpy(wl.pose_table.copy()).pin_memory().numpy()
    F = len(wl.pairs)
    o32 = torch.empty((F, _lib.REC_LINEARIZE_F32), dtype=torch.float32).pin_memory().numpy()
    o64 = torch.empty((F, 92), dtype=torch.float64).pin_memory().numpy()
    res = {"corr": wl.num_points}
    for name, fn in (("f32", lambda: b.linearize_poses_f32(poses, out=o32)),
                     ("f64", lambda: b.linearize_poses(poses, out=o64))):
        ts = []
        for k in range(reps + 3):
            torch.cuda.synchronize()
            a = time.perf_counter()
            fn()
            if k >= 3:
                ts.append((time.perf_counter() - a) * 1e3)
        res[f"{name}_ms"] = statistics.median(ts)
        res[f"{name}_gcorr"] = wl.num_points / statistics.median(ts) / 1e6
    print(json.dumps(res))


if __name__ == "__main__":
    main()
