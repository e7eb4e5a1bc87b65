#!/usr/bin/env python
"""A few config-5 steps (K-compose, K4a, K4b, K5) for ncu: the workload is built first (kNN,
covariance and map-build kernels), then `--steps` device-resident linearizations, each after
an L2 flush.  Select the step kernels with -k regex:"k_compose|k_lookup_fast|k_accumulate|k_finalize"."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_00242_b200 import _lib, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--mode", type=int, default=0)
    a = ap.parse_args()
    ctx = _lib.context(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx.set_stream(st.cuda_stream)
    wl = workloads.global_mapping()
    b = wl.batch(ctx=ctx)
    ctx.set_stream(st.cuda_stream)
    poses = torch.from_numpy(wl.pose_table).cuda()
    out = torch.zeros((len(wl.pairs), 92), dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(a.steps):
        flush.zero_()
        b.linearize_poses_device(poses.data_ptr(), poses.shape[0], a.mode, out.data_ptr())
    torch.cuda.synchronize()
    print("ncu step ok", a.steps, "steps")


if __name__ == "__main__":
    main()
