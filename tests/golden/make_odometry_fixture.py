"""Record the REFERENCE's own OdometryEstimator on the synthetic sequence of
tools/odometry_replay.py (30 frames, unmodified numpy path) as tests/golden/odometry.npz.

Run here (the container that mounts /root/reference read-only):
    python tests/golden/make_odometry_fixture.py
tests/test_gpu_odometry.py replays the same sequence through the drop-in on the GPU and
compares the per-frame states and keyframe decisions with this run.
"""
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "tools"))

import odometry_replay  # noqa: E402

FRAMES = 30

if __name__ == "__main__":
    res = odometry_replay.run(FRAMES, dropin=False)
    res.pop("seconds")
    np.savez_compressed(Path(__file__).with_name("odometry.npz"),
                        **{k: np.asarray(v) for k, v in res.items()})
    print("keyframes", res["keyframes"].tolist(), "warnings", sum(1 for w in res["warning"] if w))
