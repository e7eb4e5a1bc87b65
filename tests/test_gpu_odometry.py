"""The reference's own OdometryEstimator (odometry.py:146-300) through the drop-in.

tools/odometry_replay.py feeds a synthetic LiDAR-IMU sequence (the reference's own scene
generator) to the unmodified OdometryEstimator with integrate.patch applied — downsampling,
kNN, covariances, deskew, voxel maps, keyframe overlap gating, matching factors and the LM's
assembly all run through libvgicp — and the per-frame states and keyframe decisions must
agree with the reference's own numpy run recorded in tests/golden/odometry.npz
(tests/golden/make_odometry_fixture.py)."""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_reference_odometry_through_the_dropin_matches_the_reference_run():
    sys.path.insert(0, str(ROOT / "tools"))
    import odometry_replay

    try:
        sys.path.append(str(odometry_replay.reference_path()))
    except RuntimeError as exc:
        pytest.skip(str(exc))
    ref = np.load(ROOT / "tests" / "golden" / "odometry.npz")
    frames = len(ref["keyframes"])
    got = odometry_replay.run(frames, dropin=True)
    assert np.array_equal(got["keyframes"], ref["keyframes"])      # keyframe decisions
    assert list(got["warning"]) == list(ref["warning"])
    dt = np.abs(got["t"] - ref["t"]).max()
    dq = np.abs(np.abs((got["q"] * ref["q"]).sum(1)) - 1.0).max()  # 1 - |cos(half angle)|
    dv = np.abs(got["v"] - ref["v"]).max()
    db = np.abs(got["bias"] - ref["bias"]).max()
    print(f"odometry replay: max |dt| {dt:.2e} m, |dq| {dq:.2e}, |dv| {dv:.2e} m/s, "
          f"|dbias| {db:.2e}; median frame {np.median(got['seconds']):.3f} s")
    # measured: 9e-16 m, 2e-16, 1e-14 m/s, 2e-15 — the run reproduces the reference's
    assert dt < 1e-9 and dq < 1e-12 and dv < 1e-9 and db < 1e-10
