#!/usr/bin/env python
"""The reference's own OdometryEstimator (odometry.py:146-300) on a synthetic LiDAR-IMU
sequence, run either unmodified (`--mode reference`: numpy path) or with the drop-in patched
in (`--mode dropin`: integrate.patch — voxel downsampling, kNN, covariances, deskew, voxel
maps, overlap gating, matching factors and the LM's assembly on the GPU).

The sequence is the reference's own generator (synthetic.square_loop_scene +
generate_synthetic_scene, synthetic.py:298-432): a 20 m square loop in a box room, 128 x 16
rays per scan at 10 Hz, 200 Hz IMU, 1 s at rest for the bootstrap, 5 mm range noise.  IMU
samples are handed to process_frame up to each scan's end (the first frame also gets the
0.5 s bootstrap window).  Per frame it records the estimated state (pose, velocity, biases),
the keyframe count, the warning and the wall time; `tests/golden/make_odometry_fixture.py`
stores the reference's run, `tests/test_gpu_odometry.py` replays it through the drop-in.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def reference_path(ref_src: str | None = None) -> Path:
    """limapper's location: the installed copy in baseline/_ref, else the given source tree."""
    p = Path(ref_src) if ref_src else ROOT / "baseline" / "_ref"
    if not (p / "limapper").is_dir():
        raise RuntimeError(f"limapper not found under {p}")
    return p


def scene(n_frames: int = 60, seed: int = 3):
    import limapper.synthetic as syn

    spec = syn.square_loop_scene(perimeter=20.0, n_frames=n_frames, n_azimuth=128,
                                 n_elevation=16, range_noise=0.005, seed=seed)
    return syn.generate_synthetic_scene(spec)


def run(frames: int, dropin: bool) -> dict:
    if dropin:
        sys.path.insert(0, str(ROOT))
        from paper_2202_00242_b200 import integrate

        integrate.patch("limapper")
    from limapper.odometry import OdometryEstimator

    sc = scene()
    odo = OdometryEstimator()
    imu, j = sc.imu, 0
    out = {"t": [], "q": [], "v": [], "bias": [], "keyframes": [], "warning": [], "seconds": []}
    for scan in sc.scans[:frames]:
        horizon = max(scan.scan_end + 0.05, 0.6)
        batch = []
        while j < len(imu) and imu[j].stamp <= horizon:
            batch.append(imu[j])
            j += 1
        a = time.perf_counter()
        res = odo.process_frame(scan, batch)
        out["seconds"].append(time.perf_counter() - a)
        st = res.state
        out["t"].append(np.asarray(st.pose.translation, float))
        out["q"].append(np.asarray(st.pose.rotation.quat, float))
        out["v"].append(np.asarray(st.velocity, float))
        out["bias"].append(np.concatenate([st.bias_accel, st.bias_gyro]).astype(float))
        out["keyframes"].append(len(odo.keyframes))
        out["warning"].append(res.warning or "")
    for k in ("t", "q", "v", "bias"):
        out[k] = np.array(out[k])
    out["keyframes"] = np.array(out["keyframes"])
    out["events"] = json.dumps([{k: (v if isinstance(v, (int, float, str, bool)) else str(v))
                                 for k, v in ev.items()} for ev in odo.keyframe_events])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["reference", "dropin"], default="dropin")
    ap.add_argument("--frames", type=int, default=30)
    ap.add_argument("--ref-src", default=None, help="limapper source tree (default baseline/_ref)")
    ap.add_argument("--out", default=None, help="write the run as .npz")
    a = ap.parse_args()
    sys.path.append(str(reference_path(a.ref_src)))
    res = run(a.frames, a.mode == "dropin")
    if a.out:
        np.savez_compressed(a.out, **{k: (np.array(v) if not isinstance(v, np.ndarray) else v)
                                     for k, v in res.items()})
    sec = np.array(res["seconds"])
    print(json.dumps({"mode": a.mode, "frames": a.frames,
                      "median_frame_s": float(np.median(sec)),
                      "moving_median_frame_s": float(np.median(sec[10:])) if len(sec) > 10 else None,
                      "total_s": float(sec.sum()), "keyframes": int(res["keyframes"][-1]),
                      "warnings": sum(1 for w in res["warning"] if w)}))


if __name__ == "__main__":
    main()
