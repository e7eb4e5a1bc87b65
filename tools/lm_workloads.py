#!/usr/bin/env python
"""LM-level benchmark workloads on the REFERENCE's own factor graph (limapper from
baseline/_ref, drop-in patched in with integrate.patch) — bench infrastructure, not product.

local_mapping_lm(): BASELINE config 4 as a full local-mapping problem — 100 frame-state
variables (15-dof SensorState) on a 0.4 m-step circular PathTrajectory (the reference's
synthetic.py:176-296), 8,192-point scans (512 az x 16 el) cast at the frame poses, all-to-all
MatchingCostFactors at 0.5 m (4,950), 99 ImuFactors preintegrated (imu.py:153-226) from a
200 Hz IMU stream derived from the trajectory exactly as generate_synthetic_scene does
(synthetic.py:327-345), and 100 PriorFactors (a full-state gauge prior on frame 0, bias
priors on every other frame).  Estimates start from the truth perturbed by (0.05 m, 1 deg);
the gauge prior holds frame 0 at the truth.
"""
from __future__ import annotations

import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def _reference():
    if not (REF / "limapper").is_dir():
        raise RuntimeError("reference not installed in baseline/_ref (tools/install_reference.sh)")
    if str(REF) not in sys.path:
        sys.path.append(str(REF))
    from paper_2202_00242_b200 import integrate

    integrate.patch("limapper")
    import limapper.factor_graph as fg
    import limapper.geometry as geo
    import limapper.imu as imu
    import limapper.preprocess as pre
    import limapper.synthetic as syn

    return fg, geo, imu, pre, syn


def local_mapping_lm(frames: int = 100, step: float = 0.4, speed: float = 4.0, seed: int = 4,
                     matching: bool = True):
    """`matching=False`: the frame states, IMU and prior factors only (no scans; no GPU)."""
    sys.path.insert(0, str(ROOT))
    fg, geo, imu, pre, syn = _reference()
    rng = np.random.default_rng(seed)
    radius = frames * step / (2 * math.pi)
    traj = syn.PathTrajectory(syn.CirclePath(radius, laps=1.0), speed, settle=0.0, ramp_time=0.0)
    dt = step / speed
    stamps = [k * dt for k in range(frames)]
    truth = [traj.pose(t) for t in stamps]
    # IMU stream from the analytic derivatives (synthetic.py:333-345), noise-free
    rate = 200.0
    imu_samples = []
    for k in range(int(round(stamps[-1] * rate)) + 2):
        t = k / rate
        rot = traj.pose(t).rotation
        imu_samples.append(imu.ImuSample(t, rot.inverse().apply(traj.accel(t) - imu.GRAVITY),
                                         traj.omega_body(t)))
    g = fg.FactorGraph()
    frames_obj, maps = [], []
    if matching:
        from paper_2202_00242_b200 import _lib, synthetic
        from paper_2202_00242_b200.registration import build_voxelmap

        dirs = synthetic.ray_table(512, 16)
    for k, p in enumerate(truth):
        if matching:
            pts = synthetic.scan(p, dirs, np.random.default_rng(seed * 1000 + k))
            cloud = _lib.DeviceCloud(pts, None)
            _, covs, _ = cloud.estimate_covariances(10, 1e-3, want_neighbors=False)
            f = pre.Frame(points=pts, stamps=np.zeros(len(pts)), stamp=stamps[k], covs=covs,
                          deskewed=True)
            frames_obj.append(f)
            maps.append(build_voxelmap(f, 0.5))
        pert = np.r_[rng.normal(size=3) * (math.radians(1.0) / math.sqrt(3)),
                     rng.normal(size=3) * (0.05 / math.sqrt(3))]
        state = geo.SensorState(pose=geo.pose_retract(p, pert), velocity=traj.velocity(stamps[k]),
                                bias_accel=np.zeros(3), bias_gyro=np.zeros(3), stamp=stamps[k])
        g.add_variable(fg.frame_key(k), state)
    noise = imu.ImuNoiseParams()
    for k in range(frames):
        # the gauge: frame 0's full state at the truth; the other frames: bias priors only
        info = np.r_[np.full(6, 1e6), np.full(3, 1e2), np.full(6, 1e2)] if k == 0 \
            else np.r_[np.zeros(9), np.full(6, 1e2)]
        prior = geo.SensorState(pose=truth[k], velocity=traj.velocity(stamps[k]),
                                bias_accel=np.zeros(3), bias_gyro=np.zeros(3), stamp=stamps[k])
        g.add_factor(fg.PriorFactor(fg.frame_key(k), prior, info))
    for k in range(frames - 1):
        pim = imu.preintegrate(imu_samples, stamps[k], stamps[k + 1], np.zeros(6), noise)
        g.add_factor(fg.ImuFactor(fg.frame_key(k), fg.frame_key(k + 1), pim))
    for j in range(frames if matching else 0):
        for i in range(j + 1, frames):
            g.add_factor(fg.MatchingCostFactor(fg.frame_key(i), frames_obj[i], maps[j],
                                               key_target=fg.frame_key(j)))
    return g, fg, {"frames": frames, "scan_points": int(len(dirs)) if matching else 0,
                   "matching_factors": frames * (frames - 1) // 2 if matching else 0,
                   "imu_factors": frames - 1, "prior_factors": frames, "voxel_resolution_m": 0.5}


def global_mapping_lm(wl):
    """BASELINE config 5 as an LM problem on the reference's FactorGraph: one submap-pose
    variable per submap of `wl` (workloads.global_mapping) at its perturbed estimate, a gauge
    prior on submap 0, and the workload's MatchingCostFactors (source frame i -> map j)."""
    sys.path.insert(0, str(ROOT))
    fg, geo, imu, pre, syn = _reference()
    from paper_2202_00242_b200.registration import GaussianVoxelMap

    g = fg.FactorGraph()
    for i in range(wl.n_submaps):
        row = wl.pose_table[i]
        g.add_variable(fg.submap_key(i), geo.Se3Pose(geo.Rotation(row[:4]), row[4:7].copy()))
    g.add_factor(fg.PriorFactor(fg.submap_key(0), g.values[fg.submap_key(0)], np.full(6, 1e6)))
    frames = [pre.Frame(points=wl.scans[i][sel], stamps=np.zeros(len(sel)), stamp=0.0,
                        covs=wl.scan_covs[i][sel], deskewed=True)
              for i, sel in enumerate(wl.source_index)]
    maps = [GaussianVoxelMap._from_device(wl.resolution, m) for m in wl.maps]
    for i, j in wl.pairs:
        g.add_factor(fg.MatchingCostFactor(fg.submap_key(int(i)), frames[i], maps[j],
                                           key_target=fg.submap_key(int(j))))
    return g, fg, {"variables": wl.n_submaps, "factors": int(len(wl.pairs)), "prior_factors": 1}


def time_lm_iteration(g, fg, info: dict) -> dict:
    """One LM iteration (LmSettings(max_iterations=1)) through the reference's FactorGraph with
    the drop-in patched in — the device solve above the dense threshold (optimize_lm replaced,
    SURVEY §8f row 3) — and, from the same starting values, through the reference's own
    optimize_lm (host dense / splu solve; only total_cost / _assemble_dense replaced)."""
    from paper_2202_00242_b200 import factor_graph as vfg
    from paper_2202_00242_b200 import integrate

    slices, dim = g._slices()
    t0 = time.perf_counter()
    g.total_cost()
    g._assemble_dense(g.values, slices, dim)
    if dim > fg.LmSettings().dense_threshold:
        vfg.DeviceNormalEquations.of(g, slices, dim)  # cuSOLVER handle + device H
    setup = time.perf_counter() - t0
    parts = {}
    for name, fn in (("total_cost_s", lambda: g.total_cost()),
                     ("assemble_dense_s", lambda: g._assemble_dense(g.values, slices, dim))):
        ts = []
        for _ in range(3):
            a = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - a)
        parts[name] = float(np.median(ts))
    start = dict(g.values)
    c0 = g.total_cost()
    one = fg.LmSettings(max_iterations=1)

    def run(fn):  # one LM iteration from the same starting values
        g.values = dict(start)
        g._cached_normal = None
        a = time.perf_counter()
        res = fn()
        return time.perf_counter() - a, res

    first, res = run(lambda: g.optimize_lm(one))
    reps = [run(lambda: g.optimize_lm(one)) for _ in range(3)]
    it, res = sorted(reps, key=lambda r: r[0])[1]
    out = dict(info, seconds=it, seconds_first_call=first, iterations=res.iterations,
               initial_cost=c0, final_cost=res.final_cost, tangent_dim=dim,
               first_call_setup_s=round(setup, 2), **parts)
    if dim > fg.LmSettings().dense_threshold:
        dev_values = res.estimates
        host = integrate.ORIGINALS[(fg.FactorGraph, "optimize_lm")]
        reps_h = [run(lambda: host(g, one)) for _ in range(3)]
        t_h, res_h = sorted(reps_h, key=lambda r: r[0])[1]
        out["seconds_host_solve"] = t_h
        out["final_cost_host_solve"] = res_h.final_cost

        def trans(v):
            return v.translation if hasattr(v, "translation") else v.pose.translation

        out["max_translation_difference_m"] = float(max(
            np.max(np.abs(trans(dev_values[k]) - trans(res_h.estimates[k]))) for k in dev_values))
        out["api"] = ("limapper FactorGraph.optimize_lm(LmSettings(max_iterations=1)) with the "
                      "drop-in: device-resident H, device damped solve (vg_solver_*: cuSOLVER "
                      "Cholesky, LU fallback), reference LM control flow; seconds = median of 3 "
                      "iterations from the same values (seconds_first_call: the first, with "
                      "check_structure and the solver's first factorization); seconds_host_solve "
                      "= the reference's own optimize_lm (host splu) with only total_cost / "
                      "_assemble_dense / check_structure / MatchingCostFactor replaced, median of 3")
    else:
        out["api"] = ("limapper FactorGraph.optimize_lm(LmSettings(max_iterations=1)): reference "
                      "LM and host dense solve (dim <= dense_threshold); drop-in total_cost / "
                      "_assemble_dense / MatchingCostFactor")
    return out


if __name__ == "__main__":
    import json

    g, fg, info = local_mapping_lm()
    print(json.dumps(time_lm_iteration(g, fg, info)))
