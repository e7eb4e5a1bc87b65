#!/usr/bin/env python
"""Single-GPU BASELINE configs other than the headline one: 1 (single binary factor),
2 (preprocessing: kNN covariances + 3 voxel maps of a 131k-point scan), 3 (odometry window,
unary + 3 resolutions), 4 (local mapping, 4,950 factors), and "6": the keyframe overlap
matrix of the config-3 window (overlap gating).

One JSON line per config, with the fields of bench.py's line: device-resident linearization
step (compose + K4a + K4b + K5 replayed as one CUDA graph; CUDA events on the launching
stream, L2 flushed between steps; K4 timed separately with stream launches), e2e through DeviceBatch.linearize_poses with pinned host buffers, K4's fraction of the
HBM roofline (84 B/correspondence), and the CPU oracle on all host cores over a
bounded factor sample.  Config 5 is bench.py itself.

    python tools/bench_configs.py [--configs 1,3,4] [--steps 50] > profiles/r01_configs.jsonl
"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2202_00242_b200 import _lib, workloads  # noqa: E402

BUILDERS = {1: workloads.single_factor, 3: workloads.odometry_window, 4: workloads.local_mapping}


def cpu_sample(wl, max_points=2_000_000):
    """Oracle inputs for the first factors up to ~max_points correspondences."""
    from oracle import vgicp_oracle as O

    fids, pts = [], 0
    for f in range(len(wl.clouds)):
        if fids and pts + len(wl.host_sources[f][0]) > max_points:
            break
        fids.append(f)
        pts += len(wl.host_sources[f][0])
    maps, cache = {}, {}
    for f in fids:
        tp, tc, res = wl.host_targets[f]
        key = (id(tp), res)
        if key not in cache:
            cache[key] = O.build_voxelmap(tp, tc, res)
        maps[f] = cache[key]
    R, t = O.relative_transforms(wl.pose_table, wl.var_source[fids], wl.var_target[fids])
    sample = {"pairs": np.array([(f, f) for f in fids]), "maps": maps,
              "sources": {f: wl.host_sources[f] for f in fids},
              "R": np.zeros((max(fids) + 1, 3, 3)), "t": np.zeros((max(fids) + 1, 3)),
              "points": pts}
    sample["R"][fids] = R
    sample["t"][fids] = t
    return sample, len(fids)


def run(cfg, args, ctx, stream):
    wl = BUILDERS[cfg]()
    batch = wl.batch(ctx=ctx)
    ctx.set_stream(stream.cuda_stream)
    V = wl.pose_table.shape[0]
    F = len(wl.clouds)
    REC = _lib.RECORD_SIZE[_lib.MODE_LINEARIZE]
    poses = torch.from_numpy(wl.pose_table).cuda()
    out = torch.zeros((F, REC), dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def step(ev=None):
        if ev:
            ev[0].record()
        batch.compose_device(poses.data_ptr(), V)
        if ev:
            ev[1].record()
        batch.accumulate_device(_lib.MODE_LINEARIZE)
        if ev:
            ev[2].record()
        batch.finalize_device(_lib.MODE_LINEARIZE, out.data_ptr())
        if ev:
            ev[3].record()

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    with bench.ClockSampler(0) as clk:
        for k in range(args.steps):
            flush.zero_()
            step(evs[k])
        torch.cuda.synchronize()
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    k4_ms = [e[1].elapsed_time(e[2]) for e in evs]
    ms = statistics.median(step_ms)
    if not args.no_graph:
        # the step as one CUDA graph launch (small configs are launch-latency bound)
        batch.capture_graph(poses.data_ptr(), V, _lib.MODE_LINEARIZE, out.data_ptr())
        for _ in range(3):
            batch.launch_graph()
        gms = []
        for k in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            batch.launch_graph()
            e1.record()
            torch.cuda.synchronize()
            gms.append(e0.elapsed_time(e1))
        ms = statistics.median(gms)
    # e2e: host pose table in, host records out (pinned)
    poses_h = torch.from_numpy(wl.pose_table.copy()).pin_memory().numpy()
    out_h = torch.empty((F, REC), dtype=torch.float64).pin_memory().numpy()
    e2e = []
    for k in range(args.steps + 2):
        torch.cuda.synchronize()
        a = time.perf_counter()
        batch.linearize_poses(poses_h, _lib.MODE_LINEARIZE, out=out_h)
        if k >= 2:
            e2e.append((time.perf_counter() - a) * 1e3)
    peak, kind = bench.hbm_peak()
    achieved = bench.BYTES_PER_CORR * wl.num_points / (statistics.median(k4_ms) / 1e3) / 1e9
    cpu = None
    if not args.no_cpu:
        from oracle import cpu_baseline

        sample, nf = cpu_sample(wl)
        rate, sec, procs = cpu_baseline.time_sample(sample, steps=2, warmup=1)
        cpu = {"value": rate, "unit": bench.UNIT, "cores": procs, "kind": "port",
               "sample": f"first {nf} factors, {sample['points']} correspondences per pass, "
                         f"oracle linearization (unary factors evaluated as binary), "
                         f"{procs}-process fork pool, 2 passes"}
    hits = int(out_h[:, 91].sum())  # inlier correspondences (hits) of the e2e records
    cfgd = dict(wl.config)
    cfgd.update({"workload": wl.name, "corr_per_step": wl.num_points, "hits_per_step": hits,
                 "hit_fraction": round(hits / max(wl.num_points, 1), 4),
                 "l2": "flushed between timed steps (256 MB write)",
                 "step": "one CUDA graph (compose + K4a + K4b + K5)" if not args.no_graph
                 else "stream launches"})
    return {"metric": bench.METRIC, "value": wl.num_points / (ms / 1e3), "unit": bench.UNIT,
            "n_gpus": 1, "steps": args.steps, "ms_per_step": ms, "higher_is_better": True,
            "dtype": "f32+f64", "data": "synthetic", "config": cfgd,
            "e2e": {"value": wl.num_points / (statistics.median(e2e) / 1e3), "unit": bench.UNIT,
                    "h2d_bytes_per_step": int(wl.pose_table.nbytes),
                    "d2h_bytes_per_step": int(F * REC * 8),
                    "ms_per_step": statistics.median(e2e)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "kernel": "K4 (K4a + K4b)",
                         "kernel_ms": statistics.median(k4_ms),
                         "bytes_per_corr": bench.BYTES_PER_CORR, "peak_kind": kind},
            "clocks": clk.summary(), "cpu_baseline": cpu}


def run_preprocess(args):
    """Config 2: k-NN (k = 10) covariances + voxel maps at 0.5 / 1.0 / 2.0 m of one
    131,072-point scan (1024 az x 128 el), host points in, device cloud + maps out."""
    from paper_2202_00242_b200 import synthetic

    pts = synthetic.scan(synthetic.yaw_pose(0.2, [1.0, -2.0, 0.0]), synthetic.ray_table(1024, 128),
                         np.random.default_rng(2))
    n = len(pts)

    def once():
        cloud = _lib.DeviceCloud(pts, None)
        cloud.estimate_covariances(10, 1e-3, want_neighbors=False)
        t1 = time.perf_counter()
        maps = [_lib.DeviceMap.build(cloud, r) for r in (0.5, 1.0, 2.0)]
        torch.cuda.synchronize()
        return t1, maps

    for _ in range(2):
        once()
    knn_ms, map_ms = [], []
    for _ in range(max(3, args.steps // 10)):
        torch.cuda.synchronize()
        a = time.perf_counter()
        t1, _ = once()
        b = time.perf_counter()
        knn_ms.append((t1 - a) * 1e3)
        map_ms.append((b - t1) * 1e3)
    cpu = None
    if not args.no_cpu:
        from oracle import vgicp_oracle as O

        a = time.perf_counter()
        nb = O.knn_search(pts, 10)
        covs, _ = O.estimate_covariances(pts, nb)
        b = time.perf_counter()
        for r in (0.5, 1.0, 2.0):
            O.build_voxelmap(pts, covs, r)
        c = time.perf_counter()
        cpu = {"value": n / (b - a), "unit": "points/s", "cores": 1, "kind": "port",
               "sample": f"the same scan once: kNN + covariances {1e3 * (b - a):.0f} ms, 3 map "
                         f"builds {1e3 * (c - b):.0f} ms (single-threaded NumPy/SciPy, as the "
                         f"reference)"}
    # device-resident figure beside it: kNN + covariances of a resident cloud with the results
    # left on the device (wall clock around the call and a context synchronize: no transfers)
    cloud = _lib.DeviceCloud(pts, None)
    dev_ms = []
    for i in range(max(3, args.steps // 10) + 2):
        cloud.ctx.synchronize()
        a = time.perf_counter()
        _lib.check(cloud.ctx.lib.vg_cloud_estimate_covariances(cloud.ctx.handle, cloud.handle,
                                                               10, 1e-3, None, None, None))
        cloud.ctx.synchronize()
        if i >= 2:
            dev_ms.append((time.perf_counter() - a) * 1e3)
    k = statistics.median(knn_ms)
    m = statistics.median(map_ms)
    return {"metric": "points preprocessed/sec (kNN k=10 + covariances)", "value": n / (k / 1e3),
            "unit": "points/s", "n_gpus": 1, "ms_per_step": k, "higher_is_better": True,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "preprocessing (BASELINE config 2)", "scan_points": n,
                       "knn": 10, "resolutions_m": [0.5, 1.0, 2.0],
                       "timing": "wall clock around the host API calls (upload included)"},
            "map_build": {"value": 3 * n / (m / 1e3), "unit": "points/s", "ms_per_step": m},
            "device_resident": {"value": n / (statistics.median(dev_ms) / 1e3),
                                "unit": "points/s", "ms_per_step": statistics.median(dev_ms),
                                "what": "kNN + covariances of a device cloud, results kept on "
                                        "the device (wall clock, no host transfers)"},
            "cpu_baseline": cpu}


def run_frontend(args):
    """Scan front end either side of the path: voxel_downsample of one raw
    131,072-point spinning scan at 0.25 m (odometry downsample_resolution, config.py:21;
    stamps by azimuth over a 0.1 s sweep, so seam voxels split) and the per-point deskew of
    the downsampled frame on a 21-node trajectory, host arrays in and out."""
    from paper_2202_00242_b200 import preprocess as PP
    from paper_2202_00242_b200 import synthetic

    pts = synthetic.scan(synthetic.yaw_pose(0.2, [1.0, -2.0, 0.0]), synthetic.ray_table(1024, 128),
                         np.random.default_rng(2))
    n = len(pts)
    stamps = 50.0 + (np.arctan2(pts[:, 1], pts[:, 0]) + np.pi) / (2 * np.pi) * 0.1
    scan = PP.RawScan(pts, stamps, 50.0, 50.1)
    node_t = np.linspace(50.0, 50.1, 21)
    ang = np.linspace(0.0, 0.12, 21)
    quats = np.column_stack([0.1 * np.sin(ang / 2), np.zeros(21), np.sin(ang / 2),
                             np.cos(ang / 2)])
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    trans = np.column_stack([np.linspace(0, 0.8, 21), np.linspace(0, 0.1, 21), np.zeros(21)])

    def once():
        a = time.perf_counter()
        down = PP.voxel_downsample(scan, 0.25)
        b = time.perf_counter()
        PP.deskew_points(down.points, down.stamps, node_t, quats, trans)
        c = time.perf_counter()
        return (b - a) * 1e3, (c - b) * 1e3, len(down)

    for _ in range(3):
        once()
    ds_ms, dk_ms = [], []
    for _ in range(max(5, args.steps // 5)):
        x, y, m = once()
        ds_ms.append(x)
        dk_ms.append(y)
    cpu = None
    if not args.no_cpu:
        from oracle import vgicp_oracle as O

        a = time.perf_counter()
        dp, dt = O.voxel_downsample(pts, stamps, 0.25, 0.1)
        b = time.perf_counter()
        O.deskew_points(dp, dt, node_t, quats, trans)
        c = time.perf_counter()
        cpu = {"value": n / (b - a), "unit": "points/s", "cores": 1, "kind": "port",
               "sample": f"the same scan once: voxel_downsample {1e3 * (b - a):.0f} ms (per-voxel "
                         f"Python loop, as the reference), deskew per-point {1e3 * (c - b):.1f} ms "
                         f"(NumPy)"}
    d = statistics.median(ds_ms)
    k = statistics.median(dk_ms)
    return {"metric": "raw points downsampled/sec (voxel_downsample 0.25 m)", "value": n / (d / 1e3),
            "unit": "points/s", "n_gpus": 1, "ms_per_step": d, "higher_is_better": True,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "scan front end (voxel_downsample + deskew, SURVEY 8f row 4)",
                       "scan_points": n, "downsampled_points": m, "resolution_m": 0.25,
                       "trajectory_nodes": 21,
                       "timing": "wall clock around the host API calls (copies included)"},
            "deskew": {"value": m / (k / 1e3), "unit": "points/s", "ms_per_step": k},
            "cpu_baseline": cpu}


def run_overlap(args):
    """The keyframe overlap matrix of config 3's window (odometry.py:396-403): every ordered
    pair of the 23 frames (506 overlap_rate calls of 16,384 points each) in one
    VG_MODE_INLIERS launch, vs the oracle's per-pair loop."""
    from paper_2202_00242_b200 import registration as RG
    from paper_2202_00242_b200 import synthetic
    from paper_2202_00242_b200.preprocess import make_frame

    dirs = synthetic.ray_table(256, 64)
    traj = synthetic.circle_trajectory(23, step=0.4)
    scans = [synthetic.scan(p, dirs, np.random.default_rng(900 + k)) for k, p in enumerate(traj)]
    frames, vmaps = [], []
    for sc in scans:
        c = _lib.DeviceCloud(sc, None)
        _, covs, _ = c.estimate_covariances(10, 1e-3, want_neighbors=False)
        f = make_frame(sc, covs)
        frames.append(f)
        vmaps.append(RG.build_voxelmap(f, 1.0))
    RG.overlap_matrix(frames, vmaps, traj)  # warm: uploads + batch
    ms = []
    for _ in range(max(5, args.steps // 5)):
        torch.cuda.synchronize()
        a = time.perf_counter()
        m = RG.overlap_matrix(frames, vmaps, traj)
        ms.append((time.perf_counter() - a) * 1e3)
    n = sum(len(scans[i]) for i in range(23) for j in range(23) if i != j)
    cpu = None
    if not args.no_cpu:
        from oracle import vgicp_oracle as O
        from paper_2202_00242_b200.geometry import pose_compose, pose_inverse

        omaps = [(1.0, v.keys, v.means, v.covs, v.counts) for v in vmaps]
        a = time.perf_counter()
        for i in range(23):
            for j in range(23):
                if i != j:
                    tij = pose_compose(pose_inverse(traj[j]), traj[i])
                    O.overlap_rate(scans[i], omaps[j], tij.rotation.matrix(), tij.translation)
        sec = time.perf_counter() - a
        cpu = {"value": n / sec, "unit": "lookups/s", "cores": 1, "kind": "port",
               "sample": f"the same 506 pairs once: {1e3 * sec:.0f} ms (single-threaded NumPy)"}
    k = statistics.median(ms)
    return {"metric": "voxel lookups/sec (keyframe overlap matrix)", "value": n / (k / 1e3),
            "unit": "lookups/s", "n_gpus": 1, "ms_per_step": k, "higher_is_better": True,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "keyframe overlap matrix (config 3 window, odometry.py:396-403)",
                       "frames": 23, "pairs": 506, "scan_points": 16384,
                       "timing": "wall clock around registration.overlap_matrix (host API)"},
            "cpu_baseline": cpu}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,6,7")  # 6: overlap matrix, 7: front end
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    ctx = _lib.context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    for c in (int(x) for x in args.configs.split(",")):
        line = (run_preprocess(args) if c == 2 else run_overlap(args) if c == 6
                else run_frontend(args) if c == 7 else run(c, args, ctx, stream))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
