"""Benchmark workloads of BASELINE.json, built on the GPU with the product's own
preprocessing (device kNN + covariances, device voxel maps).

single_factor() — config 1; odometry_window() — config 3; local_mapping() — config 4 (the
single-GPU workloads, tools/bench_configs.py); global_mapping() — config 5 (bench.py).

global_mapping(): config 5 — N submaps, each a 256 x 64 = 16,384-point scan from a random
pose in the room; the source cloud of submap i is a seeded random subsample of its scan with
n ~ U[200, 600] points; the target map of submap j is its full scan at 1.0 m
(config.py:56); one binary factor per ordered pair (i -> j) for the k nearest submaps j of
each i, listed by target j; estimates are the truth perturbed by (0.05 m, 1 deg).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib, synthetic
from .geometry import pose_retract, pose_row


@dataclass
class GlobalWorkload:
    n_submaps: int
    neighbors: int
    resolution: float
    truth: list
    estimates: list
    scans: list                 # host fp32-exact points per submap
    scan_covs: list             # host covariances per submap (device kNN + covariance)
    source_index: list          # indices of each submap's source subsample in its scan
    pairs: np.ndarray           # (F, 2) (source submap i, target submap j)
    pose_table: np.ndarray      # (n_submaps, 8) estimates, quat xyzw + t
    clouds: list = field(default_factory=list)   # DeviceCloud of each source subsample
    maps: list = field(default_factory=list)     # DeviceMap of each full scan
    num_points: int = 0         # correspondences per linearization (sum of source sizes)

    def batch(self, factor_ids=None, ctx=None) -> _lib.DeviceBatch:
        ids = np.arange(len(self.pairs)) if factor_ids is None else np.asarray(factor_ids)
        p = self.pairs[ids]
        return _lib.DeviceBatch([self.clouds[i] for i in p[:, 0]], [self.maps[j] for j in p[:, 1]],
                                [False] * len(ids), [10] * len(ids), p[:, 0], p[:, 1], ctx=ctx)


def global_mapping(n_submaps: int = 1000, neighbors: int = 50, resolution: float = 1.0,
                   n_az: int = 256, n_el: int = 64, seed: int = 5, device_objects: bool = True,
                   knn: int = 10) -> GlobalWorkload:
    rng = np.random.default_rng(seed)
    truth = synthetic.random_submap_poses(rng, n_submaps)
    dirs = synthetic.ray_table(n_az, n_el)
    scans = [synthetic.scan(p, dirs, np.random.default_rng(seed * 100003 + i))
             for i, p in enumerate(truth)]
    sizes = rng.integers(200, 601, n_submaps)
    source_index = [np.sort(rng.choice(len(s), int(n), replace=False)) for s, n in zip(scans, sizes)]
    pairs = synthetic.nearest_pairs(truth, neighbors)
    # factor list ordered by target submap (stable in the source): the batch's work items are
    # target-major either way; this order also makes its staged host copies contiguous
    pairs = pairs[np.lexsort((pairs[:, 0], pairs[:, 1]))]
    est = [pose_retract(p, synthetic.perturbation(rng, 0.05, 1.0)) for p in truth]
    wl = GlobalWorkload(n_submaps, neighbors, resolution, truth, est, scans, [], source_index,
                        pairs, np.array([pose_row(p) for p in est]))
    wl.num_points = int(sum(len(source_index[i]) for i in pairs[:, 0]))
    if device_objects:
        for s, sel in zip(scans, source_index):
            full = _lib.DeviceCloud(s, None)
            _, covs, _ = full.estimate_covariances(knn, 1e-3, want_neighbors=False)
            wl.scan_covs.append(covs)
            wl.maps.append(_lib.DeviceMap.build(full, resolution))
            wl.clouds.append(_lib.DeviceCloud(s[sel], covs[sel]))
    return wl


@dataclass
class FactorWorkload:
    """A generic factor set: per-factor device clouds/maps, variables in a pose table, and
    the host inputs the CPU oracle needs for a bounded sample."""
    name: str
    config: dict
    clouds: list                 # DeviceCloud per factor
    maps: list                   # DeviceMap per factor
    unary: list
    var_source: np.ndarray
    var_target: np.ndarray
    pose_table: np.ndarray       # (V, 8): variables, then the fixed targets of unary factors
    host_sources: list           # (points, covs) per factor (host)
    host_maps: list              # oracle-format voxel map per factor (built lazily)
    host_targets: list           # (points, covs, resolution) per factor
    num_points: int = 0

    def batch(self, ctx=None) -> _lib.DeviceBatch:
        F = len(self.clouds)
        return _lib.DeviceBatch(self.clouds, self.maps, self.unary, [10] * F, self.var_source,
                                self.var_target, ctx=ctx)


def _device_frame(points, knn=10):
    cloud = _lib.DeviceCloud(points, None)
    _, covs, _ = cloud.estimate_covariances(knn, 1e-3, want_neighbors=False)
    return cloud, covs


def single_factor() -> FactorWorkload:
    """Config 1: one binary factor between two 16,384-point scans, 0.5 m target map."""
    source, target, t_i, t_j = synthetic.config1_scans()
    src, src_covs = _device_frame(source)
    tgt, tgt_covs = _device_frame(target)
    dmap = _lib.DeviceMap.build(tgt, 0.5)
    table = np.array([pose_row(t_i), pose_row(t_j)])
    return FactorWorkload("single binary factor (BASELINE config 1)",
                          {"scan_points": 16384, "voxel_resolution_m": 0.5, "factors": 1},
                          [src], [dmap], [False], np.array([0]), np.array([1]), table,
                          [(source, src_covs)], [None], [(target, tgt_covs, 0.5)],
                          num_points=len(source))


def odometry_window(seed: int = 3) -> FactorWorkload:
    """Config 3: a new 16,384-point frame against 20 keyframes + 3 recent frames, each with
    maps at 0.5 / 1.0 / 2.0 m (69 factors); the 15 oldest keyframes are unary (fixed pose)."""
    rng = np.random.default_rng(seed)
    dirs = synthetic.ray_table(256, 64)
    traj = synthetic.circle_trajectory(24, step=0.4)
    scans = [synthetic.scan(p, dirs, np.random.default_rng(seed * 1000 + k))
             for k, p in enumerate(traj)]
    est = [pose_retract(p, synthetic.perturbation(rng, 0.05, 1.0)) for p in traj]
    new = 23
    frames = [_device_frame(s) for s in scans]
    clouds, maps, unary, vs, vt, hs, ht = [], [], [], [], [], [], []
    # variables: 0 = new frame, 1..3 = recent frames 20..22, 4..8 = keyframes 15..19;
    # keyframes 0..14 are fixed (unary targets, appended to the pose table)
    var_of = {new: 0, 20: 1, 21: 2, 22: 3}
    var_of.update({15 + k: 4 + k for k in range(5)})
    fixed = []
    rows = [None] * 9
    for f, v in var_of.items():
        rows[v] = pose_row(est[f])
    for tgt in list(range(20)) + [20, 21, 22]:
        for res in (0.5, 1.0, 2.0):
            clouds.append(frames[new][0])
            maps.append(_lib.DeviceMap.build(frames[tgt][0], res))
            u = tgt < 15
            unary.append(u)
            vs.append(0)
            if u:
                vt.append(9 + len(fixed))
                fixed.append(pose_row(est[tgt]))
            else:
                vt.append(var_of[tgt])
            hs.append((scans[new], frames[new][1]))
            ht.append((scans[tgt], frames[tgt][1], res))
    table = np.vstack([np.array(rows), np.array(fixed)])
    return FactorWorkload("odometry window (BASELINE config 3)",
                          {"scan_points": 16384, "keyframes": 20, "recent_frames": 3,
                           "resolutions_m": [0.5, 1.0, 2.0], "factors": len(clouds),
                           "unary_factors": int(sum(unary))},
                          clouds, maps, unary, np.array(vs), np.array(vt), table, hs,
                          [None] * len(clouds), ht, num_points=len(scans[new]) * len(clouds))


def local_mapping(frames: int = 100, seed: int = 4) -> FactorWorkload:
    """Config 4: 100 frames of 512 x 16 = 8,192 points on a 0.4 m-step trajectory, one binary
    factor per frame pair (4,950) at 0.5 m."""
    rng = np.random.default_rng(seed)
    dirs = synthetic.ray_table(512, 16)
    traj = synthetic.circle_trajectory(frames, step=0.4)
    scans = [synthetic.scan(p, dirs, np.random.default_rng(seed * 1000 + k))
             for k, p in enumerate(traj)]
    est = [pose_retract(p, synthetic.perturbation(rng, 0.05, 1.0)) for p in traj]
    dev = [_device_frame(s) for s in scans]
    dmaps = [_lib.DeviceMap.build(c, 0.5) for c, _ in dev]
    # target-major factor list (see global_mapping): source i > target j
    pairs = np.array([(i, j) for j in range(frames) for i in range(j + 1, frames)], np.int64)
    return FactorWorkload("local mapping (BASELINE config 4)",
                          {"frames": frames, "scan_points": 8192, "voxel_resolution_m": 0.5,
                           "factors": len(pairs)},
                          [dev[i][0] for i in pairs[:, 0]], [dmaps[j] for j in pairs[:, 1]],
                          [False] * len(pairs), pairs[:, 0], pairs[:, 1],
                          np.array([pose_row(p) for p in est]),
                          [(scans[i], dev[i][1]) for i in pairs[:, 0]], [None] * len(pairs),
                          [(scans[j], dev[j][1], 0.5) for j in pairs[:, 1]],
                          num_points=int(sum(len(scans[i]) for i in pairs[:, 0])))


def lpt_shards(weights: np.ndarray, n_shards: int) -> list:
    from .sharding import lpt_shards as _lpt

    return _lpt(weights, n_shards)
