"""Benchmark workloads of BASELINE.json, built on the GPU with the product's own
preprocessing (device kNN + covariances, device voxel maps).

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


def lpt_shards(weights: np.ndarray, n_shards: int) -> list:
    from .sharding import lpt_shards as _lpt

    return _lpt(weights, n_shards)
