#!/usr/bin/env python
"""Small end-to-end exercise of every libvgicp kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run): device kNN + covariances,
voxel-map builds (k_hash_insert's atomicCAS insertion, int64-key and 32-bit-key maps), the
batched path (K-compose, K4a, K4b with its cp.async shared-memory ring, K5, K6) in every
mode through the staged host pipeline and the small-batch graph, lookups, per-point terms,
downsampling and deskew.  No torch: only the library's own kernels run."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_00242_b200 import _lib, geometry as G, registration as RG, synthetic  # noqa: E402
from paper_2202_00242_b200.preprocess import make_frame  # noqa: E402


def main():
    rng = np.random.default_rng(3)
    truth = synthetic.random_submap_poses(rng, 24)
    dirs = synthetic.ray_table(64, 32)
    scans = [synthetic.scan(p, dirs, np.random.default_rng(50 + i)) for i, p in enumerate(truth)]
    clouds, maps, srcs = [], [], []
    for s in scans:
        full = _lib.DeviceCloud(s, None)
        _, covs, _ = full.estimate_covariances(10, 1e-3, want_neighbors=True)
        maps.append(_lib.DeviceMap.build(full, 1.0))
        sel = np.sort(rng.choice(len(s), 300, replace=False))
        clouds.append(_lib.DeviceCloud(s[sel], covs[sel]))
        srcs.append((s[sel], covs[sel]))
    pairs = synthetic.nearest_pairs(truth, 6)
    F = len(pairs)
    table = np.array([G.pose_row(G.pose_retract(p, synthetic.perturbation(rng, 0.05, 1.0)))
                      for p in truth])
    unary = [(f % 5) == 0 for f in range(F)]
    b = _lib.DeviceBatch([clouds[i] for i in pairs[:, 0]], [maps[j] for j in pairs[:, 1]], unary,
                         [10] * F, pairs[:, 0], pairs[:, 1])
    for mode in (_lib.MODE_LINEARIZE, _lib.MODE_COST, _lib.MODE_COMPACT, _lib.MODE_INLIERS):
        b.linearize_poses(table, mode)
    b.linearize_poses_f32(table)
    b.lookup_rows(table)
    b.assemble_setup(len(truth))
    ne = b.assemble_poses(table)
    # a batch large enough for the staged multi-stream host pipeline (>= 8,192 factors)
    big = _lib.DeviceBatch([clouds[i] for i in pairs[:, 0]] * 220, [maps[j] for j in pairs[:, 1]] * 220,
                           [False] * (F * 220), [10] * (F * 220), np.tile(pairs[:, 0], 220),
                           np.tile(pairs[:, 1], 220))
    big.linearize_poses(table)
    big.linearize_poses_f32(table)
    big.linearize_poses(table, _lib.MODE_COST)
    # per-factor API: int64-key map (wide extent), non-fp32 points, terms, lookups
    pts = np.vstack([scans[0], [[3000.0, 1.0, 1.0]]])
    covs = np.tile(np.eye(3) * 0.01, (len(pts), 1, 1))
    wide = RG.build_voxelmap(make_frame(pts, covs), 0.5)
    src = make_frame(scans[0][:500] + 1e-7, covs[:500])
    t = G.Se3Pose(G.so3_exp([0.01, 0.02, -0.01]), np.array([0.05, 0.0, 0.02]))
    RG.match_terms(src, wide, t)
    RG.matching_cost(src, wide, t)
    RG.overlap_rate(src, wide, t)
    wide.lookup(pts[:1000])
    # scan front end: voxel downsampling (split cells) and the per-point deskew
    from paper_2202_00242_b200 import preprocess as PP

    raw = PP.RawScan(points=scans[1], stamps=np.linspace(0.0, 0.1, len(scans[1])),
                     scan_start=0.0, scan_end=0.1)
    PP.voxel_downsample(raw, 0.25)
    node_t = np.linspace(-0.01, 0.11, 7)
    quats = np.tile([0.0, 0.0, 0.0, 1.0], (7, 1))
    quats[:, 2] = np.linspace(0, 0.05, 7)
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    PP.deskew_points(scans[1], raw.stamps, node_t, quats, np.outer(np.linspace(0, 1, 7), [1, 0, 0]))
    PP.pack_voxel_keys(scans[2], 0.4)
    print(f"sanitize case ok: {F} factors, {b.num_items} items, cost {ne.cost:.6g}, "
          f"{_lib.context().launch_count()} launches")


if __name__ == "__main__":
    main()
