"""Seeded synthetic LiDAR workloads — workload generator, not product code.

Scans are ray-cast in a closed axis-aligned room (the reference's box_room world,
synthetic.py:45-58) from an az x el ray table (elevation span +-0.45 rad as
synthetic.py:307), with Gaussian range noise, expressed in the sensor frame and rounded to
fp32 so the GPU and CPU paths see identical inputs.  Everything is deterministic in the seed.
"""

from __future__ import annotations

import math

import numpy as np

from .geometry import Rotation, Se3Pose, pose_retract, so3_exp

ROOM_CENTER = (0.11, 0.13, 0.53)
ROOM_SIZE = (40.0, 30.0, 6.0)


def ray_table(n_az: int, n_el: int, el_span=(-0.45, 0.45)) -> np.ndarray:
    """Unit directions, azimuth-major (index = a * n_el + e)."""
    az = np.linspace(0.0, 2 * math.pi, n_az, endpoint=False)
    el = np.linspace(el_span[0], el_span[1], n_el)
    a, e = np.meshgrid(az, el, indexing="ij")
    return np.column_stack([(np.cos(e) * np.cos(a)).ravel(), (np.cos(e) * np.sin(a)).ravel(),
                            np.sin(e).ravel()])


def cast_box(origin: np.ndarray, dirs: np.ndarray, center=ROOM_CENTER, size=ROOM_SIZE,
             min_range=0.3, max_range=60.0):
    """Nearest wall hit per ray from an origin inside the room; (ranges, hit mask)."""
    lo = np.asarray(center, float) - np.asarray(size, float) / 2
    hi = np.asarray(center, float) + np.asarray(size, float) / 2
    best = np.full(dirs.shape[0], np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        for axis in range(3):
            d = dirs[:, axis]
            for wall in (lo[axis], hi[axis]):
                t = (wall - origin[axis]) / d
                ok = np.isfinite(t) & (t >= min_range) & (t <= max_range)
                for other in range(3):
                    if other == axis:
                        continue
                    c = origin[other] + t * dirs[:, other]
                    ok &= (c >= lo[other]) & (c <= hi[other])
                best = np.where(ok & (t < best), t, best)
    return best, np.isfinite(best)


def scan(pose: Se3Pose, dirs_body: np.ndarray, rng: np.random.Generator,
         range_noise: float = 0.01) -> np.ndarray:
    """Points of one scan in the sensor frame (fp32-exact float64 array)."""
    R = pose.rotation.matrix()
    dirs_w = dirs_body @ R.T
    rng_t, hit = cast_box(pose.translation, dirs_w)
    r = rng_t[hit] + rng.normal(scale=range_noise, size=int(hit.sum()))
    pts = dirs_body[hit] * r[:, None]
    return pts.astype(np.float32).astype(np.float64)


def yaw_pose(yaw: float, t) -> Se3Pose:
    return Se3Pose(so3_exp([0.0, 0.0, yaw]), np.asarray(t, float))


def perturbation(rng: np.random.Generator, trans: float, rot_deg: float) -> np.ndarray:
    """Tangent (phi, rho) with |phi| = rot_deg and |rho| = trans in random directions."""
    phi = rng.normal(size=3)
    phi *= math.radians(rot_deg) / np.linalg.norm(phi)
    rho = rng.normal(size=3)
    rho *= trans / np.linalg.norm(rho)
    return np.concatenate([phi, rho])


def random_submap_poses(rng: np.random.Generator, count: int) -> list:
    poses = []
    for _ in range(count):
        yaw = rng.uniform(-math.pi, math.pi)
        xy = rng.uniform([-15.0, -10.0], [15.0, 10.0])
        poses.append(yaw_pose(yaw, [xy[0] + ROOM_CENTER[0], xy[1] + ROOM_CENTER[1], 0.0]))
    return poses


def nearest_pairs(poses, k: int) -> np.ndarray:
    """(i, j) for the k nearest other submaps j of every submap i (deterministic order)."""
    pos = np.array([p.translation for p in poses])
    n = pos.shape[0]
    k = min(k, n - 1)
    d2 = ((pos[:, None, :] - pos[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d2, np.inf)
    nn = np.argsort(d2, axis=1, kind="stable")[:, :k]
    return np.column_stack([np.repeat(np.arange(n), k), nn.ravel()]).astype(np.int64)


def config1_scans(n_az: int = 256, n_el: int = 64):
    """Config 1: target scan from identity, source from (yaw 0.05, t = (0.3, 0.1, 0)),
    linearization poses T_j = P_j, T_i = retract(P_i, xi) with a seeded (0.1 m, 5 deg) xi."""
    dirs = ray_table(n_az, n_el)
    p_j = Se3Pose.identity()
    p_i = yaw_pose(0.05, [0.3, 0.1, 0.0])
    target = scan(p_j, dirs, np.random.default_rng(0))
    source = scan(p_i, dirs, np.random.default_rng(1))
    xi = perturbation(np.random.default_rng(3), 0.1, 5.0)
    return source, target, pose_retract(p_i, xi), p_j


def circle_trajectory(count: int, step: float = 0.4, center=(0.11, 0.13, 0.0)) -> list:
    """`count` poses `step` metres apart on a circle in the room, yaw along the tangent."""
    radius = max(count * step / (2 * math.pi), 3.0)
    poses = []
    for k in range(count):
        a = k * step / radius
        t = [center[0] + radius * math.cos(a), center[1] + radius * math.sin(a), center[2]]
        poses.append(yaw_pose(a + math.pi / 2, t))
    return poses
