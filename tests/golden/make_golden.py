"""Generate the golden fixtures by running the REFERENCE implementation itself.

Run here (the container that mounts /root/reference read-only):
    python tests/golden/make_golden.py
It imports limapper from /root/reference/pkg/src (no bytecode written), runs the
reference's own functions on seeded inputs and writes tests/golden/*.npz.  The GPU box never
runs this; tests there only read the committed fixtures.
"""

from __future__ import annotations

import hashlib
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

from limapper import geometry as G  # noqa: E402
from limapper import preprocess as P  # noqa: E402
from limapper import registration as RG  # noqa: E402

from paper_2202_00242_b200 import synthetic  # noqa: E402

OUT = Path(__file__).resolve().parent


def frame(points, covs=None, neighbors=None):
    pts = np.asarray(points, float).reshape(-1, 3)
    return P.Frame(points=pts, stamps=np.zeros(len(pts)), stamp=0.0, neighbors=neighbors,
                   covs=None if covs is None else np.asarray(covs, float), deskewed=True)


def plane_cov_frame(points, k=10):
    f = frame(points)
    f = replace(f, neighbors=P.knn_search(f, k))
    return P.estimate_covariances(f)


def box_points(rng, n_per_wall=120, size=(6.0, 5.0, 3.0), center=(0.17, 0.13, 0.11)):
    sx, sy, sz = size
    pts = []
    for _ in range(n_per_wall):
        u, v = rng.uniform(0, 1, 2)
        pts += [[u * sx - sx / 2, v * sy - sy / 2, -sz / 2], [u * sx - sx / 2, v * sy - sy / 2, sz / 2],
                [u * sx - sx / 2, -sy / 2, v * sz - sz / 2], [u * sx - sx / 2, sy / 2, v * sz - sz / 2],
                [-sx / 2, u * sy - sy / 2, v * sz - sz / 2], [sx / 2, u * sy - sy / 2, v * sz - sz / 2]]
    return (np.asarray(pts) + np.asarray(center)).astype(np.float32).astype(np.float64)


def blocks(lin):
    out = {"h_ii": lin.h_ii, "b_i": lin.b_i, "cost": lin.cost, "inliers": lin.inlier_count}
    if lin.h_ij is not None:
        out.update(h_ij=lin.h_ij, h_jj=lin.h_jj, b_j=lin.b_j)
    return out


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    rng = np.random.default_rng(2024)

    # ---- voxel keys, incl. exact faces and negative coordinates
    pts = np.concatenate([rng.uniform(-30, 30, (2000, 3)),
                          np.round(rng.uniform(-20, 20, (500, 3)) * 4) / 4,
                          np.array([[0.0, -0.0, 0.5], [-0.5, 0.25, -1e-300], [1.5, -2.5, 3.0]])])
    keys = {f"keys_{r}": P.pack_voxel_keys(pts, r) for r in (0.25, 0.4, 0.5, 1.0, 2.0)}
    np.savez_compressed(OUT / "keys.npz", points=pts, **keys)

    # ---- voxel maps + matching on box rooms with plane covariances
    cases = {}
    src_pts = box_points(np.random.default_rng(7), 120)
    src = plane_cov_frame(src_pts)
    tgt_pts = box_points(np.random.default_rng(8), 150)
    tgt = plane_cov_frame(tgt_pts)
    cases["src_points"], cases["src_covs"] = src.points, src.covs
    cases["tgt_points"], cases["tgt_covs"] = tgt.points, tgt.covs
    cases["src_neighbors"] = src.neighbors
    for res in (0.5, 1.0):
        vm = RG.build_voxelmap(tgt, res)
        tag = str(res).replace(".", "p")
        cases[f"map{tag}_keys"], cases[f"map{tag}_means"] = vm.keys, vm.means
        cases[f"map{tag}_covs"], cases[f"map{tag}_counts"] = vm.covs, vm.counts
    vm = RG.build_voxelmap(tgt, 0.5)
    poses = []
    prng = np.random.default_rng(11)
    for c in range(6):
        t_i = G.Se3Pose(G.so3_exp(prng.uniform(-0.05, 0.05, 3)), prng.uniform(-0.1, 0.1, 3))
        t_j = G.Se3Pose(G.so3_exp(prng.uniform(-0.05, 0.05, 3)), prng.uniform(-0.1, 0.1, 3))
        t_ij = G.pose_compose(G.pose_inverse(t_j), t_i)
        R, t = t_ij.rotation.matrix(), t_ij.translation
        terms = RG.match_terms(src, vm, t_ij)
        rows = vm.lookup(terms.moved)
        unary = c % 3 == 2
        lin = RG.linearize_matching_cost(src, vm, t_i, t_j, target_fixed=unary)
        cases[f"case{c}_R"], cases[f"case{c}_t"] = R, t
        cases[f"case{c}_unary"] = np.array(unary)
        cases[f"case{c}_rows"] = rows
        cases[f"case{c}_cost"] = np.array(terms.cost)
        cases[f"case{c}_overlap"] = np.array(RG.overlap_rate(src, vm, t_ij))
        for k, v in blocks(lin).items():
            cases[f"case{c}_{k}"] = np.asarray(v)
        poses.append(np.concatenate([t_i.rotation.quat, t_i.translation, [0.0]]))
        poses.append(np.concatenate([t_j.rotation.quat, t_j.translation, [0.0]]))
    cases["pose_table"] = np.array(poses)
    np.savez_compressed(OUT / "registration.npz", **cases)

    # ---- kNN / covariances
    knn = {}
    for n, k in [(50, 5), (400, 10), (2000, 10)]:
        p = np.random.default_rng(n).uniform(-10, 10, (n, 3))
        knn[f"rand{n}_points"] = p
        knn[f"rand{n}_k"] = np.array(k)
        knn[f"rand{n}_nbrs"] = P.knn_search(frame(p), k)
    dup = np.array([[0, 0, 0], [0, 0, 0], [5, 0, 0], [0, 0, 0], [1, 0, 0]], float)
    knn["dup_points"], knn["dup_nbrs"] = dup, P.knn_search(frame(dup), 3)
    knn["box_points"] = src_pts
    knn["box_nbrs"] = src.neighbors
    knn["box_covs"] = src.covs
    knn["box_degenerate"] = src.degenerate
    planar = np.column_stack([np.random.default_rng(4).uniform(-1, 1, (30, 2)), np.zeros(30)])
    pf = plane_cov_frame(planar)
    knn["planar_points"], knn["planar_covs"] = planar, pf.covs
    np.savez_compressed(OUT / "preprocess.npz", **knn)

    # ---- config 1 (16,384-point scans): outputs only; inputs are regenerated by the package
    source, target, t_i, t_j = synthetic.config1_scans()
    fs = plane_cov_frame(source)
    ft = plane_cov_frame(target)
    vm = RG.build_voxelmap(ft, 0.5)
    t_ij = G.pose_compose(G.pose_inverse(t_j), t_i)
    lin = RG.linearize_matching_cost(fs, vm, t_i, t_j)
    c1 = {"source_sha": np.array(sha(source)), "target_sha": np.array(sha(target)),
          "source_n": np.array(len(source)), "target_n": np.array(len(target)),
          "R": t_ij.rotation.matrix(), "t": t_ij.translation,
          "map_m": np.array(len(vm)), "map_keys_sha": np.array(sha(vm.keys)),
          "rows_sha": np.array(sha(vm.lookup(G.pose_apply(t_ij, fs.points)))),
          "src_nbrs_sha": np.array(sha(fs.neighbors))}
    for k, v in blocks(lin).items():
        c1[k] = np.asarray(v)
    np.savez_compressed(OUT / "config1.npz", **c1)
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


def downsample_cases():
    """voxel_downsample (preprocess.py:73-119) on scans that exercise the split rule, groups
    longer than NumPy's 128-element pairwise block, negative coordinates and exact faces."""
    rng = np.random.default_rng(11)
    cases = {}
    # random order stamps over the whole scan: most multi-point voxels split
    pts = rng.uniform(-2, 2, (3000, 3))
    cases["rand"] = (pts, rng.uniform(0.0, 0.1, 3000), 0.5, 0.0, 0.1)
    # one voxel holding 800 points with a stamp ramp: both cells > 128 members
    pts = np.concatenate([rng.uniform(0.01, 0.49, (800, 3)), rng.uniform(-3, 3, (700, 3))])
    ts = np.concatenate([np.linspace(0.0, 0.1, 800), rng.uniform(0.0, 0.1, 700)])
    cases["big"] = (pts, ts, 0.5, 0.0, 0.1)
    # a spinning scan: first and last azimuths share voxels
    az = np.linspace(0.0, 2 * np.pi, 4096, endpoint=False)
    r = 5.0 + rng.normal(0, 0.02, 4096)
    pts = np.column_stack([r * np.cos(az), r * np.sin(az), rng.uniform(-0.5, 0.5, 4096)])
    cases["spin"] = (pts.astype(np.float32).astype(float), 10.0 + az / (2 * np.pi) * 0.1, 0.3,
                     10.0, 10.1)
    # negative coordinates, exact faces, signed zeros, a non-power-of-two resolution
    g = rng.integers(-8, 8, (400, 3)) * 0.25
    g[:40] = -0.0
    pts = np.concatenate([g, rng.uniform(-2, 2, (300, 3))])
    cases["faces"] = (pts, rng.uniform(5.0, 5.05, 700), 0.25, 5.0, 5.05)
    pts = rng.uniform(-2, 2, (500, 3))
    cases["res04"] = (pts, np.sort(rng.uniform(0.0, 0.1, 500)), 0.4, 0.0, 0.1)
    out = {}
    for name, (p, t, res, t0, t1) in cases.items():
        d = P.voxel_downsample(P.RawScan(p, t, t0, t1), res)
        out[f"{name}_points"], out[f"{name}_stamps"] = p, t
        out[f"{name}_meta"] = np.array([res, t0, t1])
        out[f"{name}_out_points"], out[f"{name}_out_stamps"] = d.points, d.stamps
    np.savez_compressed(OUT / "downsample.npz", **out)
    print("wrote downsample.npz", {k: len(v) for k, v in out.items() if k.endswith("out_stamps")})


def deskew_cases():
    """deskew (preprocess.py:181-232) run by the reference; the node trajectory its host loop
    builds is captured through this package's make_deskew glue (driven by the reference's own
    integration_nodes / propagate_state) so the per-point kernel can be checked on the GPU box,
    where the reference is absent."""
    from limapper import imu as I
    from paper_2202_00242_b200 import preprocess as PP

    rng = np.random.default_rng(21)
    out = {}

    def run(name, n, gyro, accel, state, stamp_lo=0.0, jitter=0.0):
        pts = rng.uniform(-20, 20, (n, 3))
        ts = rng.uniform(stamp_lo, 0.1, n)
        st = np.arange(-0.01, 0.125, 0.005) + rng.uniform(-jitter, jitter, 27)
        samples = [I.ImuSample(float(t), -I.GRAVITY + np.asarray(accel(t)), np.asarray(gyro(t)))
                   for t in np.sort(st)]
        frame = P.Frame(points=pts, stamps=ts, stamp=0.0, scan_end=0.1)
        ref = P.deskew(frame, samples, state)
        cap = {}

        def capture(p, t, node_t, quats, trans):
            cap.update(node_t=node_t.copy(), quats=quats.copy(), trans=trans.copy())
            return ref.points
        PP.make_deskew(P, points_fn=capture)(frame, samples, state)
        out[f"{name}_points"], out[f"{name}_stamps"] = pts, ts
        for k, v in cap.items():
            out[f"{name}_{k}"] = v
        out[f"{name}_out"] = ref.points

    zero = G.SensorState.zero()
    run("stationary", 2000, lambda t: np.zeros(3), lambda t: np.zeros(3), zero)
    run("yaw", 4096, lambda t: np.array([0.0, 0.0, 1.0]), lambda t: np.array([0.5, 0.0, 0.0]),
        zero)
    posed = G.SensorState(pose=G.Se3Pose(G.so3_exp([0.4, -0.1, 1.2]), np.array([10.0, -3.0, 2.0])),
                          velocity=np.array([1.0, 0.5, -0.2]), bias_accel=np.zeros(3),
                          bias_gyro=np.zeros(3), stamp=0.0)
    run("tumble", 4096, lambda t: np.array([3.0 * np.sin(20 * t), -2.0, 4.0 * np.cos(9 * t)]),
        lambda t: np.array([0.3, -0.2, 0.1]) * (1 + 5 * t), posed, stamp_lo=-0.02, jitter=0.002)
    np.savez_compressed(OUT / "deskew.npz", **out)
    print("wrote deskew.npz", {k: v.shape for k, v in out.items() if k.endswith("node_t")})


if __name__ == "__main__":
    if sys.argv[1:] == ["downsample"]:
        downsample_cases()
    elif sys.argv[1:] == ["deskew"]:
        deskew_cases()
    else:
        main()
        downsample_cases()
        deskew_cases()
