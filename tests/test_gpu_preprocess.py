"""GPU kNN / covariance parity (preprocess.py:122-164) against the reference fixtures and
the oracle, plus the reference's own property tests (test_preprocess.py:83-160)."""

import numpy as np
import pytest

from oracle import vgicp_oracle as O
from paper_2202_00242_b200 import geometry as G
from paper_2202_00242_b200 import preprocess as P
from paper_2202_00242_b200.errors import FrameTooSparse

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [50, 400, 2000])
def test_knn_matches_reference(golden, n):
    g = golden("preprocess")
    pts, k = g[f"rand{n}_points"], int(g[f"rand{n}_k"])
    assert np.array_equal(P.knn_search(P.make_frame(pts), k), g[f"rand{n}_nbrs"])


def test_knn_box_room_and_bruteforce(golden):
    g = golden("preprocess")
    assert np.array_equal(P.knn_search(P.make_frame(g["box_points"]), 10), g["box_nbrs"])
    dup = g["dup_points"]
    assert np.array_equal(P.knn_search(P.make_frame(dup), 3), O.knn_bruteforce(dup, 3))


def test_knn_reference_properties():
    f = P.make_frame([[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0]])
    nb = P.knn_search(f, 2)
    assert list(nb[0]) == [0, 1] and list(nb[3]) == [3, 2]
    f = P.make_frame(np.random.default_rng(2).normal(size=(8, 3)))
    for row in P.knn_search(f, 8):
        assert sorted(row) == list(range(8))
    nb = P.knn_search(P.make_frame([[0, 0, 0], [0, 0, 0], [5, 0, 0]]), 2)
    assert list(nb[0]) == [0, 1] and list(nb[1]) == [0, 1]
    with pytest.raises(FrameTooSparse):
        P.knn_search(P.make_frame([[0, 0, 0]]), 2)


def test_knn_large_scan_vs_oracle():
    from paper_2202_00242_b200 import synthetic

    pts = synthetic.scan(synthetic.yaw_pose(0.3, [1.0, -2.0, 0.0]), synthetic.ray_table(256, 32),
                         np.random.default_rng(5))
    ours = P.knn_search(P.make_frame(pts), 10)
    ref = O.knn_search(pts, 10)
    d2o = O.squared_distances(pts, ours)
    d2r = O.squared_distances(pts, ref)
    # identical distance profiles; indices identical except inside exact distance ties
    assert np.array_equal(d2o, d2r)
    assert np.mean(np.all(ours == ref, axis=1)) > 0.999


def test_covariances_match_reference(golden):
    g = golden("preprocess")
    f = P.make_frame(g["box_points"], neighbors=g["box_nbrs"])
    out = P.estimate_covariances(f)
    np.testing.assert_allclose(out.covs, g["box_covs"], rtol=0, atol=1e-9)
    assert np.array_equal(out.degenerate, g["box_degenerate"])


def test_covariance_properties():
    rng = np.random.default_rng(4)
    pts = np.column_stack([rng.uniform(-1, 1, 30), rng.uniform(-1, 1, 30), np.zeros(30)])
    f = P.make_frame(pts)
    out = P.estimate_covariances(P.Frame(points=f.points, stamps=f.stamps, stamp=0.0,
                                         neighbors=P.knn_search(f, 10)))
    evals, evecs = np.linalg.eigh(out.covs[0])
    assert np.allclose(evals, [1e-3, 1.0, 1.0], atol=1e-9)
    assert abs(abs(evecs[2, 0]) - 1.0) < 1e-9
    pts = np.tile([[1.0, 2.0, 3.0]], (5, 1))
    f = P.make_frame(pts)
    out = P.estimate_covariances(P.Frame(points=f.points, stamps=f.stamps, stamp=0.0,
                                         neighbors=P.knn_search(f, 5)))
    assert np.allclose(out.covs[0], 1e-3 * np.eye(3)) and out.degenerate[0]
    pts = np.random.default_rng(6).normal(size=(50, 3))
    rot = G.so3_exp(np.random.default_rng(7).uniform(-2, 2, 3)).matrix()

    def covs_of(p):
        f = P.make_frame(p)
        return P.estimate_covariances(P.Frame(points=f.points, stamps=f.stamps, stamp=0.0,
                                              neighbors=P.knn_search(f, 10))).covs

    a, b = covs_of(pts), covs_of(pts @ rot.T)
    for ca, cb in zip(a, b):
        assert np.allclose(rot @ ca @ rot.T, cb, atol=1e-9)
    with pytest.raises(ValueError):
        P.estimate_covariances(P.make_frame(pts))


def test_fused_knn_covariances_vs_oracle():
    from paper_2202_00242_b200 import synthetic

    pts = synthetic.scan(G.Se3Pose.identity(), synthetic.ray_table(128, 32),
                         np.random.default_rng(8))
    out = P.knn_covariances(P.make_frame(pts), 10)
    ref, degen = O.estimate_covariances(pts, O.knn_search(pts, 10))
    # compare where the smallest eigen-direction is resolvable (eigengap >= 1e-6 relative)
    nb = pts[O.knn_search(pts, 10)]
    c = nb - nb.mean(1, keepdims=True)
    lam = np.linalg.eigvalsh(np.einsum("nki,nkj->nij", c, c) / 10)
    ok = (lam[:, 1] - lam[:, 0]) > 1e-6 * lam[:, 2]
    assert ok.mean() > 0.99
    np.testing.assert_allclose(out.covs[ok], ref[ok], rtol=0, atol=1e-6)
    assert np.array_equal(out.degenerate, degen)


def _brute_knn(pts, k, chunk=512):
    """(d2, index)-ordered brute force with the reference's d2 association (dx²+dz²)+dy²."""
    out = np.empty((len(pts), k), np.int64)
    idx = np.arange(len(pts))
    for a in range(0, len(pts), chunk):
        q = pts[a:a + chunk]
        d = pts[None, :, :] - q[:, None, :]
        sq = d * d
        d2 = (sq[..., 0] + sq[..., 2]) + sq[..., 1]
        order = np.lexsort((np.broadcast_to(idx, d2.shape), d2), axis=1)
        out[a:a + chunk] = order[:, :k]
    return out


@pytest.mark.parametrize("case", ["lattice_ties", "clusters_outliers", "flat"])
def test_grid_knn_exact_on_hard_clouds(case):
    """Clouds >= 4096 points take the grid kNN: exact (d2, index) order, including exact
    distance ties (integer lattice), duplicates, far outliers and a degenerate (flat) extent."""
    rng = np.random.default_rng(3)
    if case == "lattice_ties":
        g = np.stack(np.meshgrid(np.arange(20), np.arange(20), np.arange(12), indexing="ij"), -1)
        pts = g.reshape(-1, 3).astype(float) * 0.5
        pts = np.vstack([pts, pts[:300]])                      # exact duplicates
    elif case == "clusters_outliers":
        centers = rng.uniform(-30, 30, (12, 3))
        pts = np.vstack([c + rng.normal(scale=0.2, size=(400, 3)) for c in centers])
        pts = np.vstack([pts, rng.uniform(-500, 500, (20, 3))])  # isolated far points
    else:
        pts = np.column_stack([rng.uniform(-5, 5, 5000), rng.uniform(-5, 5, 5000), np.zeros(5000)])
    pts = pts.astype(np.float32).astype(np.float64)
    assert len(pts) >= 4096
    ours = P.knn_search(P.make_frame(pts), 10)
    assert np.array_equal(ours, _brute_knn(pts, 10))


# ---- voxel_downsample (preprocess.py:73-119) ------------------------------------------------

def _scan(points, stamps, start=0.0, end=0.1):
    return P.RawScan(np.asarray(points, float), np.asarray(stamps, float), start, end)


@pytest.mark.parametrize("case", ["rand", "big", "spin", "faces", "res04"])
def test_voxel_downsample_matches_reference(golden, case):
    """Bit-identical to the reference's own output (tests/golden/downsample.npz), order
    included: split groups, 800-member cells (pairwise stamp sums), faces, signed zeros."""
    g = golden("downsample")
    res, t0, t1 = g[f"{case}_meta"]
    out = P.voxel_downsample(_scan(g[f"{case}_points"], g[f"{case}_stamps"], t0, t1), res)
    assert np.array_equal(out.points, g[f"{case}_out_points"])
    assert np.array_equal(out.stamps, g[f"{case}_out_stamps"])
    assert out.scan_start == t0 and out.scan_end == t1


def test_voxel_downsample_reference_tests():
    """test_preprocess.py:29-79 on the GPU path."""
    out = P.voxel_downsample(_scan([[0.01, 0, 0], [0.02, 0, 0]], [0.000, 0.004]), 0.1)
    assert len(out) == 1
    assert np.allclose(out.points[0], [0.015, 0, 0]) and out.stamps[0] == pytest.approx(0.002)
    assert len(P.voxel_downsample(_scan([[0.01, 0, 0], [0.02, 0, 0]], [0.0, 0.05]), 0.1)) == 2
    out = P.voxel_downsample(_scan([[1.0, 2.0, 3.0]], [0.05]), 0.25)
    assert len(out) == 1 and np.allclose(out.points[0], [1.0, 2.0, 3.0])
    empty = _scan(np.zeros((0, 3)), np.zeros(0))
    assert len(P.voxel_downsample(empty, 0.25)) == 0
    pts = np.tile([[0.05, 0.05, 0.05]], (10, 1))
    assert len(P.voxel_downsample(_scan(pts, np.linspace(0.0, 0.1, 10)), 1.0)) == 2
    rng = np.random.default_rng(0)
    pts = rng.uniform(-2, 2, (500, 3))
    out = P.voxel_downsample(_scan(pts, rng.uniform(0.0, 0.1, 500)), 0.5)
    uniq = {tuple(k) for k in np.floor(pts / 0.5).astype(int)}
    assert len(uniq) <= len(out) <= 2 * len(uniq)
    rng = np.random.default_rng(1)
    pts = rng.uniform(-2, 2, (300, 3))
    once = P.voxel_downsample(_scan(pts, np.full(300, 0.05)), 0.5)
    twice = P.voxel_downsample(once, 0.5)
    o1, o2 = np.lexsort(once.points.T), np.lexsort(twice.points.T)
    assert len(once) == len(twice) and np.allclose(once.points[o1], twice.points[o2])
    with pytest.raises(ValueError):
        P.voxel_downsample(_scan([[0.0, 0, 0]], [0.0]), 0.0)


@pytest.mark.parametrize("res", [0.1, 0.25, 0.4, 1.0])
def test_voxel_downsample_spinning_scan_vs_oracle(res):
    """A 65,536-point spinning scan (stamps by azimuth, so the seam voxels split) against the
    oracle restatement, bit for bit."""
    rng = np.random.default_rng(int(res * 100))
    n = 65536
    az = np.linspace(0.0, 2 * np.pi, n, endpoint=False)
    el = rng.uniform(-0.4, 0.4, n)
    r = rng.uniform(2.0, 30.0, n)
    pts = np.column_stack([r * np.cos(el) * np.cos(az), r * np.cos(el) * np.sin(az),
                           r * np.sin(el)]).astype(np.float32).astype(float)
    ts = 100.0 + az / (2 * np.pi) * 0.1
    out = P.voxel_downsample(_scan(pts, ts, 100.0, 100.1), res)
    op, ot = O.voxel_downsample(pts, ts, res, out.scan_end - out.scan_start)
    assert np.array_equal(out.points, op) and np.array_equal(out.stamps, ot)


# ---- deskew, per-point half (preprocess.py:218-231) -----------------------------------------
# tolerance: 1e-9 m absolute on coordinates up to ~35 m (CUDA's acos/sin are within 2 ulp of
# NumPy's; the north_star allows 1e-6 abs for floating point)
DESKEW_ATOL = 1e-9


@pytest.mark.parametrize("case", ["stationary", "yaw", "tumble"])
def test_deskew_points_matches_reference(golden, case):
    g = golden("deskew")
    out = P.deskew_points(g[f"{case}_points"], g[f"{case}_stamps"], g[f"{case}_node_t"],
                          g[f"{case}_quats"], g[f"{case}_trans"])
    np.testing.assert_allclose(out, g[f"{case}_out"], rtol=0, atol=DESKEW_ATOL)


def _yaw_quat(a):
    return np.column_stack([np.zeros_like(a), np.zeros_like(a), np.sin(a / 2), np.cos(a / 2)])


def test_deskew_points_properties_and_edges():
    rng = np.random.default_rng(3)
    pts = rng.uniform(-10, 10, (1000, 3))
    ts = rng.uniform(-0.02, 0.12, 1000)  # some stamps outside the node range: clipped
    node_t = np.linspace(0.0, 0.1, 11)
    # identity trajectory: points unchanged, bit for bit
    out = P.deskew_points(pts, ts, node_t, _yaw_quat(np.zeros(11)), np.zeros((11, 3)))
    assert np.array_equal(out, pts)
    # constant yaw rate 1 rad/s: closed form rotation by the clipped stamp (slerp is exact)
    out = P.deskew_points(pts, ts, node_t, _yaw_quat(node_t), np.zeros((11, 3)))
    a = np.clip(ts, 0.0, 0.1)
    exp = np.column_stack([np.cos(a) * pts[:, 0] - np.sin(a) * pts[:, 1],
                           np.sin(a) * pts[:, 0] + np.cos(a) * pts[:, 1], pts[:, 2]])
    np.testing.assert_allclose(out, exp, rtol=0, atol=1e-9)
    # repeated node stamps (zero-length segments), two-node trajectories, antipodal quats
    node_t = np.array([0.0, 0.05, 0.05, 0.1])
    q = _yaw_quat(np.array([0.0, 0.3, 0.3, 0.9]))
    q[2] *= -1.0
    tr = rng.normal(size=(4, 3))
    np.testing.assert_allclose(P.deskew_points(pts, ts, node_t, q, tr),
                               O.deskew_points(pts, ts, node_t, q, tr), rtol=0, atol=DESKEW_ATOL)
    np.testing.assert_allclose(P.deskew_points(pts, ts, node_t[[0, 3]], q[[0, 3]], tr[[0, 3]]),
                               O.deskew_points(pts, ts, node_t[[0, 3]], q[[0, 3]], tr[[0, 3]]),
                               rtol=0, atol=DESKEW_ATOL)
    assert P.deskew_points(np.zeros((0, 3)), np.zeros(0), node_t, q, tr).shape == (0, 3)


def test_deskew_points_large_scan_vs_oracle(golden):
    """131,072 points against the oracle on the reference's tumbling trajectory."""
    g = golden("deskew")
    rng = np.random.default_rng(4)
    pts = rng.uniform(-30, 30, (131072, 3))
    ts = rng.uniform(-0.01, 0.1, 131072)
    args = (g["tumble_node_t"], g["tumble_quats"], g["tumble_trans"])
    np.testing.assert_allclose(P.deskew_points(pts, ts, *args), O.deskew_points(pts, ts, *args),
                               rtol=0, atol=DESKEW_ATOL)
