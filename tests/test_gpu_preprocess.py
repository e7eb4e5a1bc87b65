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
