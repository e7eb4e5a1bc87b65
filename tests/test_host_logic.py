"""CPU checks of the host-side logic and of the kernel's arithmetic design.

kernel_model restates K4/K5 in NumPy: in fp64 the compact 29-value accumulation + adjoint
expansion must reproduce the oracle's explicit-Jacobian blocks to ~1e-12 (the algebra is
exact); with the kernel's precision choices (fp64 covariances and inverse, fp32 per-point
Jacobian terms and lane sums) it must stay within the 1e-4 rel / 1e-6 abs parity bar.
"""

from pathlib import Path

import numpy as np
import pytest

import kernel_model as KM
from oracle import vgicp_oracle as O
from paper_2202_00242_b200 import geometry as G
from paper_2202_00242_b200.registration import unpack_record, unpack_sym6

NAMES = ("h_ii", "b_i", "h_ij", "h_jj", "b_j")


def _map(g, res=0.5):
    tag = str(res).replace(".", "p")
    return (res, g[f"map{tag}_keys"], g[f"map{tag}_means"], g[f"map{tag}_covs"],
            g[f"map{tag}_counts"])


@pytest.mark.parametrize("case", range(6))
def test_adjoint_expansion_exact_in_fp64(golden, case):
    g = golden("registration")
    vm = _map(g)
    R, t, unary = g[f"case{case}_R"], g[f"case{case}_t"], bool(g[f"case{case}_unary"])
    ref = O.linearize(g["src_points"], g["src_covs"], vm, R, t, target_fixed=unary)
    got = KM.expand(KM.compact(g["src_points"], g["src_covs"], vm, R, t), R, t, unary)
    for k in NAMES:
        if ref[k] is not None:
            np.testing.assert_allclose(got[k], ref[k], rtol=1e-9, atol=1e-7)
    assert got["inliers"] == ref["inliers"]


def test_fp32_designs_would_break_parity(golden):
    """Why the kernel is fp64 per correspondence: the cheaper designs (fp32 per-point math,
    fp32-stored covariances) exceed the per-element 1e-4 bar on cancelling H/b entries."""
    g = golden("registration")
    vm = _map(g)
    worst = {"fp32 math": 0.0, "fp32 storage": 0.0}
    for case in range(6):
        R, t, unary = g[f"case{case}_R"], g[f"case{case}_t"], bool(g[f"case{case}_unary"])
        ref = O.linearize(g["src_points"], g["src_covs"], vm, R, t, target_fixed=unary)
        for name, kw in (("fp32 math", {"dtype": np.float32}),
                         ("fp32 storage", {"cov_dtype": np.float32})):
            got = KM.expand(KM.compact(g["src_points"], g["src_covs"], vm, R, t, **kw), R, t,
                            unary)
            for k in NAMES:
                if ref[k] is not None:
                    worst[name] = max(worst[name], KM.within_tolerance(got[k], ref[k]))
    assert worst["fp32 math"] > 1.0 and worst["fp32 storage"] > 1.0


def test_record_unpack_layout():
    rec = np.arange(92, dtype=float)
    lin = unpack_record(rec, unary=False)
    assert lin.h_ii[0, 0] == 0 and lin.h_ii[0, 5] == 5 and lin.h_ii[5, 0] == 5
    assert lin.h_ii[5, 5] == 20 and lin.h_ij[0, 0] == 21 and lin.h_ij[5, 5] == 56
    assert lin.h_jj[0, 0] == 57 and lin.b_i[0] == 78 and lin.b_j[5] == 89
    assert lin.cost == 90 and lin.inlier_count == 91
    u = unpack_record(rec, unary=True)
    assert u.h_ij is None and u.b_j is None


def test_sym6_roundtrip():
    a = np.random.default_rng(0).normal(size=(6, 6))
    a = a + a.T
    iu = np.triu_indices(6)
    assert np.array_equal(unpack_sym6(a[iu]), a)


def test_pose_table_composition_matches_host_geometry():
    rng = np.random.default_rng(5)
    poses = [G.Se3Pose(G.so3_exp(rng.uniform(-2, 2, 3)), rng.uniform(-20, 20, 3))
             for _ in range(8)]
    table = np.array([G.pose_row(p) for p in poses])
    vs, vt = np.array([0, 3, 5, 7]), np.array([1, 2, 6, 0])
    R, t = O.relative_transforms(table, vs, vt)
    for f in range(4):
        tij = G.pose_compose(G.pose_inverse(poses[vt[f]]), poses[vs[f]])
        np.testing.assert_allclose(R[f], tij.rotation.matrix(), atol=1e-15, rtol=0)
        np.testing.assert_allclose(t[f], tij.translation, atol=1e-13, rtol=0)


def test_geometry_mirror_matches_reference_ops():
    rng = np.random.default_rng(9)
    for _ in range(20):
        xi = rng.uniform(-1, 1, 6)
        p = G.pose_retract(G.Se3Pose.identity(), xi)
        np.testing.assert_allclose(G.pose_local(p, G.Se3Pose.identity()), xi, atol=1e-12)


def test_integrate_patch_replaces_and_restores():
    import types

    from paper_2202_00242_b200 import factor_graph, integrate, registration

    sentinel = object()
    pkg = types.SimpleNamespace(
        __name__="fakepkg",
        registration=types.SimpleNamespace(build_voxelmap=sentinel, match_terms=sentinel,
                                           unrelated=sentinel),
        factor_graph=types.SimpleNamespace(MatchingCostFactor=sentinel),
        preprocess=types.SimpleNamespace(knn_search=sentinel),
        odometry=types.SimpleNamespace(overlap_rate=sentinel, OdometryEstimator=None))

    class OdometryEstimator:
        def _overlap_matrix(self):
            return "reference loop"

    pkg.odometry.OdometryEstimator = OdometryEstimator
    undo = integrate.patch(pkg)
    assert OdometryEstimator._overlap_matrix is integrate._overlap_matrix
    assert pkg.registration.build_voxelmap is registration.build_voxelmap
    assert pkg.factor_graph.MatchingCostFactor is factor_graph.MatchingCostFactor
    assert pkg.odometry.overlap_rate is registration.overlap_rate
    assert pkg.registration.unrelated is sentinel
    undo()
    assert OdometryEstimator()._overlap_matrix() == "reference loop"
    assert pkg.registration.build_voxelmap is sentinel
    assert pkg.preprocess.knn_search is sentinel


def test_normal_equations_flat_layout_and_dense():
    """NormalEquations.from_flat / dense (the host side of vg_batch_assemble_*): the flat C-ABI
    layout [cost, count, diag V x 21 (upper), grad V x 6, pairs P x 36] scatters into the dense
    system the way the reference's _assemble_dense does (factor_graph.py:529-535)."""
    from paper_2202_00242_b200._lib import NormalEquations

    rng = np.random.default_rng(4)
    V, pairs = 4, np.array([[0, 2], [1, 3]], np.int32)
    full = [rng.normal(size=(6, 6)) for _ in range(V)]
    full = [a + a.T for a in full]
    iu = np.triu_indices(6)
    off = rng.normal(size=(2, 6, 6))
    grad = rng.normal(size=(V, 6))
    flat = np.concatenate([[3.5, 7.0], np.concatenate([a[iu] for a in full]), grad.ravel(),
                           off.ravel()])
    ne = NormalEquations.from_flat(flat, V, pairs)
    assert ne.cost == 3.5 and ne.count == 7
    assert all(np.array_equal(ne.diag[v], full[v]) for v in range(V))
    h, g = ne.dense(offsets=[0, 6, 12, 18], dim=24)
    ref = np.zeros((24, 24))
    for v in range(V):
        ref[6 * v:6 * v + 6, 6 * v:6 * v + 6] += full[v]
    for (a, b), blk in zip(pairs, off):
        ref[6 * a:6 * a + 6, 6 * b:6 * b + 6] += blk
        ref[6 * b:6 * b + 6, 6 * a:6 * a + 6] += blk.T
    assert np.array_equal(h, ref) and np.array_equal(h, h.T)
    assert np.array_equal(g, grad.ravel())
    # 15-dof keys: blocks land top-left of each variable's slice
    h15, _ = ne.dense(offsets=[0, 15, 30, 45], dim=60)
    assert np.array_equal(h15[15:21, 45:51], off[1]) and not h15[21:30].any()


@pytest.mark.skipif(not Path("/root/reference/pkg/src").exists(), reason="needs the reference")
def test_make_deskew_glue_matches_reference_deskew():
    """The drop-in deskew (reference host IMU integration + per-point step) equals the
    reference's deskew on its own test scenarios (test_preprocess.py:162-231); the per-point
    step is the oracle here (no GPU), the GPU kernel is checked against the same trajectories
    in tests/test_gpu_preprocess.py."""
    import importlib
    import sys as _sys

    _sys.path.insert(0, "/root/reference/pkg/src")
    try:
        P = importlib.import_module("limapper.preprocess")
        G = importlib.import_module("limapper.geometry")
        I = importlib.import_module("limapper.imu")
        E = importlib.import_module("limapper.errors")
    finally:
        _sys.path.remove("/root/reference/pkg/src")
    from oracle import vgicp_oracle as O
    from paper_2202_00242_b200 import preprocess as PP

    dk = PP.make_deskew(P, points_fn=O.deskew_points)
    rng = np.random.default_rng(8)
    pts = rng.uniform(-3, 3, (50, 3))
    stamps = rng.uniform(0.0, 0.1, 50)
    samples = [I.ImuSample(float(t), -I.GRAVITY + [0.3, -0.2, 0.1], [0.1, 0.2, -0.3])
               for t in np.arange(-0.01, 0.12, 0.005)]
    frame = P.Frame(points=pts, stamps=stamps, stamp=0.0, scan_end=0.1)
    state = G.SensorState(pose=G.Se3Pose(G.so3_exp([0.4, -0.1, 1.2]), np.array([10.0, -3.0, 2.0])),
                          velocity=np.array([1.0, 0.5, -0.2]), bias_accel=np.zeros(3),
                          bias_gyro=np.zeros(3), stamp=0.0)
    for st in (G.SensorState.zero(), state):
        ref = P.deskew(frame, samples, st)
        got = dk(frame, samples, st)
        assert got.deskewed and type(got) is type(ref)
        np.testing.assert_allclose(got.points, ref.points, rtol=0, atol=1e-12)
    with pytest.raises(E.ImuCoverageGap):
        dk(P.Frame(points=pts[:1], stamps=np.array([0.05]), stamp=0.0, scan_end=0.1),
           [I.ImuSample(0.0, -I.GRAVITY, np.zeros(3)), I.ImuSample(0.1, -I.GRAVITY, np.zeros(3))],
           G.SensorState.zero())
    with pytest.raises(ValueError):
        dk(P.Frame(points=np.zeros((1, 3)), stamps=np.zeros(1), stamp=0.0, scan_end=0.1,
                   deskewed=True), samples, G.SensorState.zero())
    empty = P.Frame(points=np.zeros((0, 3)), stamps=np.zeros(0), stamp=0.0, scan_end=0.1)
    assert dk(empty, samples, G.SensorState.zero()).deskewed


def test_f32_record_decoding():
    """record_cost_inliers_f32 reads the compact record's fp64 cost (words 90-91, low word
    first) and int32 inlier count (word 92) — the layout K5's rec32_word writes."""
    from paper_2202_00242_b200 import _lib

    rec = np.zeros((3, _lib.REC_LINEARIZE_F32), np.float32)
    costs = np.array([1.5e5 + 1e-9, 0.0, -3.25], np.float64)
    inl = np.array([13004, 0, 7], np.int32)
    rec[:, 90:92] = costs.view(np.float32).reshape(3, 2)
    rec[:, 92] = inl.view(np.float32)
    rec[:, :90] = np.arange(90, dtype=np.float32)
    c, n = _lib.record_cost_inliers_f32(rec)
    assert np.array_equal(c, costs) and np.array_equal(n, inl.astype(np.int64))
    assert c.dtype == np.float64 and n.dtype == np.int64


def test_pose_table_builder_matches_pose_row():
    """factor_graph._PoseTable (the batch pose table at given values, with the key-order fast
    path) equals the row-by-row geometry.pose_row table for submap poses and frame states,
    whether or not `values` keeps the last call's key objects and order."""
    from types import SimpleNamespace

    from paper_2202_00242_b200.factor_graph import _PoseTable, frame_key, submap_key

    rng = np.random.default_rng(3)

    def pose():
        return G.Se3Pose(G.so3_exp(rng.normal(size=3)), rng.normal(size=3))

    keys = [submap_key(i) for i in range(5)] + [frame_key(i) for i in range(3)]
    fixed = np.array([G.pose_row(pose())])
    vals = {k: (pose() if k.kind == "submap-pose" else SimpleNamespace(pose=pose()))
            for k in keys}
    var_keys = [keys[i] for i in (3, 0, 6, 1, 5)]
    table = _PoseTable(var_keys, fixed)

    def want(values):
        rows = [G.pose_row(values[k] if k.kind == "submap-pose" else values[k].pose)
                for k in var_keys]
        return np.vstack([np.array(rows), fixed])

    assert np.array_equal(table.build(vals), want(vals))          # slow path, learns order
    moved = {k: (pose() if k.kind == "submap-pose" else SimpleNamespace(pose=pose()))
             for k in vals}                                       # same key objects/order
    assert np.array_equal(table.build(moved), want(moved))        # fast path
    shuffled = dict(reversed(list(moved.items())))                # other order
    assert np.array_equal(table.build(shuffled), want(shuffled))
    fresh = {submap_key(k.index) if k.kind == "submap-pose" else frame_key(k.index): v
             for k, v in moved.items()}                           # equal, not identical keys
    assert np.array_equal(table.build(fresh), want(fresh))
