"""The LM's damped solve on the device (vg_solver_*, csrc/solve.cu).

Checked against scipy on the same matrices (the reference's cho_factor / splu calls,
factor_graph.py:565-576, 711-722), the device scatter of a batch's normal equations against
the host NormalEquations.dense (bit for bit), and whole LM runs through the reference's own
FactorGraph: the patched optimize_lm (device solve) against the reference's optimize_lm (host
splu) from the same values, on a global-mapping graph and an IMU local-mapping graph above
the dense threshold."""

import sys
from pathlib import Path

import numpy as np
import pytest
import scipy.linalg

from paper_2202_00242_b200 import _lib
from paper_2202_00242_b200 import workloads as W

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def spd(rng, dim, rows=None):
    J = rng.normal(size=(rows or dim + 200, dim))
    return J.T @ J + 1e-3 * np.eye(dim)


def tiles(H, t=64):
    n = H.shape[0]
    return [(r, c, H[r:r + t, c:c + t]) for r in range(0, n, t) for c in range(0, n, t)]


def test_solver_matches_scipy_cholesky():
    rng = np.random.default_rng(0)
    dim = 700
    H = spd(rng, dim)
    g = rng.normal(size=dim)
    s = _lib.DeviceSolver(dim)
    s.add_blocks(tiles(H), g)
    h, gg, cost = s.export()
    assert np.array_equal(h, H) and np.array_equal(gg, g) and cost == 0.0
    assert np.array_equal(s.diagonal(), np.diag(H))
    for lam in (0.0, 1e-6, 0.25, 1e4):
        assert s.factor(lam, method=_lib.SOLVE_CHOLESKY) == 0
        got = s.solve()
        a = H + np.diag(lam * np.diag(H))            # factor_graph.py:571-573
        want = scipy.linalg.cho_solve(scipy.linalg.cho_factor(a, lower=True), -g)
        assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
    # several right-hand sides (marginal_covariance's identity columns, :711-722)
    assert s.factor(0.0, jitter=1e-6) == 0
    rhs = np.zeros((dim, 6))
    rhs[120:126] = np.eye(6)
    want = np.linalg.solve(H + 1e-6 * np.eye(dim), rhs)
    assert np.allclose(s.solve(rhs), want, rtol=1e-9, atol=1e-14)


def test_solver_lu_fallback_has_splu_semantics():
    """An indefinite nonsingular damped matrix: cho_factor fails (info > 0), splu solves; an
    exactly singular one fails both ways (the reference's LinAlgError / RuntimeError)."""
    rng = np.random.default_rng(1)
    dim = 640
    Q, _ = np.linalg.qr(rng.normal(size=(dim, dim)))
    ev = rng.uniform(0.5, 2.0, dim)
    ev[::7] *= -1.0
    H = (Q * ev) @ Q.T
    H = 0.5 * (H + H.T)
    g = rng.normal(size=dim)
    s = _lib.DeviceSolver(dim)
    s.add_blocks(tiles(H), g)
    assert s.factor(0.0, method=_lib.SOLVE_CHOLESKY) > 0
    assert s.factor(0.0, method=_lib.SOLVE_CHOLESKY_LU) == 0
    want = np.linalg.solve(H, -g)
    assert np.linalg.norm(s.solve() - want) <= 1e-9 * np.linalg.norm(want)
    s.reset()
    Hs = H.copy()
    Hs[5, :] = 0.0
    Hs[:, 5] = 0.0
    s.add_blocks(tiles(Hs), g)
    assert s.factor(0.0, method=_lib.SOLVE_CHOLESKY_LU) > 0
    with pytest.raises(ValueError):
        s.solve()  # no factorization


def test_solver_rejects_bad_blocks():
    s = _lib.DeviceSolver(700)
    with pytest.raises(ValueError):
        s.add_blocks([(690, 0, np.ones((20, 6)))])
    with pytest.raises(ValueError):
        _lib.DeviceSolver(0)


@pytest.fixture(scope="module")
def small_global():
    return W.global_mapping(n_submaps=40, neighbors=6, n_az=128, n_el=32, seed=11)


def test_batch_scatter_equals_host_dense_assembly(small_global):
    """vg_solver_add_batch scatters K6's block-sparse system into the device H exactly where
    NormalEquations.dense puts it (15-dof frame-state spacing, pose block top-left), bit for
    bit, and returns the batch's gated cost."""
    wl = small_global
    batch = wl.batch()
    V = wl.n_submaps
    batch.assemble_setup(V)
    ne = batch.assemble_poses(wl.pose_table)
    offsets = np.arange(V) * 15 + 3 * (np.arange(V) % 2)   # pose block anywhere in its slice
    dim = 15 * V
    h_ref, g_ref = ne.dense(offsets, dim)
    s = _lib.DeviceSolver(dim)
    cost = s.add_batch(batch, wl.pose_table, offsets)
    h, g, c = s.export()
    assert np.array_equal(h, h_ref) and np.array_equal(g, g_ref)
    assert cost == ne.cost == c
    with pytest.raises(ValueError):  # overlapping variable blocks
        s.add_batch(batch, wl.pose_table, np.arange(V) * 3)


# ---- whole LM runs through the reference's FactorGraph ------------------------------------

def _reference_or_skip():
    sys.path.insert(0, str(ROOT / "tools"))
    import lm_workloads

    if not (lm_workloads.REF / "limapper").is_dir():
        pytest.skip("reference not installed in baseline/_ref")
    return lm_workloads


def _trans(v):
    return v.translation if hasattr(v, "translation") else v.pose.translation


def _rot(v):
    return (v.rotation if hasattr(v, "rotation") else v.pose.rotation).matrix()


def _compare_runs(g_dev, g_host, fg, settings):
    from paper_2202_00242_b200 import integrate

    slices, dim = g_dev._slices()
    assert dim > settings.dense_threshold
    a = g_dev.optimize_lm(settings)                      # patched: device solve
    b = integrate.ORIGINALS[(fg.FactorGraph, "optimize_lm")](g_host, settings)  # host splu
    assert a.iterations == b.iterations
    assert abs(a.final_cost - b.final_cost) <= 1e-9 * abs(b.final_cost)
    for k in a.estimates:
        assert np.max(np.abs(_trans(a.estimates[k]) - _trans(b.estimates[k]))) < 1e-8
        assert np.max(np.abs(_rot(a.estimates[k]) - _rot(b.estimates[k]))) < 1e-8
    return a, b


def test_global_mapping_lm_device_solve_matches_reference_lm():
    lw = _reference_or_skip()
    wl = W.global_mapping(n_submaps=110, neighbors=8, n_az=128, n_el=32, seed=12)
    g1, fg, _ = lw.global_mapping_lm(wl)
    g2, _, _ = lw.global_mapping_lm(wl)
    c0 = g1.total_cost()
    a, _ = _compare_runs(g1, g2, fg, fg.LmSettings(max_iterations=6))
    assert a.final_cost < c0
    # marginal covariance of a submap pose: device factorization vs the reference's cho_factor
    from paper_2202_00242_b200 import integrate

    key = fg.submap_key(37)
    got = g1.marginal_covariance(key)
    g2.values = dict(g1.values)
    g2._cached_normal = None
    want = integrate.ORIGINALS[(fg.FactorGraph, "marginal_covariance")](g2, key)
    assert np.allclose(got, want, rtol=1e-8, atol=1e-14)


def test_local_mapping_with_imu_lm_device_solve_matches_reference_lm():
    lw = _reference_or_skip()
    g1, fg, _ = lw.local_mapping_lm(frames=41)      # 41 x 15 = 615 tangent dims
    g2, _, _ = lw.local_mapping_lm(frames=41)
    _compare_runs(g1, g2, fg, fg.LmSettings(max_iterations=4))


def test_small_graphs_keep_the_reference_dense_path():
    lw = _reference_or_skip()
    from paper_2202_00242_b200 import factor_graph as vfg

    wl = W.global_mapping(n_submaps=20, neighbors=4, n_az=128, n_el=32, seed=13)
    g, fg, _ = lw.global_mapping_lm(wl)
    g.optimize_lm(fg.LmSettings(max_iterations=2))
    assert "_vgicp_normal" not in g.__dict__          # no device solver for dim <= 600
    assert isinstance(vfg.DeviceNormalEquations, type)


def test_singular_graph_exhausts_damping_on_the_device():
    """Device Cholesky fails, the LU fallback meets an exactly zero pivot: the LM raises the
    reference's NotConverged("damping exhausted ...") with the same best estimates."""
    lw = _reference_or_skip()
    from test_lm_control import _run, _same, singular_graph

    from paper_2202_00242_b200 import integrate

    import limapper.factor_graph as fg

    settings = fg.LmSettings(max_iterations=5)
    a = _run(lambda: singular_graph(lw, fg).optimize_lm(settings))
    b = _run(lambda: integrate.ORIGINALS[(fg.FactorGraph, "optimize_lm")](
        singular_graph(lw, fg), settings))
    assert a[0] == "NotConverged" and "singular" in str(a[1])
    _same(a, b)
