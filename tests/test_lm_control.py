"""CPU check of the device-solve LM's control flow (factor_graph.graph_optimize_lm) against
the reference's optimize_lm (factor_graph.py:546-612): with the device normal equations
replaced by a host stand-in that assembles with the graph's own _assemble_dense and solves
with the reference's splu call, the two LMs must agree bit for bit — iterations, accepted
steps, damping, final cost and the NotConverged exits.  No GPU: an IMU + prior local-mapping
graph above the dense threshold (41 frame states, 615 tangent dims)."""

import sys
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse
import scipy.sparse.linalg

ROOT = Path(__file__).resolve().parents[1]


class HostNormalEquations:
    """Stand-in for DeviceNormalEquations with the reference's own arithmetic."""

    def __init__(self, graph, slices, dim):
        self.graph, self.slices, self.dim = graph, slices, dim

    def assemble(self, values):
        self.h, self.g, cost = self.graph._assemble_dense(values, self.slices, self.dim)
        return cost

    def damped_step(self, lam):
        a = self.h + np.diag(lam * np.diag(self.h).copy())
        try:
            delta = scipy.sparse.linalg.splu(scipy.sparse.csc_matrix(a)).solve(-self.g)
        except (np.linalg.LinAlgError, RuntimeError, ValueError):
            return None
        return delta if np.all(np.isfinite(delta)) else None


@pytest.fixture()
def lm(monkeypatch):
    sys.path.insert(0, str(ROOT / "tools"))
    import lm_workloads

    if not (lm_workloads.REF / "limapper").is_dir():
        pytest.skip("reference not installed in baseline/_ref")
    from paper_2202_00242_b200 import factor_graph as vfg
    from paper_2202_00242_b200 import integrate

    monkeypatch.setattr(vfg.DeviceNormalEquations, "of",
                        classmethod(lambda cls, g, s, d: HostNormalEquations(g, s, d)))
    g, fg, _ = lm_workloads.local_mapping_lm(frames=41, matching=False)
    return lm_workloads, fg, integrate.ORIGINALS[(fg.FactorGraph, "optimize_lm")]


def _run(fn):
    try:
        return "ok", fn()
    except Exception as exc:  # NotConverged carries estimates and cost
        return type(exc).__name__, exc


def _same(a, b):
    assert a[0] == b[0]
    if a[0] == "ok":
        ra, rb = a[1], b[1]
        assert ra.iterations == rb.iterations and ra.final_cost == rb.final_cost
        est_a, est_b = ra.estimates, rb.estimates
    else:
        assert str(a[1]) == str(b[1]) and a[1].cost == b[1].cost
        est_a, est_b = a[1].estimates, b[1].estimates
    for k in est_a:
        assert np.array_equal(est_a[k].pose.translation, est_b[k].pose.translation)
        assert np.array_equal(est_a[k].velocity, est_b[k].velocity)


@pytest.mark.parametrize("kw", [dict(max_iterations=8),
                                dict(max_iterations=3, lambda_init=10.0),
                                dict(max_iterations=50, lambda_max=1e-4)])
def test_device_lm_control_flow_equals_reference(lm, kw):
    lw, fg, original = lm
    settings = fg.LmSettings(**kw)
    g1, _, _ = lw.local_mapping_lm(frames=41, matching=False)
    g2, _, _ = lw.local_mapping_lm(frames=41, matching=False)
    assert g1._slices()[1] > settings.dense_threshold
    _same(_run(lambda: g1.optimize_lm(settings)), _run(lambda: original(g2, settings)))
    for k in g1.values:  # the graph's own values are left as the reference leaves them
        assert np.array_equal(g1.values[k].pose.translation, g2.values[k].pose.translation)


def singular_graph(lw, fg):
    """The local-mapping graph plus a frame state anchored by a bias-only prior: its pose and
    velocity directions have no information, so every damped system is exactly singular."""
    g, _, _ = lw.local_mapping_lm(frames=41, matching=False)
    last = g.values[fg.frame_key(40)]
    g.add_variable(fg.frame_key(41), last)
    g.add_factor(fg.PriorFactor(fg.frame_key(41), last, np.r_[np.zeros(9), np.full(6, 1e2)]))
    return g


def test_singular_system_exhausts_damping_like_the_reference(lm):
    lw, fg, original = lm
    settings = fg.LmSettings(max_iterations=5)
    a = _run(lambda: singular_graph(lw, fg).optimize_lm(settings))
    b = _run(lambda: original(singular_graph(lw, fg), settings))
    assert a[0] == "NotConverged" and "singular" in str(a[1])
    _same(a, b)


class _Edge:
    """A structural stand-in factor: keys and the grounding flag are all check_structure
    reads (factor_graph.py:478-510)."""

    def __init__(self, keys, grounding=False):
        self.keys = tuple(keys)
        self.grounding = grounding


@pytest.mark.parametrize("seed", range(12))
def test_check_structure_matches_reference(lm, seed):
    """graph_check_structure (connected components over integer indices) raises exactly what
    the reference's union-find raises, message included, or passes where it passes."""
    lw, fg, _ = lm
    from paper_2202_00242_b200 import integrate

    original = integrate.ORIGINALS[(fg.FactorGraph, "check_structure")]
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 40))
    g = fg.FactorGraph()
    for i in range(n):
        g.add_variable(fg.submap_key(i), None)
    for _ in range(int(rng.integers(0, 2 * n))):
        k = int(rng.integers(1, 4))
        ids = rng.choice(n, size=k, replace=False)
        g.factors.append(_Edge([fg.submap_key(int(i)) for i in ids], rng.random() < 0.15))
    a = _run(lambda: g.check_structure())
    g.__dict__.pop("_vgicp_checked", None)
    b = _run(lambda: original(g))
    assert a[0] == b[0] and (a[0] == "ok" or str(a[1]) == str(b[1]))


def test_graphs_beyond_the_device_bound_keep_the_reference_solve(lm, monkeypatch):
    """Above DEVICE_SOLVE_MAX_DIM the dense device system is not built: optimize_lm is the
    reference's own (its sparse host solve)."""
    lw, fg, original = lm
    from paper_2202_00242_b200 import factor_graph as vfg

    monkeypatch.setattr(vfg, "DEVICE_SOLVE_MAX_DIM", 100)
    monkeypatch.setattr(vfg.DeviceNormalEquations, "of",
                        classmethod(lambda cls, g, s, d: pytest.fail("device path taken")))
    settings = fg.LmSettings(max_iterations=3)
    g1, _, _ = lw.local_mapping_lm(frames=41, matching=False)
    g2, _, _ = lw.local_mapping_lm(frames=41, matching=False)
    _same(_run(lambda: g1.optimize_lm(settings)), _run(lambda: original(g2, settings)))
