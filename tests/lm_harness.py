"""TEST HARNESS — a restatement of the reference's host LM (limapper factor_graph.py:129-167,
425-612: PriorFactor, LmSettings, OptimizeResult, FactorGraph.optimize_lm), used by the GPU
tests only where the reference package itself is not importable.  The product drives the
reference's own FactorGraph (integrate.patch); see graph_api() below.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

from paper_2202_00242_b200.factor_graph import (
    Factor,
    FactorLinearization,
    Key,
    MatchingCostFactor,
    graph_assemble_dense,
    graph_total_cost,
    submap_key,
)
from paper_2202_00242_b200.geometry import pose_local, pose_retract, so3_right_jacobian_inv


def graph_api():
    """(FactorGraph, PriorFactor, LmSettings, submap_key, per-factor _assemble_dense, geometry)
    — the reference's own classes (and pose math) with the drop-in patched in when limapper is
    importable (e.g. from baseline/_ref), else this harness's restatement with the same
    replacements and the package's geometry mirror."""
    import os
    import sys
    from pathlib import Path

    ref = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
    if ref.is_dir() and str(ref) not in sys.path and not os.environ.get("VGICP_NO_REF"):
        sys.path.append(str(ref))
    try:
        import limapper.factor_graph as fg  # noqa: F401
    except Exception:
        from paper_2202_00242_b200 import geometry

        return (FactorGraph, PriorFactor, LmSettings, submap_key,
                FactorGraph._per_factor_assemble, geometry)
    import limapper.geometry as geometry

    from paper_2202_00242_b200 import integrate

    integrate.patch("limapper")
    orig = integrate.ORIGINALS[(fg.FactorGraph, "_assemble_dense")]
    return fg.FactorGraph, fg.PriorFactor, fg.LmSettings, fg.submap_key, orig, geometry


class PriorFactor(Factor):
    """Quadratic prior on a submap pose's tangent offset (factor_graph.py:129-167)."""

    grounding = True
    kind = "prior"

    def __init__(self, key: Key, prior_value, information):
        if key.kind != "submap-pose":
            raise ValueError("this restatement supports submap-pose priors only")
        self.keys = (key,)
        self.prior = prior_value
        info = np.asarray(information, dtype=float)
        self.information = np.diag(info) if info.ndim == 1 else info

    def cost(self, values) -> float:
        r = pose_local(values[self.keys[0]], self.prior)
        return float(r @ self.information @ r)

    def linearize(self, values) -> FactorLinearization:
        cur = values[self.keys[0]]
        r = pose_local(cur, self.prior)
        jac = np.eye(6)
        jac[0:3, 0:3] = so3_right_jacobian_inv(r[:3])
        jac[3:6, 3:6] = self.prior.rotation.matrix().T @ cur.rotation.matrix()
        jtw = 2.0 * jac.T @ self.information
        return FactorLinearization(self.keys, [jtw @ r], {(0, 0): jtw @ jac},
                                   float(r @ self.information @ r))


@dataclass
class LmSettings:
    max_iterations: int = 64
    rel_cost_tol: float = 1e-9
    update_tol: float = 1e-9
    lambda_init: float = 1e-6
    lambda_down: float = 0.5
    lambda_up: float = 4.0
    lambda_max: float = 1e12
    dense_threshold: int = 600


@dataclass
class OptimizeResult:
    estimates: dict
    final_cost: float
    iterations: int
    converged: bool = True


class NotConverged(RuntimeError):
    def __init__(self, message, estimates=None, cost=None):
        super().__init__(message)
        self.estimates = estimates
        self.cost = cost


class FactorGraph:
    """Variables + factors with the reference's damped Gauss-Newton (factor_graph.py:445-612)."""

    def __init__(self):
        self.values: dict = {}
        self.factors: list = []

    def add_variable(self, key: Key, initial_value) -> None:
        if key in self.values:
            raise ValueError(f"{key} already in graph")
        self.values[key] = initial_value

    def add_factor(self, factor: Factor) -> None:
        for k in factor.keys:
            if k not in self.values:
                raise KeyError(f"factor references missing {k}")
        self.factors.append(factor)
        if isinstance(factor, MatchingCostFactor):  # as graph_add_factor does when patched
            factor._graph_ref = weakref.ref(self)

    def _slices(self):
        out, off = {}, 0
        for k in self.values:
            out[k] = slice(off, off + k.dim)
            off += k.dim
        return out, off

    # the drop-in's replacements of the reference's total_cost / _assemble_dense
    total_cost = graph_total_cost
    _assemble_dense = graph_assemble_dense

    def _per_factor_assemble(self, values, slices, dim):
        """The reference's per-factor scatter (factor_graph.py:522-536)."""
        h = np.zeros((dim, dim))
        g = np.zeros(dim)
        cost = 0.0
        for f in self.factors:
            lin = f.linearize(values)
            cost += lin.cost
            sls = [slices[k] for k in lin.keys]
            for a, ga in enumerate(lin.g):
                g[sls[a]] += ga
            for (a, b), blk in lin.h.items():
                h[sls[a], sls[b]] += blk
                if a != b:
                    h[sls[b], sls[a]] += blk.T
        return h, g, cost

    def _retract_all(self, values, slices, delta):
        return {k: pose_retract(v, delta[slices[k]]) for k, v in values.items()}

    def _solve(self, h, g, lam, diag, dense):
        a = h + np.diag(lam * diag)
        if dense:
            return scipy.linalg.cho_solve(scipy.linalg.cho_factor(a, lower=True), -g)
        return scipy.sparse.linalg.splu(scipy.sparse.csc_matrix(a)).solve(-g)

    def optimize_lm(self, settings: LmSettings | None = None) -> OptimizeResult:
        s = settings or LmSettings()
        slices, dim = self._slices()
        values = dict(self.values)
        cost = self.total_cost(values)
        lam = s.lambda_init
        iterations = 0
        dense = dim <= s.dense_threshold
        for _ in range(s.max_iterations):
            h, g, cost = self._assemble_dense(values, slices, dim)
            iterations += 1
            diag = np.diag(h).copy()
            accepted = converged = False
            while True:
                try:
                    delta = self._solve(h, g, lam, diag, dense)
                    if not np.all(np.isfinite(delta)):
                        raise np.linalg.LinAlgError("non-finite update")
                except (np.linalg.LinAlgError, RuntimeError, ValueError):
                    lam *= s.lambda_up
                    if lam > s.lambda_max:
                        self.values = values
                        raise NotConverged("damping exhausted", estimates=values, cost=cost)
                    continue
                if np.max(np.abs(delta)) < s.update_tol:
                    converged = True
                    break
                candidate = self._retract_all(values, slices, delta)
                new_cost = self.total_cost(candidate)
                if np.isfinite(new_cost) and new_cost < cost:
                    values = candidate
                    accepted = True
                    lam = max(lam * s.lambda_down, 1e-12)
                    break
                lam *= s.lambda_up
                if lam > s.lambda_max:
                    self.values = values
                    raise NotConverged("no cost-reducing step", estimates=values, cost=cost)
            if converged:
                break
            if accepted and (cost - new_cost) <= s.rel_cost_tol * max(cost, 1e-30):
                cost = new_cost
                break
            cost = new_cost
        self.values = values
        _, _, final = self._assemble_dense(values, slices, dim)
        return OptimizeResult(values, final, iterations)
