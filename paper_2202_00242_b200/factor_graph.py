"""Drop-in MatchingCostFactor with a batching shim, plus the host-side LM that calls it.

``MatchingCostFactor`` keeps the reference's per-factor interface (factor_graph.py:102-126,
209-308): ``keys``, ``unary``, ``grounding``, ``kind``, ``cost(values)``,
``linearize(values) -> FactorLinearization``.  The reference ``FactorGraph`` calls it one
factor at a time (total_cost :472-474, _assemble_dense :522-536).  Behind that unchanged
interface, the first factor that misses its cache for a given set of values triggers ONE
batched GPU evaluation of every live matching factor whose variables are in ``values``;
each factor then serves its own record from an identity-keyed cache, exactly as the
reference's ``_terms_cache`` does for one factor (:253-269).  Values are immutable, so
identity of (v_i, v_j) is a safe key.

``FactorGraph`` / ``PriorFactor`` restate the reference's host LM (:425-612) so the drop-in
can be exercised end to end where the reference package is absent (the GPU box); the LM
solve stays on the host as in the reference.
"""

from __future__ import annotations

import itertools
import weakref
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

from . import _lib
from .geometry import (
    pose_local,
    pose_retract,
    pose_row,
    so3_right_jacobian_inv,
)
from .preprocess import device_cloud
from .registration import _as_device_map, unpack_sym6

VARIABLE_DIMS = {"frame-state": 15, "submap-pose": 6, "endpoint-state": 15}


@dataclass(frozen=True, order=True)
class Key:
    kind: str
    index: int

    @property
    def dim(self) -> int:
        return VARIABLE_DIMS[self.kind]

    def __repr__(self) -> str:
        return f"{self.kind}:{self.index}"


def frame_key(index: int) -> Key:
    return Key("frame-state", index)


def submap_key(index: int) -> Key:
    return Key("submap-pose", index)


def _pose_of(kind: str, value):
    return value if kind == "submap-pose" else value.pose


class FactorLinearization:
    """Gradient/Hessian blocks of one factor (factor_graph.py:102-111)."""

    __slots__ = ("keys", "g", "h", "cost")

    def __init__(self, keys, g, h, cost):
        self.keys = keys
        self.g = g
        self.h = h
        self.cost = cost


class Factor:
    keys: tuple
    grounding = False

    def cost(self, values) -> float:
        raise NotImplementedError

    def linearize(self, values) -> FactorLinearization:
        raise NotImplementedError


# ---- the batching shim ---------------------------------------------------------------------


class _Batcher:
    """Registry of live GPU matching factors and the cache of flattened device batches."""

    def __init__(self):
        self._live: "weakref.WeakValueDictionary[int, MatchingCostFactor]" = \
            weakref.WeakValueDictionary()
        self._serial = itertools.count()
        self._batches: "OrderedDict[tuple, tuple]" = OrderedDict()
        self.evaluations = 0

    def register(self, f: "MatchingCostFactor") -> None:
        f._serial = next(self._serial)
        self._live[f._serial] = f

    def _batch_for(self, group):
        sig = tuple(f._serial for f in group)
        hit = self._batches.get(sig)
        if hit is not None:
            self._batches.move_to_end(sig)
            return hit
        var_index: dict = {}
        for f in group:
            for k in f.keys:
                var_index.setdefault(k, len(var_index))
        var_keys = list(var_index)
        fixed_rows = []
        vs, vt = [], []
        for f in group:
            vs.append(var_index[f.keys[0]])
            if f.unary:
                vt.append(len(var_keys) + len(fixed_rows))
                fixed_rows.append(pose_row(f.fixed_target_pose))
            else:
                vt.append(var_index[f.keys[1]])
        batch = _lib.DeviceBatch([device_cloud(f.source) for f in group],
                                 [_as_device_map(f.target_map) for f in group],
                                 [f.unary for f in group], [f.min_inliers for f in group],
                                 vs, vt)
        fixed = np.array(fixed_rows).reshape(-1, 8)
        entry = (batch, var_keys, fixed, [weakref.ref(f) for f in group])
        self._batches[sig] = entry
        while len(self._batches) > 8:
            self._batches.popitem(last=False)
        return entry

    def evaluate(self, values, mode: int, requester: "MatchingCostFactor") -> None:
        group = []
        for serial in sorted(self._live.keys()):
            f = self._live.get(serial)
            if f is None or f._empty:
                continue
            if any(k not in values for k in f.keys):
                continue
            if f._cached(values, mode) is not None:
                continue
            group.append(f)
        if requester not in group:
            group.append(requester)
        # factors sharing a target map adjacent: the batch's item order is then target-major
        # (map reuse in L2) and its pipelined host copy moves contiguous record ranges
        group.sort(key=lambda f: id(f.target_map))
        batch, var_keys, fixed, _ = self._batch_for(group)
        poses = np.empty((len(var_keys) + fixed.shape[0], 8))
        for i, k in enumerate(var_keys):
            poses[i] = pose_row(_pose_of(k.kind, values[k]))
        if fixed.shape[0]:
            poses[len(var_keys):] = fixed
        # fp64 records into pinned memory (the staged copies overlap the compute); the compact
        # fp32 record (linearize_poses_f32) halves the PCIe bytes for callers that take fp32
        # blocks, but here the per-factor Python unpacking dominates either way
        out = batch.linearize_poses(poses, mode)
        self.evaluations += 1
        for f, rec in zip(group, out):
            f._store(values, mode, rec)


    def assemble(self, group, values, var_keys) -> "_lib.NormalEquations":
        """Device-assembled normal equations of `group` over the graph variables `var_keys`
        (FactorGraph._assemble_dense, factor_graph.py:522-536)."""
        sig = ("asm", tuple(f._serial for f in group), tuple(var_keys))
        hit = self._batches.get(sig)
        if hit is None:
            index = {k: i for i, k in enumerate(var_keys)}
            fixed_rows, vs, vt = [], [], []
            for f in group:
                vs.append(index[f.keys[0]])
                if f.unary:
                    vt.append(len(var_keys) + len(fixed_rows))
                    fixed_rows.append(pose_row(f.fixed_target_pose))
                else:
                    vt.append(index[f.keys[1]])
            batch = _lib.DeviceBatch([device_cloud(f.source) for f in group],
                                     [_as_device_map(f.target_map) for f in group],
                                     [f.unary for f in group], [f.min_inliers for f in group],
                                     vs, vt)
            batch.assemble_setup(len(var_keys))
            hit = (batch, np.array(fixed_rows).reshape(-1, 8), [weakref.ref(f) for f in group])
            self._batches[sig] = hit
            while len(self._batches) > 8:
                self._batches.popitem(last=False)
        self._batches.move_to_end(sig)
        batch, fixed, _ = hit
        poses = np.empty((len(var_keys) + fixed.shape[0], 8))
        for i, k in enumerate(var_keys):
            poses[i] = pose_row(_pose_of(k.kind, values[k]))
        if fixed.shape[0]:
            poses[len(var_keys):] = fixed
        self.evaluations += 1
        return batch.assemble_poses(poses)


_BATCHER = _Batcher()


class MatchingCostFactor(Factor):
    """Voxelized registration constraint between a source frame and a target voxel map;
    unary when the target pose is fixed (factor_graph.py:209-308).  GPU-evaluated."""

    def __init__(self, key_source: Key, source, target_map, key_target: Key | None = None,
                 fixed_target_pose=None, min_inliers: int = 10):
        if (key_target is None) == (fixed_target_pose is None):
            raise ValueError("exactly one of key_target / fixed_target_pose")
        self.keys = (key_source,) if key_target is None else (key_source, key_target)
        self.source = source
        self.target_map = target_map
        self.fixed_target_pose = fixed_target_pose
        self.min_inliers = min_inliers
        self._empty = (len(source) == 0 or len(target_map) == 0
                       or getattr(source, "covs", None) is None)
        self._cache = None  # (v_i, v_j, mode, record)
        _BATCHER.register(self)

    @property
    def unary(self) -> bool:
        return self.fixed_target_pose is not None

    @property
    def grounding(self) -> bool:
        return self.unary

    @property
    def kind(self) -> str:
        return "matching-cost-unary" if self.unary else "matching-cost-binary"

    def _vals(self, values):
        return values[self.keys[0]], (None if self.unary else values[self.keys[1]])

    def _cached(self, values, mode):
        c = self._cache
        if c is None:
            return None
        v_i, v_j = self._vals(values)
        if c[0] is v_i and c[1] is v_j and (c[2] == _lib.MODE_LINEARIZE or mode == c[2]):
            return c
        return None

    def _store(self, values, mode, rec) -> None:
        v_i, v_j = self._vals(values)
        self._cache = (v_i, v_j, mode, rec)

    def _record(self, values, mode):
        c = self._cached(values, mode)
        if c is None:
            _BATCHER.evaluate(values, mode, self)
            c = self._cache
        return c[2], c[3]

    def cost(self, values) -> float:
        if self._empty:
            return 0.0
        mode, rec = self._record(values, _lib.MODE_COST)
        cost, inl = (rec[0], rec[1]) if mode == _lib.MODE_COST else (rec[90], rec[91])
        return 0.0 if inl < self.min_inliers else float(cost)

    def linearize(self, values) -> FactorLinearization:
        zeros = [np.zeros(k.dim) for k in self.keys]
        if not self._empty:
            _, rec = self._record(values, _lib.MODE_LINEARIZE)
            cost, inl = float(rec[90]), rec[91]
        if self._empty or inl < self.min_inliers:  # DegenerateConstraint -> no-op
            h = {(a, a): np.zeros((k.dim, k.dim)) for a, k in enumerate(self.keys)}
            return FactorLinearization(self.keys, zeros, h, 0.0)
        di = self.keys[0].dim
        g_i = np.zeros(di)
        g_i[:6] = rec[78:84]
        h_ii = np.zeros((di, di))
        h_ii[:6, :6] = unpack_sym6(rec[0:21])
        if self.unary:
            return FactorLinearization(self.keys, [g_i], {(0, 0): h_ii}, cost)
        dj = self.keys[1].dim
        g_j = np.zeros(dj)
        g_j[:6] = rec[84:90]
        h_jj = np.zeros((dj, dj))
        h_jj[:6, :6] = unpack_sym6(rec[57:78])
        h_ij = np.zeros((di, dj))
        h_ij[:6, :6] = rec[21:57].reshape(6, 6)
        return FactorLinearization(self.keys, [g_i, g_j],
                                   {(0, 0): h_ii, (0, 1): h_ij, (1, 1): h_jj}, cost)


# ---- host-side graph (restated so the drop-in runs where limapper is absent) ---------------

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

    def total_cost(self, values=None) -> float:
        values = self.values if values is None else values
        return float(sum(f.cost(values) for f in self.factors))

    def _slices(self):
        out, off = {}, 0
        for k in self.values:
            out[k] = slice(off, off + k.dim)
            off += k.dim
        return out, off

    #: sum the matching factors' blocks on the device (vg_batch_assemble_*) instead of per
    #: factor on the host; results agree to fp64 rounding (block sums in factor order)
    device_assembly = True

    def _assemble_dense(self, values, slices, dim):
        h = np.zeros((dim, dim))
        g = np.zeros(dim)
        cost = 0.0
        factors = self.factors
        if self.device_assembly:
            gpu = [f for f in factors if isinstance(f, MatchingCostFactor) and not f._empty]
            if gpu:
                keys = list(self.values)
                ne = _BATCHER.assemble(gpu, values, keys)
                hd, gd = ne.dense([slices[k].start for k in keys], dim)
                h += hd
                g += gd
                cost += ne.cost
                factors = [f for f in factors
                           if not (isinstance(f, MatchingCostFactor) and not f._empty)]
        for f in factors:
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
